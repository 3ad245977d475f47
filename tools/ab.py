"""A/B timing of compile-time k_raycast variants on the GPU box (name:@lib.so times a prebuilt library).

    python tools/ab.py --variant base: --variant staged:-DDTSDF_ALWAYS_STAGED [--configs C1,C2] [--rounds 2]

Each variant is built with the product flags plus its defines into gpurun_out/ab_<name>.so, then
timed in its own process (tools/ab.py --run), round-robin over the variants `--rounds` times so
that clock drift hits all of them alike.  Every run also checks parity against the oracle on the
same frame (tests/parity.py), so a faster variant that changes results shows up at once.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


# row strips holding the slowest warp tiles of a view (tools/isolate.py): launched alone, their
# k_raycast time is the uncontended critical path
STRIPS = {"C1": "64:72,224:232", "C2": "344:352,472:480"}


def run_one(args):
    import numpy as np
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle
    import scenes
    from parity import compare
    from paper_2301_12796_b200 import Renderer

    R = Renderer(0)
    for kv in args.set:  # DTSDF_OPT_* settings "option=value"
        o, v = kv.split("=")
        R.set_option(int(o), int(v))
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for name in args.configs.split(","):
        w = scenes.CONFIGS[name]()
        R.upload_volume(w.volume)
        poses = np.asarray(w.poses[:1], np.float32)
        out = R.render(poses, w.intrinsics)
        for _ in range(5):
            R.render_into(poses, w.intrinsics, out["depth"], out["normal"], out["color"], out["mask"])
        torch.cuda.synchronize()
        R.reset_kernel_times()
        R.set_profiling(True)
        for _ in range(args.reps):
            if not args.no_flush:
                flush.fill_(1.0)
            R.render_into(poses, w.intrinsics, out["depth"], out["normal"], out["color"], out["mask"])
        torch.cuda.synchronize()
        R.set_profiling(False)
        kt = R.kernel_times()
        ms = kt["raycast_ms"] / kt["raycast_launches"]
        pre_ms = kt["range_ms"] / max(kt["range_launches"], 1)  # range pass + tile order
        strips = {}
        for sp in (STRIPS.get(name, "") if args.strips else "").split(","):
            if not sp:
                continue
            r0, r1 = map(int, sp.split(":"))
            so = R.render(poses, w.intrinsics, row0=r0, row1=r1)
            for _ in range(3):
                R.render_into(poses, w.intrinsics, so["depth"], so["normal"], so["color"], so["mask"], row0=r0, row1=r1)
            torch.cuda.synchronize()
            R.reset_kernel_times()
            R.set_profiling(True)
            for _ in range(20):
                if not args.no_flush:
                    flush.fill_(1.0)
                R.render_into(poses, w.intrinsics, so["depth"], so["normal"], so["color"], so["mask"], row0=r0, row1=r1)
            torch.cuda.synchronize()
            R.set_profiling(False)
            kt2 = R.kernel_times()
            strips[sp] = round(kt2["raycast_ms"] / kt2["raycast_launches"], 4)
        st = {}
        if not args.no_parity:
            ora = oracle.OracleVolume(w.volume).render(w.poses[0], w.intrinsics)
            st = compare({k: v[0].cpu().numpy() for k, v in out.items()}, ora)
        import hashlib
        h = hashlib.sha1()
        for k in ("depth", "normal", "color", "mask"):
            h.update(out[k].cpu().numpy().tobytes())
        print(json.dumps({"variant": args.name, "config": name, "l2": "warm" if args.no_flush else "flushed",
                          "out_sha1": h.hexdigest()[:16],
                          "options": args.set,
                          "raycast_ms": round(ms, 4), "range_order_ms": round(pre_ms, 4),
                          **({"strips_alone_ms": strips} if strips else {}),
                          "budget_used": st.get("budget_used"), "color_exact": st.get("color_exact"),
                          "depth_max": st.get("depth_max_err"), "hit_disagree": st.get("hit_disagree"),
                          "geom_bad": st.get("geom_out_of_tol")}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", action="append", default=[], help="name:-DFOO -DBAR=1")
    ap.add_argument("--configs", default="C1,C2")
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-flush", action="store_true", help="keep L2 warm between launches (an upper bound)")
    ap.add_argument("--run", action="store_true")
    ap.add_argument("--strips", action="store_true", help="also time the slow-tile row strips alone")
    ap.add_argument("--set", action="append", default=[], help="dtsdf_set_option for the --run process: opt=value")
    ap.add_argument("--name", default="")
    args = ap.parse_args()
    if args.run:
        return run_one(args)
    from paper_2301_12796_b200 import build as B
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    libs = []
    name_opts = {}
    for v in args.variant or ["base:"]:
        name, _, defs = v.partition(":")
        if "|" in defs:  # name:defines|opt=value,opt=value -> runtime options too
            defs, _, opts = defs.partition("|")
            name_opts[name] = [o for o in opts.split(",") if o]
        if defs.startswith("@"):  # a prebuilt library (e.g. an earlier build kept under gpurun_out/)
            libs.append((name, os.path.abspath(defs[1:])))
            continue
        lib = os.path.join(ROOT, "gpurun_out", f"ab_{name}.so")
        cus = sorted(os.path.join(B.CSRC, f) for f in os.listdir(B.CSRC) if f.endswith(".cu"))
        cmd = [B.NVCC, *B.NVCC_FLAGS, *defs.split(), *cus, "-o", lib]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode:
            sys.exit(res.stdout + res.stderr)
        regs = [ln.strip() for ln in (res.stdout + res.stderr).splitlines() if "registers" in ln]
        print(json.dumps({"variant": name, "defines": defs, "ptxas": regs[:2]}), flush=True)
        libs.append((name, lib))
    for r in range(args.rounds):
        for name, lib in libs:
            env = dict(os.environ, DTSDF_LIB=lib)
            cmd = [sys.executable, os.path.abspath(__file__), "--run", "--name", name, "--configs", args.configs,
                   "--reps", str(args.reps)] + (["--no-parity"] if args.no_parity or r > 0 else []) + \
                  (["--no-flush"] if args.no_flush else []) + (["--strips"] if args.strips else []) + sum((["--set", o] for o in name_opts.get(name, [])), [])
            subprocess.run(cmd, env=env, check=True)


if __name__ == "__main__":
    main()
