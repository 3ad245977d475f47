#!/usr/bin/env python
"""Benchmark of the DTSDF raycast hot path (BASELINE.json metric on configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dtsdf|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

With --gpus N > 1 and no torch.distributed environment (WORLD_SIZE unset) the script re-executes
itself under torch.distributed.run with N processes; a world size other than --gpus is an error.

One step = every rank renders one 640x480 depth+normal+colour+dirmask view of the configs[1]
room volume (seeded synthetic) through dtsdf_render_batch; per-GPU work is fixed
(weak scaling).  The volume is generated on rank 0, replicated by one NCCL broadcast per buffer
into the library-owned buffers and committed on every rank before timing.  L2 is flushed
(256 MiB write) between timed steps; each step is timed with CUDA events on the render stream,
and the job time is the max over ranks.  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "Mrays/s"
FLUSH_BYTES = 256 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["dtsdf", "reference"], default="dtsdf")
    ap.add_argument("--config", choices=["C0", "C1", "C2", "C3", "C4"], default="C1",
                    help="C1 is the bench workload (BASELINE.json metric); the others are for profiling")
    ap.add_argument("--views", type=int, default=1,
                    help="views per rank per step, taken round-robin from the config's poses "
                         "(1 = the configs[1] workload)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle time for cpu_baseline")
    ap.add_argument("--e2e-steps", type=int, default=100)
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--mode", choices=["direct", "combined"], default="direct",
                    help="direct: per-sample combination (the north-star path); combined: the paper's "
                         "view-dependent combined TSDF (NEXT-1), recombined per eqs. 10-13 inside the timed loop")
    ap.add_argument("--dist", action="store_true",
                    help="run the multi-GPU code path (NCCL process group, volume broadcast into library buffers, "
                         "checksum all-gather, max over ranks) even at world size 1")
    ap.add_argument("--shard", choices=["none", "views", "rows"], default="none",
                    help="none: every rank renders its own --views views (weak scaling, the default); views: the "
                         "--views views of one batch are split into contiguous ranges per rank (SURVEY §8(e), C3); "
                         "rows: every view's rows are split per rank via row0/row1 (C4's large view) -- strong scaling")
    ap.add_argument("--combine-mode", type=int, default=0, choices=[0, 1],
                    help="combined mode: 0 eq:combine_weight (the paper's method), 1 Algorithm 1 (NEXT-4)")
    ap.add_argument("--boxes", type=int, default=20,
                    help="C1 only: boxes in the room (20 = configs[1]; more approach configs[1]'s ~40k blocks, R30)")
    ap.add_argument("--batch-views", type=int, default=256,
                    help="views of the strong-scaling C3 batch timed after the headline (SURVEY §8(e)); 0 = skip")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check without kernels: every rank joins a gloo process group and reports; "
                         "rank 0 prints the ranks it saw")
    return ap.parse_args()


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(args) -> int:
    """--gpus N > 1 without a torch.distributed environment: run this script under
    torch.distributed.run with N processes on this node (one per GPU), same arguments."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def dry_run(args) -> int:
    """Launcher check (CPU, gloo): each rank reports (rank, world, pid); rank 0 prints them."""
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", str(free_port()))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seen = [None] * world
    dist.all_gather_object(seen, {"rank": rank, "world": world, "pid": os.getpid(),
                                  "local_rank": int(os.environ.get("LOCAL_RANK", "0"))})
    if rank == 0:
        print(json.dumps({"dry_run": True, "impl": args.impl, "n_gpus": world, "ranks": seen,
                          "comm": {"backend": dist.get_backend(), "world_size": dist.get_world_size()}}), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    return 0


def workload(name, boxes=20):
    import scenes
    if name == "C1" and boxes != 20:  # sensitivity to the block count (reading R30: configs[1] says ~40k)
        return scenes.c1_room(n_boxes=boxes)
    if name == "C0":
        return scenes.c0_sphere()
    if name == "C2":
        return scenes.c2_thin()
    if name == "C3":
        return scenes.c3_batch()
    if name == "C4":
        return scenes.c4_large()
    return scenes.c1_room()


def describe(w, views, boxes=20):
    K = w.intrinsics
    return {"workload": f"{w.name}: " + {
        "C1": f"room scale, {boxes} seeded boxes on a 4x4 m floor, 1 cm voxels, tau 4 cm, one 640x480 view at the "
              "seeded pose (fx=fy=525, cx=319.5, cy=239.5)",
        "C0": "dense sphere r=0.2 m, 64^3 voxels at 1 cm, 80x60 view",
        "C2": "200 thin plates, 5 mm voxels, 640x480 views",
        "C3": "configs[1] volume, orbit views",
        "C4": "8x8x3 m room of seeded boxes, cylinders and thin plates, 5 mm voxels, tau 2 cm, orbit views"}[w.name],
        "width": K.width, "height": K.height, "views_per_step_per_gpu": views,
        "n_blocks": int(w.volume.n_blocks if w.volume is not None else w.extra["n_blocks"]), "theta_deg": 65.0, "outputs": "depth+normal+color+dirmask",
        "l2": "flushed between timed steps (256 MiB write)"}


# ------------------------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"unavailable": "nvidia-smi not runnable"}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = [[c.strip() for c in ln.split(",")] for ln in self.lines if ln.count(",") >= 6]
        if not rows:
            return {"unavailable": "no samples"}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------------------------------
# reference arm: the CPU oracle (TEST INFRASTRUCTURE, the one other place bench may run it)
# ------------------------------------------------------------------------------------------
def oracle_sample_rate(w, n_pix, seed=0, threads=None):
    import oracle
    K = w.intrinsics
    rng = np.random.default_rng(seed)
    idx = rng.choice(K.width * K.height, size=min(n_pix, K.width * K.height), replace=False)
    px = np.stack([idx % K.width, idx // K.width], 1).astype(np.int32)
    ov = oracle.OracleVolume(w.volume)
    t0 = time.perf_counter()
    out = ov.render(w.poses[0], K, pixels=px, threads=threads)
    dt = time.perf_counter() - t0
    return len(px), dt, px, out


def cpu_baseline(w, seconds):
    """The oracle as it stands on all host cores: a seeded pixel subset sized for `seconds` of CPU
    work; when one whole frame takes less, the frame is traced again (same pixels, same result)
    until `seconds` have passed, so the rate is measured over ~10-30 s as the contract asks."""
    import oracle
    threads = os.cpu_count() or 1
    n0, dt0, _, _ = oracle_sample_rate(w, 2048, seed=1, threads=threads)
    n = int(min(w.intrinsics.width * w.intrinsics.height, max(2048, n0 * seconds / max(dt0, 1e-3))))
    n, dt, px, out = oracle_sample_rate(w, n, seed=2, threads=threads)
    passes, tot = 1, dt
    ov = oracle.OracleVolume(w.volume)
    while tot < seconds and passes < 64:
        t0 = time.perf_counter()
        ov.render(w.poses[0], w.intrinsics, pixels=px, threads=threads)
        tot += time.perf_counter() - t0
        passes += 1
    return {"value": n * passes / tot / 1e6, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{n} of {w.intrinsics.width * w.intrinsics.height} pixel rays of the {w.name} view "
                      f"(seeded uniform subset) x {passes} pass(es), fp64 brute-force march, {tot:.1f} s"}, px, out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = workload(args.config, args.boxes)
    threads = os.cpu_count() or 1
    n0, dt0, _, _ = oracle_sample_rate(w, 1024, seed=1, threads=threads)
    rate = n0 / max(dt0, 1e-3)
    per_step = min(2.0, 150.0 / max(args.steps + args.warmup, 1))
    n = int(min(w.intrinsics.width * w.intrinsics.height, max(256, rate * per_step)))
    for i in range(args.warmup):
        oracle_sample_rate(w, n, seed=100 + i, threads=threads)
    tot = 0.0
    for i in range(args.steps):
        _, dt, _, _ = oracle_sample_rate(w, n, seed=1000 + i, threads=threads)
        tot += dt
    value = n * args.steps / tot / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(describe(w, args.views, args.boxes), mode=args.mode),  # the product arm's config keys
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"each step: {n} of {w.intrinsics.width * w.intrinsics.height} pixel rays "
                                       f"of the {w.name} view (seeded uniform subset)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------
# the product arm
# ------------------------------------------------------------------------------------------
def load_json(path):
    try:
        return json.load(open(path))
    except Exception:
        return None


def run_dtsdf(args):
    import torch
    import torch.distributed as dist

    from paper_2301_12796_b200 import Renderer
    from paper_2301_12796_b200 import dist as pdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the product path has no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    use_dist = world > 1 or args.dist
    if use_dist:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=dev)
    w = workload(args.config, args.boxes) if rank == 0 else None
    R = Renderer(local)
    stream = torch.cuda.current_stream()

    # ---- replicate the volume: rank 0 fills its buffers, NCCL broadcast into the others' ----
    t_up = time.perf_counter()
    if use_dist:
        meta = None
        if rank == 0:
            v = w.volume
            meta = {"n_blocks": v.n_blocks, "voxel_size": v.voxel_size, "truncation": v.truncation,
                    "theta": v.theta, "step": v.step}
        meta = pdist.broadcast_volume_meta(dist, meta, dev)
        bufs = R.alloc(meta["voxel_size"], meta["truncation"], meta["theta"], meta["n_blocks"], meta["step"])
        if rank == 0:
            for k, t in pdist.volume_arrays_to_tensors(w.volume).items():
                bufs[k].copy_(t)
        torch.cuda.synchronize()
        dist.barrier()
        tb = time.perf_counter()
        pdist.broadcast_buffers(dist, bufs)
        torch.cuda.synchronize()
        bcast_ms = 1e3 * (time.perf_counter() - tb)
        cs = pdist.checksum(bufs)
        sums = [None] * world
        dist.all_gather_object(sums, cs)
        if len(set(sums)) != 1:
            raise SystemExit(f"volume replicas differ after broadcast: {sums}")
        R.commit(stream)
        # the rest of the workload (name, poses, intrinsics) travels as a small object
        objs = [dataclasses.replace(w, volume=None, patches=None,
                                    extra=dict(w.extra or {}, n_blocks=w.volume.n_blocks)) if rank == 0 else None]
        dist.broadcast_object_list(objs, 0)
        if rank != 0:
            w = objs[0]
    else:
        bcast_ms = 0.0
        R.upload_volume(w.volume)
    upload_ms = 1e3 * (time.perf_counter() - t_up)
    K = w.intrinsics
    # this rank's views: round-robin over the config's poses (configs[1] has one).  Weak scaling:
    # every rank renders its own --views views; --shard views / rows split one batch (strong scaling)
    row0, row1 = 0, K.height
    if args.shard == "views":
        if args.views < world:
            raise SystemExit("--shard views needs at least one view per rank")
        lo, hi = pdist.shard_range(args.views, rank, world)
        idx = [i % len(w.poses) for i in range(lo, hi)]
        total_rays = K.width * K.height * args.views
    elif args.shard == "rows":
        idx = [i % len(w.poses) for i in range(args.views)]
        row0, row1 = pdist.shard_range(K.height, rank, world)
        total_rays = K.width * K.height * args.views
    else:
        idx = [(rank * args.views + i) % len(w.poses) for i in range(args.views)]
        total_rays = world * K.width * K.height * args.views
    poses = np.ascontiguousarray(np.asarray(w.poses, np.float32)[idx])
    rays_per_step = K.width * (row1 - row0) * len(idx)  # this rank's
    out = R.render(poses, K, row0=row0, row1=row1)
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    # combined mode (NEXT-1): every view is one frame of a sequence; before rendering it the
    # recombination conditions (eqs. 10-13) decide whether the combined TSDF is
    # recomputed at its pose.  The state runs on across warm-up and timed steps.
    from paper_2301_12796_b200.dtsdf import should_recombine
    seq = {"frame": 0, "last": 0, "last_pose": None, "combines": 0}

    def step(d, n, c, m, host=False):
        if args.mode == "direct":
            R.render_into(poses, K, d, n, c, m, row0=row0, row1=row1, stream=stream)
            return
        for i in range(len(poses)):
            f = seq["frame"]
            if seq["last_pose"] is None or should_recombine(f, seq["last"], poses[i], seq["last_pose"]):
                R.combine(poses[i], K, stream=stream, mode=args.combine_mode)
                seq["last"], seq["last_pose"] = f, poses[i]
                seq["combines"] += 1
            sl = slice(i, i + 1)
            R.render_combined_into(poses[sl], K, d[sl], n[sl], c[sl], m[sl], row0=row0, row1=row1, stream=stream)
            seq["frame"] = f + 1

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        if not args.no_flush:
            flush.fill_(1.0)
        step(out["depth"], out["normal"], out["color"], out["mask"])
    torch.cuda.synchronize()
    R.reset_kernel_times()
    R.set_profiling(True)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    n_launch0 = R.launch_count()
    combines0 = seq["combines"]
    for i in range(args.steps):
        if not args.no_flush:
            flush.fill_(1.0)
        starts[i].record(stream)
        step(out["depth"], out["normal"], out["color"], out["mask"])
        ends[i].record(stream)
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    launches = R.launch_count() - n_launch0
    combines = seq["combines"] - combines0
    # the shards are checked against each other -- ranks that rendered the same poses
    # (configs[1] has one) must produce bit-identical outputs; a 64-bit checksum per rank is gathered
    out_sum = pdist.checksum({"keys": out["depth"], "sdf": out["normal"], "weight": out["color"], "rgb": out["mask"]})
    if use_dist:
        sums = [None] * world
        mine = ([int(i) for i in idx], row0, row1)
        dist.all_gather_object(sums, (out_sum, mine))
        same = [s for s, v in sums if v == mine]
        replicas_equal = len(set(same)) == 1
    else:
        replicas_equal = None
    clk = clocks.stop()
    R.set_profiling(False)
    kt = R.kernel_times()
    total_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    max_ms = pdist.max_over_ranks(dist, total_ms, dev) if use_dist else total_ms
    value = total_rays * args.steps / (max_ms / 1e3) / 1e6

    # ---- roofline of the dominant kernel (raycast) ----
    ray_ms = kt["raycast_ms"] / max(kt["raycast_launches"], 1)
    balg = load_json(os.path.join(ROOT, "profiles", "b_alg.json")) or {}
    b_ray = balg.get(w.name, {}).get("bytes_per_ray") if args.mode == "direct" else None
    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json")) or {}
    peak = peaks.get("hbm_gbs", 6650.0)
    ncu = load_json(os.path.join(ROOT, "profiles", "ncu_summary.json")) or {}
    traffic = ncu.get(w.name, {}).get("raycast_dram_bytes_per_launch") if args.mode == "direct" else None
    achieved = (b_ray * rays_per_step / (ray_ms / 1e3) / 1e9) if b_ray else None
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": (achieved / peak) if achieved else None, "traffic": traffic,
            "kernel": "k_raycast", "kernel_ms": ray_ms, "bytes_per_ray_alg": b_ray,
            "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)" if "hbm_gbs" in peaks else "fallback 6.65 TB/s",
            "range_pass_ms": kt["range_ms"] / max(kt["range_launches"], 1),  # k_range + k_order
            "range_pass_note": "range pass + tile order (k_range_*, k_order), per launch"}
    # what actually bounds k_raycast: instruction issue.  Warp instructions per launch
    # from the committed ncu capture of this config (a property of the workload), divided by this
    # run's live kernel time, against 148 SMs x 4 schedulers x 1 instruction per clock.
    ins = ncu.get(w.name, {}).get("raycast_warp_insts_per_launch") if args.mode == "direct" and args.views == 1 else None
    if ins:
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        mhz = (clk.get("sm_mhz") if isinstance(clk, dict) else None) or 1965.0
        ach = ins / (ray_ms / 1e3) / 1e12
        pk = sms * 4 * mhz * 1e6 / 1e12
        roof["issue"] = {"achieved": ach, "peak": pk, "unit": "Tinst/s (warp instructions)", "frac": ach / pk,
                         "insts_per_launch": ins, "source": ncu.get(w.name, {}).get("source")}
    # the on-chip side: L1 load demand of one launch (sectors from the committed capture of this config)
    # over this run's live kernel time, and the L1 wavefront utilisation ncu measured
    ncu_c = ncu.get(w.name, {}) if args.mode == "direct" and args.views == 1 else {}
    if ncu_c.get("raycast_l1_load_sectors_per_launch"):
        dem = ncu_c["raycast_l1_load_sectors_per_launch"] * 32.0
        roof["l1"] = {"demand_bytes_per_launch": dem, "demand_bytes_per_ray": dem / rays_per_step,
                      "achieved_TBps": dem / (ray_ms / 1e3) / 1e12,
                      "l2_bytes_per_launch": (ncu_c.get("raycast_l2_sectors_per_launch") or 0) * 32.0,
                      "wavefront_pct_of_peak": ncu_c.get("raycast_l1_wavefronts_pct_of_peak"),
                      "source": ncu_c.get("source")}
    if args.mode == "combined":
        roof["combine_ms_per_step"] = kt["combine_ms"] / args.steps
        roof["recombinations_per_step"] = combines / args.steps

    # ---- end to end through the C ABI with pinned HOST outputs (copies inside the timing) ----
    H, W = row1 - row0, K.width  # this rank's share
    V = len(idx)
    hd = torch.empty((V, H, W), dtype=torch.float32).pin_memory()
    hn = torch.empty((V, H, W, 3), dtype=torch.float32).pin_memory()
    hc = torch.empty((V, H, W, 3), dtype=torch.uint8).pin_memory()
    hm = torch.empty((V, H, W), dtype=torch.uint8).pin_memory()
    pose_host = torch.from_numpy(np.ascontiguousarray(poses)).pin_memory()
    e2e_steps = min(args.e2e_steps, args.steps)

    def e2e_run():
        for _ in range(3):
            step(hd, hn, hc, hm)
        tot = 0.0
        if use_dist:
            dist.barrier()
        for _ in range(e2e_steps):
            if not args.no_flush:
                flush.fill_(1.0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            step(hd, hn, hc, hm)  # synchronizes (host outputs)
            tot += time.perf_counter() - t0
        return pdist.max_over_ranks(dist, tot, dev) if use_dist else tot

    from paper_2301_12796_b200.dtsdf import OPT_HOST_WRITE
    R.set_option(OPT_HOST_WRITE, 0)  # context: render into device scratch, then copy engine D2H
    e2e_copy = e2e_run()
    R.set_option(OPT_HOST_WRITE, 1)  # default: the kernel writes the pinned outputs directly
    e2e_max = e2e_run()
    e2e = {"value": total_rays * e2e_steps / e2e_max / 1e6, "unit": UNIT,
           "h2d_bytes_per_step": int(pose_host.numel() * 4 + 32),
           "d2h_bytes_per_step": int(hd.numel() * 4 + hn.numel() * 4 + hc.numel() + hm.numel()),
           "timing": "host wall clock per dtsdf_render_batch call into pinned host outputs, written by the "
                     "raycast across the host link (DTSDF_OPT_HOST_WRITE)",
           "copy_path_value": total_rays * e2e_steps / e2e_copy / 1e6}

    # ---- SURVEY §8(e) strong scaling: the configs[3] batch (orbit views of this volume) split into
    # contiguous per-rank view ranges, timed like the headline (events, flushed L2, max over ranks) ----
    c3 = None
    if args.batch_views > 0 and w.name == "C1" and args.mode == "direct" and args.shard == "none":
        import scenes
        allp = scenes.orbit_poses(np.random.default_rng([3, 0]), args.batch_views)  # c3_batch's poses
        lo, hi = pdist.shard_range(args.batch_views, rank, world)
        bp = np.ascontiguousarray(np.asarray(allp, np.float32)[lo:hi])
        bo = R.render(bp, K) if hi > lo else None
        c3_steps = 5
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(c3_steps)]
        for i in range(2 + c3_steps):
            if not args.no_flush:
                flush.fill_(1.0)
            if i >= 2:
                ev[i - 2][0].record(stream)
            if bo is not None:
                R.render_into(bp, K, bo["depth"], bo["normal"], bo["color"], bo["mask"], stream=stream)
            if i >= 2:
                ev[i - 2][1].record(stream)
        torch.cuda.synchronize()
        c3_ms = sum(a.elapsed_time(b) for a, b in ev)
        c3_max = pdist.max_over_ranks(dist, c3_ms, dev) if use_dist else c3_ms
        c3 = {"workload": f"C3: the {args.batch_views} configs[3] orbit views of this volume, split into contiguous "
                          f"per-rank view ranges (strong scaling)", "views": args.batch_views,
              "views_this_rank": hi - lo, "value": K.width * K.height * args.batch_views * c3_steps / (c3_max / 1e3) / 1e6,
              "unit": UNIT, "ms_per_batch": c3_max / c3_steps, "steps": c3_steps, "scaling": "strong"}
        del bo

    if rank != 0:
        dist.barrier() if use_dist else None
        dist.destroy_process_group() if use_dist else None
        return 0

    # ---- CPU oracle baseline (rank 0, N = 1 only) + a sampled parity check of this run ----
    cpu = None
    parity = None
    if world == 1 and not args.no_cpu_baseline and args.mode == "direct":
        cpu, px, ora = cpu_baseline(w, args.cpu_seconds)
        g = {k: v[0].cpu().numpy()[px[:, 1], px[:, 0]] for k, v in out.items()}
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from parity import compare
        parity = compare(g, ora)
    st = R.stats()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if args.shard == "none" else "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded scene, DESIGN.md §3)",
        "config": dict(describe(w, args.views, args.boxes), mode=args.mode,
                       **({"combine_mode": args.combine_mode} if args.mode == "combined" else {}),
                       **({"shard": args.shard, "views_per_step_total": args.views,
                           "views_per_step_per_gpu": len(idx), "rows_per_gpu": row1 - row0}
                          if args.shard != "none" else {})),
        "frames_per_s": total_rays / (K.width * K.height) * args.steps / (max_ms / 1e3),
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
        "clocks": clk,
        "comm": ({"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                  "nccl_version": ".".join(str(x) for x in torch.cuda.nccl.version())} if use_dist else
                 {"backend": None, "world_size": 1, "note": "single process, no process group"}),
        "extra": {"c3_strong_scaling": c3, "upload_and_index_ms": upload_ms, "broadcast_ms": bcast_ms, "n_locations": st["n_locations"],
                  "output_checksum": out_sum, "ranks_with_same_views_bit_identical": replicas_equal,
                  "device_bytes": st["bytes"], "parity_sample_vs_oracle": parity,
                  "device": torch.cuda.get_device_name(dev)},
    }
    print(json.dumps(line), flush=True)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.gpus < 1:
        raise SystemExit("bench.py: --gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but the process group has {world} ranks", file=sys.stderr, flush=True)
        return 2
    if args.dry_run:
        return dry_run(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_dtsdf(args)


if __name__ == "__main__":
    sys.exit(main())
