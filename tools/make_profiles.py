"""Copy the judged evidence of one GPU pass from gpurun_out/ into profiles/ (tracked).

    python tools/make_profiles.py <tag> [--config C1]

Writes profiles/<tag>_ncu_k_raycast.txt (key `ncu --set full` metrics of one k_raycast launch),
profiles/<tag>_launches.txt (per-kernel shares of the `gpu__time_duration.sum` launch list),
profiles/<tag>_bench.jsonl (bench lines of that pass) and merges the raycast DRAM bytes per
launch into profiles/ncu_summary.json, which bench.py reads for roofline.traffic.
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from ncu_summary import summary  # noqa: E402

OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    unit = rows[hi + 1][ui]
    for r in rows[hi + 1:]:
        agg[r[ki]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold cache, serialised; unit {unit})",
             f"{'kernel':70s} {'launches':>8s} {'mean':>12s} {'share':>7s}"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{k[:70]:70s} {len(v):8d} {sum(v) / len(v):12.1f} {sum(v) / tot:7.3f}")
    return "\n".join(lines) + "\n"


def main():
    tag = sys.argv[1]
    cfg = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else "C1"
    os.makedirs(PROF, exist_ok=True)
    rep = os.path.join(OUT, f"prof_{tag}.ncu-rep")
    if os.path.exists(rep):
        s = summary(rep)
        with open(os.path.join(PROF, f"{tag}_ncu_k_raycast.txt"), "w") as fh:
            fh.write(f"# ncu --set full --clock-control none -k regex:k_raycast -s 5 -c 1, workload {cfg}\n")
            for k, v in s.items():
                fh.write(f"{k:60s} {v}\n")
        rd = float(s.get("dram__bytes_read.sum [Mbyte]", "nan")) * 1e6 if "dram__bytes_read.sum [Mbyte]" in s else None
        wk = [k for k in s if k.startswith("dram__bytes_write.sum")]
        wr = None
        if wk:
            unit = wk[0].split("[")[1].rstrip("]")
            wr = float(s[wk[0]]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
        rk = [k for k in s if k.startswith("dram__bytes_read.sum")]
        if rk:
            unit = rk[0].split("[")[1].rstrip("]")
            rd = float(s[rk[0]]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
        path = os.path.join(PROF, "ncu_summary.json")
        js = json.load(open(path)) if os.path.exists(path) else {}
        ins = s.get("Executed Instructions [inst]")
        js[cfg] = {"raycast_dram_bytes_per_launch": (rd or 0) + (wr or 0), "source": f"profiles/{tag}_ncu_k_raycast.txt",
                   "duration_us": float(s.get("Duration [us]", "nan")),
                   "raycast_warp_insts_per_launch": float(ins.replace(",", "")) if ins else None}
        for key, name in (("raycast_l1_load_sectors_per_launch", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum"),
                          ("raycast_l2_sectors_per_launch", "lts__t_sectors.sum"),
                          ("raycast_l1_wavefronts_pct_of_peak", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed")):
            k = [x for x in s if x.startswith(name + " ")]
            if k:
                js[cfg][key] = float(s[k[0]].replace(",", ""))
        json.dump(js, open(path, "w"), indent=1)
    lc = os.path.join(OUT, f"launches_{tag}.csv")
    if os.path.exists(lc):
        open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write(launch_shares(lc))
    lines = []
    for name in (f"bench_{tag}.log", f"bench_ref_{tag}.log"):
        p = os.path.join(OUT, name)
        if os.path.exists(p):
            lines += [ln for ln in open(p).read().splitlines() if ln.startswith("{")]
    if lines:
        open(os.path.join(PROF, f"{tag}_bench.jsonl"), "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
