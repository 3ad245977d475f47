"""Per-kernel durations of the last fused frame in an ncu launch list (--metrics gpu__time_duration.sum
--csv) of tools/bench_fusion.py: python tools/ncu_frame.py launches.csv"""
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
i = [j for j, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[i:]))
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
ks = [(r[ki].split("(")[0], float(r[vi])) for r in rows[1:]]
fp = [j for j, (n, _) in enumerate(ks) if n.startswith("k_frame_points") or n.startswith("k_fuse_alloc")]
tot = 0.0
for n, v in ks[fp[-2]:fp[-1]]:
    print(f"{n:36s} {v / 1000:8.1f} us")
    tot += v
print(f"{'frame total':36s} {tot / 1000:8.1f} us")
