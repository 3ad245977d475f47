"""Aggregate an ncu source page (cuda,sass) by CUDA source line: instructions and samples."""
import csv
import sys
from collections import defaultdict


def f(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return 0.0


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur_file, h, line = None, None, None
    agg = defaultdict(lambda: [0.0, 0.0, ""])
    stall = defaultdict(float)
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            h = {k: j for j, k in enumerate(r)}
            continue
        if h is None or len(r) < 5:
            continue
        if r[0].strip():
            line = (cur_file, r[0])
            agg[line][2] = r[1][:100]
        agg[line][0] += f(r[h["Instructions Executed"]])
        agg[line][1] += f(r[h["# Samples"]])
        for k, j in h.items():
            if k.startswith("stall_") and "Not Issued" not in k:
                stall[k] += f(r[j])
    T = sum(v[0] for v in agg.values())
    S = sum(v[1] for v in agg.values())
    St = sum(stall.values())
    print(f"warp instructions {T:.3e}  samples {S:.0f}")
    print("stalls:", ", ".join(f"{k[6:]} {v / St * 100:.1f}%" for k, v in sorted(stall.items(), key=lambda kv: -kv[1])[:8]))
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{k[0][:10]}:{k[1]:<5} instr {v[0] / T * 100:5.1f}% samp {v[1] / S * 100:5.1f}%  {v[2]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
