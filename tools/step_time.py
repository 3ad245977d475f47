"""Whole-step time of dtsdf_render_batch (range pass + tile order + raycast) with CUDA events around
each call and the library's own tracing OFF (its per-kernel events would sit between the launches).

    DTSDF_LIB=... python tools/step_time.py [--configs C1,C2] [--reps 200]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import scenes  # noqa: E402
from paper_2301_12796_b200 import Renderer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C1,C2")
ap.add_argument("--reps", type=int, default=200)
ap.add_argument("--name", default=os.path.basename(os.environ.get("DTSDF_LIB", "libdtsdf.so")))
ap.add_argument("--views", type=int, default=1, help="views per call (round-robin over the config's poses)")
ap.add_argument("--set", action="append", default=[], help="dtsdf_set_option opt=value")
args = ap.parse_args()
R = Renderer(0)
for kv in args.set:
    o, v = kv.split("=")
    R.set_option(int(o), int(v))
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for name in args.configs.split(","):
    w = scenes.CONFIGS[name]()
    R.upload_volume(w.volume)
    poses = np.asarray(w.poses, np.float32)[[i % len(w.poses) for i in range(args.views)]]
    out = R.render(poses, w.intrinsics)
    ts = []
    for i in range(args.reps + 5):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        R.render_into(poses, w.intrinsics, out["depth"], out["normal"], out["color"], out["mask"])
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    ms = np.array([a.elapsed_time(b) for a, b in ts[5:]])
    print(json.dumps({"lib": args.name, "config": name, "views": args.views, "options": args.set,
                      "ms_per_view": round(float(ms.mean()) / args.views, 4),
                      "step_ms_mean": round(float(ms.mean()), 4),
                      "step_ms_median": round(float(np.median(ms)), 4)}), flush=True)
