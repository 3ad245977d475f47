"""k_raycast on row strips of one view, alone: how long the slow warp tiles take without the rest of
the frame contending for the SMs (the whole-view span vs the span of the strips holding its slowest
warp tiles).

    python tools/isolate.py [C1] [--strips 64:72,224:232,0:8]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import scenes  # noqa: E402
from paper_2301_12796_b200 import Renderer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", nargs="?", default="C1")
ap.add_argument("--strips", default="64:72,224:232,40:48,0:8,240:248")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()

R = Renderer(0)
w = scenes.CONFIGS[a.config]()
R.upload_volume(w.volume)
poses = np.asarray(w.poses[:1], np.float32)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def timed(r0, r1):
    out = R.render(poses, w.intrinsics, row0=r0, row1=r1)
    for _ in range(3):
        R.render_into(poses, w.intrinsics, out["depth"], out["normal"], out["color"], out["mask"], row0=r0, row1=r1)
    torch.cuda.synchronize()
    R.reset_kernel_times()
    R.set_profiling(True)
    for _ in range(a.reps):
        flush.fill_(1.0)
        R.render_into(poses, w.intrinsics, out["depth"], out["normal"], out["color"], out["mask"], row0=r0, row1=r1)
    torch.cuda.synchronize()
    R.set_profiling(False)
    kt = R.kernel_times()
    return 1e3 * kt["raycast_ms"] / kt["raycast_launches"]


H = w.intrinsics.height
print(f"{a.config} whole view rows 0:{H}: k_raycast {timed(0, H):.1f} us")
for s in a.strips.split(","):
    r0, r1 = map(int, s.split(":"))
    print(f"{a.config} strip rows {r0}:{r1} alone: k_raycast {timed(r0, r1):.1f} us")
