"""Render one 16x8-pixel CTA tile of a view alone (intrinsics shifted so that the tile is a whole
16x8 image): the launch holds just that CTA's four warps, for ncu instruction / stall attribution of
the slowest tiles.

    python tools/one_tile.py C1 448 64 [reps]
"""
import dataclasses
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import scenes  # noqa: E402
from paper_2301_12796_b200 import Renderer  # noqa: E402

name, u0, v0 = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
w = scenes.CONFIGS[name]()
K = dataclasses.replace(w.intrinsics, cx=w.intrinsics.cx - u0, cy=w.intrinsics.cy - v0, width=16, height=8)
R = Renderer(0)
R.upload_volume(w.volume)
poses = np.asarray(w.poses[:1], np.float32)
full = R.render(poses, w.intrinsics)
for _ in range(reps):
    out = R.render(poses, K)
torch.cuda.synchronize()
same = torch.equal(out["depth"][0].cpu(), full["depth"][0, v0:v0 + 8, u0:u0 + 16].cpu())
R.reset_kernel_times()
R.set_profiling(True)
for _ in range(20):
    R.render(poses, K)
torch.cuda.synchronize()
kt = R.kernel_times()
print(f"{name} tile ({u0},{v0}) alone: k_raycast {1e3 * kt['raycast_ms'] / kt['raycast_launches']:.1f} us; "
      f"depth equal to the full view's: {same}")
