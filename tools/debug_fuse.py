"""Debug helper: C1 room fused from 6 frames, GPU volume -> gpurun_out/fuse_dbg.npz."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import scenes  # noqa
from paper_2301_12796_b200 import Renderer  # noqa
K = scenes.Intrinsics(fx=262.5, fy=262.5, cx=159.5, cy=119.5, width=320, height=240)
w = scenes.c1_room()
poses = scenes.room_scan_poses(np.random.default_rng([7, 0]), 6)
R = Renderer(0)
R.upload(0.01, 0.04, scenes.THETA, np.zeros((0, 4), np.int32), np.zeros((0, 512), np.float32), np.zeros((0, 512), np.float32))
R.fusion_reserve(60000)
for P in poses:
    fr = scenes.analytic_frame(w.patches, P, K)
    R.fuse(fr.depth, fr.normal, fr.color, P, K)
k, s, wt, c = R.get_volume()
np.savez(os.path.join(ROOT, "gpurun_out", "fuse_dbg.npz"), k=k, s=s, w=wt, c=c)
print("ok", len(k))
