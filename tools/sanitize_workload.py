"""Small workload touching every kernel of libdtsdf.so, for compute-sanitizer (SURVEY.md §4
memory-safety gate): index build, range pass + raycast (row shards, host outputs), combined TSDF (both modes) + its raycast, fusion (normals, allocation,
fusion, incremental and full re-commit), ICP."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import scenes  # noqa: E402
from paper_2301_12796_b200 import Renderer  # noqa: E402
from paper_2301_12796_b200.dtsdf import OPT_LOCATION_GRID  # noqa: E402

w = scenes.c0_sphere()
R = Renderer(0)
R.upload_volume(w.volume)
K = w.intrinsics
out = R.render(w.poses, K)
R.render(w.poses, K, row0=3, row1=41)
R.set_option(OPT_LOCATION_GRID, 0)
R.render(w.poses, K)
R.set_option(OPT_LOCATION_GRID, 1)
hd = np.zeros((1, K.height, K.width), np.float32)
R.render_into(w.poses, K, hd)
for mode in (0, 1):
    R.combine(w.poses[0], K, mode=mode)
    R.render(w.poses, K, combined=True)
    R.get_combined()
# fusion into the sphere volume from a room-like frame of two walls
c1 = scenes.c1_room()
Kc = scenes.Intrinsics(fx=65.6, fy=65.6, cx=39.5, cy=29.5, width=80, height=60)
R.fusion_reserve(w.volume.n_blocks + 4000)
fr = scenes.analytic_frame(c1.patches, c1.poses[0], Kc)
nrm = R.depth_normals(torch.from_numpy(fr.depth).cuda(), Kc)
R.fuse(fr.depth, fr.normal, fr.color, c1.poses[0], Kc)
R.render(c1.poses[:1], Kc)
ref = R.render(c1.poses[:1], Kc)
R.icp(torch.from_numpy(fr.depth).cuda(), ref["depth"][0], ref["normal"][0], c1.poses[0], Kc, max_iters=3,
      outlier=0.05, raise_singular=False)
torch.cuda.synchronize()
R.close()
print("sanitize workload done")
