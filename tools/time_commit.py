import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, scenes
from paper_2301_12796_b200 import Renderer
w = scenes.c1_room()
R = Renderer(0)
R.upload_volume(w.volume)
R.fusion_reserve(80000)
for _ in range(3): R.commit()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20): R.commit()
print("commit ms", (time.perf_counter() - t) / 20 * 1e3)
fr = scenes.analytic_frame(w.patches, w.poses[0], w.intrinsics)
d = {k: torch.from_numpy(getattr(fr, k)).cuda() for k in ("depth", "normal", "color")}
for _ in range(3): R.fuse(d["depth"], d["normal"], d["color"], w.poses[0], w.intrinsics)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20): R.fuse(d["depth"], d["normal"], d["color"], w.poses[0], w.intrinsics)
print("fuse ms", (time.perf_counter() - t) / 20 * 1e3)
