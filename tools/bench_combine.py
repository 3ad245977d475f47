"""Time the combined-TSDF precompute (NEXT-1) on a config: dtsdf_combine at the config's first
pose, repeated, with the library's per-kind kernel timing (CUDA events on the stream).

    python tools/bench_combine.py [C1] [--mode 0|1] [--reps 20]"""
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
ap.add_argument("config", nargs="?", default="C1")
ap.add_argument("--mode", type=int, default=0)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
w = scenes.CONFIGS[a.config]()
R = Renderer(0)
R.upload_volume(w.volume)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for _ in range(3):
    R.combine(w.poses[0], w.intrinsics, mode=a.mode)
torch.cuda.synchronize()
R.reset_kernel_times()
R.set_profiling(True)
for _ in range(a.reps):
    flush.fill_(1.0)
    R.combine(w.poses[0], w.intrinsics, mode=a.mode)
torch.cuda.synchronize()
R.set_profiling(False)
kt = R.kernel_times()
# checksum of the combined TSDF in location order (the slot order depends on an atomic counter)
import hashlib  # noqa: E402
g = R.get_combined()
locs = np.asarray(g["locs"]).reshape(-1, 3)
order = np.lexsort((locs[:, 2], locs[:, 1], locs[:, 0]))
h = hashlib.sha1(locs[order].tobytes())
for k in ("sdf", "weight", "rgb", "mask"):
    h.update(np.ascontiguousarray(np.asarray(g[k])[order]).tobytes())
print(json.dumps({"config": a.config, "mode": a.mode, "combine_ms": kt["combine_ms"] / a.reps, "sha1": h.hexdigest()[:16],
                  "locations": R.combined_stats()["n_locations"], "l2": "flushed (256 MiB write) before each combine"}))
