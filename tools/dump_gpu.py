"""Render configs on the GPU and save the outputs (gpurun_out/gpu_<cfg>.npz) for offline analysis."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import scenes  # noqa: E402
from paper_2301_12796_b200 import Renderer  # noqa: E402

R = Renderer(0)
for name in sys.argv[1:] or ["C1"]:
    w = scenes.CONFIGS[name]()
    R.upload_volume(w.volume)
    n = 2 if name == "C2" else 1
    g = R.render(w.poses[:n], w.intrinsics)
    np.savez_compressed(os.path.join(ROOT, "gpurun_out", f"gpu_{name}.npz"), **{k: v.cpu().numpy() for k, v in g.items()})
    print("saved", name)
