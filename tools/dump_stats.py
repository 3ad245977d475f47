"""Per-ray sample counts from the DTSDF_STATS debug build (normal channel = march/refine/skip)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DTSDF_LIB"] = os.path.join(ROOT, "paper_2301_12796_b200", "libdtsdf_stats.so")
import scenes  # noqa
from paper_2301_12796_b200 import Renderer  # noqa
R = Renderer(0)
for name in sys.argv[1:] or ["C1"]:
    w = scenes.CONFIGS[name]()
    R.upload_volume(w.volume)
    g = R.render(w.poses[:1], w.intrinsics)
    n = g["normal"][0].cpu().numpy().reshape(-1, 3)
    d = g["depth"][0].cpu().numpy().reshape(-1)
    hit = d > 0
    print(name, "rays", len(d), "hits", hit.sum())
    for i, nm in enumerate(["march_evals", "refine_evals", "skip_steps"]):
        print(f"  {nm}: mean {n[:, i].mean():.2f}  hit-mean {n[hit, i].mean():.2f}  miss-mean {n[~hit, i].mean():.2f} "
              f"p50 {np.median(n[:, i]):.0f} p99 {np.quantile(n[:, i], 0.99):.0f} max {n[:, i].max():.0f}")
