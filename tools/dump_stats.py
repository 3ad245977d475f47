"""Per-ray counters of the DTSDF_STATS debug build (libdtsdf_stats.so): the normal channel holds
clock64 cycles (outside evaluations, march evaluations, refinement evaluations) and the colour
channel the counts (march evaluations, refinement evaluations, advance steps)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("DTSDF_LIB", os.path.join(ROOT, "paper_2301_12796_b200", "libdtsdf_stats.so"))
import scenes  # noqa: E402
from paper_2301_12796_b200 import Renderer  # noqa: E402

R = Renderer(0)
for name in sys.argv[1:] or ["C1"]:
    w = scenes.CONFIGS[name]()
    R.upload_volume(w.volume)
    g = R.render(w.poses[:1], w.intrinsics)
    cyc = g["normal"][0].cpu().numpy().astype(np.float64)
    cnt = g["color"][0].cpu().numpy().astype(np.float64)
    d = g["depth"][0].cpu().numpy()
    H, W = d.shape
    print(name, "rays", d.size, "hits", int((d > 0).sum()))
    cnt[..., 2] = cnt[..., 2]
    cpi = g["mask"][0].cpu().numpy().astype(np.float64)
    print(f"  cpi_skips      mean {cpi.mean():6.2f} p50 {np.median(cpi):5.0f} p99 {np.quantile(cpi, 0.99):5.0f}")
    for i, nm in enumerate(["march_evals", "refine_evals", "empty_block_steps"]):
        x = cnt[..., i]
        print(f"  {nm:14s} mean {x.mean():6.2f} p50 {np.median(x):5.0f} p99 {np.quantile(x, 0.99):5.0f} max {x.max():5.0f}")

    def tiles(a):
        return a[: H // 4 * 4, : W // 8 * 8].reshape(H // 4, 4, W // 8, 8).transpose(0, 2, 1, 3).reshape(-1, 32)
    tot = cyc.sum(-1)
    tt = tiles(tot)
    print(f"  cycles/ray mean {tot.mean():.0f}; per warp tile max {tt.max(1).mean():.0f} (lanes run together)")
    for i, nm in enumerate(["outside evals", "march evals", "refine evals"]):
        t = tiles(cyc[..., i])
        print(f"  {nm:14s} share of warp cycles {t.max(1).sum() / tt.max(1).sum():.3f}  mean/ray {cyc[..., i].mean():.0f}")
    np.save(os.path.join(ROOT, "gpurun_out", f"stats_{name}.npy"), np.concatenate([cyc, cnt], -1))

# per-warp step efficiency: a warp runs as many steps as its slowest lane needs
for name in sys.argv[1:] or ["C1"]:
    a = np.load(os.path.join(ROOT, "gpurun_out", f"stats_{name}.npy"))
    H, W = a.shape[:2]
    ev = a[..., 3] + a[..., 4]  # march + refinement evaluations per ray

    def tiles(x):
        return x[: H // 4 * 4, : W // 8 * 8].reshape(H // 4, 4, W // 8, 8).transpose(0, 2, 1, 3).reshape(-1, 32)
    t = tiles(ev)
    print(f"{name}: evaluations per ray mean {ev.mean():.2f}; per warp max {t.max(1).mean():.2f}; "
          f"lane efficiency of the step loop {t.mean(1).sum() / t.max(1).sum():.3f}")
