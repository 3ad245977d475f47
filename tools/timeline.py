"""Per-ray start/end timestamps (%globaltimer) and SM ids from the DTSDF_STATS debug build:
how busy the SMs are over the kernel's duration, and how long the slowest warps run."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("DTSDF_LIB", os.path.join(ROOT, "paper_2301_12796_b200", "libdtsdf_stats.so"))
import scenes  # noqa: E402
from paper_2301_12796_b200 import Renderer, dtsdf  # noqa: E402

R = Renderer(0)
for name in sys.argv[1:] or ["C1"]:
    w = scenes.CONFIGS[name]()
    R.upload_volume(w.volume)
    for _ in range(3):
        g = R.render(w.poses[:1], w.intrinsics)
    torch.cuda.synchronize()
    ptr = ctypes.c_void_p.in_dll(dtsdf.lib(), "dtsdf_debug_timeline").value
    H, W = w.intrinsics.height, w.intrinsics.width
    n = H * W * 3

    class CAI:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<u8", "data": (ptr, False), "version": 3}
    tl = torch.as_tensor(CAI(), device="cuda").cpu().numpy().reshape(H, W, 3).astype(np.int64)
    st, en, sm = tl[..., 0], tl[..., 1], tl[..., 2]
    t0 = st.min()
    st, en = (st - t0) / 1e3, (en - t0) / 1e3  # microseconds
    span = en.max()
    dur = en - st
    print(f"{name}: kernel span {span:.1f} us; ray durations us p50 {np.median(dur):.1f} p90 {np.quantile(dur, .9):.1f} "
          f"p99 {np.quantile(dur, .99):.1f} max {dur.max():.1f}")
    # warps = 8x4 tiles
    tiles = lambda a: a[: H // 4 * 4, : W // 8 * 8].reshape(H // 4, 4, W // 8, 8).transpose(0, 2, 1, 3).reshape(-1, 32)
    wst, wen = tiles(st).min(1), tiles(en).max(1)
    wd = wen - wst
    print(f"  warp durations us p50 {np.median(wd):.1f} p90 {np.quantile(wd, .9):.1f} p99 {np.quantile(wd, .99):.1f} "
          f"max {wd.max():.1f}; warp starts: last start at {wst.max():.1f} us")
    # active warps over time
    bins = np.linspace(0, span, 21)
    act = [int(((wst <= b) & (wen > b)).sum()) for b in bins[:-1]]
    print("  active warps over time (20 bins):", act)
    print(f"  total warp-time / (span * max active) = {wd.sum() / (span * max(act)):.3f}")
    np.save(os.path.join(ROOT, "gpurun_out", f"timeline_{name}.npy"), np.stack([st, en, sm.astype(np.float64)], -1))
