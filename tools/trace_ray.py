"""Step-by-step trace of the slowest ray of a warp tile (DTSDF_STATS build, libdtsdf_stats.so):
per step the cycles spent, how many of them in the advance loop, the mode, the lattice index, the
block locations newly located and the certainly-positive lookahead scans -- once in the whole view,
once with only the tile's row strip launched (no contention from the rest of the frame).

    python tools/trace_ray.py C1 68,448 [224,424 ...]
"""
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

MODES = "MBIS"
name = sys.argv[1]
R = Renderer(0)
w = scenes.CONFIGS[name]()
R.upload_volume(w.volume)
poses = np.asarray(w.poses[:1], np.float32)
H = w.intrinsics.height
g = R.render(poses, w.intrinsics)
cnt = g["color"][0].cpu().numpy().astype(np.int64)
lib = dtsdf.lib()
pix = ctypes.c_int.in_dll(lib, "dtsdf_debug_trace_pix")


def trace(u0, v0, r0, r1):
    pix.value = u0 | ((v0 - r0) << 16)
    for _ in range(3):
        R.render(poses, w.intrinsics, row0=r0, row1=r1)
    torch.cuda.synchronize()
    ptr = ctypes.c_void_p.in_dll(lib, "dtsdf_debug_trace").value

    class CAI:
        __cuda_array_interface__ = {"shape": (32 * 128 * 8,), "typestr": "<i8", "data": (ptr, False), "version": 3}
    t = torch.as_tensor(CAI(), device="cuda").cpu().numpy().reshape(32, 128, 8)
    n = np.array([int(np.argmax(t[l, :, 0] == -1)) for l in range(32)])
    return t, n


for spec in sys.argv[2:]:
    row, col = map(int, spec.split(","))
    ev = cnt[row:row + 4, col:col + 8, 0] + cnt[row:row + 4, col:col + 8, 1]
    print(f"== {name} warp tile {row},{col}: evaluations per lane max {ev.max()} mean {ev.mean():.1f}")
    r0 = row // 8 * 8
    for label, (a, b) in (("whole view", (0, H)), (f"strip {r0}:{r0 + 8} alone", (r0, r0 + 8))):
        t, n = trace(col, row, a, b)
        L = int(np.argmax(n))
        steps = int(n.max())
        cyc = np.array([max(t[l, i, 1] for l in range(32) if i < n[l]) for i in range(steps)])
        locs = [[t[l, i, 6] >> 16 for l in range(32) if i < n[l]] for i in range(steps)]
        tot = lambda sh: int(sum(((t[l, :n[l], 7] >> sh) & 0xffff).sum() for l in range(32)))
        print(f"  {label}: lane totals: scans {tot(0)}, jumps {tot(16)}, empty-block steps {tot(32)}")
        print(f"  {label}: {steps} warp steps, {cyc.sum()} cycles ({cyc.sum() / steps:.0f}/step); "
              f"locates per step (max lane) {sum(max(x) for x in locs)}, (all lanes) {sum(sum(x) for x in locs)}")
        if label == "whole view":
            print("    step  cycles  adv(slowest lane)  lanes M/B/I  locates max/mean  newblk max  scans max  jumps max  empty max")
            for i in range(steps):
                act = [l for l in range(32) if i < n[l]]
                md = [t[l, i, 3] & 255 for l in act]
                lc = np.array([t[l, i, 6] >> 16 for l in act])
                nb = np.array([t[l, i, 6] & 0xffff for l in act])
                sc = np.array([t[l, i, 7] & 0xffff for l in act])
                jm = np.array([(t[l, i, 7] >> 16) & 0xffff for l in act])
                em = np.array([(t[l, i, 7] >> 32) & 0xffff for l in act])
                adv = max(t[l, i, 2] for l in act)
                print(f"    {i:4d} {cyc[i]:7d} {adv:7d}   {md.count(0):2d}/{md.count(1):2d}/{md.count(2):2d}   "
                      f"{lc.max():3d}/{lc.mean():5.2f}   {nb.max():3d}  {sc.max():3d}  {jm.max():3d}  {em.max():3d}")
