"""Host-side cost of one dtsdf_render_batch call (enqueue only, device outputs) and of the
synchronous call into pinned host outputs, split into binding and library time.

    python tools/call_overhead.py
"""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import scenes  # noqa: E402
from paper_2301_12796_b200 import Renderer, dtsdf  # noqa: E402

w = scenes.c1_room()
R = Renderer(0)
R.upload_volume(w.volume)
poses = np.ascontiguousarray(np.asarray(w.poses[:1], np.float32).reshape(-1, 16))
K = w.intrinsics
out = R.render(poses, K)
H, W = K.height, K.width
k = dtsdf.make_intrinsics(K)
stream = torch.cuda.current_stream().cuda_stream
args = (R._h, 1, poses.ctypes.data, C.byref(k), 0, H, out["depth"].data_ptr(), out["normal"].data_ptr(),
        out["color"].data_ptr(), out["mask"].data_ptr(), stream)
lib = dtsdf.lib()


def per_call(fn, n=300):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / n * 1e6


n64, b64 = C.c_int64(), C.c_int64()
print(f"trivial library call (dtsdf_volume_stats): {per_call(lambda: lib.dtsdf_volume_stats(R._h, C.byref(n64), C.byref(b64), C.byref(b64))):.1f} us")
print(f"dtsdf_render_batch, prepared ctypes args, device outputs (enqueue): {per_call(lambda: lib.dtsdf_render_batch(*args)):.1f} us")
print(f"Renderer.render_into, device outputs (enqueue): {per_call(lambda: R.render_into(poses, K, out['depth'], out['normal'], out['color'], out['mask'])):.1f} us")
hd = torch.empty((1, H, W), dtype=torch.float32).pin_memory()
hn = torch.empty((1, H, W, 3)).pin_memory()
hc = torch.empty((1, H, W, 3), dtype=torch.uint8).pin_memory()
hm = torch.empty((1, H, W), dtype=torch.uint8).pin_memory()
ts = []
for i in range(110):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    R.render_into(poses, K, hd, hn, hc, hm)
    if i >= 10:
        ts.append(time.perf_counter() - t0)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
R.render_into(poses, K, out["depth"], out["normal"], out["color"], out["mask"])
ev[1].record()
torch.cuda.synchronize()
print(f"synchronous call into pinned host outputs: median {np.median(ts) * 1e6:.1f} us; device time of one step "
      f"{ev[0].elapsed_time(ev[1]) * 1e3:.1f} us")
