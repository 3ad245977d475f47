"""ICP throughput on the GPU: configs[1] 640x480 frame displaced by 1 cm + 2 deg from the rendered
pose, tracked against the renderer's depth + normals (coarse 0.05 m / 20 it, fine 0.005 m / 50 it).
Prints one JSON line: wall ms per tracked frame, iterations, ms per iteration (CUDA events)."""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa
import scenes  # noqa
from paper_2301_12796_b200 import Renderer  # noqa


def exp_se3(xi):  # input generator only: a known displacement (Rodrigues)
    w, v = np.asarray(xi[3:]), np.asarray(xi[:3])
    a = np.linalg.norm(w)
    W = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
    Rm = np.eye(3) + np.sin(a) / a * W + (1 - np.cos(a)) / a ** 2 * W @ W
    V = np.eye(3) + (1 - np.cos(a)) / a ** 2 * W + (a - np.sin(a)) / a ** 3 * W @ W
    T = np.eye(4)
    T[:3, :3], T[:3, 3] = Rm, V @ v
    return T


w = scenes.c1_room()
K, pose = w.intrinsics, w.poses[0]
R = Renderer(0)
R.upload_volume(w.volume)
out = R.render(pose[None], K)
E = exp_se3(np.r_[np.array([0.6, 0.2, -0.77]) / np.linalg.norm([0.6, 0.2, -0.77]) * 0.01,
                  np.array([0.3, -0.5, 0.8]) / np.linalg.norm([0.3, -0.5, 0.8]) * np.deg2rad(2)])
fr = scenes.analytic_frame(w.patches, np.asarray(pose) @ E, K)
d = torch.from_numpy(fr.depth).cuda()
rd, rn = out["depth"][0], out["normal"][0]
for _ in range(3):
    D, _ = R.icp(d, rd, rn, pose, K, outlier=0.05, max_iters=20)
    D, info = R.icp(d, rd, rn, pose, K, init_delta=D, outlier=0.005, max_iters=50)
ts, its = [], []
for _ in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    D, i1 = R.icp(d, rd, rn, pose, K, outlier=0.05, max_iters=20)
    D, i2 = R.icp(d, rd, rn, pose, K, init_delta=D, outlier=0.005, max_iters=50)
    ts.append(time.perf_counter() - t0)
    its.append(i1["iterations"] + i2["iterations"])
# one iteration's kernels timed with events (normal equations call = reduce + solve)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
R.set_profiling(True)
R.reset_kernel_times()
for _ in range(50):
    R.icp_normal_equations(d, rd, rn, pose, K, D, outlier=0.005)
kt = R.kernel_times()
R.set_profiling(False)
print(json.dumps({"what": "icp", "config": "C1 640x480, 1 cm + 2 deg, coarse 20 + fine 50 max iterations",
                  "ms_per_frame_median": 1e3 * float(np.median(ts)), "iterations": int(np.median(its)),
                  "kernel_ms_per_linearisation": kt["other_ms"] / 50, "inliers": int(info["inliers"]),
                  "device": torch.cuda.get_device_name(0)}))
