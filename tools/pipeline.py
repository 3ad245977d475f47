"""The paper's tracking-and-mapping loop (Fig. 1) on the GPU path only:

    frame t: render the model at the last pose estimate (direct, or the combined TSDF when the
    recombination conditions fire, eqs. 10-13) -> ICP of the new depth frame against the render
    (coarse 0.05 m / fine 0.005 m) -> fuse the frame at the tracked pose.

Input: seeded ideal depth frames of the configs[1] room along a smooth orbit (scenes module).
Prints one JSON line with the per-stage wall times and the tracking error against the ground truth.

    python tools/pipeline.py [--frames 60] [--combined]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import scenes  # noqa: E402
from paper_2301_12796_b200 import Renderer  # noqa: E402
from paper_2301_12796_b200.dtsdf import should_recombine  # noqa: E402


def run(frames=60, combined=False, step_m=0.02, step_deg=0.8, seed=3):
    w = scenes.c1_room()
    K = w.intrinsics
    rng = np.random.default_rng([seed, 0])
    gt = scenes.orbit_poses(rng, n_views=frames, step_m=step_m, step_deg=step_deg, height=1.5)
    data = [scenes.analytic_frame(w.patches, P, K) for P in gt]
    dev = [{k: torch.from_numpy(getattr(f, k)).cuda() for k in ("depth", "normal", "color")} for f in data]
    R = Renderer(0)
    R.fusion_reserve(120000, voxel_size=0.01, truncation=0.04, theta=scenes.THETA)
    est = [np.asarray(gt[0], np.float64)]
    R.fuse(dev[0]["depth"], dev[0]["normal"], dev[0]["color"], est[0], K)
    out = R.render(est[0][None], K)
    last, last_pose = 0, est[0]
    times = {"render": [], "track": [], "fuse": [], "combine": []}
    for t in range(1, frames):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ref = est[-1]
        if combined:
            tc = time.perf_counter()
            if should_recombine(t, last, ref, last_pose):
                R.combine(ref, K)
                last, last_pose = t, ref
            times["combine"].append(time.perf_counter() - tc)
            R.render_combined_into(ref[None], K, out["depth"], out["normal"], out["color"], out["mask"])
        else:
            R.render_into(ref[None], K, out["depth"], out["normal"], out["color"], out["mask"])
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        D, _ = R.icp(dev[t]["depth"], out["depth"][0], out["normal"][0], ref, K, outlier=0.05, max_iters=20)
        D, info = R.icp(dev[t]["depth"], out["depth"][0], out["normal"][0], ref, K, init_delta=D, outlier=0.005,
                        max_iters=50)
        pose = ref @ D
        est.append(pose)
        t2 = time.perf_counter()
        R.fuse(dev[t]["depth"], dev[t]["normal"], dev[t]["color"], pose, K)
        t3 = time.perf_counter()
        times["render"].append(t1 - t0)
        times["track"].append(t2 - t1)
        times["fuse"].append(t3 - t2)
    err_t = [float(np.linalg.norm(e[:3, 3] - np.asarray(g)[:3, 3])) for e, g in zip(est, gt)]
    err_r = [float(np.degrees(np.arccos(np.clip((np.trace(e[:3, :3].T @ np.asarray(g)[:3, :3]) - 1) / 2, -1, 1))))
             for e, g in zip(est, gt)]
    res = {"what": "pipeline", "frames": frames, "mode": "combined" if combined else "direct",
           "ms_render": 1e3 * float(np.median(times["render"])), "ms_track": 1e3 * float(np.median(times["track"])),
           "ms_fuse": 1e3 * float(np.median(times["fuse"])),
           "fps": 1.0 / float(np.median(np.add(np.add(times["render"], times["track"]), times["fuse"]))),
           "final_translation_error_m": err_t[-1], "max_translation_error_m": max(err_t),
           "max_rotation_error_deg": max(err_r), "blocks": R.stats()["n_blocks"]}
    R.close()
    return res


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=60)
    ap.add_argument("--combined", action="store_true")
    a = ap.parse_args()
    print(json.dumps(run(a.frames, a.combined)))
