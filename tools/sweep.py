"""Tuning sweep on the GPU: raycast kernel time and parity vs the oracle per option setting.

    python tools/sweep.py [--configs C1,C2] [--reps 200]
"""
import argparse
import itertools
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import scenes  # noqa: E402
from parity import compare  # noqa: E402
from paper_2301_12796_b200 import Renderer  # noqa: E402
from paper_2301_12796_b200.dtsdf import OPT_BISECT_STEPS, OPT_REFINE_TOL_NM  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C1,C2")
ap.add_argument("--reps", type=int, default=200)
ap.add_argument("--schedules", default="0", help="(the persistent schedule 1 was removed in round 2)")
ap.add_argument("--bisect", default="-1,6,5,4,3")
ap.add_argument("--views", type=int, default=1)
ap.add_argument("--tol", default="0")
ap.add_argument("--no-parity", action="store_true")
args = ap.parse_args()

R = Renderer(0)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for name in args.configs.split(","):
    w = scenes.CONFIGS[name]()
    R.upload_volume(w.volume)
    ora = None if args.no_parity else oracle.OracleVolume(w.volume).render(w.poses[0], w.intrinsics)
    poses = np.repeat(np.asarray(w.poses[:1], np.float32), args.views, axis=0)
    for sch, nb, tol in itertools.product([int(x) for x in args.schedules.split(",")],
                                          [int(x) for x in args.bisect.split(",")],
                                          [int(x) for x in args.tol.split(",")]):
        R.set_option(OPT_REFINE_TOL_NM, tol)
        R.set_option(OPT_BISECT_STEPS, nb)
        out = R.render(poses, w.intrinsics)
        for _ in range(5):
            R.render_into(poses, w.intrinsics, out["depth"], out["normal"], out["color"], out["mask"])
        torch.cuda.synchronize()
        R.reset_kernel_times()
        R.set_profiling(True)
        for _ in range(args.reps):
            flush.fill_(1.0)
            R.render_into(poses, w.intrinsics, out["depth"], out["normal"], out["color"], out["mask"])
        torch.cuda.synchronize()
        R.set_profiling(False)
        kt = R.kernel_times()
        ms = kt["raycast_ms"] / kt["raycast_launches"]
        st = compare({k: v[0].cpu().numpy() for k, v in out.items()}, ora) if ora is not None else {
            "budget_used": None, "color_exact": None, "depth_max_err": None, "hit_disagree": None, "geom_out_of_tol": None}
        rays = w.intrinsics.width * w.intrinsics.height * args.views
        print(json.dumps({"config": name, "views": args.views, "schedule": sch, "bisect": nb, "tol_nm": tol, "raycast_ms": round(ms, 4),
                          "Mrays_s_kernel": round(rays / ms / 1e3, 1), "budget_used": st["budget_used"],
                          "color_exact": st["color_exact"], "depth_max": st["depth_max_err"],
                          "hit_disagree": st["hit_disagree"], "geom_bad": st["geom_out_of_tol"]}), flush=True)
R.set_option(OPT_BISECT_STEPS, -1)
R.set_option(OPT_REFINE_TOL_NM, 0)
