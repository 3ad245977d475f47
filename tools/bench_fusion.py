"""Fusion throughput on the GPU: configs[1] room scanned by seeded 640x480 ideal depth frames,
fused frame by frame through dtsdf_fuse (allocation + fusion + re-commit of the index).

    python tools/bench_fusion.py [--frames 30]
Prints one JSON line: wall ms per frame (host clock around the synchronous call) and the summed
kernel times of the last frames (dtsdf_kernel_times, CUDA events)."""
import argparse, json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa
import scenes  # noqa
from paper_2301_12796_b200 import Renderer  # noqa

ap = argparse.ArgumentParser()
ap.add_argument("--frames", type=int, default=30)
ap.add_argument("--warmup", type=int, default=5)
ap.add_argument("--start", choices=["c1", "empty"], default="c1",
                help="c1: fuse into the uploaded configs[1] volume; empty: scan the room from nothing")
ap.add_argument("--incremental", type=int, default=1, help="DTSDF_OPT_INCREMENTAL")
args = ap.parse_args()
w = scenes.c1_room()
K = w.intrinsics
poses = scenes.room_scan_poses(np.random.default_rng([9, 0]), args.frames + args.warmup)
frames = [scenes.analytic_frame(w.patches, P, K) for P in poses]
dev = [{k: torch.from_numpy(getattr(f, k)).cuda() for k in ("depth", "normal", "color")} for f in frames]
R = Renderer(0)
from paper_2301_12796_b200.dtsdf import OPT_INCREMENTAL  # noqa: E402
R.set_option(OPT_INCREMENTAL, args.incremental)
if args.start == "c1":
    R.upload_volume(w.volume)
    R.fusion_reserve(w.volume.n_blocks + 60000)
else:
    R.upload(0.01, 0.04, scenes.THETA, np.zeros((0, 4), np.int32), np.zeros((0, 512), np.float32),
             np.zeros((0, 512), np.float32))
    R.fusion_reserve(80000)
for i in range(args.warmup):
    R.fuse(dev[i]["depth"], dev[i]["normal"], dev[i]["color"], poses[i], K)
torch.cuda.synchronize()
t = []
new = 0
for i in range(args.warmup, args.warmup + args.frames):
    t0 = time.perf_counter()
    new += R.fuse(dev[i]["depth"], dev[i]["normal"], dev[i]["color"], poses[i], K)
    t.append(time.perf_counter() - t0)
st = R.stats()
# kernel times from a second pass over the same frames with event tracing on (tracing adds host
# overhead, so it is not on during the wall-clock pass above)
R.reset_kernel_times()
R.set_profiling(True)
for i in range(args.warmup, args.warmup + args.frames):
    R.fuse(dev[i]["depth"], dev[i]["normal"], dev[i]["color"], poses[i], K)
R.set_profiling(False)
kt = R.kernel_times()
print(json.dumps({"what": "fusion", "config": "C1 room, 640x480 ideal depth frames, 1 cm voxels, tau 4 cm",
                  "start": args.start, "incremental": args.incremental,
                  "frames": args.frames, "ms_per_frame_median": 1e3 * float(np.median(t)),
                  "frames_per_s": 1.0 / float(np.median(t)), "kernel_ms_per_frame": kt["other_ms"] / args.frames,
                  "kernel_launches_per_frame": kt["other_launches"] / args.frames, "new_blocks": new,
                  "blocks": st["n_blocks"], "device": torch.cuda.get_device_name(0)}))
