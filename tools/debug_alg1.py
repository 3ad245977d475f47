"""Debug helper: Algorithm-1 combined TSDF of configs[2] view 0 exported (grid and hash location
paths) -> gpurun_out/alg1_dbg.npz."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import scenes  # noqa
from paper_2301_12796_b200 import Renderer  # noqa
from paper_2301_12796_b200.dtsdf import OPT_LOCATION_GRID  # noqa
w = scenes.c2_thin()
R = Renderer(0)
R.upload_volume(w.volume)
R.combine(w.poses[0], w.intrinsics, mode=1)
ex = R.get_combined()
R.set_option(OPT_LOCATION_GRID, 0)
R.combine(w.poses[0], w.intrinsics, mode=1)
ex2 = R.get_combined()
i1, i2 = np.lexsort(ex["locs"].T), np.lexsort(ex2["locs"].T)
print("grid vs hash sdf equal:", np.array_equal(ex["sdf"][i1], ex2["sdf"][i2], equal_nan=True))
np.savez_compressed(os.path.join(ROOT, "gpurun_out", "alg1_dbg.npz"), **ex)
