"""Debug helper: dump combined-render GPU vs oracle mismatches (C1) to gpurun_out/comb_dbg.npz."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle, scenes  # noqa
from paper_2301_12796_b200 import Renderer  # noqa
w = scenes.c1_room()
R = Renderer(0)
R.upload_volume(w.volume)
R.combine(w.poses[0], w.intrinsics)
g = R.render(w.poses, w.intrinsics, combined=True)
g = {k: v[0].cpu().numpy() for k, v in g.items()}
o = oracle.render_combined(oracle.OracleVolume(w.volume), w.poses[0], w.intrinsics, w.poses[0], w.intrinsics)
ex = R.get_combined()
np.savez_compressed(os.path.join(ROOT, "gpurun_out", "comb_dbg.npz"), **{"g_" + k: v for k, v in g.items()},
                    **{"o_" + k: v for k, v in o.items()}, **{"x_" + k: v for k, v in ex.items()})
print("saved")
