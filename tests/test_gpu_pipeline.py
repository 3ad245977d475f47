"""The paper's tracking-and-mapping loop (Fig. 1) run end to end on the GPU path:
render at the last estimate (direct or the conditionally recombined combined TSDF) -> ICP ->
fusion at the tracked pose, on seeded ideal depth frames of the configs[1] room along a smooth
orbit.  The expected values are the analytic ground-truth poses.  Needs a B200."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


@pytest.mark.parametrize("combined", [False, True])
def test_track_and_map_loop_stays_on_the_ground_truth(combined):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from pipeline import run
    res = run(frames=30, combined=combined)
    print(res)
    assert res["max_translation_error_m"] < 0.01
    assert res["max_rotation_error_deg"] < 0.2


def test_combined_tsdf_survives_fusion(c1):
    """A fused frame re-commits the volume; the combined TSDF is kept (stale until recombined,
    P:256-262) except where voxels received data for the first time (reading R58): every
    combined voxel that was valid before the frame is bit-identical after it, no slot is lost, and
    rendering through it still works."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import scenes
    from paper_2301_12796_b200 import Renderer
    R = Renderer(0)
    R.upload_volume(c1.volume)
    R.fusion_reserve(c1.volume.n_blocks + 20000)
    K = scenes.Intrinsics(fx=262.5, fy=262.5, cx=159.5, cy=119.5, width=320, height=240)
    R.combine(c1.poses[0], K)
    a = R.get_combined()
    P = scenes.room_scan_poses(np.random.default_rng([8, 0]), 1)[0]
    fr = scenes.analytic_frame(c1.patches, P, K)
    assert R.fuse(fr.depth, fr.normal, fr.color, P, K) > 0
    b = R.get_combined()
    assert len(b["locs"]) >= len(a["locs"])
    pos = {tuple(l): i for i, l in enumerate(b["locs"])}
    idx = np.array([pos[tuple(l)] for l in a["locs"]])
    valid = ~np.isnan(a["sdf"])
    for k in ("sdf", "weight", "rgb", "mask"):
        assert np.array_equal(a[k][valid], b[k][idx][valid]), k
    out = R.render(c1.poses, K, combined=True)
    assert (out["depth"] > 0).sum() > 0.5 * K.width * K.height
    R.close()
