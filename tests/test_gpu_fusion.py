"""GPU parity of voxel-projection fusion: the CUDA
allocation + fusion through the C ABI against the fp64 oracle (fusion.c) on the same seeded
synthetic depth frames (scenes.analytic_frame), then the fused volumes rendered on both sides.
Needs a B200."""
import numpy as np
import pytest

import oracle
import scenes
from parity import assert_parity, to_np

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

K_HALF = scenes.Intrinsics(fx=262.5, fy=262.5, cx=159.5, cy=119.5, width=320, height=240)
S, TAU = 0.01, 0.04
SDF_TOL = 1e-5
BUDGET = 1e-3


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2301_12796_b200 import Renderer
    r = Renderer(0)
    yield r
    r.close()


def _sorted(keys, *arrs):
    idx = np.lexsort(keys.T[::-1])
    return (keys[idx],) + tuple(a[idx] for a in arrs)


def _compare_volumes(R, F):
    gk, gs, gw, gc = R.get_volume()
    ov = F.volume()
    gk, gs, gw, gc = _sorted(gk, gs, gw, gc)
    ok, os_, ow, oc = _sorted(ov.keys, ov.sdf, ov.weight, ov.rgb)
    assert np.array_equal(gk, ok), (len(gk), len(ok))  # allocation: identical key sets (R40)
    upd = (ow > 0) | (gw > 0)
    n = upd.sum()
    sdf_bad = (np.abs(gs - os_) > SDF_TOL) & upd
    # fp32 weight products (w_ICP w_angle w_dir; acosf near the membership band edge) vs fp64
    w_bad = (np.abs(gw - ow) > 1e-5 + 1e-4 * ow) & upd
    c_bad = (gc != oc).any(-1) & upd
    st = {"blocks": len(gk), "updated_voxels": int(n), "sdf_bad": int(sdf_bad.sum()), "w_bad": int(w_bad.sum()),
          "rgb_bad": int(c_bad.sum()), "sdf_max_err": float(np.abs(gs - os_)[upd].max()),
          "w_max_abs_err": float(np.abs(gw - ow)[upd].max()),
          "w_bad_examples": list(zip(gw[w_bad][:4].tolist(), ow[w_bad][:4].tolist()))}
    assert sdf_bad.sum() <= BUDGET * n and w_bad.sum() <= BUDGET * n and c_bad.sum() <= BUDGET * n, st
    return st


def test_depth_normals_match_oracle(R, c1):
    fr = scenes.analytic_frame(c1.patches, c1.poses[0], c1.intrinsics)
    g = R.depth_normals(fr.depth, c1.intrinsics)
    o = oracle.depth_normals(fr.depth, c1.intrinsics)
    gv, ov = (g != 0).any(-1), (o != 0).any(-1)
    assert np.array_equal(gv, ov)
    # component difference (arccos of a float32 dot product near 1 cannot resolve below ~3e-4 rad)
    assert np.abs(g[gv].astype(np.float64) - o[gv]).max() < 1e-5


def test_fused_room_matches_oracle_and_renders_alike(R, c1):
    """configs[1] room fused from 6 seeded frames (320x240) on both sides: identical key sets,
    voxels within tolerance, then the fused volumes rendered (BJ tolerances)."""
    poses = scenes.room_scan_poses(np.random.default_rng([7, 0]), 6)
    R.upload(S, TAU, scenes.THETA, np.zeros((0, 4), np.int32), np.zeros((0, 512), np.float32),
             np.zeros((0, 512), np.float32))
    R.fusion_reserve(60000)
    F = oracle.OracleFusion(S, TAU, scenes.THETA, 60000)
    for P in poses:
        fr = scenes.analytic_frame(c1.patches, P, K_HALF)
        ng = R.fuse(fr.depth, fr.normal, fr.color, P, K_HALF)
        no = F.fuse(fr.depth, fr.normal, fr.color, P, K_HALF)
        assert ng == no
    st = _compare_volumes(R, F)
    print("fused room", st)
    g = R.render(poses[:1], K_HALF)
    o = oracle.OracleVolume(F.volume()).render(poses[0], K_HALF)
    print("fused room render", assert_parity({k: to_np(v[0]) for k, v in g.items()}, o, what="fused C1"))


def test_fuse_into_uploaded_volume_and_device_frames(R, c1):
    """Fusion into an existing volume (configs[1]) with device-resident frames equals the oracle
    initialised from the same volume (colour weights start at the depth weights, R45)."""
    R.upload_volume(c1.volume)
    R.fusion_reserve(c1.volume.n_blocks + 20000)
    F = oracle.OracleFusion(S, TAU, scenes.THETA, c1.volume.n_blocks + 20000, vol=c1.volume)
    P = scenes.room_scan_poses(np.random.default_rng([8, 0]), 1)[0]
    fr = scenes.analytic_frame(c1.patches, P, K_HALF)
    dev = {k: torch.from_numpy(getattr(fr, k)).cuda() for k in ("depth", "normal", "color")}
    R.fuse(dev["depth"], dev["normal"], dev["color"], P, K_HALF)
    F.fuse(fr.depth, fr.normal, fr.color, P, K_HALF)
    print("fused into C1", _compare_volumes(R, F))


def test_fusion_capacity_exhaustion(R):
    from paper_2301_12796_b200.dtsdf import OUT_OF_MEMORY, DtsdfError
    pat = scenes.Patches.empty()
    pat.extend(np.array([0.8, 0, 0]), np.array([-1.0, 0, 0]), np.array([0, 1.0, 0]), np.array([0, 0, 1.0]), 1, 1,
               [1, 2, 3])
    K = scenes.Intrinsics(fx=30.0, fy=30.0, cx=15.5, cy=11.5, width=32, height=24)
    pose = scenes.look_at([0, 0, 0], [1, 0, 0])
    fr = scenes.analytic_frame(pat, pose, K)
    R.upload(S, TAU, scenes.THETA, np.zeros((0, 4), np.int32), np.zeros((0, 512), np.float32),
             np.zeros((0, 512), np.float32))
    R.fusion_reserve(3)
    with pytest.raises(DtsdfError) as e:
        R.fuse(fr.depth, fr.normal, fr.color, pose, K)
    assert e.value.code == OUT_OF_MEMORY
    assert R.stats()["n_blocks"] == 3


@pytest.mark.parametrize("start", ["c1", "empty"])
def test_incremental_index_equals_full_recommit(c1, start):
    """DTSDF_OPT_INCREMENTAL: after every fused frame the incrementally updated index (bricks, cell
    masks, surface bits, location grid, empty-space distances of the locations within one block of a
    changed block) renders exactly what a full re-commit of the same pool renders, and the pools
    hold the same blocks -- into the uploaded configs[1] volume and from an empty volume (whose
    growing AABB takes the full path)."""
    from paper_2301_12796_b200 import Renderer
    from paper_2301_12796_b200.dtsdf import OPT_INCREMENTAL
    poses = scenes.room_scan_poses(np.random.default_rng([7, 0]), 6)
    outs = {}
    for inc in (1, 0):
        Q = Renderer(0)
        Q.set_option(OPT_INCREMENTAL, inc)
        if start == "c1":
            Q.upload_volume(c1.volume)
            Q.fusion_reserve(c1.volume.n_blocks + 30000)
        else:
            Q.upload(S, TAU, scenes.THETA, np.zeros((0, 4), np.int32), np.zeros((0, 512), np.float32),
                     np.zeros((0, 512), np.float32))
            Q.fusion_reserve(60000)
        renders = []
        for P in poses:
            fr = scenes.analytic_frame(c1.patches, P, K_HALF)
            Q.fuse(fr.depth, fr.normal, fr.color, P, K_HALF)
            renders.append({k: v.cpu() for k, v in Q.render(poses[:2], K_HALF).items()})
        outs[inc] = (renders, _sorted(*Q.get_volume()), Q.stats())
        Q.close()
    assert outs[1][2]["n_blocks"] == outs[0][2]["n_blocks"] and outs[1][2]["n_locations"] == outs[0][2]["n_locations"]
    for a, b in zip(outs[1][1], outs[0][1]):
        assert np.array_equal(a, b)
    for i, (a, b) in enumerate(zip(outs[1][0], outs[0][0])):
        for k in a:
            assert torch.equal(a[k], b[k]), (i, k)
