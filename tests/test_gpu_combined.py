"""GPU parity of the view-dependent combined TSDF: the
CUDA combine + combined raycast through the C ABI against the fp64 oracle (oracle.c
combine_voxel / render_pixel_combined) on the same seeded inputs.  Needs a B200."""
import numpy as np
import pytest

import oracle
import scenes
from parity import assert_parity, to_np

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

SDF_TOL = 2e-5     # normalised sdf: fp32 sum of <= 6 products / S (|phi| <= 1)
WEIGHT_RTOL = 1e-4


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2301_12796_b200 import Renderer
    r = Renderer(0)
    yield r
    r.close()


def _sel(gpu, view, pixels=None):
    out = {}
    for k, v in gpu.items():
        a = to_np(v[view])
        if pixels is not None:
            a = a[pixels[:, 1], pixels[:, 0]]
        out[k] = a
    return out


def _voxels(locs):
    off = scenes.local_offsets().astype(np.int64)
    return (locs.astype(np.int64)[:, None, :] * 8 + off[None]).reshape(-1, 3)


def _compare_voxels(R, w, pose, budget=1e-3, mode=0, vol=None, before=None):
    """Every exported combined voxel against the oracle's combine_voxel at the same position, and
    sampled non-exported locations hold no valid oracle voxel.  vol: the volume (default
    w.volume); before: the OracleVolume the combined TSDF was computed from when fusion has since
    changed it (reading R58)."""
    vol = w.volume if vol is None else vol
    ex = R.get_combined()
    n = len(ex["locs"])
    assert n > 0
    ov = oracle.OracleVolume(vol)
    ijk = _voxels(ex["locs"])
    o = oracle.combined_voxels(ov, pose, w.intrinsics, ijk, mode=mode, before=before)
    g_valid = ~np.isnan(ex["sdf"].reshape(-1))
    assert np.array_equal(g_valid, ex["weight"].reshape(-1) > 0)
    disagree = (g_valid != o["valid"]).sum()
    both = g_valid & o["valid"]
    sdf_err = np.abs(ex["sdf"].reshape(-1)[both] - o["sdf"][both])
    w_rel = np.abs(ex["weight"].reshape(-1)[both] - o["weight"][both]) / o["weight"][both]
    rgb_eq = (ex["rgb"].reshape(-1, 3)[both] == o["rgb"][both]).all(1).mean()
    mask_eq = (ex["mask"].reshape(-1)[both] == o["mask"][both]).mean()
    st = {"locations": n, "voxels_valid": int(both.sum()), "valid_disagree": int(disagree),
          "sdf_max_err": float(sdf_err.max()), "weight_max_rel": float(w_rel.max()), "rgb_exact": float(rgb_eq),
          "mask_exact": float(mask_eq)}
    assert disagree <= budget * both.sum(), st
    assert (sdf_err > SDF_TOL).sum() <= budget * both.sum(), st
    assert (w_rel > WEIGHT_RTOL).sum() <= budget * both.sum(), st
    assert rgb_eq >= 0.999 and mask_eq >= 0.999, st
    # completeness: allocated locations the GPU did not combine have no valid oracle voxel
    locs_all = np.unique(vol.keys[:, :3], axis=0)
    got = {tuple(l) for l in ex["locs"]}
    rest = np.array([l for l in locs_all if tuple(l) not in got])
    if len(rest):
        rng = np.random.default_rng(0)
        pick = rest[rng.choice(len(rest), min(len(rest), 400), replace=False)]
        assert oracle.combined_voxels(ov, pose, w.intrinsics, _voxels(pick), mode=mode, before=before)["valid"].sum() <= \
            budget * both.sum()
    return st


def test_c0_combined_voxels_and_render(R, c0):
    R.upload_volume(c0.volume)
    R.combine(c0.poses[0], c0.intrinsics)
    st = _compare_voxels(R, c0, c0.poses[0])
    g = R.render(c0.poses, c0.intrinsics, combined=True)
    o = oracle.render_combined(oracle.OracleVolume(c0.volume), c0.poses[0], c0.intrinsics, c0.poses[0],
                               c0.intrinsics)
    rs = assert_parity(_sel(g, 0), o, what="C0 combined")
    assert rs["hits_gpu"] > 1800
    print("C0 combined", st, rs)


def test_c1_combined_voxels_and_full_frame(R, c1):
    """configs[1] at full size: combined TSDF of the bench pose, every combined voxel compared,
    and the full 640x480 render through it."""
    R.upload_volume(c1.volume)
    R.combine(c1.poses[0], c1.intrinsics)
    st = _compare_voxels(R, c1, c1.poses[0])
    g = R.render(c1.poses, c1.intrinsics, combined=True)
    o = oracle.render_combined(oracle.OracleVolume(c1.volume), c1.poses[0], c1.intrinsics, c1.poses[0],
                               c1.intrinsics)
    rs = assert_parity(_sel(g, 0), o, what="C1 combined")
    assert rs["hits_gpu"] > 100000
    print("C1 combined", st, rs)


def test_c2_combined_thin_plates(R, c2):
    """configs[2]: combined TSDFs of 4 of the 20 views (both sides of two plate clusters)."""
    R.upload_volume(c2.volume)
    ov = oracle.OracleVolume(c2.volume)
    for v in (0, 1, 10, 11):
        R.combine(c2.poses[v], c2.intrinsics)
        g = R.render(c2.poses[v:v + 1], c2.intrinsics, combined=True)
        o = oracle.render_combined(ov, c2.poses[v], c2.intrinsics, c2.poses[v], c2.intrinsics)
        print("C2 combined", v, assert_parity(_sel(g, 0), o, what=f"C2 combined view {v}"))


def test_c3_render_from_moved_poses(R, c1):
    """configs[3] trajectory: combined at view 0, rendered from views 1..3 (the poses the
    recombination conditions keep using it for), on a 1/4 pixel grid."""
    w = scenes.c3_batch(n_views=4, room=c1)
    R.upload_volume(w.volume)
    R.combine(w.poses[0], w.intrinsics)
    g = R.render(w.poses, w.intrinsics, combined=True)
    ov = oracle.OracleVolume(w.volume)
    v, u = np.mgrid[1:w.intrinsics.height:4, 2:w.intrinsics.width:4]
    px = np.stack([u.ravel(), v.ravel()], 1).astype(np.int32)
    for i in range(4):
        o = oracle.render_combined(ov, w.poses[0], w.intrinsics, w.poses[i], w.intrinsics, pixels=px)
        print("C3 moved", i, assert_parity(_sel(g, i, px), o, what=f"C3 moved view {i}"))


def test_recombination_is_bit_identical_and_accelerations_invisible(R, c1):
    """SPEC invariant 'recombination invariance': combining again for the same camera yields the
    same voxels (slot order aside) and the same render bits; the range pass and skips stay exact."""
    from paper_2301_12796_b200.dtsdf import OPT_BLOCK_SKIP, OPT_LOCATION_GRID, OPT_RANGE_PASS
    R.upload_volume(c1.volume)
    K = scenes.Intrinsics(fx=262.5, fy=262.5, cx=159.5, cy=119.5, width=320, height=240)
    R.combine(c1.poses[0], K)
    a = R.get_combined()
    ref = R.render(c1.poses, K, combined=True)
    R.combine(c1.poses[0], K)
    b = R.get_combined()
    ia, ib = np.lexsort(a["locs"].T), np.lexsort(b["locs"].T)
    for k in a:
        assert np.array_equal(a[k][ia], b[k][ib], equal_nan=True), k
    g = R.render(c1.poses, K, combined=True)
    for k in ref:
        assert torch.equal(ref[k], g[k]), k
    for opt, val in ((OPT_RANGE_PASS, 0), (OPT_BLOCK_SKIP, 0), (OPT_LOCATION_GRID, 0)):
        R.set_option(opt, val)
        if opt == OPT_LOCATION_GRID:
            R.combine(c1.poses[0], K)
        g = R.render(c1.poses, K, combined=True)
        R.set_option(opt, 1)
        for k in ref:
            assert torch.equal(ref[k], g[k]), (opt, k)
    R.combine(c1.poses[0], K)


def test_combined_errors_and_invalidation(R, c0):
    from paper_2301_12796_b200.dtsdf import NO_COMBINED, DtsdfError
    R.upload_volume(c0.volume)
    with pytest.raises(DtsdfError) as e:
        R.render(c0.poses, c0.intrinsics, combined=True)
    assert e.value.code == NO_COMBINED
    R.combine(c0.poses[0], c0.intrinsics)
    R.render(c0.poses, c0.intrinsics, combined=True)
    R.upload_volume(c0.volume)  # a new volume invalidates the combined TSDF
    with pytest.raises(DtsdfError) as e:
        R.render(c0.poses, c0.intrinsics, combined=True)
    assert e.value.code == NO_COMBINED
    with pytest.raises(DtsdfError):
        R.combine(c0.poses[0], c0.intrinsics, margin=-1.0)


def test_combined_host_outputs_equal_device(R, c1):
    R.upload_volume(c1.volume)
    K = scenes.Intrinsics(fx=262.5, fy=262.5, cx=159.5, cy=119.5, width=320, height=240)
    R.combine(c1.poses[0], K)
    g = R.render(c1.poses, K, combined=True)
    hd = np.zeros((1, 240, 320), np.float32)
    hn = np.zeros((1, 240, 320, 3), np.float32)
    hc = np.zeros((1, 240, 320, 3), np.uint8)
    hm = np.zeros((1, 240, 320), np.uint8)
    R.render_combined_into(c1.poses, K, hd, hn, hc, hm)
    assert np.array_equal(hd, to_np(g["depth"])) and np.array_equal(hn, to_np(g["normal"]))
    assert np.array_equal(hc, to_np(g["color"])) and np.array_equal(hm, to_np(g["mask"]))


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_algorithm1_voxels_and_render(R, cfg, c1, c2):
    """NEXT-4: the Algorithm-1 combined TSDF (mode 1, readings R53-R57) -- every combined voxel
    against the oracle, then the render through it (BJ tolerances)."""
    w = c1 if cfg == "C1" else c2
    v = 0
    R.upload_volume(w.volume)
    R.combine(w.poses[v], w.intrinsics, mode=1)
    st = _compare_voxels(R, w, w.poses[v], mode=1)
    g = R.render(w.poses[v:v + 1], w.intrinsics, combined=True)
    o = oracle.render_combined(oracle.OracleVolume(w.volume), w.poses[v], w.intrinsics, w.poses[v], w.intrinsics,
                               mode=1)
    rs = assert_parity(_sel(g, 0), o, what=f"{cfg} algorithm 1")
    print(cfg, "algorithm 1", st, rs)


def test_combined_host_outputs_equal_device_outputs(R, c1):
    """The combined raycast into pinned host outputs (written by the kernel, DTSDF_OPT_HOST_WRITE)
    and via the copy path equals the device render bit for bit, on a ragged row range."""
    from paper_2301_12796_b200.dtsdf import OPT_HOST_WRITE
    R.upload_volume(c1.volume)
    K = c1.intrinsics
    R.combine(c1.poses[0], K)
    r0, r1 = 3, 470
    g = R.render(c1.poses, K, row0=r0, row1=r1, combined=True)
    H, W = r1 - r0, K.width
    for host_write in (1, 0):
        R.set_option(OPT_HOST_WRITE, host_write)
        hd = torch.full((1, H, W), 7.0, dtype=torch.float32).pin_memory()
        hn = torch.full((1, H, W, 3), 7.0, dtype=torch.float32).pin_memory()
        hc = torch.full((1, H, W, 3), 7, dtype=torch.uint8).pin_memory()
        hm = torch.full((1, H, W), 7, dtype=torch.uint8).pin_memory()
        R.render_combined_into(c1.poses, K, hd, hn, hc, hm, row0=r0, row1=r1)
        for k, h in (("depth", hd), ("normal", hn), ("color", hc), ("mask", hm)):
            assert torch.equal(g[k].cpu(), h), (k, host_write)
    R.set_option(OPT_HOST_WRITE, 1)


@pytest.mark.parametrize("mode", [0, 1])
def test_fused_frame_adds_first_time_voxels(R, c1, mode):
    """Reading R58: the combined TSDF of the bench pose is computed from the room
    without its last 8 boxes; a frame of the whole room (ideal depth camera) is then fused.  Every
    combined voxel equals the oracle's: voxels that received data for the first time (the missing
    boxes' new blocks, zero-weight voxels that gained weight) combined from the fused volume, all
    others kept from the combination before the frame; the render through it likewise.  The fused
    volume on the oracle side is the oracle's own fusion (oracle/fusion.c) of the same frame."""
    import dataclasses
    S, TAU = 0.01, 0.04
    pat = c1.patches
    keep = 1 + 5 * 12  # floor + 12 of the 20 boxes (5 patches each)
    sub = dataclasses.replace(pat, **{f: getattr(pat, f)[:keep] for f in ("q", "n", "u", "v", "hu", "hv", "color", "kind")})
    before = scenes.patch_fill(sub, voxel_size=S, truncation=TAU, theta=scenes.THETA)
    pose, K = c1.poses[0], c1.intrinsics
    K_half = scenes.Intrinsics(fx=262.5, fy=262.5, cx=159.5, cy=119.5, width=320, height=240)
    fr = scenes.analytic_frame(pat, pose, K_half)
    cap = before.n_blocks + 30000
    R.upload_volume(before)
    R.fusion_reserve(cap)
    R.combine(pose, K, mode=mode)
    n_before = R.combined_stats()["n_locations"]
    new_blocks = R.fuse(fr.depth, fr.normal, fr.color, pose, K_half)
    F = oracle.OracleFusion(S, TAU, scenes.THETA, cap, vol=before)
    assert F.fuse(fr.depth, fr.normal, fr.color, pose, K_half) == new_blocks > 500
    after = F.volume()
    n_after = R.combined_stats()["n_locations"]
    assert n_after > n_before
    ob = oracle.OracleVolume(before)
    st = _compare_voxels(R, c1, pose, mode=mode, vol=after, before=ob)
    g = R.render(c1.poses, K, combined=True)
    o = oracle.render_combined(oracle.OracleVolume(after), pose, K, pose, K, mode=mode, before=ob)
    rs = assert_parity(_sel(g, 0), o, what=f"C1 combined after a fused frame (mode {mode})")
    # the added boxes are visible: more hits than the combination before the frame rendered
    print("R58", mode, n_before, n_after, st, rs)
