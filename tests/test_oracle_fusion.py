"""Pins of the fusion oracle (readings R39-R46 in DESIGN.md §4).

Voxel-projection fusion of depth frames into the DTSDF.  The pins are
closed-form geometry (planes seen by an ideal depth camera), the running-average fixed point
(SPEC fusion invariant), membership special cases (eq:angular_threshold / eq:direction_weight),
carving and its depth-edge guard, the paper's printed weight values, and the closed
fuse -> render loop against analytic ray hits."""
import numpy as np
import pytest

import oracle
import scenes
from helpers import angle_between, pinhole
from scenes import DIRECTION_VECTORS, look_at

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")
TH = np.deg2rad(65.0)
S, TAU = 0.01, 0.04


def _wall_patches(x0=0.8, color=(10, 200, 30), n=(-1.0, 0.0, 0.0), half=1.0):
    pat = scenes.Patches.empty()
    n = np.asarray(n, np.float64)
    n /= np.linalg.norm(n)
    u = np.cross(n, [0.0, 0.0, 1.0])
    if np.linalg.norm(u) < 1e-6:
        u = np.cross(n, [1.0, 0.0, 0.0])
    u /= np.linalg.norm(u)
    v = np.cross(n, u)
    pat.extend(-n * x0, n, u, v, half, half, color)
    return pat


def _voxel_centres(vol):
    off = scenes.local_offsets().astype(np.int64)
    return (vol.keys[:, None, :3].astype(np.int64) * 8 + off[None]) * np.float64(np.float32(S))


# ---------------------------------------------------------------------------------------
# R39: depth normals
# ---------------------------------------------------------------------------------------
def test_depth_normals_planes():
    """Fronto-parallel plane -> (0,0,-1); a tilted plane -> its analytic normal (cross products of
    exact plane points are exact up to the float32 depth rounding); border and pixels next to a
    missing depth -> invalid (0)."""
    K = pinhole(40, 30, 35.0)
    fr = scenes.analytic_frame(_wall_patches(0.9, n=(0, 0, -1)), np.eye(4), K)
    nm = oracle.depth_normals(fr.depth, K)
    inner = nm[1:-1, 1:-1].reshape(-1, 3)
    assert np.abs(inner - [0, 0, -1]).max() < 1e-5
    assert (nm[0] == 0).all() and (nm[:, -1] == 0).all()
    nw = np.array([0.3, -0.2, -1.0])
    nw /= np.linalg.norm(nw)
    fr = scenes.analytic_frame(_wall_patches(0.9, n=nw, half=3.0), np.eye(4), K)
    nm = oracle.depth_normals(fr.depth, K)
    ang = angle_between(nm[1:-1, 1:-1].reshape(-1, 3).astype(np.float64), np.tile(nw, (38 * 28, 1)))
    assert np.median(ang) < 1e-5 and ang.max() < 1e-3  # float32 depth rounding over a 2-pixel baseline
    d = fr.depth.copy()
    d[10, 10] = 0.0
    nm = oracle.depth_normals(d, K)
    for (v, u) in ((10, 10), (10, 9), (10, 11), (9, 10), (11, 10)):
        assert (nm[v, u] == 0).all()
    assert (nm[9, 9] != 0).any()


# ---------------------------------------------------------------------------------------
# R40-R42: allocation and the first observation of a plane
# ---------------------------------------------------------------------------------------
def _fused_wall(x0=0.8, frames=1, n=(-1.0, 0.0, 0.0), K=None, pose=None):
    K = K or pinhole(32, 24, 30.0)
    pose = look_at([0, 0, 0], [1, 0, 0]) if pose is None else pose
    fr = scenes.analytic_frame(_wall_patches(x0, n=n), pose, K)
    F = oracle.OracleFusion(S, TAU, TH, 20000)
    news = [F.fuse(fr.depth, fr.normal, fr.color, pose, K) for _ in range(frames)]
    return F, fr, news, pose, K


def test_plane_allocates_only_admitted_directions_and_is_idempotent():
    """A plane with normal -x admits only X- (w_dir^D(n) > 0 iff the angle to v^D is below theta,
    eq:angular_threshold P:80); re-fusing the same frame allocates nothing (SPEC allocate
    idempotence); every allocated block holds a point within tau of the plane."""
    F, fr, news, pose, K = _fused_wall(frames=2)
    vol = F.volume()
    assert news[0] > 0 and news[1] == 0
    assert (vol.keys[:, 3] == 1).all()
    lo = vol.keys[:, 0].astype(np.float64) * 8 * S
    assert np.all(lo - 0.8 <= TAU + 1e-9) and np.all(lo + 7 * S - 0.8 >= -TAU - 1e-9)


def test_first_observation_is_the_point_to_plane_distance():
    """eq:point-to-plane with the sign of reading R6: after one frame every
    updated voxel holds clamp((x0 - x)/tau, -1, 1), positive in front of the wall; voxels more
    than tau behind are untouched (weight 0)."""
    x0 = 0.8037
    F, fr, news, pose, K = _fused_wall(x0)
    vol = F.volume()
    X = _voxel_centres(vol)
    upd = vol.weight > 0
    d = (x0 - X[..., 0]) / TAU
    band = upd & (np.abs(d) <= 1.0)
    assert band.sum() > 500
    assert np.abs(vol.sdf[band] - d[band]).max() < 2e-6
    assert not (upd & (d < -1.0 - 1e-6)).any()


def test_weights_follow_the_printed_factors_on_the_optical_axis():
    """On the optical axis of a camera facing the wall, w_angle = 1 and w_dir = 1, so the fused
    weight is w_ICP(z) = 1 / (z + (1 - z_min))^2 (eq:ICP_weight) with z the depth."""
    x0 = 0.8
    K = pinhole(33, 25, 30.0, z_min=0.1)
    F, fr, news, pose, K = _fused_wall(x0, K=K)
    vol = F.volume()
    X = _voxel_centres(vol)
    on_axis = (np.abs(X[..., 1]) < 1e-9) & (np.abs(X[..., 2]) < 1e-9) & (vol.weight > 0) & \
              (np.abs(X[..., 0] - x0) < TAU)
    assert on_axis.sum() >= 4
    assert np.allclose(vol.weight[on_axis], 1.0 / (x0 + (1 - 0.1)) ** 2, rtol=1e-6)


def test_running_average_fixed_point_and_weight_cap():
    """SPEC fusion invariant: after k identical observations the sdf equals the observation and
    the weight is min(k w_1, w_max) (weighted cumulative moving average)."""
    F1, _, _, _, _ = _fused_wall(frames=1)
    F5, _, _, _, _ = _fused_wall(frames=5)
    a, b = F1.volume(), F5.volume()
    assert np.array_equal(a.keys, b.keys)
    upd = a.weight > 0
    assert np.abs(a.sdf[upd] - b.sdf[upd]).max() < 1e-6
    assert np.allclose(b.weight[upd], np.minimum(5 * a.weight[upd], 128.0), rtol=1e-5)
    # the cap: 300 observations of weight w ~ 0.3 saturate at 128
    F = oracle.OracleFusion(S, TAU, TH, 20000)
    K = pinhole(8, 6, 8.0)
    pose = look_at([0, 0, 0], [1, 0, 0])
    fr = scenes.analytic_frame(_wall_patches(0.3), pose, K)
    for _ in range(300):
        F.fuse(fr.depth, fr.normal, fr.color, pose, K)
    assert F.volume().weight.max() == pytest.approx(128.0)


def test_blending_band_splits_membership():
    """A plane at 45 degrees between -x and -y lies in the overlap of X- and Y- (w_dir = 1/2 each,
    eq:direction_weight with reading R1): both directions get blocks, and a voxel fused in both
    gets equal weights and equal distances."""
    n = np.array([-1.0, -1.0, 0.0]) / np.sqrt(2)
    pose = look_at([0, 0, 0], [0.5, 0.5, 0.0])
    F, fr, news, _, K = _fused_wall(0.7, n=n, pose=pose)
    vol = F.volume()
    assert set(vol.keys[:, 3]) == {1, 3}
    idx = {tuple(k): b for b, k in enumerate(vol.keys)}
    pairs = 0
    for b, k in enumerate(vol.keys):
        if k[3] == 1 and (k[0], k[1], k[2], 3) in idx:
            o = idx[(k[0], k[1], k[2], 3)]
            both = (vol.weight[b] > 0) & (vol.weight[o] > 0)
            assert np.allclose(vol.weight[b][both], vol.weight[o][both], rtol=1e-6)
            assert np.allclose(vol.sdf[b][both], vol.sdf[o][both], atol=1e-7)
            pairs += both.sum()
    assert pairs > 100


def test_every_admitted_direction_is_allocated_at_any_height():
    """A plane whose normal (cos 38.7 deg to +x, cos 51.3 deg to +y) admits X+ and Y+, placed above
    z = 0: both directions are allocated over the same block locations (a direction must never
    alias another one's key)."""
    n = np.array([0.78, 0.625, 0.0])
    n /= np.linalg.norm(n)
    c = np.array([0.0, 0.0, 1.3])
    pat = scenes.Patches.empty()
    u = np.cross(n, [0, 0, 1.0])
    pat.extend(c, n, u / np.linalg.norm(u), np.array([0, 0, 1.0]), 0.6, 0.6, [5, 6, 7])
    K = pinhole(40, 30, 30.0)
    pose = look_at(c + 0.9 * n, c)
    fr = scenes.analytic_frame(pat, pose, K)
    F = oracle.OracleFusion(S, TAU, TH, 40000)
    F.fuse(fr.depth, fr.normal, fr.color, pose, K)
    keys = F.volume().keys
    assert set(keys[:, 3]) == {0, 2}
    assert {tuple(k[:3]) for k in keys if k[3] == 0} == {tuple(k[:3]) for k in keys if k[3] == 2}
    assert (keys[:, 2] > 0).all()


# ---------------------------------------------------------------------------------------
# R43: free-space carving and its depth-edge guard
# ---------------------------------------------------------------------------------------
def test_carving_removes_a_spurious_surface_but_not_at_depth_edges():
    """A spurious blob (negative sdf) in front of a wall is carved towards +1 by repeated
    observations of the wall behind it; voxels whose pixel has a depth jump > tau within two
    pixels are not carved."""
    K = pinhole(40, 30, 30.0)
    pose = look_at([0, 0, 0], [1, 0, 0])
    F = oracle.OracleFusion(S, TAU, TH, 40000)
    blob = _wall_patches(0.5, half=0.05)  # a small square at x = 0.5 (the "spurious" surface)
    fr_blob = scenes.analytic_frame(blob, pose, K)
    F.fuse(fr_blob.depth, fr_blob.normal, fr_blob.color, pose, K)
    wall = _wall_patches(1.2)
    fr = scenes.analytic_frame(wall, pose, K)
    for _ in range(20):
        F.fuse(fr.depth, fr.normal, fr.color, pose, K)
    vol = F.volume()
    X = _voxel_centres(vol)
    near_blob = (np.abs(X[..., 0] - 0.5) < 0.005) & (np.abs(X[..., 1]) < 0.03) & (np.abs(X[..., 2]) < 0.03)
    assert near_blob.sum() > 10 and (vol.sdf[near_blob] > 0).all()
    # guard: a depth edge (blob and wall in the same frame) keeps the blob's rim from carving
    F2 = oracle.OracleFusion(S, TAU, TH, 40000)
    F2.fuse(fr_blob.depth, fr_blob.normal, fr_blob.color, pose, K)
    both = scenes.Patches.empty()
    for p in (blob, wall):
        both.extend(p.q[0], p.n[0], p.u[0], p.v[0], p.hu[0], p.hv[0], p.color[0])
    fr2 = scenes.analytic_frame(both, pose, K)
    w_before = F2.volume().weight.copy()
    F2.fuse(fr2.depth, fr2.normal, fr2.color, pose, K)
    v2 = F2.volume()
    X2 = _voxel_centres(v2)
    # voxels of the blob volume far in front of the wall that project onto wall pixels within two
    # pixels of the blob's silhouette: d > 1 (free space) but guarded
    xc = X2[..., 0]
    u = 30.0 * (-X2[..., 1]) / xc + 19.5
    v = 30.0 * (-X2[..., 2]) / xc + 14.5
    sil = fr2.depth > 1.0
    edge = np.zeros_like(sil)
    for dv in range(-2, 3):
        for du in range(-2, 3):
            edge |= np.roll(np.roll(fr2.depth < 1.0, dv, 0), du, 1)
    iu, iv = np.floor(u + 0.5).astype(int), np.floor(v + 0.5).astype(int)
    ok = (iu >= 2) & (iu < 38) & (iv >= 2) & (iv < 28) & (np.abs(xc - 0.5) > TAU + 0.01) & (xc < 1.2 - TAU - 0.01)
    guarded = ok.copy()
    guarded[ok] = sil[iv[ok], iu[ok]] & edge[iv[ok], iu[ok]]
    assert guarded.sum() > 0
    n0 = v2.n_blocks if w_before.shape[0] == v2.n_blocks else w_before.shape[0]
    assert np.array_equal(v2.weight[:n0][guarded[:n0]], w_before[guarded[:n0]])


# ---------------------------------------------------------------------------------------
# R46: the closed loop fuse -> render against closed-form geometry
# ---------------------------------------------------------------------------------------
def test_fused_room_renders_the_analytic_scene(c1):
    """configs[1] room fused from 6 seeded ideal depth frames, then rendered (direct oracle) from
    one of them: depth equals the analytic ray hit to 1e-5 m on >= 88 % of the pixels both see
    (within 1 cm on >= 95 %: near edges and corners voxel projection blends surfaces),
    normals within 1e-4 rad on 95 % of those, colours exact on 90 %."""
    K = scenes.Intrinsics(fx=262.5, fy=262.5, cx=159.5, cy=119.5, width=320, height=240)
    poses = scenes.room_scan_poses(np.random.default_rng([7, 0]), 6)
    F = oracle.OracleFusion(S, TAU, TH, 60000)
    for P in poses:
        fr = scenes.analytic_frame(c1.patches, P, K)
        F.fuse(fr.depth, fr.normal, fr.color, P, K)
    out = oracle.OracleVolume(F.volume()).render(poses[0], K)
    fr = scenes.analytic_frame(c1.patches, poses[0], K)
    both = (out["depth"] > 0) & (fr.depth > 0)
    assert both.mean() > 0.7
    err = np.abs(out["depth"] - fr.depth)
    good = err < 1e-5  # face interiors: the fused band is the exact point-to-plane distance
    assert good[both].mean() > 0.88 and (err[both] < 0.01).mean() > 0.95  # edges/corners blend
    R = np.asarray(poses[0], np.float64)[:3, :3]
    nw = fr.normal.reshape(-1, 3) @ R.T
    sel = (both & good).reshape(-1)
    assert np.quantile(angle_between(out["normal"].reshape(-1, 3)[sel], nw[sel]), 0.95) < 1e-4  # edge pixels excepted
    assert (out["color"][both & good] == fr.color[both & good]).all(1).mean() > 0.9


def test_capacity_exhaustion_raises():
    K = pinhole(16, 12, 15.0)
    pose = look_at([0, 0, 0], [1, 0, 0])
    fr = scenes.analytic_frame(_wall_patches(0.8), pose, K)
    F = oracle.OracleFusion(S, TAU, TH, 3)
    with pytest.raises(MemoryError):
        F.fuse(fr.depth, fr.normal, fr.color, pose, K)


def test_carve_weight_zero_means_no_carving():
    """R43 with carve_weight 0 (include/dtsdf.h: 0 = no carving): voxels in front of the surface
    keep their values -- a fresh block's free-space voxels stay at sdf 1, weight 0 (the running
    average would otherwise be 0/0) -- and everything else equals the fusion with carving on."""
    K = pinhole(40, 30, 30.0)
    pose = look_at([0, 0, 0], [1, 0, 0])
    fr = scenes.analytic_frame(_wall_patches(0.8), pose, K)
    F0 = oracle.OracleFusion(S, TAU, TH, 40000)
    F1 = oracle.OracleFusion(S, TAU, TH, 40000)
    F0.fuse(fr.depth, fr.normal, fr.color, pose, K, carve_weight=0.0)
    F1.fuse(fr.depth, fr.normal, fr.color, pose, K)
    v0, v1 = F0.volume(), F1.volume()
    assert np.array_equal(v0.keys, v1.keys)
    assert np.isfinite(v0.sdf).all() and np.isfinite(v0.weight).all()
    carved = v1.weight != v0.weight
    free = (v0.weight == 0) & (v0.sdf == 1.0)
    assert carved.any() and (carved <= free).all()  # carving touched only free-space voxels
    assert np.array_equal(v0.sdf[~carved], v1.sdf[~carved])
