"""Pins of the combined-TSDF oracle (readings R33-R38 in DESIGN.md §4).

The combined TSDF is the view-dependent regular TSDF of Lemma 1, computed per
voxel of the (widened) view frustum with the combination weights and the
6-neighbour gradient, then raycast like a regular TSDF.  The pins
are closed-form geometry, special cases with known answers, invariants, and the paper's own
statements of the recombination conditions."""
import numpy as np
import pytest

import oracle
import scenes
from helpers import angle_between, block_cube, field_volume, pinhole, project
from scenes import DIRECTION_VECTORS, look_at
from test_oracle_pins import _plate, _wall

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")
TH = np.deg2rad(65.0)


def _vox_grid(vol):
    """Integer positions of every voxel of every allocated block location, with their keys."""
    locs = np.unique(vol.keys[:, :3], axis=0).astype(np.int64)
    off = scenes.local_offsets().astype(np.int64)  # [512, 3] (lx, ly, lz) in l order
    return (locs[:, None, :] * 8 + off[None]).reshape(-1, 3)


def _stored(vol, D, ijk):
    """Stored (sdf, weight) of direction D at voxels ijk (NaN where unallocated) -- input lookup."""
    index = {tuple(k[:3]): b for b, k in enumerate(vol.keys) if k[3] == D}
    off = scenes.local_offsets()
    lidx = {tuple(o): l for l, o in enumerate(off)}
    sdf = np.full(len(ijk), np.nan)
    w = np.full(len(ijk), np.nan)
    for q, (i, j, k) in enumerate(ijk):
        b = index.get((i // 8, j // 8, k // 8))
        if b is None:
            continue
        l = lidx[(i % 8, j % 8, k % 8)]
        sdf[q] = vol.sdf[b, l]
        w[q] = vol.weight[b, l]
    return sdf, w


# ---------------------------------------------------------------------------------------
# R34: combined voxels -- special cases with known answers
# ---------------------------------------------------------------------------------------
def test_single_direction_combined_equals_its_sdf():
    """SPEC build_combined example 1: a volume with a single direction populated -> the combined
    sdf equals that direction's sdf wherever it is visible (W > 0); the mask is that direction."""
    vol = _wall()  # wall x = 0.5303 facing -x, stored in X- only
    ov = oracle.OracleVolume(vol)
    K = pinhole(32, 24, 40.0)
    pose = look_at([0, 0, 0], [1, 0, 0])
    ijk = _vox_grid(vol)
    cv = oracle.combined_voxels(ov, pose, K, ijk)
    sdf, w = _stored(vol, 1, ijk)
    v = cv["valid"]
    assert v.sum() > 1000
    assert np.abs(cv["sdf"][v] - sdf[v]).max() < 1e-12  # W phi / W, one rounding
    assert (cv["mask"][v] == 2).all() and (cv["mask"][~v] == 0).all()
    assert (cv["rgb"][v] == [10, 200, 30]).all()


def test_agreeing_directions_give_either_input():
    """SPEC build_combined example 3: two directions mapping the same plane with equal data ->
    the combined sdf equals either input, whatever the combination weights."""
    n = np.array([1.0, 1.0, 0.0]) / np.sqrt(2)  # a 45-degree plane stored in X- and Y- alike

    def field(D, X):
        return np.clip((0.6 - X @ n) / 0.04, -1, 1), np.full(len(X), 2.0), np.tile([7, 8, 9], (len(X), 1))
    vol = field_volume(block_cube((2, 2, -2), (7, 7, 1), [1, 3]), field, 0.01, truncation=0.04)
    ov = oracle.OracleVolume(vol)
    K = pinhole(40, 30, 30.0)
    pose = look_at([0, 0, 0], [0.42, 0.42, 0.0])
    ijk = _vox_grid(vol)
    cv = oracle.combined_voxels(ov, pose, K, ijk)
    sdf, _ = _stored(vol, 1, ijk)
    v = cv["valid"]
    assert v.sum() > 1000
    assert np.abs(cv["sdf"][v] - sdf[v]).max() < 1e-12
    assert (cv["rgb"][v] == [7, 8, 9]).all()
    # both directions face the camera and admit the 45-degree normal (w_dir = 1/2 each)
    assert (cv["mask"][v] == 0b1010).mean() > 0.9


def test_back_face_and_foreign_direction_get_no_weight():
    """eq:combine_weight factors: a plane seen from behind (<n,-r> <= 0) and a
    plane stored in a direction whose axis is beyond theta from its normal contribute nothing."""
    vol = _wall()
    ov = oracle.OracleVolume(vol)
    K = pinhole(32, 24, 40.0)
    behind = look_at([1.2, 0, 0], [0.5, 0, 0])  # looks at the wall's back (-x facing wall, camera at +x)
    cv = oracle.combined_voxels(ov, behind, K, _vox_grid(vol))
    assert not cv["valid"].any()

    def field(D, X):  # a +z-facing floor stored in X+ (foreign: angle 90 deg > theta)
        return np.clip((X[:, 2] + 0.3) / 0.04, -1, 1), np.ones(len(X)), np.zeros((len(X), 3))
    foreign = field_volume(block_cube((-2, -2, -5), (1, 1, -3), [0]), field, 0.01, truncation=0.04)
    ijk = _vox_grid(foreign)
    cv = oracle.combined_voxels(oracle.OracleVolume(foreign), look_at([0, 0, 0.5], [0, 0.01, -0.3]), K, ijk)
    # gradient present: inside the band and off the allocation's rim (clipped and rim voxels have
    # no gradient and fall back to eq. 9)
    band = (np.abs(ijk[:, 2] * 0.01 + 0.3) < 0.04 - 0.015) & (np.abs(ijk[:, :2] + 0.5) < 15).all(1)
    assert band.sum() > 1000 and not cv["valid"][band].any()


def test_no_gradient_fallback_combined_voxel():
    """eq:combine_tsdf_weight (SPEC combine_weight_nograd): with constant fields
    (no gradient anywhere) a direction whose axis faces the camera (<v^D,-r> > 0) gives its own
    sdf; one facing away gives nothing."""
    def field(D, X):
        return np.full(len(X), 0.25), np.ones(len(X)), np.zeros((len(X), 3))
    vol = field_volume(block_cube((2, -1, -1), (3, 0, 0), [1]), field, 0.01, truncation=0.04)  # X- = (-1,0,0)
    ov = oracle.OracleVolume(vol)
    K = pinhole(32, 24, 20.0)
    ijk = _vox_grid(vol)
    cv = oracle.combined_voxels(ov, look_at([0, 0, 0], [1, 0, 0]), K, ijk)  # camera at -x side: <v,-r> > 0
    assert cv["valid"].sum() > 500 and np.all(cv["sdf"][cv["valid"]] == 0.25)
    cv = oracle.combined_voxels(ov, look_at([1.0, 0, 0], [0, 0, 0]), K, ijk)  # camera at +x: facing away
    assert not cv["valid"].any()


def test_convex_combination_on_c1_voxels(c1):
    """SPEC invariant: the combined sdf lies in [min_D sdf^D, max_D sdf^D] over the contributing
    directions (mask bits), and the colour in the hull of their colours."""
    vol = c1.volume
    ov = oracle.OracleVolume(vol)
    rng = np.random.default_rng(5)
    ijk = _vox_grid(vol)
    ijk = ijk[rng.choice(len(ijk), 40000, replace=False)]
    cv = oracle.combined_voxels(ov, c1.poses[0], c1.intrinsics, ijk)
    v = cv["valid"]
    assert v.sum() > 3000
    per = np.stack([_stored(vol, D, ijk[v])[0] for D in range(6)], 1)
    m = cv["mask"][v]
    bits = ((m[:, None] >> np.arange(6)) & 1).astype(bool)
    assert bits.any(1).all()
    lo = np.where(bits, per, np.inf).min(1)
    hi = np.where(bits, per, -np.inf).max(1)
    s = cv["sdf"][v]
    assert np.all(s >= lo - 1e-12) and np.all(s <= hi + 1e-12)


# ---------------------------------------------------------------------------------------
# R33: the widened frustum
# ---------------------------------------------------------------------------------------
def test_frustum_margin_is_one_eighth_of_the_image():
    """Voxels projecting up to W/8 (H/8) pixels beyond the image border are combined, voxels
    further out or outside [z_min, z_max] are not."""
    def field(D, X):
        return np.full(len(X), 0.5), np.ones(len(X)), np.zeros((len(X), 3))
    vol = field_volume(block_cube((-20, -20, 9), (19, 19, 10), [5]), field, 0.01, truncation=0.04)  # Z- faces a +z camera
    ov = oracle.OracleVolume(vol)
    K = pinhole(64, 48, 50.0, z_min=0.1, z_max=0.8)
    pose = np.eye(4)  # camera at the origin looking +z
    ijk = _vox_grid(vol)
    cv = oracle.combined_voxels(ov, pose, K, ijk)
    u, v, z = project(pose, K, ijk * 0.01)
    inside = (u >= -8) & (u <= 63 + 8) & (v >= -6) & (v <= 47 + 6) & (z >= 0.1) & (z <= 0.8)
    clear = (np.abs(u + 8) > 1e-6) & (np.abs(u - 71) > 1e-6) & (np.abs(v + 6) > 1e-6) & (np.abs(v - 53) > 1e-6) \
        & (np.abs(z - 0.8) > 1e-9)
    assert inside.sum() > 5000 and (~inside).sum() > 5000
    assert np.array_equal(cv["valid"][clear], inside[clear])


# ---------------------------------------------------------------------------------------
# R36-R37: raycast of the combined TSDF -- closed forms
# ---------------------------------------------------------------------------------------
def test_combined_plane_depth_normal_color_closed_form():
    """Wall x = x0 rendered through its combined TSDF from the source pose: depth = x0 (camera z)
    to 1e-6, normal (-1,0,0), colour exact, mask {X-} (PAPER.md:253 'used like a regular TSDF')."""
    x0 = 0.5303
    ov = oracle.OracleVolume(_wall(x0))
    K = pinhole(32, 24, 40.0)
    pose = look_at([0, 0, 0], [1, 0, 0])
    out = oracle.render_combined(ov, pose, K, pose, K)
    d = out["depth"]
    assert (d > 0).all() and np.abs(d - x0).max() < 1e-6
    assert np.allclose(out["normal"], [-1, 0, 0], atol=1e-9)
    assert (out["color"] == [10, 200, 30]).all() and (out["mask"] == 2).all()


def test_combined_c0_sphere_closed_form(c0):
    """configs[0] through the combined TSDF: every direction stores the same field, so the
    combined voxels equal the stored sdf; depth within 0.5 mm of the closed-form sphere below
    75 deg incidence, radial normals within 0.1 deg, disagreements only at the silhouette."""
    K = c0.intrinsics
    pose = c0.poses[0]
    ov = oracle.OracleVolume(c0.volume)
    ijk = _vox_grid(c0.volume)
    cv = oracle.combined_voxels(ov, pose, K, ijk)
    sdf0, _ = _stored(c0.volume, 0, ijk)
    assert cv["valid"].sum() > 20000
    assert np.abs(cv["sdf"][cv["valid"]] - sdf0[cv["valid"]]).max() < 1e-12
    out = oracle.render_combined(ov, pose, K, pose, K)
    d = out["depth"]
    o, r, L = oracle.ray_dirs(pose, K)
    b = r @ o
    disc = b * b - (o @ o - 0.04)
    t = -b - np.sqrt(np.maximum(disc, 0))
    z = np.where(disc >= 0, t / L, 0.0).reshape(d.shape)
    hit_cf, hit = z > 0, d > 0
    pad = np.pad(hit_cf, 1, mode="edge")
    edge = np.zeros_like(hit_cf)
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            edge |= pad[1 + dy:61 + dy, 1 + dx:81 + dx] != hit_cf
    assert not ((hit != hit_cf) & ~edge).any()
    X = o + t[:, None] * r
    n = X / np.linalg.norm(X, axis=1, keepdims=True)
    inc = (-(n * r).sum(1)).reshape(d.shape)
    sel = hit & hit_cf & (inc > np.cos(np.deg2rad(75)))
    assert sel.sum() > 1700
    assert np.abs(d - z)[sel].max() < 5e-4
    Xr = (o + (d.ravel() * L)[:, None] * r).reshape(60, 80, 3)
    assert np.max(angle_between(out["normal"][sel], Xr[sel])) < np.deg2rad(0.1)
    assert ((out["mask"] > 0) == hit).all()


def test_combined_thin_plate_lemma1():
    """Lemma 1 (Fig. 3): the combined TSDF computed for a camera in front of a
    3 mm plate holds only the front face (its back-face directions get zero weight), so the
    render shows the front face at the closed-form depth with its colour; from behind, the back
    face.  A combined TSDF is view-dependent: the front camera's one shows no back face."""
    pat, c, n = _plate()
    vol = scenes.patch_fill(pat, voxel_size=0.005, truncation=0.02, theta=TH)
    ov = oracle.OracleVolume(vol)
    K = pinhole(48, 36, 60.0)
    band = 0.02 + 2 * 0.005
    for side, pid, col in ((1, 0, [200, 30, 40]), (-1, 1, [20, 90, 250])):
        pose = look_at(c + side * 0.5 * n, c)
        out = oracle.render_combined(ov, pose, K, pose, K)
        o, r, L = oracle.ray_dirs(pose, K)
        t, hitp = pat.ray_hit(o, r)
        X = o + np.where(np.isfinite(t), t, 0)[:, None] * r
        rel = X - pat.q[pid]
        interior = ((hitp == pid) & (np.abs(rel @ pat.u[pid]) < pat.hu[pid] - band) &
                    (np.abs(rel @ pat.v[pid]) < pat.hv[pid] - band)).reshape(36, 48)
        assert interior.sum() > 200 and (out["depth"][interior] > 0).all()
        zc = np.where(np.isfinite(t), t / L, 0).reshape(36, 48)
        # occupied voxels inside the plate average the front and back distances by their stored
        # weights (R57), which moves the root by a fraction of a voxel (the paper's "dents")
        err = np.abs(out["depth"] - zc)[interior]
        print("alg1 plate", side, err.max(), err.mean(), (out["color"][interior] == col).all(1).mean())
        assert err.max() < 0.5 * 0.005 and err.mean() < 1e-3
        other = [20, 90, 250] if pid == 0 else [200, 30, 40]
        cpx = out["color"][interior].astype(int)
        nearer = np.abs(cpx - col).sum(1) < np.abs(cpx - other).sum(1)
        print("alg1 nearer", nearer.mean())
        assert nearer.mean() > 0.9  # blended, but the visible face dominates
        assert np.max(angle_between(out["normal"][interior], np.tile(side * n, (interior.sum(), 1)))) < 1e-6
        admit = sum(1 << D for D in range(6) if side * n @ DIRECTION_VECTORS[D] > np.cos(TH))
        assert ((out["mask"][interior].astype(int) & ~admit) == 0).all()
        # the other side's combined TSDF, looked at from this side, has no surface facing here
        other = look_at(c - side * 0.5 * n, c)
        cv = oracle.combined_voxels(ov, other, K, _vox_grid(vol))
        assert ((cv["mask"][cv["valid"]].astype(int) & admit & ~sum(
            1 << D for D in range(6) if -side * n @ DIRECTION_VECTORS[D] > np.cos(TH))) == 0).all()


def test_combined_equals_direct_on_affine_single_direction_fields():
    """Where one direction carries an affine field and is the only contributor, combining then
    interpolating equals interpolating then combining: the combined render equals the direct
    render (depth 1e-9, normal 1e-9, colour and mask exact) -- a reduction to the direct path."""
    ov = oracle.OracleVolume(_wall(0.61))
    K = pinhole(24, 18, 30.0)
    pose = look_at([0.02, -0.01, 0.01], [1, 0.05, -0.03])
    a = oracle.render_combined(ov, pose, K, pose, K)
    b = ov.render(pose, K)
    assert (a["depth"] > 0).all()
    assert np.abs(a["depth"] - b["depth"]).max() < 1e-9
    assert np.abs(a["normal"] - b["normal"]).max() < 1e-9
    assert (a["color"] == b["color"]).all() and (a["mask"] == b["mask"]).all()


def test_combined_render_from_moved_pose_uses_source_weights():
    """The combined TSDF belongs to its source pose (Lemma 1): rendering a nearby pose through it
    differs from combining at the nearby pose only through the weights, so on a single-direction
    plane (weights irrelevant) both give the same closed-form depth."""
    x0 = 0.5303
    ov = oracle.OracleVolume(_wall(x0))
    K = pinhole(32, 24, 40.0)
    src = look_at([0, 0, 0], [1, 0, 0])
    moved = look_at([0.03, 0.01, -0.02], [1, 0.02, 0])
    out = oracle.render_combined(ov, src, K, moved, K)
    o, r, L = oracle.ray_dirs(moved, K)
    t = (x0 - o[0]) / r[:, 0]
    z = (t / L).reshape(24, 32)
    hit = out["depth"] > 0
    assert hit.mean() > 0.9
    assert np.abs(out["depth"] - z)[hit].max() < 1e-6


# ---------------------------------------------------------------------------------------
# R38: conditional combination (eqs. condition_1-4)
# ---------------------------------------------------------------------------------------
def _pose(tx=0.0, angle=0.0):
    T = np.eye(4)
    c, s = np.cos(angle), np.sin(angle)
    T[:3, :3] = [[c, -s, 0], [s, c, 0], [0, 0, 1]]
    T[0, 3] = tx
    return T


@pytest.mark.parametrize("frame,last,tx,ang,want", [
    (3, 3, 0.0, 0.0, True),                        # boot up: framesSinceStart < 5
    (4, 4, 0.0, 0.0, True),
    (5, 4, 0.0, 0.0, False),
    (60, 9, 0.0, 0.0, True),                       # stale: 51 frames since the update
    (59, 9, 0.0, 0.0, False),                      # exactly 50 is not > 50
    (30, 20, 0.04, 0.02 * np.pi / 2, False),       # all four conditions false (SPEC example 3)
    (30, 20, 0.06, 0.0, True),                     # translation > 0.05 m
    (30, 20, 0.0, 0.06 * np.pi / 2, True),         # rotation > 0.05 pi/2
])
def test_should_recombine_conditions(frame, last, tx, ang, want):
    assert oracle.should_recombine(frame, last, _pose(tx, ang), _pose()) is want


# ---------------------------------------------------------------------------------------
# NEXT-4: Algorithm 1 (readings R53-R57) as combination mode 1
# ---------------------------------------------------------------------------------------
def _one_sided_wall(facing):
    """Wall x = 0.6 whose stored face normal is `facing` (+1: +x, stored in X+; -1: -x, in X-)."""
    D = 0 if facing > 0 else 1

    def field(Dq, X):
        return np.clip(facing * (X[:, 0] - 0.6) / 0.04, -1, 1), np.ones(len(X)), np.tile([40, 50, 60], (len(X), 1))
    return field_volume(block_cube((6, -3, -3), (8, 2, 2), [D]), field, 0.01, truncation=0.04)


def test_algorithm1_free_space_without_transition_keeps_the_field():
    """q = none ("if q = empty then freespace = 1"): in front of a camera-facing wall the
    back-march towards the camera leaves the direction's data without a transition, so the voxel
    is free space and keeps its stored distance; behind the face it is occupied space."""
    vol = _one_sided_wall(-1)
    ov = oracle.OracleVolume(vol)
    K = pinhole(32, 24, 30.0)
    pose = look_at([0, 0, 0], [1, 0, 0])
    ijk = _vox_grid(vol)
    cv = oracle.combined_voxels(ov, pose, K, ijk, mode=1)
    sdf, _ = _stored(vol, 1, ijk)
    band = np.abs(sdf) < 0.74  # gradient present (inside the band, R53)
    inner = band & (np.abs(ijk[:, 1:] + 0.5) < 20).all(1)
    assert inner.sum() > 1000 and cv["valid"][inner].all()
    assert np.abs(cv["sdf"][inner] - sdf[inner]).max() < 1e-12
    assert (cv["mask"][inner] == 2).all()


def test_algorithm1_transition_in_free_space_is_free():
    """Fig. 4's p2: behind a wall whose stored face looks away from the camera, the back-march
    finds the face (q) but no other direction is occupied there, so the voxel stays free space --
    where eq:combine_weight gives it no weight at all (<n, -r> < 0)."""
    vol = _one_sided_wall(+1)
    ov = oracle.OracleVolume(vol)
    K = pinhole(32, 24, 30.0)
    pose = look_at([0, 0, 0], [1, 0, 0])
    ijk = _vox_grid(vol)
    sdf, _ = _stored(vol, 0, ijk)
    a1 = oracle.combined_voxels(ov, pose, K, ijk, mode=1)
    w8 = oracle.combined_voxels(ov, pose, K, ijk, mode=0)
    free = (sdf > 0) & (sdf < 0.74) & (np.abs(ijk[:, 1:] + 0.5) < 20).all(1)
    assert free.sum() > 500
    assert a1["valid"][free].all() and np.abs(a1["sdf"][free] - sdf[free]).max() < 1e-12
    assert not w8["valid"][free].any()
    # rendering from that camera sees no surface: a back face is never a +->- transition
    out = oracle.render_combined(ov, pose, K, pose, K, mode=1)
    assert (out["depth"] == 0).all()


def test_algorithm1_hidden_point_is_occupied_and_thin_plate_renders():
    """Fig. 4's p1 / Lemma 1: behind a thin plate seen from the front, the back
    direction's free space ends at the back face, which lies in the occupied space of the visible
    front face -> not free; the render through the Algorithm-1 TSDF shows the front face at the
    closed-form depth with its colour, from either side."""
    pat, c, n = _plate()
    vol = scenes.patch_fill(pat, voxel_size=0.005, truncation=0.02, theta=TH)
    ov = oracle.OracleVolume(vol)
    K = pinhole(48, 36, 60.0)
    band = 0.02 + 2 * 0.005
    for side, pid, col in ((1, 0, [200, 30, 40]), (-1, 1, [20, 90, 250])):
        pose = look_at(c + side * 0.5 * n, c)
        # hidden voxels: beyond the plate (from this camera), within 1 cm of its far face
        ijk = _vox_grid(vol)
        X = ijk * np.float64(np.float32(0.005))
        h = (X - c) @ (side * n)
        lat = np.abs((X - c) @ pat.u[0]) < 0.05
        hidden = (h < -0.004) & (h > -0.012) & lat & (np.abs((X - c) @ pat.v[0]) < 0.04)
        cv = oracle.combined_voxels(ov, pose, K, ijk[hidden], mode=1)
        assert cv["valid"].sum() > 50 and (cv["sdf"][cv["valid"]] < 0).all()
        out = oracle.render_combined(ov, pose, K, pose, K, mode=1)
        o, r, L = oracle.ray_dirs(pose, K)
        t, hitp = pat.ray_hit(o, r)
        Xh = o + np.where(np.isfinite(t), t, 0)[:, None] * r
        rel = Xh - pat.q[pid]
        interior = ((hitp == pid) & (np.abs(rel @ pat.u[pid]) < pat.hu[pid] - band) &
                    (np.abs(rel @ pat.v[pid]) < pat.hv[pid] - band)).reshape(36, 48)
        assert interior.sum() > 200 and (out["depth"][interior] > 0).all()
        zc = np.where(np.isfinite(t), t / L, 0).reshape(36, 48)
        # occupied voxels inside the plate average the front and back distances by their stored
        # weights (R57), which moves the root by a fraction of a voxel (the paper's "dents")
        err = np.abs(out["depth"] - zc)[interior]
        print("alg1 plate", side, err.max(), err.mean(), (out["color"][interior] == col).all(1).mean())
        assert err.max() < 0.5 * 0.005 and err.mean() < 1e-3
        other = [20, 90, 250] if pid == 0 else [200, 30, 40]
        cpx = out["color"][interior].astype(int)
        nearer = np.abs(cpx - col).sum(1) < np.abs(cpx - other).sum(1)
        print("alg1 nearer", nearer.mean())
        assert nearer.mean() > 0.9  # blended, but the visible face dominates


def _facing_walls(delta):
    """X+ (D = 0) stores a wall at x = 0.6 facing +x (away from a camera at the origin looking
    +x); X- (D = 1) stores a wall at x = 0.6 - delta facing the camera.  Input fields only."""
    def field(D, X):
        if D == 0:
            return np.clip((X[:, 0] - 0.6) / 0.04, -1, 1), np.ones(len(X)), np.tile([10, 20, 30], (len(X), 1))
        return np.clip(-(X[:, 0] - (0.6 - delta)) / 0.04, -1, 1), np.ones(len(X)), np.tile([200, 100, 50], (len(X), 1))
    return field_volume(block_cube((6, -3, -3), (8, 2, 2), [0, 1]), field, 0.01, truncation=0.04)


@pytest.mark.parametrize("delta,occupied", [(4e-3, True), (2e-8, True), (-2e-8, False), (-4e-3, False)])
def test_algorithm1_conflict_test_is_strictly_negative(delta, occupied):
    """P:203-204, Algorithm 1: D's free space fails iff another direction D~ has
    "Phi^D~(q) < 0 and <n^D~(q), -r> > 0" at D's first zero transition q towards the camera.
    Voxels p just behind x = 0.6 are free in X+ (phi > 0, its transition q at x = 0.6) and
    occupied in X- (phi < 0, a camera-facing surface at 0.6 - delta).  q lies delta inside X-'s
    occupied space: for every delta > 0 -- even 2e-8 m, Phi^X-(q) = -5e-7 -- the free space
    conflicts and p takes the occupied direction's value; for delta < 0 (q in front of X-'s
    surface, Phi^X-(q) > 0) it stays free.  The 2e-8 cases pin the strict "< 0" against any
    threshold (a "< -1e-6" reading keeps them free)."""
    vol = _facing_walls(delta)
    ov = oracle.OracleVolume(vol)
    K = pinhole(32, 24, 30.0)
    pose = look_at([0, 0, 0], [1, 0, 0])
    ijk = np.array([[i, j, k] for i in (61, 62, 63) for j in (-3, 0, 2) for k in (-2, 0, 3)], np.int64)
    cv = oracle.combined_voxels(ov, pose, K, ijk, mode=1)
    s0, _ = _stored(vol, 0, ijk)
    s1, _ = _stored(vol, 1, ijk)
    assert cv["valid"].all() and (s0 > 0).all() and (s1 < 0).all()
    want, mask = (s1, 2) if occupied else (s0, 1)
    assert np.abs(cv["sdf"] - want).max() < 1e-12, (delta, cv["sdf"], want)
    assert (cv["mask"] == mask).all()


def _floor_with_tagged_layer():
    """Z+ (D = 4) holds the floor phi = z / tau (weight 1).  Y+ (D = 2) holds phi = z / tau +
    20 (y - 0.06) with weight 1 only on the voxel layer k = -1 (z = -s) for y in [0.02, 0.05),
    weight 0 elsewhere: its 6-neighbour gradient (0, 20, 25) lies 51 deg from +y (membership > 0,
    P:88-96), so combined voxels of that layer carry the mask {Z+, Y+}; layers k = 0, 1 carry
    {Z+} and layer 0 is exactly 0 (the floor lies on the voxel plane z = 0)."""
    s = 0.01

    def field(D, X):
        if D == 4:
            return X[:, 2] / 0.04, np.ones(len(X)), np.tile([50, 60, 70], (len(X), 1))
        k = np.round(X[:, 2] / s).astype(int)
        j = np.round(X[:, 1] / s).astype(int)
        w = ((k == -1) & (j >= 2) & (j <= 4)).astype(float)
        return X[:, 2] / 0.04 + 20 * (X[:, 1] - 0.06), w, np.tile([200, 10, 10], (len(X), 1))
    return field_volume(block_cube((-1, -1, -1), (0, 0, 0), [4, 2]), field, s, truncation=0.04)


def test_combined_mask_on_a_voxel_plane_root():
    """Reading R37: the combined render's mask is the OR of the masks of the corners with
    trilinear weight >= 1/8.  The floor's root lies exactly on the voxel plane z = 0 (combined
    sdf 0 there), so the shading point b (f <= 0) sits at the top of a cell of layers -1/0 with
    fz -> 1: the layer -1 corners have weight ~0 and the mask is layer 0's {Z+}.  A plain OR over
    all 8 corners would add layer -1's Y+ bit -- whereas b just above the plane would add layer 1's
    mask: which side a root on a voxel plane is refined to must not decide the mask."""
    vol = _floor_with_tagged_layer()
    ov = oracle.OracleVolume(vol)
    K = pinhole(16, 16, 100.0)
    pose = look_at([0.003, 0.035, 0.3], [0.003, 0.035, 0.0], up=(0, 1, 0))
    # the premise: layer -1 voxels of the window are {Z+, Y+}, layers 0 and 1 are {Z+}
    ijk = np.array([[i, j, k] for i in (-1, 0, 1) for j in (2, 3) for k in (-1, 0, 1)], np.int64)
    cv = oracle.combined_voxels(ov, pose, K, ijk)
    assert cv["valid"].all()
    assert (cv["mask"][ijk[:, 2] == -1] == (1 << 4) | (1 << 2)).all()
    assert (cv["mask"][ijk[:, 2] >= 0] == 1 << 4).all()
    assert (cv["sdf"][ijk[:, 2] == 0] == 0).all() and (cv["sdf"][ijk[:, 2] == -1] < 0).all()
    out = oracle.render_combined(ov, pose, K, pose, K)
    o, r, L = oracle.ray_dirs(pose, K)
    y_hit = (o[1] - o[2] / r[:, 2] * r[:, 1]).reshape(16, 16)  # ray / plane z = 0
    win = (y_hit > 0.0205) & (y_hit < 0.0395)
    win[:, :2] = win[:, -2:] = False  # cells reaching beyond the widened frustum (R33) are invalid
    assert win.sum() >= 20 and (out["depth"][win] > 0).all()
    assert np.abs(out["depth"][win] - 0.3).max() < 1e-6  # camera height above the floor
    assert (out["mask"][out["depth"] > 0] == 1 << 4).all()
    assert (out["color"][win] == [50, 60, 70]).all()


# ---------------------------------------------------------------------------------------
# R58: voxels receiving data for the first time are added to the combined TSDF
# ---------------------------------------------------------------------------------------
def _wall_volume(x_old, x_new, by_hi, w_zero_above=None):
    """X- (D = 1) walls facing a camera at the origin: blocks by in [-3, by_hi], bx 6..8, bz -3..2.
    Voxels with y < 0 hold the wall at x_old, y >= 0 at x_new; with w_zero_above, voxels with
    z > w_zero_above store weight 0 (allocated, no data).  Input fields only."""
    def field(D, X):
        x0 = np.where(X[:, 1] < 0, x_old, x_new)
        w = np.ones(len(X)) if w_zero_above is None else (X[:, 2] <= w_zero_above).astype(float)
        return np.clip(-(X[:, 0] - x0) / 0.04, -1, 1), w, np.tile([30, 60, 90], (len(X), 1))
    return field_volume(block_cube((6, -3, -3), (8, by_hi, 2), [1]), field, 0.01, truncation=0.04)


def test_first_time_voxels_are_added_and_stale_voxels_kept():
    """R58 ("Voxels that receive data for the first time are always directly added to the
    combined TSDF"; P:254-256 conditional combination).  The combined TSDF was computed from
    `before`: a wall at x = 0.60 over y < 0, weight 0 above z = 0.05.  Fusion produced `after`:
    the wall at 0.62 everywhere, new blocks over y >= 0, weights 1.  Voxels that had data before
    keep the value combined from `before` (the wall at 0.60, stale); voxels of the new blocks and
    the zero-weight voxels above z = 0.05 take the value combined from `after` (0.62).  Rendered
    from the source camera: depth 0.60 where the old data lies, 0.62 elsewhere (closed forms)."""
    before = _wall_volume(0.60, 0.60, -1, w_zero_above=0.05)
    after = _wall_volume(0.62, 0.62, 2)
    ob, oa = oracle.OracleVolume(before), oracle.OracleVolume(after)
    K = pinhole(48, 36, 40.0)
    pose = look_at([0, 0, 0], [1, 0, 0])
    ijk = _vox_grid(after)
    cv = oracle.combined_voxels(oa, pose, K, ijk, before=ob)
    s_old, w_old = _stored(before, 1, ijk)
    s_new, _ = _stored(after, 1, ijk)
    had = w_old > 0  # NaN (unallocated before) compares False
    inner = (np.abs(s_new) < 0.74) & (np.abs(ijk[:, 1:] + 0.5) < 20).all(1)
    inner &= ~had | (np.abs(s_old) < 0.74)
    assert (inner & had).sum() > 200 and (inner & ~had).sum() > 200
    assert cv["valid"][inner].all()
    assert np.abs(cv["sdf"][inner & had] - s_old[inner & had]).max() < 1e-12   # stale
    assert np.abs(cv["sdf"][inner & ~had] - s_new[inner & ~had]).max() < 1e-12  # added
    # without `before` the same call is the fresh combination of `after`
    fresh = oracle.combined_voxels(oa, pose, K, ijk)
    assert np.abs(fresh["sdf"][inner] - s_new[inner]).max() < 1e-12
    # render from the source camera
    out = oracle.render_combined(oa, pose, K, pose, K, before=ob)
    o, r, L = oracle.ray_dirs(pose, K)
    hit = out["depth"].ravel() > 0
    X = (o + (out["depth"].ravel() * L)[:, None] * r)
    old = hit & (X[:, 1] < -0.03) & (X[:, 2] < 0.02) & (X[:, 2] > -0.02)
    new = hit & ((X[:, 1] > 0.03) | (X[:, 2] > 0.08)) & (np.abs(X[:, 1]) < 0.18) & (np.abs(X[:, 2]) < 0.18)
    assert old.sum() > 20 and new.sum() > 20
    assert np.abs(out["depth"].ravel()[old] - 0.60).max() < 1e-6
    assert np.abs(out["depth"].ravel()[new] - 0.62).max() < 1e-6


def test_first_time_voxels_outside_the_frustum_stay_invalid():
    """R58 with R33: a first-time voxel outside the source camera's widened frustum is not added
    (such pixels stay invalid until the next recombination)."""
    before = _wall_volume(0.60, 0.60, -1)
    after = _wall_volume(0.60, 0.60, 2)
    ob, oa = oracle.OracleVolume(before), oracle.OracleVolume(after)
    K = pinhole(8, 8, 40.0, z_max=15.0)  # narrow view: the new blocks (y >= 0.16) lie outside it
    pose = look_at([0, -0.1, 0], [1, -0.1, 0])
    ijk = np.array([[61, j, 0] for j in range(16, 24)], np.int64)
    cv = oracle.combined_voxels(oa, pose, K, ijk, before=ob)
    assert not cv["valid"].any()
