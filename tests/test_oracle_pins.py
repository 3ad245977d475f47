"""Pins of the CPU oracle against what the paper and mathematics fix (no GPU needed).

Each test names the oracle part it pins and the passage or closed
form it uses.  None of them re-types the oracle's arithmetic: they use closed-form geometry,
invariants, special cases with known answers and library reductions (scipy)."""
import os

import numpy as np
import pytest

import oracle
import scenes
from helpers import angle_between, block_cube, field_volume, pinhole, project
from scenes import DIRECTION_VECTORS, look_at

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TH = np.deg2rad(65.0)


def _golden(name):
    rows = []
    for line in open(os.path.join(GOLDEN, name)):
        line = line.split("#")[0].strip()
        if line:
            rows.append(line.split())
    return rows


# ---------------------------------------------------------------------------------------
# O3(d) membership function (eq:direction_weight, reading R1)
# ---------------------------------------------------------------------------------------
def test_w_dir_prose_values():
    """golden/w_dir_prose.txt: values fixed by the prose of PAPER.md:96 and Fig. 2."""
    for th, al, want in _golden("w_dir_prose.txt"):
        got = oracle.w_dir(np.cos(np.deg2rad(float(al))), np.deg2rad(float(th)))
        assert got == pytest.approx(float(want), abs=1e-12), (th, al)


@pytest.mark.parametrize("theta_deg", [50, 60, 65, 70, 80, 90])
def test_w_dir_partition_and_linearity(theta_deg):
    """Two neighbouring axes in one plane (Fig. 2): the weights blend linearly and sum to one
    across the overlap [pi/2 - theta, theta] ("blends linearly on the full [0,1] range")."""
    th = np.deg2rad(theta_deg)
    al = np.linspace(np.pi / 2 - th, th, 41)
    w1 = np.array([oracle.w_dir(np.cos(a), th) for a in al])
    w2 = np.array([oracle.w_dir(np.cos(np.pi / 2 - a), th) for a in al])
    assert np.allclose(w1 + w2, 1.0, atol=1e-12)
    assert np.allclose(np.diff(w1, 2), 0.0, atol=1e-12)  # linear in the angle
    assert w1[0] == pytest.approx(1.0) and w1[-1] == pytest.approx(0.0, abs=1e-12)


def test_w_dir_printed_formula_rejected():
    """Reading R1: the printed eq:direction_weight is not 1 at alpha = 0 for
    theta = 65 deg, contradicting the prose; the oracle follows the prose."""
    printed = min(max((1 - 0.0) / (2 * TH - np.pi / 4), 0), 1)
    assert abs(printed - 1.0) > 0.3
    assert oracle.w_dir(1.0, TH) == 1.0


@pytest.mark.parametrize("theta_deg", [56, 60, 65, 70, 80, 90])
def test_active_direction_count_3d(theta_deg):
    """'every surface point matches at least one and at most three directions'
    (holds for theta >= arccos(1/sqrt(3)) = 54.74 deg; reading R2)."""
    th = np.deg2rad(theta_deg)
    rng = np.random.default_rng(7)
    n = rng.normal(size=(20000, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    n = np.vstack([n, np.ones((1, 3)) / np.sqrt(3)])  # worst case: the cube diagonal
    cnt = np.zeros(len(n), int)
    for D in range(6):
        c = n @ DIRECTION_VECTORS[D]
        cnt += np.array([oracle.w_dir(ci, th) > 0 for ci in c])
    assert cnt.min() >= 1 and cnt.max() <= 3


def test_active_direction_count_fails_below_5474():
    """Reading R2: at theta = 50 deg the cube diagonal belongs to no direction."""
    d = 1 / np.sqrt(3)
    assert all(oracle.w_dir(d * s, np.deg2rad(50)) == 0.0 for s in (1, -1))


# ---------------------------------------------------------------------------------------
# O3(a)/(c) trilinear + gradient: exact on affine fields (dyadic grid -> exact f32 inputs)
# ---------------------------------------------------------------------------------------
S_DY = 0.0625
A, B, Cc, Dd = 0.25, -0.5, 0.125, 0.75


def _affine_vol():
    def field(D, X):
        phi = A * X[:, 0] + B * X[:, 1] + Cc * X[:, 2] + Dd
        w = 1.0 + 0.5 * X[:, 0]
        return phi, w, np.zeros((len(X), 3))
    return field_volume(block_cube((-1, -1, -1), (1, 1, 1), [0, 3]), field, S_DY, truncation=0.25)


def test_trilinear_exact_on_affine_field():
    ov = oracle.OracleVolume(_affine_vol())
    rng = np.random.default_rng(1)
    for x in rng.uniform(-0.49, 0.93, size=(200, 3)):
        for D in (0, 3):
            phi, om = ov.trilinear(D, x)
            assert phi == pytest.approx(A * x[0] + B * x[1] + Cc * x[2] + Dd, abs=1e-12)
            assert om == pytest.approx(1.0 + 0.5 * x[0], abs=1e-12)
        assert ov.trilinear(1, x) is None  # D=1 never allocated


def test_trilinear_presence_needs_all_corners():
    """O3(a): a direction is present only if all 8 corners lie in allocated blocks (R11)."""
    ov = oracle.OracleVolume(_affine_vol())
    assert ov.trilinear(0, [0.93, 0.0, 0.0]) is not None   # cell 14, corners 14/15 allocated
    assert ov.trilinear(0, [0.94, 0.0, 0.0]) is None       # cell 15 needs voxel 16 (block 2)
    assert ov.trilinear(0, [-0.5, 0.0, 0.0]) is not None   # cell -8
    assert ov.trilinear(0, [-0.501, 0.0, 0.0]) is None     # cell -9 (block -2)


def test_gradient_exact_on_affine_field():
    ov = oracle.OracleVolume(_affine_vol())
    rng = np.random.default_rng(2)
    for x in rng.uniform(-0.43, 0.81, size=(200, 3)):
        g = ov.gradient(0, x)
        assert np.allclose(g, [A, B, Cc], atol=1e-12)
    assert ov.gradient(0, [0.81, 0, 0]) is not None  # cell 12: stencil up to voxel 15
    assert ov.gradient(0, [0.88, 0, 0]) is None  # cell 14: stencil reaches voxel 16
    assert ov.gradient(0, [-0.44, 0, 0]) is None  # stencil reaches voxel -9


def test_gradient_sphere_normals():
    """O3(c): central differences of the C0 sphere field give the radial normal (< 0.1 deg)."""
    vol = scenes.sphere_volume()
    ov = oracle.OracleVolume(vol)
    rng = np.random.default_rng(3)
    d = rng.normal(size=(300, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    pts = d * rng.uniform(0.18, 0.22, size=(300, 1))
    ang = [angle_between(ov.gradient(0, p), p) for p in pts]
    assert np.max(ang) < np.deg2rad(0.1)


# ---------------------------------------------------------------------------------------
# O3(d)/(e) combination: special cases with known answers
# ---------------------------------------------------------------------------------------
def _two_dir_vol(f1, f2, d1, d2, w1=1.0, w2=1.0, s=0.01):
    def field(D, X):
        fn, w = (f1, w1) if D == d1 else (f2, w2)
        return fn(X), np.full(len(X), w), np.zeros((len(X), 3))
    return field_volume(block_cube((-1, -1, -1), (1, 1, 1), [d1, d2]), field, s, truncation=0.04)


def _inner_points(rng, n=60):
    return rng.uniform(-0.05, 0.05, size=(n, 3))


def test_combination_is_stored_weight_average():
    """Two directions with planes along their own axes (w_dir = 1) seen under the same angle:
    f is the weighted cumulative average of the stored distances by the stored weights w_d
    (third factor of eq:combine_weight)."""
    vol = _two_dir_vol(lambda X: (X[:, 0] - 0.01) / 0.04, lambda X: (X[:, 1] + 0.02) / 0.04, 0, 2, 0.25, 0.75)
    ov = oracle.OracleVolume(vol)
    r = -np.array([1.0, 1.0, 0.0]) / np.sqrt(2)
    for x in _inner_points(np.random.default_rng(4)):
        e = ov.eval(x, r)
        p1, p2 = (x[0] - 0.01) / 0.04, (x[1] + 0.02) / 0.04
        assert e["valid"] and e["regime"] == 1
        assert e["f"] == pytest.approx(0.25 * p1 + 0.75 * p2, abs=1e-6)
        assert e["W"][0] / e["W"][2] == pytest.approx(1 / 3, rel=1e-9)


def test_membership_gates_foreign_normals():
    """First factor of eq:combine_weight: a surface stored in X+ whose normal is
    70 deg from +x (> theta) gets zero weight; only the Z+ surface is used."""
    n1 = np.array([np.cos(np.deg2rad(70)), np.sin(np.deg2rad(70)), 0.0])
    vol = _two_dir_vol(lambda X: (X @ n1 - 0.003) / 0.04, lambda X: (X[:, 2] + 0.004) / 0.04, 0, 4)
    ov = oracle.OracleVolume(vol)
    r = -np.array([0.3, 0.3, 0.9])
    r /= np.linalg.norm(r)
    for x in _inner_points(np.random.default_rng(5)):
        e = ov.eval(x, r)
        assert e["valid"] and e["W"][0] == 0.0 and e["W"][4] > 0
        assert e["f"] == pytest.approx((x[2] + 0.004) / 0.04, abs=1e-6)


def test_back_faces_are_excluded():
    """Second factor <n^D, -r> (reading R10): of two opposite surfaces at the same
    place only the one facing the camera is used -- from either side."""
    vol = _two_dir_vol(lambda X: (X[:, 0] - 0.002) / 0.04, lambda X: (0.002 - X[:, 0] - 0.004) / 0.04, 0, 1)
    ov = oracle.OracleVolume(vol)
    for x in _inner_points(np.random.default_rng(6)):
        e = ov.eval(x, np.array([1.0, 0, 0]))  # looking +x: sees the X- surface
        assert e["W"][0] == 0.0 and e["f"] == pytest.approx((-0.002 - x[0]) / 0.04, abs=1e-6)
        e = ov.eval(x, np.array([-1.0, 0, 0]))  # looking -x: sees the X+ surface
        assert e["W"][1] == 0.0 and e["f"] == pytest.approx((x[0] - 0.002) / 0.04, abs=1e-6)


def test_no_gradient_fallback():
    """eq:combine_tsdf_weight: with constant fields (no gradient in any
    direction) the weights are w^D <v^D, -r> (clamped at 0, reading R10)."""
    vol = _two_dir_vol(lambda X: np.full(len(X), 0.3), lambda X: np.full(len(X), -0.2), 0, 2)
    ov = oracle.OracleVolume(vol)
    x = np.array([0.011, -0.02, 0.003])
    e = ov.eval(x, np.array([-1.0, 0, 0]))  # ray along -v^X+: weight = w_d
    assert e["regime"] == 2 and e["W"][0] == pytest.approx(1.0) and e["W"][2] == 0.0
    assert e["f"] == pytest.approx(0.3, abs=1e-7)
    e = ov.eval(x, -np.array([1.0, 1.0, 0]) / np.sqrt(2))
    assert e["f"] == pytest.approx(0.05, abs=1e-7)
    assert np.allclose(e["nt"][0], [1, 0, 0]) and np.allclose(e["nt"][2], [0, 1, 0])
    e = ov.eval(x, np.array([0, 0, 1.0]))  # orthogonal to both v^D: no weight, invalid
    assert not e["valid"]


def test_fallback_ignores_directions_without_data():
    """Reading R8: a direction with stored weight 0 at x holds no data there, so its gradient
    does not suppress the fallback ("absence of gradients in all directions")."""
    def field(D, X):
        if D == 0:
            return np.full(len(X), 0.3), np.ones(len(X)), np.zeros((len(X), 3))
        return (X[:, 2] - 0.001) / 0.04, np.zeros(len(X)), np.zeros((len(X), 3))  # gradient, no data
    vol = field_volume(block_cube((-1, -1, -1), (1, 1, 1), [0, 4]), field, 0.01, truncation=0.04)
    e = oracle.OracleVolume(vol).eval(np.array([0.0, 0.01, 0.02]), np.array([-1.0, 0, 0]))
    assert e["valid"] and e["regime"] == 2 and e["f"] == pytest.approx(0.3)


def test_zero_weight_is_invalid():
    """O3(b): no stored weight anywhere -> no sample (W_D is proportional to w_d in both regimes)."""
    vol = _two_dir_vol(lambda X: X[:, 0], lambda X: X[:, 1], 0, 2, 0.0, 0.0)
    e = oracle.OracleVolume(vol).eval(np.zeros(3) + 0.001, -np.ones(3) / np.sqrt(3))
    assert not e["valid"]


# ---------------------------------------------------------------------------------------
# O1-O8 end to end: closed-form geometry
# ---------------------------------------------------------------------------------------
def _wall(x0=0.5303, color=(10, 200, 30)):
    def field(D, X):
        return np.clip((x0 - X[:, 0]) / 0.04, -1, 1), np.ones(len(X)), np.tile(color, (len(X), 1))
    return field_volume(block_cube((3, -4, -4), (9, 3, 3), [1]), field, 0.01, truncation=0.04)


def test_plane_depth_normal_color_closed_form():
    """A wall x = x0 facing -x stored in X- (O1-O8): depth = camera z = x0 for every pixel,
    normal (-1,0,0), colour exact, mask = {X-}; projection round trip (eq:reprojection)."""
    x0 = 0.5303
    ov = oracle.OracleVolume(_wall(x0))
    K = pinhole(32, 24, 40.0)
    pose = look_at([0, 0, 0], [1, 0, 0])
    out = ov.render(pose, K)
    d = out["depth"]
    assert (d > 0).all()
    assert np.abs(d - x0).max() < 1e-6
    assert np.allclose(out["normal"], [-1, 0, 0], atol=1e-9)
    assert (out["color"] == [10, 200, 30]).all() and (out["mask"] == 2).all()
    o, r, L = oracle.ray_dirs(pose, K)
    X = o + (d.ravel() * L)[:, None] * r
    u, v, z = project(pose, K, X)
    vv, uu = np.mgrid[0:24, 0:32]
    assert np.allclose(u, uu.ravel(), atol=1e-6) and np.allclose(v, vv.ravel(), atol=1e-6)
    assert np.allclose(z, d.ravel(), atol=1e-9)


def test_camera_inside_negative_space_is_not_a_hit():
    """Reading R19: a ray starting behind the wall (negative run first) has no +->- transition."""
    ov = oracle.OracleVolume(_wall(0.2))
    K = pinhole(8, 6, 10.0, z_min=0.05)
    out = ov.render(look_at([0.45, 0, 0], [1, 0, 0]), K)
    assert (out["depth"] == 0).all() and (out["mask"] == 0).all()


def test_c0_sphere_closed_form(c0):
    """configs[0] against the closed-form ray-sphere intersection (golden/c0_sphere.txt)."""
    g = dict((k, float(v)) for k, v in _golden("c0_sphere.txt"))
    ov = oracle.OracleVolume(c0.volume)
    out = ov.render(c0.poses[0], c0.intrinsics)
    d = out["depth"]
    o, r, L = oracle.ray_dirs(c0.poses[0], c0.intrinsics)
    b = r @ o
    disc = b * b - (o @ o - 0.04)
    t = -b - np.sqrt(np.maximum(disc, 0))
    z = np.where(disc >= 0, t / L, 0.0).reshape(d.shape)
    assert int((z > 0).sum()) == g["closed_form_hits"]
    assert d[30, 40] == pytest.approx(g["center_depth"], abs=2e-8)
    hit_cf, hit = z > 0, d > 0
    # disagreements only on the closed-form silhouette (a pixel with a neighbour of the other kind)
    pad = np.pad(hit_cf, 1, mode="edge")
    edge = np.zeros_like(hit_cf)
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            edge |= pad[1 + dy:61 + dy, 1 + dx:81 + dx] != hit_cf
    assert not ((hit != hit_cf) & ~edge).any()
    # depth within 0.5 mm where the incidence angle is below 75 deg
    X = o + (t[:, None]) * r
    n = X / np.linalg.norm(X, axis=1, keepdims=True)
    inc = (-(n * r).sum(1)).reshape(d.shape)
    sel = hit & hit_cf & (inc > np.cos(np.deg2rad(75)))
    assert sel.sum() > 1700
    assert np.abs(d - z)[sel].max() < 5e-4
    # normals radial (at the rendered point) within 0.1 deg on the same pixels; mask nonempty iff hit
    Xr = (o + (d.ravel() * L)[:, None] * r).reshape(60, 80, 3)
    assert np.max(angle_between(out["normal"][sel], Xr[sel])) < np.deg2rad(0.1)
    assert ((out["mask"] > 0) == hit).all()


def test_c0_reduces_to_textbook_single_tsdf_raycaster(c0):
    """When every direction stores the same distance field, f = phi whatever the weights, so the
    DTSDF render must equal a plain single-TSDF raycaster built from library routines:
    scipy.ndimage.map_coordinates(order=1) for the trilinear field and scipy.optimize.brentq for
    the root in the first +->- lattice bracket."""
    from scipy.ndimage import map_coordinates
    from scipy.optimize import brentq

    vol = c0.volume
    s = vol.voxel_size
    grid = np.zeros((64, 64, 64))  # [x, y, z] voxel index + 32
    for b in np.flatnonzero(vol.keys[:, 3] == 0):
        bx, by, bz, _ = vol.keys[b]
        blk = vol.sdf[b].astype(np.float64).reshape(8, 8, 8)  # [lz, ly, lx]
        grid[8 * bx + 32:8 * bx + 40, 8 * by + 32:8 * by + 40, 8 * bz + 32:8 * bz + 40] = blk.transpose(2, 1, 0)

    def phi(X):
        return map_coordinates(grid, (np.atleast_2d(X) / s + 32).T, order=1, mode="nearest")

    K = c0.intrinsics
    o, r, L = oracle.ray_dirs(c0.poses[0], K)
    want = np.zeros(len(r))
    for i in range(len(r)):
        k = np.arange(int(np.ceil(np.float32(K.z_min) * L[i] / s)), int(np.floor(np.float32(K.z_max) * L[i] / s)) + 1)
        X = o + (k * s)[:, None] * r[i]
        inside = np.all((X / s >= -32) & (X / s < 31), axis=1)
        k, X = k[inside], X[inside]
        if len(k) < 2:
            continue
        f = phi(X)
        cross = np.flatnonzero((f[:-1] > 0) & (f[1:] <= 0) & (np.diff(k) == 1))
        if len(cross):
            j = cross[0]
            t = brentq(lambda tt: phi(o + tt * r[i])[0], k[j] * s, k[j + 1] * s, xtol=1e-13)
            want[i] = t / L[i]
    got = oracle.OracleVolume(vol).render(c0.poses[0], K)["depth"].ravel()
    both = (got > 0) & (want > 0)
    assert both.sum() >= 0.99 * (want > 0).sum()
    assert np.abs(got[both] - want[both]).max() < 1e-7


def _plate():
    pat = scenes.Patches.empty()
    n = np.array([0.2, -0.1, 1.0])
    n /= np.linalg.norm(n)
    u = np.cross(n, [1.0, 0, 0])
    u /= np.linalg.norm(u)
    v = np.cross(n, u)
    c = np.array([0.013, -0.021, 0.407])
    thick = 0.003
    pat.extend(c + thick / 2 * n, n, u, v, 0.1, 0.08, [200, 30, 40])
    pat.extend(c - thick / 2 * n, -n, u, v, 0.1, 0.08, [20, 90, 250])
    return pat, c, n


def test_thin_plate_both_sides():
    """Lemma 1 / thin-object motivation: a 3 mm plate at 5 mm voxels renders
    its front face from the front and its back face from the back, with the face colours;
    the same faces merged into ONE regular TSDF lose most of the surface (the control: only
    voxels that happen to fall inside the 3 mm slab carry a negative value)."""
    pat, c, n = _plate()
    vol = scenes.patch_fill(pat, voxel_size=0.005, truncation=0.02, theta=TH)
    ov = oracle.OracleVolume(vol)
    K = pinhole(48, 36, 60.0)
    band = 0.02 + 2 * 0.005
    interiors = {}
    for side, pid, col in ((1, 0, [200, 30, 40]), (-1, 1, [20, 90, 250])):
        pose = look_at(c + side * 0.5 * n, c)
        out = ov.render(pose, K)
        o, r, L = oracle.ray_dirs(pose, K)
        t, hitp = pat.ray_hit(o, r)
        X = o + np.where(np.isfinite(t), t, 0)[:, None] * r
        rel = X - pat.q[pid]
        interior = (hitp == pid) & (np.abs(rel @ pat.u[pid]) < pat.hu[pid] - band) & \
                   (np.abs(rel @ pat.v[pid]) < pat.hv[pid] - band)
        interior = interior.reshape(36, 48)
        interiors[side] = interior
        assert interior.sum() > 200 and (out["depth"][interior] > 0).all()
        zc = np.where(np.isfinite(t), t / L, 0).reshape(36, 48)
        assert np.abs(out["depth"] - zc)[interior].max() < 1e-6
        assert (out["color"][interior] == col).all()
        assert np.max(angle_between(out["normal"][interior], np.tile(side * n, (interior.sum(), 1)))) < 1e-6
        # only directions that admit the visible face's normal contribute
        admit = sum(1 << D for D in range(6) if side * n @ DIRECTION_VECTORS[D] > np.cos(TH))
        assert ((out["mask"][interior].astype(int) & ~admit) == 0).all()
    # control: one regular TSDF holding both faces (nearest face wins) -> no zero crossing
    def merged(D, Xv):
        s_f = (Xv - pat.q[0]) @ pat.n[0]
        s_b = (Xv - pat.q[1]) @ pat.n[1]
        s_ = np.where(np.abs(s_f) <= np.abs(s_b), s_f, s_b)
        return np.clip(s_ / 0.02, -1, 1), np.ones(len(Xv)), np.zeros((len(Xv), 3))
    locs = np.unique(vol.keys[:, :3], axis=0)
    ctrl = field_volume([tuple(k) + (D,) for k in locs for D in range(6)], merged, 0.005, truncation=0.02)
    cov = oracle.OracleVolume(ctrl)
    for side in (1, -1):
        out = cov.render(look_at(c + side * 0.5 * n, c), K)
        assert (out["depth"][interiors[side]] > 0).mean() < 0.25


def _face_interior_pixels(w, pose, K, margin):
    pat = w.patches
    o, r, L = oracle.ray_dirs(pose, K)
    t, pid = pat.ray_hit(o, r)
    ok = np.isfinite(t)
    X = o + np.where(ok, t, 0)[:, None] * r
    good = ok.copy()
    idx = np.flatnonzero(ok)
    for i in idx:
        p = pid[i]
        rel = X[i] - pat.q[p]
        if abs(rel @ pat.u[p]) > pat.hu[p] - margin or abs(rel @ pat.v[p]) > pat.hv[p] - margin:
            good[i] = False
    # far from every other patch
    for p in range(len(pat)):
        sel = good & (pid != p)
        if sel.any():
            from helpers import point_rect_distance
            dist = point_rect_distance(X[sel], pat.q[p], pat.n[p], pat.u[p], pat.v[p], pat.hu[p], pat.hv[p])
            g2 = good[sel]
            g2[dist < margin] = False
            good[sel] = g2
    return good.reshape(K.height, K.width), np.where(ok, t / L, 0).reshape(K.height, K.width), pid.reshape(
        K.height, K.width)


def test_c1_face_interiors_closed_form(c1):
    """configs[1] geometry at reduced resolution: on face interiors (>= tau + 4s from every face
    edge and every other face) depth equals the closed-form plane intersection, the normal is the
    face normal and the colour is the face colour; dirmask is nonempty iff hit."""
    K = scenes.Intrinsics(fx=131.25, fy=131.25, cx=79.5, cy=59.5, width=160, height=120)
    pose = c1.poses[0]
    out = oracle.OracleVolume(c1.volume).render(pose, K)
    margin = c1.volume.truncation + 4 * c1.volume.voxel_size
    good, zc, pid = _face_interior_pixels(c1, pose, K, margin)
    assert good.sum() > 3000
    err = np.abs(out["depth"] - zc)[good]
    assert (err < 1e-6).mean() > 0.995, np.sort(err)[-10:]
    n_face = c1.patches.n[pid[good]]
    assert (angle_between(out["normal"][good], n_face) < 1e-5).mean() > 0.995
    assert (out["color"][good] == c1.patches.color[pid[good]]).all(1).mean() > 0.995
    hit = out["depth"] > 0
    assert ((out["mask"] > 0) == hit).all()
    assert np.allclose(np.linalg.norm(out["normal"][hit], axis=-1), 1.0, atol=1e-9)
    o, r, L = oracle.ray_dirs(pose, K)
    assert ((out["normal"].reshape(-1, 3) * r).sum(1)[hit.ravel()] < 0).all()  # faces the camera


def test_convex_combination_on_c1_samples(c1):
    """f lies in [min phi_D, max phi_D] over the contributing directions."""
    ov = oracle.OracleVolume(c1.volume)
    rng = np.random.default_rng(9)
    keys = c1.volume.keys
    n_checked = 0
    for b in rng.choice(len(keys), 300, replace=False):
        x = (keys[b, :3] * 8 + rng.uniform(0, 7, 3)) * 0.01
        r = rng.normal(size=3)
        r /= np.linalg.norm(r)
        e = ov.eval(x, r)
        if e["valid"]:
            contrib = e["W"] > 0
            assert e["phi"][contrib].min() - 1e-12 <= e["f"] <= e["phi"][contrib].max() + 1e-12
            n_checked += 1
    assert n_checked > 30


def test_volume_errors():
    keys = np.array([[0, 0, 0, 0], [0, 0, 0, 0]], np.int32)
    vol = scenes.BlockVolume(0.01, 0.04, TH, keys, np.zeros((2, 512)), np.zeros((2, 512)), np.zeros((2, 512, 3)))
    with pytest.raises(ValueError):
        oracle.OracleVolume(vol)
    vol.keys = np.array([[0, 0, 0, 0], [0, 0, 0, 6]], np.int32)
    with pytest.raises(ValueError):
        oracle.OracleVolume(vol)


# ---------------------------------------------------------------------------------------
# O7 shading point (reading R32) and colour rounding (reading R13)
# ---------------------------------------------------------------------------------------
def _jump_volume():
    """X- (D = 1) holds phi = +0.5, omega = 1, colour A over block locations x in [0.40, 0.80);
    Y- (D = 3) holds phi = -1, omega = 3, colour B only over x in [0.56, 0.80).  Both fields are
    constant (no gradient anywhere: eq:combine_tsdf_weight), so along a ray F is
    +0.5 until Y- becomes present -- base cell i >= 56, x >= 0.56 -- and negative after: F jumps
    from + to - at the root."""
    A, B = (10, 20, 30), (201, 101, 61)

    def field(D, X):
        if D == 1:
            return np.full(len(X), 0.5), np.ones(len(X)), np.tile(A, (len(X), 1))
        return np.full(len(X), -1.0), np.full(len(X), 3.0), np.tile(B, (len(X), 1))
    keys = block_cube((5, 5, -1), (9, 9, 0), [1]) + block_cube((7, 5, -1), (9, 9, 0), [3])
    return field_volume(keys, field, 0.01), np.array(A, float), np.array(B, float)


def test_shading_at_the_surface_side_of_a_jump():
    """Reading R32: O7 shades at the final bracket end b (valid, f <= 0).  Where F jumps at the
    root the two sides shade differently; hand-derived from eq:combine_tsdf_weight with
    W_X- = omega_A <v^X-, -r> = r_x and W_Y- = 3 r_y: on the surface side the normal is
    normalize(-r_x, -3 r_y, 0) and the colour (r_x A + 3 r_y B) / (r_x + 3 r_y); on the free side
    (-1, 0, 0) and A.  The depth is the jump, x = 56 s.  For rays whose midpoint x* = (a+b)/2 of
    the final fp64 bracket rounds onto the free side, shading "at x*" would give the free-side
    values: at least one such ray is checked."""
    vol, A, B = _jump_volume()
    ov = oracle.OracleVolume(vol)
    K = pinhole(41, 1, 200.0)  # one row: rays in the z = 0 plane, within 6 deg of (1, 1, 0)
    pose = look_at([0, 0, 0], [1, 1, 0])
    px = np.stack([np.arange(41), np.zeros(41, int)], 1).astype(np.int32)
    out = ov.render(pose, K, pixels=px)
    o, r, L = oracle.ray_dirs(pose, K, px)
    assert np.abs(r[:, 2]).max() == 0.0 and (out["depth"] > 0).all()
    t_jump = 56 * float(np.float32(0.01)) / r[:, 0]  # the voxel size reaches both paths as float32
    assert np.abs(out["depth"] * L - t_jump).max() < 1e-12
    n_surf = np.stack([-r[:, 0], -3 * r[:, 1], 0 * r[:, 0]], 1)
    n_surf /= np.linalg.norm(n_surf, axis=1, keepdims=True)
    assert np.abs(out["normal"] - n_surf).max() < 1e-12
    c_surf = (r[:, :1] * A + 3 * r[:, 1:2] * B) / (r[:, :1] + 3 * r[:, 1:2])
    clear = np.abs(c_surf - np.floor(c_surf) - 0.5) > 1e-9  # ties are pinned below (R13)
    assert clear.mean() > 0.9 and (out["color"] == np.floor(c_surf + 0.5))[clear].all()
    assert (out["mask"] == (1 << 1) | (1 << 3)).all()
    # the free-side values differ, and for some rays x* lies on the free side
    assert np.abs(out["normal"] - [-1, 0, 0]).max(1).min() > 0.5
    free_side = [ov.eval(o + out["depth"][i] * L[i] * r[i], r[i]) for i in range(len(px))]
    assert any(s["valid"] and s["f"] > 0 for s in free_side)


def _colour_ramp(lo, hi):
    """Z- (D = 5) plane z = 0.3 facing a camera at the origin looking +z, on a voxel grid of
    s = 2^-7 m (exact binary positions); colour channel 0 = lo at even x voxels, hi at odd."""
    s = 2.0 ** -7

    def field(D, X):
        i = np.round(X[:, 0] / s).astype(np.int64)
        c = np.where(i % 2 == 0, lo, hi)
        rgb = np.stack([c, np.full(len(X), 7), np.full(len(X), 255)], 1)
        return np.clip(-(X[:, 2] - 0.3) / (4 * s), -1, 1), np.ones(len(X)), rgb
    return field_volume(block_cube((-2, -2, 3), (1, 1, 6), [5]), field, s, truncation=4 * s)


@pytest.mark.parametrize("lo,hi,want", [(10, 11, 11), (11, 12, 12), (254, 255, 255), (0, 1, 1), (255, 255, 255)])
def test_colour_rounds_half_up_and_stays_in_range(lo, hi, want):
    """Reading R13: colour = min(255, floor(c + 1/2)).  A camera at x = s/2 (exact in binary)
    looks along +z at a camera-facing plane: at the hit the x fraction is exactly 1/2 between
    voxels of channel-0 colours lo and hi, y/z fractions and the single direction's weight are
    exact, so c = (lo + hi)/2 exactly: a tie that rounds up (10.5 -> 11, 11.5 -> 12; banker's
    rounding would give 10 and 12, truncation 10 and 11).  The other channels are exact (7, 255)."""
    s = 2.0 ** -7
    ov = oracle.OracleVolume(_colour_ramp(lo, hi))
    K = pinhole(9, 9, 10.0)
    pose = look_at([s / 2, 0, 0], [s / 2, 0, 1], up=(0, 1, 0))
    o, r, L = oracle.ray_dirs(pose, K, np.array([[4, 4]], np.int32))
    assert np.array_equal(r[0], [0, 0, 1]) and o[0] == s / 2
    out = ov.render(pose, K, pixels=np.array([[4, 4]], np.int32))
    assert abs(out["depth"][0] - 0.3) < 1e-9  # float32 stored distances
    assert np.allclose(out["normal"][0], [0, 0, -1], atol=1e-12)
    assert list(out["color"][0]) == [want, 7, 255]
