"""Pins of the ICP oracle (readings R47-R52 in DESIGN.md §4).

Weighted geometric point-to-plane ICP of a depth frame against a rendered view.
Pins: the SE(3) exponential against scipy's matrix exponential (library reduction), the Cholesky
solve against numpy, the zero-motion fixed point, a plane displaced along its normal (closed-form
residual), g as the gradient of the weighted objective (finite differences), and recovery of a
known relative pose on the configs[1] room (SPEC track_frame example)."""
import numpy as np
import pytest
from scipy.linalg import expm

import oracle
import scenes
from helpers import pinhole
from scenes import look_at

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


def _hat(xi):
    nu, w = xi[:3], xi[3:]
    M = np.zeros((4, 4))
    M[:3, :3] = [[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]]
    M[:3, 3] = nu
    return M


def test_se3_exp_is_the_matrix_exponential():
    rng = np.random.default_rng(3)
    for scale in (1e-10, 1e-4, 0.1, 1.0, 2.5):
        xi = rng.normal(size=6) * scale
        assert np.allclose(oracle.se3_exp(xi), expm(_hat(xi)), atol=1e-12, rtol=1e-10)
    T = oracle.se3_exp([0.1, -0.2, 0.3, 0, 0, 0])
    assert np.allclose(T[:3, :3], np.eye(3)) and np.allclose(T[:3, 3], [0.1, -0.2, 0.3])


def test_cholesky_solve_matches_numpy():
    rng = np.random.default_rng(4)
    for _ in range(20):
        A = rng.normal(size=(6, 6))
        H = A @ A.T + 0.1 * np.eye(6)
        b = rng.normal(size=6)
        assert np.allclose(oracle.cholesky_solve6(H, b), np.linalg.solve(H, b), rtol=1e-10, atol=1e-12)
    assert oracle.cholesky_solve6(np.zeros((6, 6)), np.ones(6)) is None


def _room_view(w, pose, K):
    fr = scenes.analytic_frame(w.patches, pose, K)
    R = np.asarray(pose, np.float32).astype(np.float64)[:3, :3]
    nw = (fr.normal.reshape(-1, 3).astype(np.float64) @ R.T).astype(np.float32).reshape(fr.normal.shape)
    return fr, nw


K_HALF = scenes.Intrinsics(fx=262.5, fy=262.5, cx=159.5, cy=119.5, width=320, height=240)


def test_zero_motion_is_a_fixed_point(c1):
    """A frame rendered from the reference pose itself: every residual is 0, g = 0, the first step
    is 0 and DeltaT stays the identity (SPEC track_frame example 1)."""
    pose = c1.poses[0]
    fr, nw = _room_view(c1, pose, K_HALF)
    H, g, n, res = oracle.icp_normal_equations(fr.depth, fr.depth, nw, pose, K_HALF)
    assert n > 0.7 * (fr.depth > 0).sum()
    assert res < 1e-20 and np.abs(g).max() < 1e-9
    D, info = oracle.icp(fr.depth, fr.depth, nw, pose, K_HALF)
    assert info["ok"] and info["iterations"] == 1 and info["step"] < 1e-9
    assert np.allclose(D, np.eye(4), atol=1e-9)


def test_plane_displaced_along_its_normal():
    """A wall seen 1 mm further than in the rendered view: every associated residual is +1 mm
    (r = <q - x, n> with n facing the camera, eq:geometric_ICP), so sum w r^2 = 1e-6 sum w."""
    K = pinhole(40, 30, 30.0)
    pose = look_at([0, 0, 0], [1, 0.1, 0.05])

    def wall(x0):
        pat = scenes.Patches.empty()
        pat.extend(np.array([x0, 0, 0]), np.array([-1.0, 0, 0]), np.array([0, 1.0, 0]), np.array([0, 0, 1.0]), 3, 3,
                   [9, 9, 9])
        return scenes.analytic_frame(pat, pose, K)
    ref = wall(0.8)
    R = np.asarray(pose, np.float32).astype(np.float64)[:3, :3]
    nw = (ref.normal.reshape(-1, 3).astype(np.float64) @ R.T).astype(np.float32).reshape(ref.normal.shape)
    fr = wall(0.801)
    H, g, n, res = oracle.icp_normal_equations(fr.depth, ref.depth, nw, pose, K)
    z = fr.depth[fr.depth > 0].astype(np.float64)
    wsum = (1.0 / (z + 0.9) ** 2).sum()  # eq:ICP_weight with z_min = 0.1
    assert n == (fr.depth > 0).sum()
    assert res == pytest.approx(1e-6 * wsum, rel=1e-4)
    # outlier threshold: a 6 mm displacement is rejected at the fine 5 mm threshold
    fr6 = wall(0.806)
    assert oracle.icp_normal_equations(fr6.depth, ref.depth, nw, pose, K)[2] == 0
    assert oracle.icp_normal_equations(fr6.depth, ref.depth, nw, pose, K, outlier=0.05)[2] == n


def test_g_is_the_gradient_of_the_weighted_objective(c1):
    """g = 2 sum w J r is dE/dxi of E(xi) = sum w r(exp(xi) DeltaT)^2 (eq:ICP_geometric_dx,
    eq:ICP_Hessian): central finite differences of E agree to 1e-3 relative."""
    pose = c1.poses[0]
    ref, nw = _room_view(c1, pose, K_HALF)
    E_true = oracle.se3_exp([0.004, -0.003, 0.002, 0.01, -0.005, 0.008])
    fr, _ = _room_view(c1, np.asarray(pose, np.float64) @ E_true, K_HALF)
    D0 = oracle.se3_exp([0.001, 0.001, -0.001, 0.002, 0.0, -0.001])
    H, g, n, E0 = oracle.icp_normal_equations(fr.depth, ref.depth, nw, pose, K_HALF, D0, outlier=0.05)
    eps = 1e-7
    fd = np.zeros(6)
    for k in range(6):
        e = np.zeros(6)
        e[k] = eps
        Ep = oracle.icp_normal_equations(fr.depth, ref.depth, nw, pose, K_HALF, oracle.se3_exp(e) @ D0, 0.05)[3]
        Em = oracle.icp_normal_equations(fr.depth, ref.depth, nw, pose, K_HALF, oracle.se3_exp(-e) @ D0, 0.05)[3]
        fd[k] = (Ep - Em) / (2 * eps)
    assert np.allclose(g, fd, rtol=2e-3, atol=1e-3 * np.abs(g).max())
    assert np.all(np.linalg.eigvalsh(H) > 0)


def test_recovers_a_known_relative_pose(c1):
    """SPEC track_frame example 2: configs[1] room, frame displaced by 1 cm and 2 degrees from the
    rendered pose; coarse (0.05 m, 20 iterations) then fine (0.005 m, 50 iterations)
    recovers the relative pose within 1 mm and 0.1 degree."""
    pose = c1.poses[0]
    ref, nw = _room_view(c1, pose, K_HALF)
    ax = np.array([0.3, -0.5, 0.8])
    ax /= np.linalg.norm(ax)
    E_true = oracle.se3_exp(np.r_[np.array([0.6, 0.2, -0.77]) / np.linalg.norm([0.6, 0.2, -0.77]) * 0.01,
                                  ax * np.deg2rad(2.0)])
    fr, _ = _room_view(c1, np.asarray(pose, np.float64) @ E_true, K_HALF)
    D, info = oracle.icp(fr.depth, ref.depth, nw, pose, K_HALF, outlier=0.05, max_iters=20)
    D, info = oracle.icp(fr.depth, ref.depth, nw, pose, K_HALF, D, outlier=0.005, max_iters=50)
    assert info["ok"]
    Rerr = D[:3, :3] @ E_true[:3, :3].T
    ang = np.arccos(np.clip((np.trace(Rerr) - 1) / 2, -1, 1))
    assert np.linalg.norm(D[:3, 3] - E_true[:3, 3]) < 1e-3
    assert ang < np.deg2rad(0.1)
