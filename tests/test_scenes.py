"""Input generators (scenes/): the C fill (gen.c) against the numpy fill and closed forms.
These pin the inputs, not the method."""
import numpy as np

import scenes
from scenes.fill import CYL, DISK, Patches, cylinder_patches, patch_fill, patch_fill_c


def _same(a, b):
    assert a.n_blocks == b.n_blocks
    for k in ("keys", "sdf", "weight", "rgb"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


def test_gen_c_equals_numpy_fill_room(c1):
    _same(c1.volume, patch_fill_c(c1.patches, 0.01, 0.04, scenes.THETA))


def test_gen_c_equals_numpy_fill_thin_plates():
    w = scenes.c2_thin(n_clusters=2, plates_per_cluster=10)
    _same(w.volume, patch_fill_c(w.patches, 0.005, 0.02, scenes.THETA, threads=3))


def test_gen_c_thread_count_invariant(c1):
    _same(patch_fill_c(c1.patches, 0.01, 0.04, scenes.THETA, threads=1),
          patch_fill_c(c1.patches, 0.01, 0.04, scenes.THETA, threads=7))


def test_cylinder_fill_closed_form():
    """Every written voxel of a lone cylinder holds clamp((rho - r)/tau, -1, 1) and the
    direction factor <radial, v^D>, and lies within tau + 2s of the side or the cap."""
    pat = Patches.empty()
    r, h, s, tau = 0.15, 0.4, 0.01, 0.04
    cylinder_patches(pat, [0.03, -0.02, 0.0], r, h, [[10, 20, 30], [40, 50, 60]])
    assert list(pat.kind) == [CYL, DISK]
    vol = patch_fill_c(pat, s, tau, scenes.THETA)
    loc = scenes.local_offsets()
    vox = (vol.keys[:, None, :3] * 8 + loc[None]) * s
    written = vol.weight > 0
    side = (vol.rgb[..., 0] == 10) & written
    cap = (vol.rgb[..., 0] == 40) & written
    assert side.sum() > 1000 and cap.sum() > 100
    assert not (written & ~side & ~cap).any()
    p = vox[side] - np.array([0.03, -0.02, 0.0])
    rho = np.hypot(p[:, 0], p[:, 1])
    np.testing.assert_allclose(vol.sdf[side], np.clip((rho - r) / tau, -1, 1), atol=1e-6)
    D = np.repeat(vol.keys[:, 3][:, None], 512, 1)[side]
    radial = np.stack([p[:, 0] / rho, p[:, 1] / rho, np.zeros_like(rho)], 1)
    om = (radial * scenes.DIRECTION_VECTORS[D]).sum(1)
    np.testing.assert_allclose(vol.weight[side], om, atol=1e-6)
    assert (om > np.cos(scenes.THETA)).all()  # eq:angular_threshold admits the direction
    assert (np.abs(p[:, 2] - h / 2) <= h / 2 + 1e-12).all()
    zc = vox[cap][:, 2]
    np.testing.assert_allclose(vol.sdf[cap], np.clip((zc - h) / tau, -1, 1), atol=1e-6)
    assert (vol.keys[:, 3][np.nonzero(cap.any(1))[0]] == 4).all()  # the cap is Z+ only


def test_c4_counts_scale():
    """A 1/10-count configs[4] builds, spans the 8 x 8 x 3 m room, and has all six directions."""
    w = scenes.c4_large(n_views=4, counts=dict(n_boxes=20, n_cylinders=10, n_plates=20))
    k = w.volume.keys
    assert w.volume.n_blocks > 300_000
    bsz = 8 * 0.005
    assert k[:, 0].min() * bsz <= -4.0 and (k[:, 0].max() + 1) * bsz >= 4.0
    assert k[:, 2].min() * bsz <= 0.0 and (k[:, 2].max() + 1) * bsz >= 3.0
    assert set(np.unique(k[:, 3])) == set(range(6))
    assert w.poses.shape == (4, 4, 4)
    assert w.extra["large_intrinsics"].width == 1280
