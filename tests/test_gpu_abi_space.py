"""GPU coverage of the C ABI's own parameter space (SPEC.md:217-238 volume parameters, S:438-446
raycast) and of its argument checks.  Every render is compared with the fp64
oracle on the same inputs with the north-star tolerances (tests/parity.py).  Needs a B200.

* theta in {50 (accepted with a warning, reading R2), 55, 80, 90} degrees, lattice step
  Delta in {0.5 s, 2 s} (reading R4), depth ranges other than [0.1, 15] m (reading R24) --
  the configs[1] room re-parameterised, full 640x480 frames;
* a camera inside a box of the room (reading R19: a leading negative run is not a hit);
* the single-view call dtsdf_render into device, pinned-host and pageable-host buffers;
* commit-time value checks (finite sdf, finite non-negative weight) and a usable context after
  a rejected commit; fusion with carve_weight 0 (carving off, no 0/0);
* a combined TSDF over more than 65535 block locations (grid-size limit of the combine launch).
"""
import dataclasses

import numpy as np
import pytest

import oracle
import scenes
from parity import assert_parity, compare, to_np

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2301_12796_b200 import Renderer
    r = Renderer(0)
    yield r
    r.close()


def _sel(gpu, view=0, pixels=None):
    out = {}
    for k, v in gpu.items():
        a = to_np(v[view])
        if pixels is not None:
            a = a[pixels[:, 1], pixels[:, 0]]
        out[k] = a
    return out


def _parity(R, w, vol, K, pose, what):
    R.upload_volume(vol)
    g = R.render(pose[None], K)
    o = oracle.OracleVolume(vol).render(pose, K)
    st = assert_parity(_sel(g), o, what=what)
    print(what, st)
    return st


@pytest.mark.parametrize("deg", [50.0, 55.0, 80.0, 90.0])
def test_theta(R, c1, deg):
    """eq:direction_weight's threshold theta across (pi/4, pi/2]."""
    from paper_2301_12796_b200.dtsdf import last_warning
    vol = dataclasses.replace(c1.volume, theta=float(np.deg2rad(deg)))
    st = _parity(R, c1, vol, c1.intrinsics, c1.poses[0], f"theta {deg}")
    # reading R2: accepted below 54.74 deg, with a warning
    assert (last_warning() != "") == (deg < 54.74)
    assert st["hits_gpu"] > 100000


@pytest.mark.parametrize("frac", [0.5, 2.0])
def test_lattice_step(R, c1, frac):
    """Lattice step Delta = 0.5 s and 2 s (reading R4: t_k = k Delta, anchored at the camera)."""
    vol = dataclasses.replace(c1.volume, step=float(frac * c1.volume.voxel_size))
    st = _parity(R, c1, vol, c1.intrinsics, c1.poses[0], f"step {frac} s")
    assert st["hits_gpu"] > 100000


@pytest.mark.parametrize("zr", [(0.5, 3.0), (2.6, 15.0), (0.1, 2.4), (1.0, 1.5)])
def test_depth_range(R, c1, zr):
    """[z_min, z_max] other than the default (S:40 depth range; reading R24): the lattice starts
    at ceil(z_min L / Delta) and ends at floor(z_max L / Delta) -- surfaces outside are misses."""
    K = dataclasses.replace(c1.intrinsics, z_min=zr[0], z_max=zr[1])
    st = _parity(R, c1, c1.volume, K, c1.poses[0], f"z range {zr}")
    assert st["hits_gpu"] > 0


def _largest_box(pat):
    """(centre, in-plane axis u, half extents) of the box whose smallest half extent is largest:
    box tops are the RECT patches with normal +z above the floor (scenes.box_patches)."""
    best = None
    for i in range(len(pat.hu)):
        if pat.kind[i] != 0 or pat.n[i][2] < 0.99 or pat.q[i][2] <= 1e-6:
            continue
        h = pat.q[i][2] / 2
        m = min(pat.hu[i], pat.hv[i], h)
        if best is None or m > best[0]:
            best = (m, pat.q[i] - np.array([0, 0, h]), pat.u[i], (pat.hu[i], pat.hv[i], h))
    return best


def test_camera_inside_a_box(R, c1):
    """Reading R19: a ray starting in negative space (inside a box) is not a hit where it leaves
    it (a - -> + transition); it may hit other geometry after a + -> - crossing."""
    m, centre, u, half = _largest_box(c1.patches)
    assert m > 0.1, "configs[1] has a box large enough to stand a camera in"
    pose = scenes.look_at(centre, centre + u)
    st = _parity(R, c1, c1.volume, c1.intrinsics, pose, "camera inside a box")
    g = R.render(pose[None], c1.intrinsics)
    d = to_np(g["depth"][0])
    K = c1.intrinsics
    # the centre pixel looks along u: the box face it exits is half[0] away; no hit before it
    c = d[int(K.cy), int(K.cx)]
    assert c == 0 or c > half[0] - 2 * c1.volume.truncation, (c, half)
    assert st["hits_gpu"] < K.width * K.height


def test_single_view_call_device_pinned_pageable(R, c1):
    """dtsdf_render (the north star's single-view call) into device, pinned and pageable host
    buffers: the same bits as dtsdf_render_batch, and oracle parity."""
    K, pose = c1.intrinsics, c1.poses[0]
    R.upload_volume(c1.volume)
    ref = R.render(pose[None], K)
    shp = (K.height, K.width)
    dev = {"depth": torch.empty(shp, dtype=torch.float32, device="cuda"),
           "normal": torch.empty(shp + (3,), dtype=torch.float32, device="cuda"),
           "color": torch.empty(shp + (3,), dtype=torch.uint8, device="cuda"),
           "mask": torch.empty(shp, dtype=torch.uint8, device="cuda")}
    pinned = {k: torch.empty(v.shape, dtype=v.dtype).pin_memory() for k, v in dev.items()}
    pageable = {k: np.zeros(tuple(v.shape), dtype=np.float32 if v.dtype == torch.float32 else np.uint8)
                for k, v in dev.items()}
    R.render_view(pose, K, dev["depth"], dev["normal"], dev["color"], dev["mask"])
    torch.cuda.synchronize()
    R.render_view(pose, K, pinned["depth"], pinned["normal"], pinned["color"], pinned["mask"])
    R.render_view(pose, K, pageable["depth"], pageable["normal"], pageable["color"], pageable["mask"])
    for k in dev:
        r = to_np(ref[k][0])
        assert np.array_equal(to_np(dev[k]), r), k
        assert np.array_equal(to_np(pinned[k]), r), k
        assert np.array_equal(pageable[k], r), k
    o = oracle.OracleVolume(c1.volume).render(pose, K)
    print("dtsdf_render", assert_parity({k: pageable[k] for k in dev}, o, what="dtsdf_render pageable"))


def test_commit_rejects_bad_values_and_stays_usable(R, c0):
    """NaN is the apron bricks' "unallocated" sentinel, so a non-finite sdf (or a negative /
    non-finite weight) is rejected at commit with INVALID_ARGUMENT; the context still works."""
    from paper_2301_12796_b200.dtsdf import INVALID_ARGUMENT, DtsdfError
    v = c0.volume
    for field, val in (("sdf", np.nan), ("sdf", np.inf), ("weight", -1.0), ("weight", np.inf), ("weight", np.nan)):
        arr = getattr(v, field).copy()
        arr[17, 100] = val
        bad = dataclasses.replace(v, **{field: arr})
        with pytest.raises(DtsdfError) as e:
            R.upload_volume(bad)
        assert e.value.code == INVALID_ARGUMENT, (field, val)
        assert "finite" in str(e.value)
    R.upload_volume(v)
    g = R.render(c0.poses, c0.intrinsics)
    assert_parity(_sel(g), oracle.OracleVolume(v).render(c0.poses[0], c0.intrinsics), what="C0 after rejects")


def test_fuse_with_carving_off_writes_no_nan(R):
    """carve_weight 0 turns carving off (include/dtsdf.h); on fresh blocks (weight 0) the carve
    update would otherwise be 0/0."""
    from paper_2301_12796_b200.dtsdf import FusionParams, lib
    pat = scenes.Patches.empty()
    pat.extend(np.array([0.8, 0, 0]), np.array([-1.0, 0, 0]), np.array([0, 1.0, 0]), np.array([0, 0, 1.0]), 0.5, 0.5,
               [10, 20, 30])
    K = scenes.Intrinsics(fx=60.0, fy=60.0, cx=31.5, cy=23.5, width=64, height=48)
    pose = scenes.look_at([0, 0, 0], [1, 0, 0])
    fr = scenes.analytic_frame(pat, pose, K)
    R.upload(0.01, 0.04, scenes.THETA, np.zeros((0, 4), np.int32), np.zeros((0, 512), np.float32),
             np.zeros((0, 512), np.float32))
    R.fusion_reserve(4096)
    prm = FusionParams()
    lib().dtsdf_default_fusion_params(prm)
    prm.carve_weight = 0.0
    assert R.fuse(fr.depth, fr.normal, fr.color, pose, K, params=prm) > 0
    _, sdf, w, _ = R.get_volume()
    assert np.isfinite(sdf).all() and np.isfinite(w).all()
    # the same frame with carving on: voxels in front of the band move towards +1
    prm.carve_weight = 1.0
    R.fuse(fr.depth, fr.normal, fr.color, pose, K, params=prm)
    _, sdf2, w2, _ = R.get_volume()
    assert np.isfinite(sdf2).all() and (w2 >= w).all()


def _slab_volume(nx, ny, nz, s=0.01, z0=0.803):
    """One direction (Z+) over a dense nx x ny x nz box of block locations holding the plane
    z = z0 (phi = clamp((z - z0) / tau, -1, 1), weight 1): input only, no rendering arithmetic."""
    tau = 4 * s
    bx, by, bz = np.meshgrid(np.arange(nx) - nx // 2, np.arange(ny) - ny // 2, np.arange(nz), indexing="ij")
    keys = np.stack([bx.ravel(), by.ravel(), bz.ravel(), np.full(bx.size, 4)], 1).astype(np.int32)
    loc = scenes.local_offsets()
    z = (keys[:, 2:3].astype(np.int64) * 8 + loc[None, :, 2]) * s
    sdf = np.clip((z - z0) / tau, -1, 1).astype(np.float32)
    w = np.ones_like(sdf)
    rgb = np.zeros(sdf.shape + (3,), np.uint8)
    rgb[..., 0] = 200
    return scenes.BlockVolume(s, tau, scenes.THETA, keys, sdf, w, rgb)


def test_combine_more_than_65535_locations(R):
    """a combine over > 65535 selected block locations (one grid row per slot would
    exceed gridDim.y): combined voxels sampled against the oracle and a sampled render."""
    vol = _slab_volume(64, 64, 20)
    assert vol.n_locations() > 65535
    R.upload_volume(vol)
    K = scenes.Intrinsics(fx=500.0, fy=500.0, cx=319.5, cy=239.5, width=640, height=480)
    pose = scenes.look_at([0.013, 0.021, 6.0], [0.0, 0.0, 0.0], up=(0.0, 1.0, 0.0))
    R.combine(pose, K)
    n = R.combined_stats()["n_locations"]
    assert n > 65535, n
    ex = R.get_combined()
    rng = np.random.default_rng(5)
    pick = rng.choice(n, size=64, replace=False)
    off = scenes.local_offsets().astype(np.int64)
    ijk = (ex["locs"][pick].astype(np.int64)[:, None, :] * 8 + off[None]).reshape(-1, 3)
    ov = oracle.OracleVolume(vol)
    o = oracle.combined_voxels(ov, pose, K, ijk)
    gs = ex["sdf"][pick].reshape(-1)
    gv = ~np.isnan(gs)
    assert np.array_equal(gv, o["valid"])
    assert np.abs(gs[gv] - o["sdf"][gv]).max() < 2e-5
    g = R.render(pose[None], K, combined=True)
    v, u = np.mgrid[3:K.height:24, 5:K.width:24]
    px = np.stack([u.ravel(), v.ravel()], 1).astype(np.int32)
    oc = oracle.render_combined(ov, pose, K, pose, K, pixels=px)
    st = compare(_sel(g, 0, px), oc)
    assert st["budget_used"] <= 1e-3 and st["hits_gpu"] > 0.5 * len(px), st
    print("combine > 65535", n, st)


def test_out_of_device_memory_is_reported_and_the_context_stays_usable(R, c0):
    """a volume whose record bricks do not fit in device memory fails with
    DTSDF_ERR_OUT_OF_MEMORY (not the sticky CUDA error), and the context renders the next volume.
    The context first holds a tiny volume (an upload frees the previous one), then device memory is
    filled with a torch tensor, leaving 2 GiB free."""
    from paper_2301_12796_b200.dtsdf import OUT_OF_MEMORY, DtsdfError
    vol = _slab_volume(96, 96, 24)  # 221k blocks: 1.2 GB pool + 3.9 GB record bricks + index
    R.upload_volume(c0.volume)
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    hog = torch.empty(max(free - (2 << 30), 0), dtype=torch.uint8, device="cuda")
    try:
        with pytest.raises(DtsdfError) as e:
            R.upload_volume(vol)
        assert e.value.code == OUT_OF_MEMORY, str(e.value)
    finally:
        del hog
        torch.cuda.empty_cache()
    R.upload_volume(c0.volume)
    g = R.render(c0.poses, c0.intrinsics)
    assert_parity(_sel(g), oracle.OracleVolume(c0.volume).render(c0.poses[0], c0.intrinsics), what="C0 after OOM")
