"""GPU parity: the CUDA path (through the C ABI) against the fp64 CPU oracle on the same seeded
inputs, plus the exactness invariants of the accelerations.  Needs a B200 (run via gpurun)."""
import numpy as np
import pytest

import oracle
import scenes
from helpers import block_cube, field_volume, pinhole
from parity import assert_parity, to_np

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


def _sel(gpu, view, pixels=None):
    out = {}
    for k, v in gpu.items():
        a = to_np(v[view])
        if pixels is not None:
            a = a[pixels[:, 1], pixels[:, 0]]
        out[k] = a
    return out


def _grid_pixels(K, step, offset=0):
    v, u = np.mgrid[offset:K.height:step, offset:K.width:step]
    return np.stack([u.ravel(), v.ravel()], 1).astype(np.int32)


def test_c0_full_frame(R, c0):
    R.upload_volume(c0.volume)
    g = R.render(c0.poses, c0.intrinsics)
    o = oracle.OracleVolume(c0.volume).render(c0.poses[0], c0.intrinsics)
    st = assert_parity(_sel(g, 0), o, what="C0")
    assert st["hits_gpu"] > 1800
    print("C0", st)


def test_c1_full_frame(R, c1):
    """configs[1] at full size in the launch configuration bench.py times (one 640x480 view)."""
    R.upload_volume(c1.volume)
    g = R.render(c1.poses, c1.intrinsics)
    o = oracle.OracleVolume(c1.volume).render(c1.poses[0], c1.intrinsics)
    st = assert_parity(_sel(g, 0), o, what="C1")
    assert st["hits_gpu"] > 100000
    print("C1", st)


def test_c2_thin_plates(R, c2):
    """configs[2]: 4 of the 20 views at full frame, all 20 on a 1/64 pixel grid."""
    R.upload_volume(c2.volume)
    g = R.render(c2.poses, c2.intrinsics)
    ov = oracle.OracleVolume(c2.volume)
    for v in (0, 1, 10, 11):
        st = assert_parity(_sel(g, v), ov.render(c2.poses[v], c2.intrinsics), what=f"C2 view {v}")
        print("C2", v, st)
    px = _grid_pixels(c2.intrinsics, 8, 3)
    for v in range(len(c2.poses)):
        assert_parity(_sel(g, v, px), ov.render(c2.poses[v], c2.intrinsics, pixels=px), what=f"C2 grid view {v}")


def test_c3_batch(R, c1):
    """configs[3]: 256 orbit views in one dtsdf_render_batch call; 8 evenly spaced views checked
    on a 1/4 pixel grid."""
    w = scenes.c3_batch(room=c1)
    R.upload_volume(w.volume)
    g = R.render(w.poses, w.intrinsics)
    ov = oracle.OracleVolume(w.volume)
    px = _grid_pixels(w.intrinsics, 2, 1)
    for v in range(0, 256, 32):
        st = assert_parity(_sel(g, v, px), ov.render(w.poses[v], w.intrinsics, pixels=px), what=f"C3 view {v}")
    print("C3", st)


def test_large_view_1280x960_sampled(R, c1):
    """The 1280x960 view of configs[4] (intrinsics per reading R31) over the C1 volume, on a 1/16
    pixel grid; a ragged row shard [37, 901) checked on the same pixels."""
    K = scenes.Intrinsics(fx=1050.0, fy=1050.0, cx=639.5, cy=479.5, width=1280, height=960)
    R.upload_volume(c1.volume)
    g = R.render(c1.poses, K)
    px = _grid_pixels(K, 4, 1)
    o = oracle.OracleVolume(c1.volume).render(c1.poses[0], K, pixels=px)
    assert_parity(_sel(g, 0, px), o, what="1280x960")
    gs = R.render(c1.poses, K, row0=37, row1=901)
    full = {k: to_np(v[0])[37:901] for k, v in g.items()}
    for k in full:
        assert np.array_equal(full[k], to_np(gs[k][0])), k


def test_ragged_sizes_and_rows(R, c1):
    """Image sizes that are not multiples of the 16x16 CTA / 8x8 range tile, with a row shard."""
    K = scenes.Intrinsics(fx=131.0, fy=129.0, cx=40.3, cy=31.7, width=83, height=61)
    R.upload_volume(c1.volume)
    g = R.render(c1.poses, K, row0=7, row1=50)
    o = oracle.OracleVolume(c1.volume).render(c1.poses[0], K, row0=7, row1=50)
    assert_parity(_sel(g, 0), o, budget=3e-3, what="ragged")  # 3053 px: 0.1 % would be < 4 pixels


def test_batch_equals_single_and_deterministic(R, c1):
    w = scenes.c3_batch(n_views=5, room=c1)
    R.upload_volume(w.volume)
    gb = R.render(w.poses, w.intrinsics)
    for v in range(5):
        gs = R.render(w.poses[v:v + 1], w.intrinsics)
        for k in gb:
            assert torch.equal(gb[k][v], gs[k][0]), (v, k)
    gb2 = R.render(w.poses, w.intrinsics)
    for k in gb:
        assert torch.equal(gb[k], gb2[k])


def test_row_shards_concatenate_bitexact(R, c1):
    R.upload_volume(c1.volume)
    K = c1.intrinsics
    full = R.render(c1.poses, K)
    a = R.render(c1.poses, K, row0=0, row1=240)
    b = R.render(c1.poses, K, row0=240, row1=480)
    for k in full:
        assert torch.equal(full[k], torch.cat([a[k], b[k]], 1)), k


def test_accelerations_are_result_invisible(R, c1, c2):
    """Range pass, block skipping, the live-direction cell masks and the tile order are exact
    (DESIGN.md §2 O2, §5, §6): switching them off changes no bit (C1 room and the C2 thin plates, where opposing
    directions share block locations)."""
    from paper_2301_12796_b200.dtsdf import OPT_BLOCK_SKIP, OPT_CELL_DIRS, OPT_RANGE_PASS, OPT_TILE_ORDER
    K = scenes.Intrinsics(fx=262.5, fy=262.5, cx=159.5, cy=119.5, width=320, height=240)
    for w in (c1, c2):
        R.upload_volume(w.volume)
        ref = R.render(w.poses[:2], K)
        for rng_on, skip_on, live_on, order_on in ((0, 1, 1, 1), (1, 0, 1, 1), (0, 0, 1, 1), (1, 1, 0, 1),
                                                   (1, 1, 1, 0), (0, 0, 0, 0)):
            R.set_option(OPT_RANGE_PASS, rng_on)
            R.set_option(OPT_BLOCK_SKIP, skip_on)
            R.set_option(OPT_CELL_DIRS, live_on)
            R.set_option(OPT_TILE_ORDER, order_on)
            g = R.render(w.poses[:2], K)
            for k in ref:
                assert torch.equal(ref[k], g[k]), (w.name, rng_on, skip_on, live_on, order_on, k)
        R.set_option(OPT_RANGE_PASS, 1)
        R.set_option(OPT_BLOCK_SKIP, 1)
        R.set_option(OPT_CELL_DIRS, 1)
        R.set_option(OPT_TILE_ORDER, 1)


def test_grown_empty_boxes_skip_exactly(R):
    """Empty-space skipping through the grown boxes (k_empty_box) is exact: a room
    with 64 boxes seen from 16 seeded scan poses -- inside the room, far outside it, grazing the
    floor -- renders bit-identically with block skipping on (boxes) and off (every lattice
    point located)."""
    from paper_2301_12796_b200.dtsdf import OPT_BLOCK_SKIP
    w = scenes.c1_room(n_boxes=64)
    R.upload_volume(w.volume)
    K = scenes.Intrinsics(fx=131.25, fy=131.25, cx=79.5, cy=59.5, width=160, height=120)
    rng = np.random.default_rng([2301, 12796])
    poses = np.concatenate([np.asarray(scenes.room_scan_poses(rng, n=8), np.float32),
                            np.asarray(scenes.room_scan_poses(rng, n=4, radius=(5.0, 9.0), height=(0.1, 4.0)), np.float32),
                            np.asarray(scenes.room_scan_poses(rng, n=4, radius=(1.0, 2.0), height=(0.05, 0.2)), np.float32)])
    ref = R.render(poses, K)
    assert (ref["depth"] > 0).float().mean() > 0.2
    R.set_option(OPT_BLOCK_SKIP, 0)
    try:
        g = R.render(poses, K)
    finally:
        R.set_option(OPT_BLOCK_SKIP, 1)
    for k in ref:
        assert torch.equal(ref[k], g[k]), k


def test_location_grid_and_hash_paths_agree(R, c1):
    """The dense location grid and the bitmap + hash-probe path resolve the same slots."""
    from paper_2301_12796_b200.dtsdf import OPT_LOCATION_GRID
    R.upload_volume(c1.volume)
    K = scenes.Intrinsics(fx=262.5, fy=262.5, cx=159.5, cy=119.5, width=320, height=240)
    ref = R.render(c1.poses, K)
    R.set_option(OPT_LOCATION_GRID, 0)
    g = R.render(c1.poses, K)
    R.set_option(OPT_LOCATION_GRID, 1)
    for k in ref:
        assert torch.equal(ref[k], g[k]), k


def test_host_outputs_equal_device_outputs(R, c1):
    """Pinned host outputs written by the kernel (DTSDF_OPT_HOST_WRITE), pinned via the copy path,
    and pageable host outputs all equal the device render bit for bit -- full frame, and a ragged
    width / row range / multi-view batch whose tile rows are neither full nor 16-B aligned."""
    from paper_2301_12796_b200.dtsdf import OPT_HOST_WRITE
    R.upload_volume(c1.volume)
    K1 = c1.intrinsics
    Kr = scenes.Intrinsics(fx=262.5, fy=262.5, cx=159.5, cy=119.5, width=321, height=243)
    w3 = scenes.c3_batch(n_views=3, room=c1)
    for poses, K, r0, r1 in ((c1.poses, K1, 0, K1.height), (w3.poses, Kr, 5, 240)):
        g = R.render(poses, K, row0=r0, row1=r1)
        V, H, W = len(poses), r1 - r0, K.width
        for pinned, host_write in ((True, 1), (True, 0), (False, 1)):
            R.set_option(OPT_HOST_WRITE, host_write)
            mk = (lambda t: t.pin_memory()) if pinned else (lambda t: t)
            hd = mk(torch.full((V, H, W), 7.0, dtype=torch.float32))
            hn = mk(torch.full((V, H, W, 3), 7.0, dtype=torch.float32))
            hc = mk(torch.full((V, H, W, 3), 7, dtype=torch.uint8))
            hm = mk(torch.full((V, H, W), 7, dtype=torch.uint8))
            R.render_into(poses, K, hd, hn, hc, hm, row0=r0, row1=r1)
            for k, h in (("depth", hd), ("normal", hn), ("color", hc), ("mask", hm)):
                assert torch.equal(g[k].cpu(), h), (k, W, pinned, host_write)
    R.set_option(OPT_HOST_WRITE, 1)


def test_alloc_fill_commit_equals_upload(R, c0):
    """Zero-copy path used by the multi-GPU broadcast: fill library-owned buffers, then commit."""
    vol = c0.volume
    R.upload_volume(vol)
    ref = R.render(c0.poses, c0.intrinsics)
    bufs = R.alloc(vol.voxel_size, vol.truncation, vol.theta, vol.n_blocks)
    bufs["keys"].copy_(torch.from_numpy(vol.keys))
    bufs["sdf"].copy_(torch.from_numpy(vol.sdf))
    bufs["weight"].copy_(torch.from_numpy(vol.weight))
    bufs["rgb"].copy_(torch.from_numpy(vol.rgb))
    torch.cuda.synchronize()
    R.commit()
    g = R.render(c0.poses, c0.intrinsics)
    for k in ref:
        assert torch.equal(ref[k], g[k]), k
    assert R.stats()["n_blocks"] == vol.n_blocks and R.stats()["n_locations"] == 512


def test_device_tensor_upload(R, c0):
    vol = c0.volume
    R.upload(vol.voxel_size, vol.truncation, vol.theta, torch.from_numpy(vol.keys).cuda(),
             torch.from_numpy(vol.sdf).cuda(), torch.from_numpy(vol.weight).cuda(), torch.from_numpy(vol.rgb).cuda())
    g = R.render(c0.poses, c0.intrinsics)
    o = oracle.OracleVolume(vol).render(c0.poses[0], c0.intrinsics)
    assert_parity(_sel(g, 0), o)


def test_errors(R, c0):
    from paper_2301_12796_b200 import DtsdfError, Renderer
    fresh = Renderer(0)
    with pytest.raises(DtsdfError) as e:
        fresh.render(c0.poses, c0.intrinsics)
    assert e.value.code == -3  # NO_VOLUME
    vol = c0.volume
    keys = vol.keys[:4].copy()
    keys[1] = keys[0]
    with pytest.raises(DtsdfError) as e:
        fresh.upload(0.01, 0.04, vol.theta, keys, vol.sdf[:4], vol.weight[:4], vol.rgb[:4])
    assert e.value.code == -2  # DUPLICATE_KEY
    keys = vol.keys[:4].copy()
    keys[2, 3] = 6
    with pytest.raises(DtsdfError) as e:
        fresh.upload(0.01, 0.04, vol.theta, keys, vol.sdf[:4], vol.weight[:4], vol.rgb[:4])
    assert e.value.code == -1
    with pytest.raises(DtsdfError):
        fresh.upload(0.01, 0.015, vol.theta, vol.keys[:4], vol.sdf[:4], vol.weight[:4], vol.rgb[:4])  # tau < 2s
    with pytest.raises(DtsdfError):
        fresh.upload(0.01, 0.04, 0.5, vol.keys[:4], vol.sdf[:4], vol.weight[:4], vol.rgb[:4])  # theta <= pi/4
    fresh.upload_volume(vol)
    bad = scenes.Intrinsics(fx=-1.0, fy=70.0, cx=40, cy=30, width=80, height=60)
    with pytest.raises(DtsdfError):
        fresh.render(c0.poses, bad)
    bad = scenes.Intrinsics(fx=70.0, fy=70.0, cx=40, cy=30, width=80, height=60, z_min=2.0, z_max=1.0)
    with pytest.raises(DtsdfError):
        fresh.render(c0.poses, bad)
    with pytest.raises(DtsdfError):
        fresh.render(c0.poses, c0.intrinsics, row0=30, row1=30)
    bad = scenes.Intrinsics(fx=70.0, fy=70.0, cx=40, cy=0, width=40000, height=1)  # > 32768 columns
    with pytest.raises(DtsdfError):
        fresh.render(c0.poses, bad)
    fresh.close()


def test_empty_volume_renders_misses(R, c0):
    R.upload(0.01, 0.04, c0.volume.theta, np.zeros((0, 4), np.int32), np.zeros((0, 512), np.float32),
             np.zeros((0, 512), np.float32), np.zeros((0, 512, 3), np.uint8))
    g = R.render(c0.poses, c0.intrinsics)
    assert all(int(torch.count_nonzero(v)) == 0 for v in g.values())


def test_batch_larger_than_one_launch(R, c1):
    """300 views > DTSDF_VIEWS_PER_LAUNCH: split launches give the same bits as single renders."""
    w = scenes.c3_batch(n_views=300, room=c1)
    K = scenes.Intrinsics(fx=65.6, fy=65.6, cx=39.5, cy=29.5, width=80, height=60)
    R.upload_volume(w.volume)
    n0 = R.launch_count()
    g = R.render(w.poses, K)
    assert R.launch_count() - n0 == 6  # 2 x (range pass + tile order + raycast)
    for v in (0, 255, 256, 299):
        s = R.render(w.poses[v:v + 1], K)
        for k in g:
            assert torch.equal(g[k][v], s[k][0]), (v, k)


def test_hand_built_cases_match_oracle(R):
    """Wall and thin plate of the oracle pins: GPU == oracle (and so == the closed forms)."""
    def field(D, X):
        return np.clip((0.5303 - X[:, 0]) / 0.04, -1, 1), np.ones(len(X)), np.tile([10, 200, 30], (len(X), 1))
    vol = field_volume(block_cube((3, -4, -4), (9, 3, 3), [1]), field, 0.01, truncation=0.04)
    K = pinhole(32, 24, 40.0)
    pose = scenes.look_at([0, 0, 0], [1, 0, 0])
    R.upload_volume(vol)
    g = R.render(pose[None], K)
    assert_parity(_sel(g, 0), oracle.OracleVolume(vol).render(pose, K))
    assert np.abs(to_np(g["depth"][0]) - 0.5303).max() < 1e-5
    pat = scenes.Patches.empty()
    n = np.array([0.2, -0.1, 1.0])
    n /= np.linalg.norm(n)
    u = np.cross(n, [1.0, 0, 0])
    u /= np.linalg.norm(u)
    v = np.cross(n, u)
    c = np.array([0.013, -0.021, 0.407])
    pat.extend(c + 0.0015 * n, n, u, v, 0.1, 0.08, [200, 30, 40])
    pat.extend(c - 0.0015 * n, -n, u, v, 0.1, 0.08, [20, 90, 250])
    vol = scenes.patch_fill(pat, voxel_size=0.005, truncation=0.02, theta=scenes.THETA)
    R.upload_volume(vol)
    K = pinhole(48, 36, 60.0)
    ov = oracle.OracleVolume(vol)
    for side in (1, -1):
        pose = scenes.look_at(c + side * 0.5 * n, c)
        g = R.render(pose[None], K)
        assert_parity(_sel(g, 0), ov.render(pose, K), budget=2e-3)


def test_random_and_axis_aligned_poses_inside_the_room(R, c1):
    """Cameras inside the volume's AABB at seeded random positions and directions (looking up,
    down, along the floor), plus exactly axis-aligned views whose central rays have components
    that are exactly 0 (the empty-space and AABB-entry skips divide by them): full-frame parity."""
    R.upload_volume(c1.volume)
    rng = np.random.default_rng([7, 1])
    poses = []
    for _ in range(6):
        p = np.array([rng.uniform(-1.8, 1.8), rng.uniform(-1.8, 1.8), rng.uniform(0.05, 1.6)])
        d = rng.normal(size=3)
        d[2] = -abs(d[2]) if len(poses) % 3 else abs(d[2])  # mostly towards the floor and boxes
        poses.append(scenes.look_at(p, p + d / np.linalg.norm(d)))
    poses.append(scenes.look_at((0.013, -0.021, 1.5), (0.013, -0.021, 0.0)))   # straight down
    poses.append(scenes.look_at((-1.9, 0.0, 0.3), (1.0, 0.0, 0.3)))            # along +x
    poses.append(scenes.look_at((0.4, 1.9, 0.25), (0.4, -1.0, 0.25)))          # along -y
    ov = oracle.OracleVolume(c1.volume)
    for K in (scenes.Intrinsics(fx=131.25, fy=131.25, cx=80.0, cy=60.0, width=160, height=120),
              scenes.Intrinsics(fx=131.25, fy=131.25, cx=79.5, cy=59.5, width=161, height=121)):
        g = R.render(np.stack(poses), K)
        for i, P in enumerate(poses):
            o = ov.render(P, K)
            st = assert_parity(_sel(g, i), o, what=f"pose {i} {K.width}x{K.height}")
            print("inside-room pose", i, K.width, st["hits_gpu"], st["budget_used"], st["depth_max_err"])


def test_range_epoch_wrap_is_result_invisible(R, c1):
    """The range keys carry a per-pass epoch so the buffers are never cleared between calls; passes
    just below and across the wrap (buffers cleared, epoch restarts at 1) render the same bits, and so
    do passes whose tiles hold keys of many earlier epochs."""
    from paper_2301_12796_b200.dtsdf import OPT_RANGE_EPOCH
    R.upload_volume(c1.volume)
    K = scenes.Intrinsics(fx=262.5, fy=262.5, cx=159.5, cy=119.5, width=320, height=240)
    w3 = scenes.c3_batch(n_views=4, room=c1)
    ref = [R.render(w3.poses[i:i + 1], K) for i in range(4)]
    for start in (0xFFFFFFEC, 0xFFFFFFEE):  # passes run through 0xFFFFFFF0 and wrap
        R.set_option(OPT_RANGE_EPOCH, start)
        for rep in range(6):
            i = rep % 4
            g = R.render(w3.poses[i:i + 1], K)
            for k in ref[i]:
                assert torch.equal(ref[i][k], g[k]), (hex(start), rep, k)
