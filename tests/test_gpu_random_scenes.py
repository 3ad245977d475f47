"""GPU parity on freshly seeded scenes beyond the five configs: rooms (configs[1] recipe), thin-plate
clusters (configs[2] recipe) and dense spheres (configs[0] recipe at random radii and viewpoints),
one full frame each at reduced resolution, against the fp64 oracle with the BASELINE.json
tolerances.  (tools/seed_sweep.py runs the same recipes at 640x480 over more seeds.)  Needs a B200."""
import numpy as np
import pytest

import oracle
import scenes
from parity import assert_parity, to_np
from scenes.configs import THETA, plate_cluster, room_patches, room_pose

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

HALF_K = scenes.Intrinsics(fx=262.5, fy=262.5, cx=159.5, cy=119.5, width=320, height=240)


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2301_12796_b200 import Renderer
    r = Renderer(0)
    yield r
    r.close()


def _check(R, vol, pose, K, what):
    R.upload_volume(vol)
    g = R.render(np.asarray(pose)[None], K)
    o = oracle.OracleVolume(vol).render(pose, K)
    st = assert_parity({k: to_np(v[0]) for k, v in g.items()}, o, what=what)
    return st


@pytest.mark.parametrize("seed", [200, 201, 202])
def test_random_room(R, seed):
    rng = np.random.default_rng([7, seed])
    pat, pose = room_patches(rng, n_boxes=20), room_pose(rng)
    vol = scenes.patch_fill_c(pat, voxel_size=0.01, truncation=0.04, theta=THETA)
    st = _check(R, vol, pose, HALF_K, f"room {seed}")
    assert st["hits_gpu"] > 10000


@pytest.mark.parametrize("seed", [200, 201])
def test_random_plate_cluster(R, seed):
    rng = np.random.default_rng([8, seed])
    pat, pose = plate_cluster(rng)
    vol = scenes.patch_fill_c(pat, voxel_size=0.005, truncation=0.02, theta=THETA)
    st = _check(R, vol, pose, HALF_K, f"plates {seed}")
    assert st["hits_gpu"] > 1000


@pytest.mark.parametrize("seed", [200, 201])
def test_random_sphere(R, seed):
    rng = np.random.default_rng([9, seed])
    vol = scenes.sphere_volume(radius=rng.uniform(0.12, 0.28), voxel_size=0.01, truncation=0.04, theta=THETA)
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    pose = scenes.look_at(d * rng.uniform(0.45, 0.9), rng.uniform(-0.05, 0.05, size=3))
    K = scenes.Intrinsics(fx=140.0, fy=140.0, cx=79.5, cy=59.5, width=160, height=120)
    st = _check(R, vol, pose, K, f"sphere {seed}")
    assert st["hits_gpu"] > 1000
