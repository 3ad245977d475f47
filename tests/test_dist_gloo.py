"""Multi-process host logic of the N>1 path on CPU (gloo, world size 2): view/row sharding, the
volume replication by broadcast into preallocated receive buffers, checksum agreement and the
max-over-ranks timing reduction that bench.py uses."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2301_12796_b200 import dist as pdist  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import scenes
        vol = scenes.c0_sphere().volume if rank == 0 else None
        meta = None
        if rank == 0:
            meta = {"n_blocks": vol.n_blocks, "voxel_size": vol.voxel_size, "truncation": vol.truncation,
                    "theta": vol.theta, "step": vol.step}
        meta = pdist.broadcast_volume_meta(dist, meta, "cpu")
        n = meta["n_blocks"]
        # receivers' buffers stand in for the library-owned buffers of dtsdf_alloc_volume
        bufs = {"keys": torch.zeros((n, 4), dtype=torch.int32), "sdf": torch.zeros((n, 512)),
                "weight": torch.zeros((n, 512)), "rgb": torch.zeros((n, 512, 3), dtype=torch.uint8)}
        if rank == 0:
            for k, t in pdist.volume_arrays_to_tensors(vol).items():
                bufs[k].copy_(t)
        pdist.broadcast_buffers(dist, bufs)
        cs = pdist.checksum(bufs)
        sums = [None] * world
        dist.all_gather_object(sums, cs)
        lo, hi = pdist.shard_range(256, rank, world)
        t = pdist.max_over_ranks(dist, 1.0 + rank, "cpu")
        tot = pdist.sum_over_ranks(dist, float(hi - lo), "cpu")
        q.put((rank, meta, sums, (lo, hi), t, tot, bufs["sdf"][17, 33].item(), int(bufs["keys"][5, 3])))
    finally:
        dist.destroy_process_group()


def test_broadcast_shard_and_reduce_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import scenes
    vol = scenes.c0_sphere().volume
    for rank, meta, sums, shard, tmax, tot, probe, key in res:
        assert meta["n_blocks"] == vol.n_blocks
        assert len(set(sums)) == 1  # replicas identical
        assert tmax == 2.0 and tot == 256.0
        assert probe == pytest.approx(float(vol.sdf[17, 33])) and key == int(vol.keys[5, 3])
    assert [r[3] for r in res] == [(0, 128), (128, 256)]


@pytest.mark.parametrize("n,world", [(256, 1), (256, 2), (256, 8), (480, 8), (7, 3), (1, 4)])
def test_shard_range_partitions(n, world):
    parts = [pdist.shard_range(n, r, world) for r in range(world)]
    assert parts[0][0] == 0 and parts[-1][1] == n
    assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
    sizes = [hi - lo for lo, hi in parts]
    assert max(sizes) - min(sizes) <= 1
    assert np.sum(sizes) == n


def test_bench_launcher_spawns_the_requested_ranks():
    """bench.py --gpus 2 without a torch.distributed environment re-executes itself under
    torch.distributed.run with 2 processes (the form the driver uses for N > 1); --dry-run joins
    a gloo group without kernels and rank 0 reports every rank it saw."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=240, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["comm"]["world_size"] == 2
    assert sorted(r["rank"] for r in line["ranks"]) == [0, 1]
    assert len({r["pid"] for r in line["ranks"]}) == 2


def test_bench_rejects_a_world_size_other_than_gpus():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dry-run"],
                         capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode == 2 and "--gpus 2" in out.stderr
