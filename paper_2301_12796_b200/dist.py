"""Multi-GPU plumbing: one process per GPU, torch.distributed for the
process group.  The volume is replicated with ONE broadcast per buffer from rank 0 straight into
the library-owned device buffers (dtsdf_alloc_volume -> broadcast -> dtsdf_commit_volume); views
are sharded in contiguous ranges (rows of a single large view likewise).  No collective runs on
the render path itself.  Device-agnostic so the host logic is testable with gloo on CPU."""
from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int):
    """Contiguous shard [lo, hi) of n units for this rank: [floor(r n / P), floor((r+1) n / P))."""
    return (rank * n) // world, ((rank + 1) * n) // world


def broadcast_volume_meta(dist, meta: dict | None, device, src: int = 0):
    """Broadcast the scalar volume parameters (n_blocks, voxel_size, truncation, theta, step)."""
    import torch
    t = torch.zeros(5, dtype=torch.float64, device=device)
    if dist.get_rank() == src:
        t[:] = torch.tensor([meta["n_blocks"], meta["voxel_size"], meta["truncation"], meta["theta"],
                             meta["step"]], dtype=torch.float64)
    dist.broadcast(t, src)
    v = t.cpu().numpy()
    return {"n_blocks": int(v[0]), "voxel_size": float(v[1]), "truncation": float(v[2]), "theta": float(v[3]),
            "step": float(v[4])}


def broadcast_buffers(dist, bufs: dict, src: int = 0):
    """In-place broadcast of each tensor (keys, sdf, weight, rgb) from src: the receivers' tensors
    are the library's own buffers, so there is no staging copy."""
    for name in ("keys", "sdf", "weight", "rgb"):
        if bufs[name].numel():
            dist.broadcast(bufs[name], src)


def checksum(bufs: dict) -> int:
    """Order-dependent 64-bit checksum of the volume bytes (verifies the replicas match)."""
    import torch
    total = 0
    for i, name in enumerate(("keys", "sdf", "weight", "rgb")):
        t = bufs[name].contiguous().view(-1)
        if t.numel() == 0:
            continue
        b = t.view(torch.uint8)
        n4 = (b.numel() // 4) * 4
        w = b[:n4].view(torch.int32).to(torch.int64)
        idx = torch.arange(w.numel(), device=w.device, dtype=torch.int64) % 65521 + 1
        total = (total * 1000003 + int((w * idx).sum().item()) + i) & ((1 << 63) - 1)
    return total


def max_over_ranks(dist, value: float, device) -> float:
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(dist, value: float, device) -> float:
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def volume_arrays_to_tensors(vol) -> dict:
    import torch
    return {"keys": torch.from_numpy(np.ascontiguousarray(vol.keys)),
            "sdf": torch.from_numpy(np.ascontiguousarray(vol.sdf)),
            "weight": torch.from_numpy(np.ascontiguousarray(vol.weight)),
            "rgb": torch.from_numpy(np.ascontiguousarray(vol.rgb))}
