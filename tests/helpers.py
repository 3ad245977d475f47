"""Test-side input builders (hand-made volumes) and closed-form geometry helpers.

These construct INPUTS (fields written into blocks) and analytic expectations; they do not
implement the rendering method."""
from __future__ import annotations

import numpy as np

from scenes import BLOCK, BlockVolume, Intrinsics, local_offsets

_LOC = local_offsets()


def field_volume(blocks, field, voxel_size, truncation=None, theta=np.deg2rad(65.0), step=0.0, dtype_exact=True):
    """Build a BlockVolume from block keys [(bx,by,bz,D), ...] and field(D, X[...,3]) ->
    (sdf, weight, rgb) evaluated at voxel world positions X (voxel (i,j,k) at (i,j,k)*s)."""
    keys = np.asarray(blocks, np.int32).reshape(-1, 4)
    X = (keys[:, None, :3].astype(np.int64) * BLOCK + _LOC[None]).astype(np.float64) * voxel_size
    sdf = np.zeros((len(keys), 512), np.float32)
    w = np.zeros((len(keys), 512), np.float32)
    rgb = np.zeros((len(keys), 512, 3), np.uint8)
    for b, (bx, by, bz, D) in enumerate(keys):
        s_, w_, c_ = field(int(D), X[b])
        sdf[b] = s_
        w[b] = w_
        rgb[b] = c_
    return BlockVolume(voxel_size, truncation or 4 * voxel_size, float(theta), keys, sdf, w, rgb, step)


def block_cube(lo, hi, dirs):
    """Keys of all block locations in [lo, hi] (inclusive, per axis) for the given directions."""
    out = []
    for D in dirs:
        for bz in range(lo[2], hi[2] + 1):
            for by in range(lo[1], hi[1] + 1):
                for bx in range(lo[0], hi[0] + 1):
                    out.append((bx, by, bz, D))
    return out


def pinhole(width, height, f, z_min=0.1, z_max=15.0):
    return Intrinsics(fx=f, fy=f, cx=(width - 1) / 2, cy=(height - 1) / 2, width=width, height=height, z_min=z_min,
                      z_max=z_max)


def project(pose, K, X):
    """World points -> (u, v, camera z) with the convention of reading R16."""
    pose = np.asarray(pose, np.float32).astype(np.float64)
    Xc = (np.asarray(X) - pose[:3, 3]) @ pose[:3, :3]
    z = Xc[..., 2]
    return K.fx * Xc[..., 0] / z + K.cx, K.fy * Xc[..., 1] / z + K.cy, z


def point_rect_distance(P, q, n, u, v, hu, hv):
    """Euclidean distance from points P [M,3] to a 3D rectangle."""
    rel = P - q
    a = np.clip(rel @ u, -hu, hu)
    b = np.clip(rel @ v, -hv, hv)
    closest = q + a[:, None] * u + b[:, None] * v
    return np.linalg.norm(P - closest, axis=1)


def angle_between(a, b):
    a = a / np.linalg.norm(a, axis=-1, keepdims=True)
    b = b / np.linalg.norm(b, axis=-1, keepdims=True)
    c = np.clip((a * b).sum(-1), -1.0, 1.0)
    return np.arccos(c)
