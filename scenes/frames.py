"""Seeded synthetic depth frames (fusion inputs): the closed-form first
hit of each pixel ray with a scene's rectangle patches -- camera-z depth, the hit patch's unit
normal in the camera frame (facing the camera) and its colour.  Stand-ins for the RGB-D sequences
the paper fuses (TUM, ICL-NUIM, ...), none of which is reproduced.

Holds no arithmetic of the fusion method (projection, weights, averaging live in oracle/ and
csrc/)."""
from __future__ import annotations

import dataclasses

import numpy as np

from .fill import Patches
from .volume import Intrinsics, look_at


@dataclasses.dataclass
class Frame:
    depth: np.ndarray   # float32 [H, W] camera z in metres, 0 = no return
    normal: np.ndarray  # float32 [H, W, 3] unit camera-frame normal facing the camera, 0 = invalid
    color: np.ndarray   # uint8 [H, W, 3]
    pose: np.ndarray    # float64 [4, 4] world-from-camera (float32-representable)


def analytic_frame(patches: Patches, pose, K: Intrinsics, noise_m: float = 0.0, rng=None) -> Frame:
    """Ideal depth camera: per pixel the first front-facing rectangle hit (Patches.ray_hit)."""
    pose = np.asarray(pose, np.float32).astype(np.float64)
    v, u = np.mgrid[0:K.height, 0:K.width]
    fx, fy, cx, cy = (float(np.float32(a)) for a in (K.fx, K.fy, K.cx, K.cy))
    dt = np.stack([(u.ravel() - cx) / fx, (v.ravel() - cy) / fy, np.ones(u.size)], -1)
    L = np.linalg.norm(dt, axis=1)
    R, o = pose[:3, :3], pose[:3, 3]
    r = (dt / L[:, None]) @ R.T
    t, pid = patches.ray_hit(o, r)
    hit = np.isfinite(t)
    z = np.where(hit, t / L, 0.0)
    if noise_m > 0:
        z = np.where(hit, z + rng.normal(scale=noise_m, size=z.shape), 0.0)
    ok = hit & (z >= K.z_min) & (z <= K.z_max)
    n_world = np.where(ok[:, None], patches.n[np.maximum(pid, 0)], 0.0)
    n_cam = n_world @ R  # R^T n
    col = np.where(ok[:, None], patches.color[np.maximum(pid, 0)], 0).astype(np.uint8)
    return Frame(np.where(ok, z, 0.0).astype(np.float32).reshape(K.height, K.width),
                 n_cam.astype(np.float32).reshape(K.height, K.width, 3),
                 col.reshape(K.height, K.width, 3), pose)


def room_scan_poses(rng, n=8, radius=(1.6, 2.4), height=(1.2, 1.8)):
    """Seeded cameras around the configs[1] room looking at its centre region (fusion inputs)."""
    poses = []
    for _ in range(n):
        rho, psi, h = rng.uniform(*radius), rng.uniform(0, 2 * np.pi), rng.uniform(*height)
        tgt = (rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), 0.3)
        poses.append(look_at((rho * np.cos(psi), rho * np.sin(psi), h), tgt))
    return np.stack(poses)
