"""The five BASELINE.json configs as seeded synthetic inputs.

Every config draws from ``numpy.random.default_rng([config_id, 0])`` in the order written
in its builder, so the same call always yields the same bytes.
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

from .fill import Patches, box_patches, cylinder_patches, patch_fill, patch_fill_c, sphere_volume
from .volume import BlockVolume, Intrinsics, look_at

THETA = float(np.deg2rad(65.0))  # reading R2
ROOM_K = dict(fx=525.0, fy=525.0, cx=319.5, cy=239.5, width=640, height=480)


@dataclasses.dataclass
class Workload:
    name: str
    volume: BlockVolume
    intrinsics: Intrinsics
    poses: np.ndarray  # float64 [V, 4, 4] world-from-camera (values exactly representable in f32)
    patches: Optional[Patches] = None  # analytic geometry for closed-form pins (None for C0)
    extra: Optional[dict] = None


def _rand_color(rng):
    return rng.integers(0, 256, size=3)


def c0_sphere() -> Workload:
    """configs[0]: tiny dense sphere, one 80x60 camera 0.6 m from the centre looking at it."""
    vol = sphere_volume(radius=0.2, voxel_size=0.01, truncation=0.04, theta=THETA)
    K = Intrinsics(fx=70.0, fy=70.0, cx=40.0, cy=30.0, width=80, height=60)
    pose = np.eye(4)
    pose[2, 3] = -0.6  # camera at (0,0,-0.6), R = I: looks along +z at the centre
    return Workload("C0", vol, K, pose[None], None, {"radius": 0.2})


def room_patches(rng, n_boxes=20, floor_half=2.0) -> Patches:
    """configs[1] geometry: floor top [-2,2]^2 at z=0 plus n_boxes boxes resting on it.

    Draw order: floor colour; then per box: size U(0.1,1)^3, centre xy U(-1.5,1.5)^2,
    yaw (0 for the first half, U(0, pi/2) for the second half), 6 face colours."""
    pat = Patches.empty()
    pat.extend([0.0, 0.0, 0.0], [0, 0, 1.0], [1.0, 0, 0], [0, 1.0, 0], floor_half, floor_half, _rand_color(rng))
    for i in range(n_boxes):
        size = rng.uniform(0.1, 1.0, size=3)
        cxy = rng.uniform(-1.5, 1.5, size=2)
        yaw = 0.0 if i < n_boxes // 2 else rng.uniform(0.0, np.pi / 2)
        colors = [_rand_color(rng) for _ in range(6)]
        box_patches(pat, [cxy[0], cxy[1], size[2] / 2], size, yaw, colors)
    return pat


def room_pose(rng) -> np.ndarray:
    """configs[1] camera: position (rho cos psi, rho sin psi, h), rho~U(1.5,2.5), psi~U(0,2pi),
    h~U(1.2,1.8), looking at (U(-.3,.3), U(-.3,.3), 0.3), up +z."""
    rho, psi, h = rng.uniform(1.5, 2.5), rng.uniform(0, 2 * np.pi), rng.uniform(1.2, 1.8)
    tgt = [rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), 0.3]
    return look_at([rho * np.cos(psi), rho * np.sin(psi), h], tgt)


def c1_room(n_boxes=20) -> Workload:
    """configs[1]: room scale, 1 cm voxels, tau 4 cm, single 640x480 view at a seeded pose.

    20 boxes as configs[1] states; this fill allocates N ~ 20k (block, direction) pairs, not
    the ~40k configs[1] estimates (reading R30) -- the bench reports the actual N."""
    rng = np.random.default_rng([1, 0])
    pat = room_patches(rng, n_boxes=n_boxes)
    pose = room_pose(rng)
    vol = patch_fill(pat, voxel_size=0.01, truncation=0.04, theta=THETA)
    return Workload("C1", vol, Intrinsics(**ROOM_K), pose[None], pat)


def _orthonormal(n, rng):
    a = np.array([1.0, 0, 0]) if abs(n[0]) < 0.9 else np.array([0, 1.0, 0])
    u = np.cross(n, a)
    u /= np.linalg.norm(u)
    v = np.cross(n, u)
    ang = rng.uniform(0, 2 * np.pi)
    return np.cos(ang) * u + np.sin(ang) * v, -np.sin(ang) * u + np.cos(ang) * v


def _unit_sphere(rng):
    x = rng.normal(size=3)
    return x / np.linalg.norm(x)


def c2_thin(n_clusters=10, plates_per_cluster=20) -> Workload:
    """configs[2]: 200 thin plates (2-6 mm) in 10 clusters, 5 mm voxels, tau 2 cm; two views
    per cluster from both sides (cluster centre +- 0.8 m * cluster normal)."""
    rng = np.random.default_rng([2, 0])
    pat = Patches.empty()
    poses, plates = [], []
    for c in range(n_clusters):
        cc = rng.uniform(-0.6, 0.6, size=3)
        nc = _unit_sphere(rng)
        for _ in range(plates_per_cluster):
            # plate normal within a 20 degree cap around the cluster normal
            while True:
                n = _unit_sphere(rng)
                if n @ nc >= np.cos(np.deg2rad(20.0)):
                    break
            center = cc + rng.uniform(-0.25, 0.25, size=3)
            hu, hv = 0.5 * rng.uniform(0.1, 0.3, size=2)
            thick = rng.uniform(0.002, 0.006)
            while True:
                cf, cb = rng.integers(0, 256, 3), rng.integers(0, 256, 3)
                if np.abs(cf.astype(int) - cb.astype(int)).sum() >= 96:
                    break
            u, v = _orthonormal(n, rng)
            pat.extend(center + 0.5 * thick * n, n, u, v, hu, hv, cf)  # front face
            pat.extend(center - 0.5 * thick * n, -n, u, v, hu, hv, cb)  # back face
            plates.append((center, n, thick))
        poses.append(look_at(cc + 0.8 * nc, cc))
        poses.append(look_at(cc - 0.8 * nc, cc))
    vol = patch_fill(pat, voxel_size=0.005, truncation=0.02, theta=THETA)
    return Workload("C2", vol, Intrinsics(**ROOM_K), np.stack(poses), pat, {"plates": plates})


def plate_cluster(rng, n_plates=40):
    """One configs[2]-style cluster (plates 2-6 mm thick within 20 degrees of a random cluster normal,
    front/back faces with their own colours) and a camera 0.8 m out on a random side of it."""
    pat = Patches.empty()
    cc = rng.uniform(-0.2, 0.2, size=3)
    nc = _unit_sphere(rng)
    for _ in range(n_plates):
        while True:
            n = _unit_sphere(rng)
            if n @ nc >= np.cos(np.deg2rad(20.0)):
                break
        center = cc + rng.uniform(-0.25, 0.25, size=3)
        hu, hv = 0.5 * rng.uniform(0.1, 0.3, size=2)
        thick = rng.uniform(0.002, 0.006)
        cf, cb = rng.integers(0, 256, 3), rng.integers(0, 256, 3)
        u, v = _orthonormal(n, rng)
        pat.extend(center + 0.5 * thick * n, n, u, v, hu, hv, cf)
        pat.extend(center - 0.5 * thick * n, -n, u, v, hu, hv, cb)
    side = 1.0 if rng.uniform() < 0.5 else -1.0
    return pat, look_at(cc + side * 0.8 * nc, cc)


def orbit_poses(rng, n_views=256, step_m=0.05, step_deg=2.0, height=1.5, target=(0, 0, 0)):
    """configs[3] trajectory: an orbit whose 2-degree steps are 0.05 m chords."""
    radius = step_m / np.deg2rad(step_deg)
    a0 = rng.uniform(0, 2 * np.pi)
    out = []
    for i in range(n_views):
        a = a0 + np.deg2rad(step_deg) * i
        out.append(look_at([radius * np.cos(a), radius * np.sin(a), height], target))
    return np.stack(out)


def c3_batch(n_views=256, room: Optional[Workload] = None) -> Workload:
    """configs[3]: the configs[1] volume with n_views orbit views."""
    room = room or c1_room()
    rng = np.random.default_rng([3, 0])
    return Workload("C3", room.volume, room.intrinsics, orbit_poses(rng, n_views), room.patches)


LARGE_K = dict(fx=1050.0, fy=1050.0, cx=639.5, cy=479.5, width=1280, height=960)  # reading R31


def large_patches(rng, n_boxes, n_cylinders, n_plates, keep_out=(0.83, 2.03)) -> Patches:
    """configs[4] geometry in an 8 x 8 x 3 m room: floor, four walls and a ceiling (inward
    normals), then n_boxes boxes (sides U(0.1,1) m; first half resting on the floor, second
    half floating with a bottom face; every other one yawed U(0, pi/2)), n_cylinders upright
    cylinders (r U(0.05,0.3) m, h U(0.2,2) m, side + top cap) and n_plates thin plates
    (2-6 mm, sides U(0.1,0.5) m, uniform normal, front/back colours >= 96 apart in L1).
    Objects whose horizontal extent reaches into the annulus keep_out (m from the room's
    vertical axis) are redrawn so the camera orbit stays in free space.

    Draw order: room colours (6); boxes; cylinders; plates, each as written below."""
    pat = Patches.empty()
    room = [([0, 0, 0.0], [0, 0, 1.0], [1.0, 0, 0], [0, 1.0, 0], 4.0, 4.0),      # floor
            ([0, 0, 3.0], [0, 0, -1.0], [1.0, 0, 0], [0, 1.0, 0], 4.0, 4.0),     # ceiling
            ([-4.0, 0, 1.5], [1.0, 0, 0], [0, 1.0, 0], [0, 0, 1.0], 4.0, 1.5),   # walls
            ([4.0, 0, 1.5], [-1.0, 0, 0], [0, 1.0, 0], [0, 0, 1.0], 4.0, 1.5),
            ([0, -4.0, 1.5], [0, 1.0, 0], [1.0, 0, 0], [0, 0, 1.0], 4.0, 1.5),
            ([0, 4.0, 1.5], [0, -1.0, 0], [1.0, 0, 0], [0, 0, 1.0], 4.0, 1.5)]
    for q, n, u, v, hu, hv in room:
        pat.extend(q, n, u, v, hu, hv, _rand_color(rng))

    def free(xy, ext):
        r = float(np.hypot(*xy))
        return r + ext < keep_out[0] or r - ext > keep_out[1]

    for i in range(n_boxes):
        while True:
            size = rng.uniform(0.1, 1.0, size=3)
            cxy = rng.uniform(-3.5, 3.5, size=2)
            if free(cxy, 0.5 * float(np.hypot(size[0], size[1]))):
                break
        floating = i >= n_boxes // 2
        cz = rng.uniform(size[2] / 2 + 0.3, 3.0 - size[2] / 2) if floating else size[2] / 2
        yaw = rng.uniform(0.0, np.pi / 2) if i % 2 else 0.0
        colors = [_rand_color(rng) for _ in range(6)]
        box_patches(pat, [cxy[0], cxy[1], cz], size, yaw, colors, with_bottom=floating)
    for _ in range(n_cylinders):
        while True:
            r, h = rng.uniform(0.05, 0.3), rng.uniform(0.2, 2.0)
            cxy = rng.uniform(-3.5, 3.5, size=2)
            if free(cxy, r):
                break
        cylinder_patches(pat, [cxy[0], cxy[1], 0.0], r, h, [_rand_color(rng), _rand_color(rng)])
    for _ in range(n_plates):
        while True:
            center = rng.uniform([-3.5, -3.5, 0.2], [3.5, 3.5, 2.8])
            hu, hv = 0.5 * rng.uniform(0.1, 0.5, size=2)
            if free(center[:2], float(np.hypot(hu, hv))):
                break
        n = _unit_sphere(rng)
        thick = rng.uniform(0.002, 0.006)
        while True:
            cf, cb = rng.integers(0, 256, 3), rng.integers(0, 256, 3)
            if np.abs(cf.astype(int) - cb.astype(int)).sum() >= 96:
                break
        u, v = _orthonormal(n, rng)
        pat.extend(center + 0.5 * thick * n, n, u, v, hu, hv, cf)
        pat.extend(center - 0.5 * thick * n, -n, u, v, hu, hv, cb)
    return pat


C4_COUNTS = dict(n_boxes=520, n_cylinders=220, n_plates=450)


def c4_large(n_views=64, counts=None) -> Workload:
    """configs[4]: 8 x 8 x 3 m at 5 mm voxels (tau 2 cm) of seeded boxes, cylinders and thin
    plates, counts tuned towards ~2.5 M blocks (the bench reports the actual N); n_views
    640x480 views on an orbit of 0.05 m / 2 degree steps at 1.5 m height inside the room
    looking at its centre, plus one 1280x960 view (reading R31) from the first pose
    (``extra['large_pose']``, ``extra['large_intrinsics']``)."""
    rng = np.random.default_rng([4, 0])
    pat = large_patches(rng, **(counts or C4_COUNTS))
    poses = orbit_poses(rng, n_views, height=1.5, target=(0.0, 0.0, 0.8))
    vol = patch_fill_c(pat, voxel_size=0.005, truncation=0.02, theta=THETA)
    return Workload("C4", vol, Intrinsics(**ROOM_K), poses, pat,
                    {"large_pose": poses[0], "large_intrinsics": Intrinsics(**LARGE_K)})


CONFIGS = {"C0": c0_sphere, "C1": c1_room, "C2": c2_thin, "C3": c3_batch, "C4": c4_large}
