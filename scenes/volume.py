"""Block-volume container, camera types and the snapshot file format.

This module is INPUT plumbing shared by the CPU oracle (``oracle/``) and the
CUDA path (``paper_2301_12796_b200``).  It holds none of the rendering
method's arithmetic: no interpolation, gradient, combination weight, march or
refinement lives here.

Conventions (readings R15-R17):
  * voxel (i, j, k) sits at world position (i, j, k) * voxel_size;
  * block coordinate = floor(i / 8) per axis, local index
    l = lx + 8*ly + 64*lz (x fastest);
  * direction index D in 0..5 = X+, X-, Y+, Y-, Z+, Z- (PAPER.md:79);
  * camera frame x right, y down, z forward; poses are world-from-camera
    4x4 row-major.
"""
from __future__ import annotations

import dataclasses
import struct

import numpy as np

BLOCK = 8
VOXELS_PER_BLOCK = BLOCK ** 3
DIRECTIONS = ("X+", "X-", "Y+", "Y-", "Z+", "Z-")
# v^D of PAPER.md:79, indexed by D
DIRECTION_VECTORS = np.array(
    [[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]], dtype=np.float64
)


@dataclasses.dataclass
class Intrinsics:
    """Pinhole intrinsics plus the march depth range (readings R15/R24)."""

    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    z_min: float = 0.1
    z_max: float = 15.0

    def as_tuple(self):
        return (self.fx, self.fy, self.cx, self.cy, self.width, self.height, self.z_min, self.z_max)


@dataclasses.dataclass
class BlockVolume:
    """A six-direction DTSDF stored as a list of 8^3 voxel blocks keyed by (bx, by, bz, D).

    PAPER.md:603-606: blocks of 8x8x8 voxels allocated only where needed, one index over
    (x, y, z, D).  Each voxel stores the normalised signed distance (positive in front of
    the surface), the distance weight and an RGB colour.
    """

    voxel_size: float
    truncation: float
    theta: float  # angular threshold of eq:angular_threshold / eq:direction_weight (radians)
    keys: np.ndarray  # int32 [N, 4] = (bx, by, bz, D)
    sdf: np.ndarray  # float32 [N, 512]
    weight: np.ndarray  # float32 [N, 512]
    rgb: np.ndarray  # uint8 [N, 512, 3]
    step: float = 0.0  # lattice step Delta; 0 -> voxel_size (reading R4)

    def __post_init__(self):
        self.keys = np.ascontiguousarray(self.keys, dtype=np.int32).reshape(-1, 4)
        n = self.keys.shape[0]
        self.sdf = np.ascontiguousarray(self.sdf, dtype=np.float32).reshape(n, VOXELS_PER_BLOCK)
        self.weight = np.ascontiguousarray(self.weight, dtype=np.float32).reshape(n, VOXELS_PER_BLOCK)
        self.rgb = np.ascontiguousarray(self.rgb, dtype=np.uint8).reshape(n, VOXELS_PER_BLOCK, 3)

    @property
    def n_blocks(self) -> int:
        return int(self.keys.shape[0])

    @property
    def delta(self) -> float:
        return self.step if self.step > 0 else self.voxel_size

    def n_locations(self) -> int:
        return int(np.unique(self.keys[:, :3], axis=0).shape[0]) if self.n_blocks else 0

    def nbytes(self) -> int:
        return self.keys.nbytes + self.sdf.nbytes + self.weight.nbytes + self.rgb.nbytes


# ----------------------------------------------------------------------------------------
# Snapshot file: header (magic, version, voxel_size, tau, theta, step,
# block count) then, per block, the key and its 512 voxel records.  Little-endian.
# ----------------------------------------------------------------------------------------
_MAGIC = b"DTSDFSNP"
_VERSION = 1
_HEADER = struct.Struct("<8sIIddddq")
_REC = np.dtype([("sdf", "<f4"), ("weight", "<f4"), ("rgb", "u1", (3,))])


def save_snapshot(vol: BlockVolume, path: str) -> None:
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(_MAGIC, _VERSION, 0, vol.voxel_size, vol.truncation, vol.theta,
                              vol.step, vol.n_blocks))
        recs = np.empty((vol.n_blocks, VOXELS_PER_BLOCK), dtype=_REC)
        recs["sdf"] = vol.sdf
        recs["weight"] = vol.weight
        recs["rgb"] = vol.rgb
        blk = np.dtype([("key", "<i4", (4,)), ("rec", _REC, (VOXELS_PER_BLOCK,))])
        out = np.empty(vol.n_blocks, dtype=blk)
        out["key"] = vol.keys
        out["rec"] = recs
        out.tofile(fh)


def load_snapshot(path: str) -> BlockVolume:
    with open(path, "rb") as fh:
        head = fh.read(_HEADER.size)
        magic, version, _pad, s, tau, theta, step, n = _HEADER.unpack(head)
        if magic != _MAGIC or version != _VERSION:
            raise ValueError(f"{path}: not a DTSDF snapshot v{_VERSION}")
        blk = np.dtype([("key", "<i4", (4,)), ("rec", _REC, (VOXELS_PER_BLOCK,))])
        data = np.fromfile(fh, dtype=blk, count=n)
    if data.shape[0] != n:
        raise ValueError(f"{path}: truncated snapshot")
    return BlockVolume(voxel_size=s, truncation=tau, theta=theta, step=step,
                       keys=data["key"], sdf=data["rec"]["sdf"], weight=data["rec"]["weight"],
                       rgb=data["rec"]["rgb"])


# ----------------------------------------------------------------------------------------
# Camera helpers (input construction only)
# ----------------------------------------------------------------------------------------
def look_at(position, target, up=(0.0, 0.0, 1.0)) -> np.ndarray:
    """World-from-camera pose (camera x right, y down, z forward) looking from position at target."""
    p = np.asarray(position, dtype=np.float64)
    f = np.asarray(target, dtype=np.float64) - p
    f /= np.linalg.norm(f)
    upv = np.asarray(up, dtype=np.float64)
    if abs(float(np.dot(f, upv))) > 0.99:
        upv = np.array([1.0, 0.0, 0.0]) if abs(f[0]) < 0.9 else np.array([0.0, 1.0, 0.0])
    r = np.cross(f, upv)
    r /= np.linalg.norm(r)
    d = np.cross(f, r)
    T = np.eye(4)
    T[:3, 0], T[:3, 1], T[:3, 2], T[:3, 3] = r, d, f, p
    return T.astype(np.float32).astype(np.float64)  # poses are exchanged as float32
