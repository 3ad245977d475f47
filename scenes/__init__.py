"""Seeded synthetic inputs shared by the CPU oracle and the CUDA path.

Holds no arithmetic of the rendering method (input recipe)."""
from .volume import (BLOCK, DIRECTIONS, DIRECTION_VECTORS, VOXELS_PER_BLOCK, BlockVolume, Intrinsics,
                     load_snapshot, look_at, save_snapshot)
from .fill import Patches, box_patches, cylinder_patches, local_offsets, patch_fill, patch_fill_c, sphere_volume
from .frames import Frame, analytic_frame, room_scan_poses
from .configs import CONFIGS, THETA, Workload, c0_sphere, c1_room, c2_thin, c3_batch, c4_large, orbit_poses

__all__ = [
    "BLOCK", "DIRECTIONS", "DIRECTION_VECTORS", "VOXELS_PER_BLOCK", "BlockVolume", "Intrinsics",
    "load_snapshot", "save_snapshot", "look_at", "Patches", "box_patches", "local_offsets", "patch_fill",
    "sphere_volume", "cylinder_patches", "patch_fill_c", "c4_large", "CONFIGS", "THETA", "Workload", "c0_sphere", "c1_room", "c2_thin", "c3_batch",
    "orbit_poses", "Frame", "analytic_frame", "room_scan_poses",
]
