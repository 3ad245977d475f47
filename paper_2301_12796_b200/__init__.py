"""B200-native DTSDF raycast renderer (arxiv 2301.12796).

The product is ``libdtsdf.so`` (CUDA for sm_100a behind the C ABI in ``include/dtsdf.h``);
this package holds its sources (``csrc/``), the nvcc build (``build.py``) and a thin ctypes
binding (``dtsdf.py``).  There is no CPU fallback: rendering needs the built library and a
CUDA device, and fails loudly otherwise."""
from .dtsdf import (EXPORTS, DtsdfError, Intrinsics, Renderer, VolumeParams, lib, make_intrinsics)

__all__ = ["EXPORTS", "DtsdfError", "Intrinsics", "Renderer", "VolumeParams", "lib", "make_intrinsics"]
