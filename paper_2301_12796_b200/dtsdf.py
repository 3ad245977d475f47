"""Thin ctypes binding of libdtsdf.so (include/dtsdf.h) -- argument marshalling only.

Every step of the render runs in the CUDA kernels of ``csrc/``; this module passes torch
tensors' device pointers, host structs and the current CUDA stream.  There is no CPU
fallback: if ``libdtsdf.so`` is missing or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DTSDF_LIB") or os.path.join(_HERE, "libdtsdf.so")

OK, INVALID_ARGUMENT, DUPLICATE_KEY, NO_VOLUME, OUT_OF_MEMORY, CUDA_ERROR, NO_COMBINED, SINGULAR = \
    0, -1, -2, -3, -4, -5, -6, -7
VIEWS_PER_LAUNCH = 256

EXPORTS = [
    "dtsdf_create", "dtsdf_destroy", "dtsdf_alloc_volume", "dtsdf_commit_volume", "dtsdf_upload_volume",
    "dtsdf_render", "dtsdf_render_batch", "dtsdf_volume_stats", "dtsdf_set_profiling", "dtsdf_kernel_times",
    "dtsdf_reset_kernel_times", "dtsdf_set_option", "dtsdf_launch_count", "dtsdf_last_error", "dtsdf_last_warning",
    "dtsdf_combine", "dtsdf_combine_mode", "dtsdf_render_combined", "dtsdf_combined_stats", "dtsdf_get_combined", "dtsdf_default_policy",
    "dtsdf_should_recombine", "dtsdf_default_fusion_params", "dtsdf_fusion_reserve", "dtsdf_depth_normals",
    "dtsdf_fuse", "dtsdf_get_volume", "dtsdf_default_icp_params", "dtsdf_icp", "dtsdf_icp_normal_equations",
]
MARGIN = 0.125  # PAPER.md:262 "(±1/8 image size)"
OPT_RANGE_PASS, OPT_BLOCK_SKIP, OPT_BISECT_STEPS, OPT_LOCATION_GRID, OPT_REFINE_TOL_NM = 1, 2, 4, 5, 6
OPT_HOST_WRITE = 7
OPT_CELL_DIRS = 8
OPT_TILE_ORDER = 9
OPT_RANGE_EPOCH = 10
OPT_INCREMENTAL = 11


class DtsdfError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"dtsdf error {code}: {msg}")
        self.code = code


class Intrinsics(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32),
                ("height", C.c_int32), ("z_min", C.c_float), ("z_max", C.c_float)]


class VolumeParams(C.Structure):
    _fields_ = [("voxel_size", C.c_float), ("truncation", C.c_float), ("theta", C.c_float), ("step", C.c_float),
                ("n_blocks", C.c_int64)]


class CombinePolicy(C.Structure):
    _fields_ = [("boot_frames", C.c_int32), ("stale_frames", C.c_int32), ("translation", C.c_float),
                ("rotation", C.c_float)]


class FusionParams(C.Structure):
    _fields_ = [("max_weight", C.c_float), ("carve_weight", C.c_float), ("carve_radius", C.c_int32),
                ("reserved", C.c_int32)]


class IcpParams(C.Structure):
    _fields_ = [("max_iters", C.c_int32), ("min_step", C.c_float), ("outlier", C.c_float), ("reserved", C.c_int32)]


class IcpResult(C.Structure):
    _fields_ = [("delta", C.c_float * 16), ("delta64", C.c_double * 16), ("iterations", C.c_int32),
                ("status", C.c_int32), ("inliers", C.c_int64), ("step", C.c_double), ("residual", C.c_double)]


class VolumeBuffers(C.Structure):
    _fields_ = [("keys", C.c_void_p), ("sdf", C.c_void_p), ("weight", C.c_void_p), ("rgb", C.c_void_p)]


_lib = None


def lib():
    """Load libdtsdf.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2301_12796_b200.build` "
                              "or __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        P, I32, I64 = C.c_void_p, C.c_int32, C.c_int64
        L.dtsdf_create.argtypes = [C.c_int, C.POINTER(P)]
        L.dtsdf_destroy.argtypes = [P]
        L.dtsdf_alloc_volume.argtypes = [P, C.POINTER(VolumeParams), C.POINTER(VolumeBuffers)]
        L.dtsdf_commit_volume.argtypes = [P, P]
        L.dtsdf_upload_volume.argtypes = [P, C.POINTER(VolumeParams), P, P, P, P]
        L.dtsdf_render.argtypes = [P, P, C.POINTER(Intrinsics), P, P, P, P, P]
        L.dtsdf_render_batch.argtypes = [P, I32, P, C.POINTER(Intrinsics), I32, I32, P, P, P, P, P]
        L.dtsdf_volume_stats.argtypes = [P, C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)]
        L.dtsdf_set_profiling.argtypes = [P, C.c_int]
        L.dtsdf_kernel_times.argtypes = [P, P, P]
        L.dtsdf_reset_kernel_times.argtypes = [P]
        L.dtsdf_set_option.argtypes = [P, C.c_int, C.c_int]
        L.dtsdf_launch_count.argtypes = [P]
        L.dtsdf_launch_count.restype = I64
        L.dtsdf_combine.argtypes = [P, P, C.POINTER(Intrinsics), C.c_float, P]
        L.dtsdf_combine_mode.argtypes = [P, P, C.POINTER(Intrinsics), C.c_float, C.c_int32, C.c_float, P]
        L.dtsdf_render_combined.argtypes = [P, I32, P, C.POINTER(Intrinsics), I32, I32, P, P, P, P, P]
        L.dtsdf_combined_stats.argtypes = [P, C.POINTER(I64), C.POINTER(I64)]
        L.dtsdf_get_combined.argtypes = [P, I64, P, P, P, P, P, C.POINTER(I64)]
        L.dtsdf_default_policy.argtypes = [C.POINTER(CombinePolicy)]
        L.dtsdf_default_policy.restype = None
        L.dtsdf_should_recombine.argtypes = [C.POINTER(CombinePolicy), I64, I64, P, P]
        L.dtsdf_default_fusion_params.argtypes = [C.POINTER(FusionParams)]
        L.dtsdf_default_fusion_params.restype = None
        L.dtsdf_fusion_reserve.argtypes = [P, C.POINTER(VolumeParams), I64]
        L.dtsdf_depth_normals.argtypes = [P, P, C.POINTER(Intrinsics), P, P]
        L.dtsdf_fuse.argtypes = [P, P, P, P, P, C.POINTER(Intrinsics), C.POINTER(FusionParams), C.POINTER(I64), P]
        L.dtsdf_get_volume.argtypes = [P, I64, P, P, P, P, C.POINTER(I64)]
        L.dtsdf_default_icp_params.argtypes = [C.POINTER(IcpParams)]
        L.dtsdf_default_icp_params.restype = None
        L.dtsdf_icp.argtypes = [P, P, P, P, P, C.POINTER(Intrinsics), P, C.POINTER(IcpParams), C.POINTER(IcpResult), P]
        L.dtsdf_icp_normal_equations.argtypes = [P, P, P, P, P, C.POINTER(Intrinsics), P, C.c_float, P, P,
                                                 C.POINTER(I64), C.POINTER(C.c_double), P]
        L.dtsdf_last_error.argtypes = []
        L.dtsdf_last_error.restype = C.c_char_p
        L.dtsdf_last_warning.argtypes = []
        L.dtsdf_last_warning.restype = C.c_char_p
        _lib = L
    return _lib


def last_warning() -> str:
    """dtsdf_last_warning: the warning the last parameter check on this thread left ("" if none)."""
    return lib().dtsdf_last_warning().decode()


def _check(rc):
    if rc != OK:
        raise DtsdfError(rc, lib().dtsdf_last_error().decode())


def _ptr(x) -> Optional[int]:
    """Device/host address of a torch tensor or numpy array (None passes NULL)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensors must be contiguous")
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays must be C-contiguous")
        return x.ctypes.data
    raise TypeError(f"unsupported buffer type {type(x)}")


def _stream_ptr(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    return getattr(stream, "cuda_stream", stream)


def make_intrinsics(K) -> Intrinsics:
    """From any object with fx fy cx cy width height z_min z_max."""
    return Intrinsics(K.fx, K.fy, K.cx, K.cy, int(K.width), int(K.height), K.z_min, K.z_max)


class Renderer:
    """One libdtsdf context on one CUDA device."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        _check(lib().dtsdf_create(int(device), C.byref(self._h)))
        self.device = device

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().dtsdf_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- volume -------------------------------------------------------------------------
    def upload(self, voxel_size, truncation, theta, keys, sdf, weight, rgb=None, step=0.0):
        """dtsdf_upload_volume: arrays may be numpy (host) or torch tensors (host or device)."""
        n = int(keys.shape[0])
        p = VolumeParams(voxel_size, truncation, theta, step, n)
        _check(lib().dtsdf_upload_volume(self._h, C.byref(p), _ptr(keys), _ptr(sdf), _ptr(weight), _ptr(rgb)))

    def upload_volume(self, vol):
        """Upload a scenes.BlockVolume (host arrays)."""
        self.upload(vol.voxel_size, vol.truncation, vol.theta, vol.keys, vol.sdf, vol.weight, vol.rgb, vol.step)

    def alloc(self, voxel_size, truncation, theta, n_blocks, step=0.0):
        """dtsdf_alloc_volume: returns torch tensors aliasing the library-owned device buffers."""
        import torch
        p = VolumeParams(voxel_size, truncation, theta, step, int(n_blocks))
        b = VolumeBuffers()
        _check(lib().dtsdf_alloc_volume(self._h, C.byref(p), C.byref(b)))
        return {"keys": _wrap_device(b.keys, (n_blocks, 4), torch.int32, self.device),
                "sdf": _wrap_device(b.sdf, (n_blocks, 512), torch.float32, self.device),
                "weight": _wrap_device(b.weight, (n_blocks, 512), torch.float32, self.device),
                "rgb": _wrap_device(b.rgb, (n_blocks, 512, 3), torch.uint8, self.device)}

    def commit(self, stream=None):
        _check(lib().dtsdf_commit_volume(self._h, _stream_ptr(stream)))

    def stats(self):
        n, u, b = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib().dtsdf_volume_stats(self._h, C.byref(n), C.byref(u), C.byref(b)))
        return {"n_blocks": n.value, "n_locations": u.value, "bytes": b.value}

    # -- render -------------------------------------------------------------------------
    def render_into(self, poses, K, depth, normal=None, color=None, mask=None, row0=0, row1=None, stream=None):
        """dtsdf_render_batch into caller-owned outputs (all device tensors -> async on the stream;
        all host arrays/tensors -> synchronous)."""
        poses = np.ascontiguousarray(np.asarray(poses, np.float32).reshape(-1, 16))
        row1 = K.height if row1 is None else row1
        k = make_intrinsics(K)
        _check(lib().dtsdf_render_batch(self._h, poses.shape[0], poses.ctypes.data, C.byref(k), int(row0), int(row1),
                                        _ptr(depth), _ptr(normal), _ptr(color), _ptr(mask), _stream_ptr(stream)))

    def render_view(self, pose, K, depth, normal=None, color=None, mask=None, stream=None):
        """dtsdf_render: one view (pose = world-from-camera 4x4) into caller-owned outputs (device
        tensors -> async on the stream; host arrays / tensors, pinned or pageable -> synchronous)."""
        pose = np.ascontiguousarray(np.asarray(pose, np.float32).reshape(16))
        k = make_intrinsics(K)
        _check(lib().dtsdf_render(self._h, pose.ctypes.data, C.byref(k), _ptr(depth), _ptr(normal), _ptr(color),
                                  _ptr(mask), _stream_ptr(stream)))

    def render(self, poses, K, row0=0, row1=None, stream=None, outputs=("normal", "color", "mask"),
               combined=False):
        """Allocate device outputs and render (the combined TSDF if combined=True); returns dict of
        torch tensors [V, rows, W, ...]."""
        import torch
        poses = np.asarray(poses, np.float32).reshape(-1, 4, 4)
        row1 = K.height if row1 is None else row1
        V, rows, W = poses.shape[0], row1 - row0, K.width
        dev = torch.device("cuda", self.device)
        out = {"depth": torch.empty((V, rows, W), dtype=torch.float32, device=dev)}
        if "normal" in outputs:
            out["normal"] = torch.empty((V, rows, W, 3), dtype=torch.float32, device=dev)
        if "color" in outputs:
            out["color"] = torch.empty((V, rows, W, 3), dtype=torch.uint8, device=dev)
        if "mask" in outputs:
            out["mask"] = torch.empty((V, rows, W), dtype=torch.uint8, device=dev)
        fn = self.render_combined_into if combined else self.render_into
        fn(poses, K, out["depth"], out.get("normal"), out.get("color"), out.get("mask"), row0, row1, stream)
        return out

    # -- fusion (NEXT-2) --------------------------------------------------------------------
    def fusion_reserve(self, capacity, voxel_size=0.01, truncation=0.04, theta=None, step=0.0):
        """dtsdf_fusion_reserve: room for `capacity` blocks (an empty volume if none is loaded)."""
        theta = float(np.deg2rad(65.0)) if theta is None else theta
        p = VolumeParams(voxel_size, truncation, theta, step, 0)
        _check(lib().dtsdf_fusion_reserve(self._h, C.byref(p), int(capacity)))

    def depth_normals(self, depth, K, out=None, stream=None):
        """dtsdf_depth_normals: camera-frame normals [H, W, 3] of a depth map (host or device)."""
        if out is None:
            out = np.zeros(tuple(depth.shape) + (3,), np.float32) if isinstance(depth, np.ndarray) else \
                depth.new_zeros(tuple(depth.shape) + (3,))
        k = make_intrinsics(K)
        _check(lib().dtsdf_depth_normals(self._h, _ptr(depth), C.byref(k), _ptr(out), _stream_ptr(stream)))
        return out

    def fuse(self, depth, normal, color, pose, K, params: Optional[FusionParams] = None, stream=None) -> int:
        """dtsdf_fuse: allocate + fuse one frame (host or device buffers); returns new blocks."""
        pose = np.ascontiguousarray(np.asarray(pose, np.float32).reshape(16))
        k = make_intrinsics(K)
        nb = C.c_int64()
        prm = C.byref(params) if params is not None else None
        _check(lib().dtsdf_fuse(self._h, _ptr(depth), _ptr(normal), _ptr(color), pose.ctypes.data, C.byref(k), prm,
                                C.byref(nb), _stream_ptr(stream)))
        return nb.value

    def get_volume(self):
        """dtsdf_get_volume -> (keys [n,4], sdf [n,512], weight [n,512], rgb [n,512,3]) host arrays."""
        n = self.stats()["n_blocks"]
        keys = np.zeros((n, 4), np.int32)
        sdf = np.zeros((n, 512), np.float32)
        w = np.zeros((n, 512), np.float32)
        rgb = np.zeros((n, 512, 3), np.uint8)
        got = C.c_int64()
        _check(lib().dtsdf_get_volume(self._h, n, _ptr(keys), _ptr(sdf), _ptr(w), _ptr(rgb), C.byref(got)))
        return keys, sdf, w, rgb

    # -- ICP (NEXT-3) -----------------------------------------------------------------------
    def icp(self, depth, ref_depth, ref_normal, ref_pose, K, init_delta=None, max_iters=50, min_step=1e-6,
            outlier=0.005, stream=None, raise_singular=True):
        """dtsdf_icp: DeltaT (frame camera -> rendered view camera, float64 [4,4]) and a result dict."""
        prm = IcpParams(int(max_iters), float(min_step), float(outlier), 0)
        res = IcpResult()
        ref_pose = np.ascontiguousarray(np.asarray(ref_pose, np.float32).reshape(16))
        init = None if init_delta is None else np.ascontiguousarray(np.asarray(init_delta, np.float32).reshape(16))
        k = make_intrinsics(K)
        rc = lib().dtsdf_icp(self._h, _ptr(depth), _ptr(ref_depth), _ptr(ref_normal), ref_pose.ctypes.data,
                             C.byref(k), None if init is None else init.ctypes.data, C.byref(prm), C.byref(res),
                             _stream_ptr(stream))
        if rc != OK and (rc != SINGULAR or raise_singular):
            _check(rc)
        info = dict(iterations=res.iterations, status=res.status, inliers=res.inliers, step=res.step,
                    residual=res.residual)
        return np.array(res.delta64[:], np.float64).reshape(4, 4), info

    def icp_normal_equations(self, depth, ref_depth, ref_normal, ref_pose, K, delta=None, outlier=0.005,
                             stream=None):
        """dtsdf_icp_normal_equations -> (H [6,6], g [6], inliers, sum w r^2)."""
        delta = np.ascontiguousarray(np.eye(4) if delta is None else delta, np.float64).reshape(16)
        ref_pose = np.ascontiguousarray(np.asarray(ref_pose, np.float32).reshape(16))
        H, g = np.zeros(36), np.zeros(6)
        n, r = C.c_int64(), C.c_double()
        k = make_intrinsics(K)
        _check(lib().dtsdf_icp_normal_equations(self._h, _ptr(depth), _ptr(ref_depth), _ptr(ref_normal),
                                                ref_pose.ctypes.data, C.byref(k), delta.ctypes.data,
                                                float(outlier), H.ctypes.data, g.ctypes.data, C.byref(n),
                                                C.byref(r), _stream_ptr(stream)))
        return H.reshape(6, 6), g, n.value, r.value

    # -- combined TSDF (NEXT-1) -----------------------------------------------------------
    def combine(self, pose, K, margin=MARGIN, stream=None, mode=0, w_floor=0.0):
        """dtsdf_combine_mode: the view-dependent combined TSDF of the source camera (pose, K);
        mode 0 = eq:combine_weight (the paper's method), 1 = Algorithm 1."""
        pose = np.ascontiguousarray(np.asarray(pose, np.float32).reshape(16))
        k = make_intrinsics(K)
        _check(lib().dtsdf_combine_mode(self._h, pose.ctypes.data, C.byref(k), float(margin), int(mode),
                                        float(w_floor), _stream_ptr(stream)))

    def render_combined_into(self, poses, K, depth, normal=None, color=None, mask=None, row0=0, row1=None,
                             stream=None):
        """dtsdf_render_combined into caller-owned outputs (layout as render_into)."""
        poses = np.ascontiguousarray(np.asarray(poses, np.float32).reshape(-1, 16))
        row1 = K.height if row1 is None else row1
        k = make_intrinsics(K)
        _check(lib().dtsdf_render_combined(self._h, poses.shape[0], poses.ctypes.data, C.byref(k), int(row0),
                                           int(row1), _ptr(depth), _ptr(normal), _ptr(color), _ptr(mask),
                                           _stream_ptr(stream)))

    def combined_stats(self):
        u, b = C.c_int64(), C.c_int64()
        _check(lib().dtsdf_combined_stats(self._h, C.byref(u), C.byref(b)))
        return {"n_locations": u.value, "bytes": b.value}

    def get_combined(self):
        """dtsdf_get_combined -> dict(locs [n,3], sdf [n,512], weight [n,512], rgb [n,512,3], mask [n,512])."""
        n = self.combined_stats()["n_locations"]
        out = {"locs": np.zeros((n, 3), np.int32), "sdf": np.zeros((n, 512), np.float32),
               "weight": np.zeros((n, 512), np.float32), "rgb": np.zeros((n, 512, 3), np.uint8),
               "mask": np.zeros((n, 512), np.uint8)}
        got = C.c_int64()
        _check(lib().dtsdf_get_combined(self._h, n, _ptr(out["locs"]), _ptr(out["sdf"]), _ptr(out["weight"]),
                                        _ptr(out["rgb"]), _ptr(out["mask"]), C.byref(got)))
        return out

    # -- tracing ------------------------------------------------------------------------
    def set_profiling(self, enable: bool):
        _check(lib().dtsdf_set_profiling(self._h, int(bool(enable))))

    def kernel_times(self):
        t = np.zeros(4, np.float64)
        n = np.zeros(4, np.int64)
        _check(lib().dtsdf_kernel_times(self._h, t.ctypes.data, n.ctypes.data))
        return {"range_ms": t[0], "raycast_ms": t[1], "other_ms": t[2], "combine_ms": t[3],
                "range_launches": int(n[0]), "raycast_launches": int(n[1]), "other_launches": int(n[2]),
                "combine_launches": int(n[3])}

    def reset_kernel_times(self):
        _check(lib().dtsdf_reset_kernel_times(self._h))

    def set_option(self, option: int, value: int):
        value = int(value)
        if value > 0x7FFFFFFF:  # options read as uint32 (DTSDF_OPT_RANGE_EPOCH) pass their bits
            value -= 1 << 32
        _check(lib().dtsdf_set_option(self._h, int(option), value))

    def launch_count(self) -> int:
        return int(lib().dtsdf_launch_count(self._h))


def default_policy() -> CombinePolicy:
    p = CombinePolicy()
    lib().dtsdf_default_policy(C.byref(p))
    return p


def should_recombine(frame: int, last: int, pose, last_pose, policy: Optional[CombinePolicy] = None) -> bool:
    """dtsdf_should_recombine: eqs. condition_1-4."""
    policy = policy or default_policy()
    a = np.ascontiguousarray(np.asarray(pose, np.float32).reshape(16))
    b = np.ascontiguousarray(np.asarray(last_pose, np.float32).reshape(16))
    rc = lib().dtsdf_should_recombine(C.byref(policy), int(frame), int(last), a.ctypes.data, b.ctypes.data)
    if rc < 0:
        _check(rc)
    return bool(rc)


def _wrap_device(ptr, shape, dtype, device):
    """A torch tensor view of library-owned device memory (no copy, no ownership)."""
    import torch
    nbytes = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
    if nbytes == 0:
        return torch.empty(shape, dtype=dtype, device=f"cuda:{device}")
    # __cuda_array_interface__ lets torch alias external device memory without taking ownership
    typestr = {torch.int32: "<i4", torch.float32: "<f4", torch.uint8: "|u1"}[dtype]

    class _CAI:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                    "version": 3, "strides": None}

    with torch.cuda.device(device):
        return torch.as_tensor(_CAI(), device=f"cuda:{device}")
