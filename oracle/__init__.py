"""CPU oracle for the DTSDF raycast hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2301_12796_b200``) never imports it, and it never imports the product path.

``liboracle.so`` is plain C in fp64 (``oracle.c`` raycast and combined TSDF, ``fusion.c``
voxel-projection fusion, ``icp.c`` point-to-plane ICP); this module only marshals arguments.
Every function cites the passage it follows in ``oracle.c``; DESIGN.md §4 lists the readings.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRCS = [os.path.join(_HERE, "oracle.c"), os.path.join(_HERE, "fusion.c"), os.path.join(_HERE, "icp.c")]
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

CFLAGS = ["-O2", "-std=c11", "-D_GNU_SOURCE", "-ffp-contract=off", "-fno-fast-math", "-Wall", "-shared", "-fPIC",
          "-pthread"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no -ffast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB_PATH) or any(os.path.getmtime(_LIB_PATH) < os.path.getmtime(s)
                                                     for s in _SRCS):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, *_SRCS, "-lm", "-o", tmp])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        P, D, I64, I32 = C.c_void_p, C.c_double, C.c_int64, C.c_int
        L.oracle_volume_create.argtypes = [D, D, D, D, I64, P, P, P, P, C.POINTER(P)]
        L.oracle_volume_create.restype = I32
        L.oracle_volume_destroy.argtypes = [P]
        L.oracle_enable_counting.argtypes = [P]
        L.oracle_counts.argtypes = [P, P]
        L.oracle_trilinear.argtypes = [P, I32, P, P, P]
        L.oracle_gradient.argtypes = [P, I32, P, P]
        L.oracle_w_dir.argtypes = [D, D]
        L.oracle_w_dir.restype = D
        L.oracle_eval.argtypes = [P, P, P, P]
        L.oracle_render.argtypes = [P, P, P, I64, P, I32, I32, P, P, P, P, P]
        L.oracle_render.restype = None
        L.oracle_combined_voxels_mode.argtypes = [P, P, P, D, I32, D, I64, P, P, P, P, P, P]
        L.oracle_combined_voxels_mode.restype = None
        L.oracle_render_combined_mode.argtypes = [P, P, P, D, I32, D, P, P, I64, P, I32, I32, P, P, P, P]
        L.oracle_render_combined_mode.restype = None
        L.oracle_combined_voxels_update.argtypes = [P, P, P, P, D, I32, D, I64, P, P, P, P, P, P]
        L.oracle_combined_voxels_update.restype = None
        L.oracle_render_combined_update.argtypes = [P, P, P, P, D, I32, D, P, P, I64, P, I32, I32, P, P, P, P]
        L.oracle_render_combined_update.restype = None
        L.oracle_should_recombine.argtypes = [I64, I64, P, P, I64, I64, D, D]
        L.oracle_should_recombine.restype = I32
        L.oracle_fuse_create.argtypes = [D, D, D, I64, I64, P, P, P, P, C.POINTER(P)]
        L.oracle_fuse_create.restype = I32
        L.oracle_fuse_destroy.argtypes = [P]
        L.oracle_fuse_count.argtypes = [P]
        L.oracle_fuse_count.restype = I64
        L.oracle_fuse_get.argtypes = [P, P, P, P, P, P]
        L.oracle_fuse_get.restype = None
        L.oracle_fuse_frame.argtypes = [P, P, P, P, P, P, P]
        L.oracle_fuse_frame.restype = I64
        L.oracle_depth_normals.argtypes = [P, P, P]
        L.oracle_depth_normals.restype = None
        L.oracle_se3_exp.argtypes = [P, P]
        L.oracle_se3_exp.restype = None
        L.oracle_icp_normal_equations.argtypes = [P, P, P, P, P, P, D, P, P, P]
        L.oracle_icp_normal_equations.restype = None
        L.oracle_cholesky_solve6.argtypes = [P, P, P]
        L.oracle_cholesky_solve6.restype = I32
        L.oracle_icp.argtypes = [P, P, P, P, P, D, I32, D, P, P]
        L.oracle_icp.restype = I32
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def w_dir(cosang: float, theta: float) -> float:
    """eq:direction_weight with reading R1."""
    return lib().oracle_w_dir(float(cosang), float(theta))


class OracleVolume:
    """Dense per-direction block grid over a BlockVolume (keeps references to its arrays)."""

    def __init__(self, vol, counting: bool = False):
        self.vol = vol
        self._keys = np.ascontiguousarray(vol.keys, np.int32)
        self._sdf = np.ascontiguousarray(vol.sdf, np.float32)
        self._w = np.ascontiguousarray(vol.weight, np.float32)
        self._rgb = np.ascontiguousarray(vol.rgb, np.uint8)
        h = C.c_void_p()
        # the scalar parameters as the float32 values the C ABI receives (dtsdf_volume_params)
        f32 = lambda a: float(np.float32(a))  # noqa: E731
        rc = lib().oracle_volume_create(f32(vol.voxel_size), f32(vol.truncation), f32(vol.theta), f32(vol.step),
                                        vol.n_blocks,
                                        _ptr(self._keys), _ptr(self._sdf), _ptr(self._w), _ptr(self._rgb),
                                        C.byref(h))
        if rc != 0:
            raise ValueError(f"oracle_volume_create failed: {rc}")
        self.h = h
        if counting and lib().oracle_enable_counting(self.h) != 0:
            raise MemoryError("oracle counting buffers")

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and _lib is not None:
            _lib.oracle_volume_destroy(h)
            self.h = None

    def counts(self):
        out = np.zeros(3, np.int64)
        lib().oracle_counts(self.h, _ptr(out))
        return {"voxel_records": int(out[0]), "rgb_records": int(out[1]), "locations": int(out[2])}

    def trilinear(self, D, x):
        x = np.asarray(x, np.float64)
        phi, om = C.c_double(), C.c_double()
        ok = lib().oracle_trilinear(self.h, D, _ptr(x), C.byref(phi), C.byref(om))
        return (phi.value, om.value) if ok else None

    def gradient(self, D, x):
        x = np.asarray(x, np.float64)
        g = np.zeros(3)
        ok = lib().oracle_gradient(self.h, D, _ptr(x), _ptr(g))
        return g if ok else None

    def eval(self, x, r):
        """O3 F(x, r): dict(valid, f, S, regime, W[6], nt[6,3], phi[6], omega[6], present[6], has_grad[6])."""
        x = np.asarray(x, np.float64)
        r = np.asarray(r, np.float64)
        out = np.zeros(52)
        lib().oracle_eval(self.h, _ptr(x), _ptr(r), _ptr(out))
        return dict(valid=bool(out[0]), f=out[1], S=out[2], regime=int(out[3]), W=out[4:10].copy(),
                    nt=out[10:28].reshape(6, 3).copy(), phi=out[28:34].copy(), omega=out[34:40].copy(),
                    present=out[40:46].astype(bool), has_grad=out[46:52].astype(bool))

    def render(self, pose, K, pixels=None, row0=0, row1=None, threads=None, nsamples=False):
        """Render one view.  pixels: int [P, 2] (u, v) list, or None for rows [row0, row1).

        Inputs are the float32 values the GPU path receives (pose and intrinsics are rounded
        to float32 first).  Returns dict(depth [P] or [h,W], normal, color, mask[, nsamples])."""
        pose32 = np.asarray(pose, np.float32).astype(np.float64).reshape(16)
        intr = np.array([np.float32(K.fx), np.float32(K.fy), np.float32(K.cx), np.float32(K.cy), K.width, K.height,
                         np.float32(K.z_min), np.float32(K.z_max)], np.float64)
        if pixels is None:
            row1 = K.height if row1 is None else row1
            npix = (row1 - row0) * K.width
            uv = None
            shape = (row1 - row0, K.width)
        else:
            uv = np.ascontiguousarray(pixels, np.int32).reshape(-1, 2)
            npix = uv.shape[0]
            shape = (npix,)
        depth = np.zeros(npix)
        normal = np.zeros((npix, 3))
        color = np.zeros((npix, 3), np.uint8)
        mask = np.zeros(npix, np.uint8)
        ns = np.zeros(npix, np.int32) if nsamples else None
        threads = threads or os.cpu_count() or 1
        lib().oracle_render(self.h, _ptr(pose32), _ptr(intr), npix, _ptr(uv), row0, threads, _ptr(depth),
                            _ptr(normal), _ptr(color), _ptr(mask), _ptr(ns))
        out = dict(depth=depth.reshape(shape), normal=normal.reshape(shape + (3,)),
                   color=color.reshape(shape + (3,)), mask=mask.reshape(shape))
        if nsamples:
            out["nsamples"] = ns.reshape(shape)
        return out


MARGIN = 1.0 / 8.0  # PAPER.md:262 "slightly beyond the camera frustum (±1/8 image size)"


def _pose32(pose):
    return np.ascontiguousarray(np.asarray(pose, np.float32).astype(np.float64).reshape(16))


def _intr32(K):
    return np.array([np.float32(K.fx), np.float32(K.fy), np.float32(K.cx), np.float32(K.cy), K.width, K.height,
                     np.float32(K.z_min), np.float32(K.z_max)], np.float64)


def combined_voxels(ov: "OracleVolume", pose, K, ijk, margin: float = MARGIN, mode: int = 0, w_floor: float = 0.0,
                    before: "OracleVolume" = None):
    """Combined TSDF voxels (oracle.c combine_voxel, readings R33-R35; mode 1: Algorithm 1,
    R53-R57) at integer positions ijk [n, 3] for the source camera (pose, K).  before: the volume
    the combined TSDF was computed from when fusion has since changed it to ov (reading R58:
    first-time voxels from ov, the others from before).  Returns dict(valid, sdf, weight, rgb, mask)."""
    ijk = np.ascontiguousarray(ijk, np.int64).reshape(-1, 3)
    n = len(ijk)
    valid = np.zeros(n, np.int32)
    sdf, S = np.zeros(n), np.zeros(n)
    rgb = np.zeros((n, 3), np.uint8)
    mask = np.zeros(n, np.uint8)
    args = (_ptr(_pose32(pose)), _ptr(_intr32(K)), float(np.float32(margin)), int(mode), float(np.float32(w_floor)),
            n, _ptr(ijk), _ptr(valid), _ptr(sdf), _ptr(S), _ptr(rgb), _ptr(mask))
    if before is None:
        lib().oracle_combined_voxels_mode(ov.h, *args)
    else:
        lib().oracle_combined_voxels_update(before.h, ov.h, *args)
    return dict(valid=valid.astype(bool), sdf=sdf, weight=S, rgb=rgb, mask=mask)


def render_combined(ov: "OracleVolume", src_pose, src_K, pose, K, pixels=None, row0=0, row1=None, threads=None,
                    margin: float = MARGIN, mode: int = 0, w_floor: float = 0.0, before: "OracleVolume" = None):
    """Raycast (pose, K) through the combined TSDF of the source camera (src_pose, src_K)
    (oracle.c render_pixel_combined, readings R36-R37; before: as combined_voxels, R58).
    Output layout as OracleVolume.render."""
    if pixels is None:
        row1 = K.height if row1 is None else row1
        npix = (row1 - row0) * K.width
        uv = None
        shape = (row1 - row0, K.width)
    else:
        uv = np.ascontiguousarray(pixels, np.int32).reshape(-1, 2)
        npix = uv.shape[0]
        shape = (npix,)
    depth = np.zeros(npix)
    normal = np.zeros((npix, 3))
    color = np.zeros((npix, 3), np.uint8)
    mask = np.zeros(npix, np.uint8)
    threads = threads or os.cpu_count() or 1
    args = (_ptr(_pose32(src_pose)), _ptr(_intr32(src_K)), float(np.float32(margin)), int(mode),
            float(np.float32(w_floor)), _ptr(_pose32(pose)), _ptr(_intr32(K)), npix, _ptr(uv), row0, threads,
            _ptr(depth), _ptr(normal), _ptr(color), _ptr(mask))
    if before is None:
        lib().oracle_render_combined_mode(ov.h, *args)
    else:
        lib().oracle_render_combined_update(before.h, ov.h, *args)
    return dict(depth=depth.reshape(shape), normal=normal.reshape(shape + (3,)), color=color.reshape(shape + (3,)),
                mask=mask.reshape(shape))


def should_recombine(frame: int, last: int, pose, last_pose, boot: int = 5, stale: int = 50, trans: float = 0.05,
                     rot: float = 0.05 * np.pi / 2) -> bool:
    """Conditional combination, eqs. condition_1-4, reading R38."""
    return bool(lib().oracle_should_recombine(int(frame), int(last), _ptr(_pose32(pose)), _ptr(_pose32(last_pose)),
                                              int(boot), int(stale), float(trans), float(rot)))


def ray_dirs(pose, K, pixels=None):
    """O1 in numpy for test-side closed forms: camera-centre o and unit world rays r per pixel
    plus L = |d~| (depth = t / L).  pose/intrinsics rounded to float32 like the render inputs."""
    pose = np.asarray(pose, np.float32).astype(np.float64)
    if pixels is None:
        v, u = np.mgrid[0:K.height, 0:K.width]
        u, v = u.ravel(), v.ravel()
    else:
        u, v = np.asarray(pixels)[:, 0], np.asarray(pixels)[:, 1]
    fx, fy, cx, cy = (float(np.float32(a)) for a in (K.fx, K.fy, K.cx, K.cy))
    dt = np.stack([(u - cx) / fx, (v - cy) / fy, np.ones_like(u, dtype=np.float64)], -1)
    L = np.linalg.norm(dt, axis=-1)
    r = (dt / L[:, None]) @ pose[:3, :3].T
    return pose[:3, 3], r, L


# ------------------------------------------------------------------------------------------
# NEXT-2: voxel-projection fusion (fusion.c, readings R39-R46)
# ------------------------------------------------------------------------------------------
W_MAX, CARVE_WEIGHT, CARVE_RADIUS = 128.0, 1.0, 2


def depth_normals(depth, K):
    """Camera-frame normals of a depth map (fusion.c oracle_depth_normals, reading R39)."""
    depth = np.ascontiguousarray(depth, np.float32)
    out = np.zeros(depth.shape + (3,), np.float32)
    lib().oracle_depth_normals(_ptr(depth), _ptr(_intr32(K)), _ptr(out))
    return out


class OracleFusion:
    """A growable DTSDF fused from depth frames (fusion.c).  Parameters as the float32 values the
    C ABI receives."""

    def __init__(self, voxel_size, truncation, theta, capacity, vol=None):
        f32 = lambda a: float(np.float32(a))  # noqa: E731
        h = C.c_void_p()
        n0 = 0 if vol is None else vol.n_blocks
        self._init = None
        if vol is not None:
            self._init = (np.ascontiguousarray(vol.keys, np.int32), np.ascontiguousarray(vol.sdf, np.float32),
                          np.ascontiguousarray(vol.weight, np.float32), np.ascontiguousarray(vol.rgb, np.uint8))
        args = [_ptr(a) for a in self._init] if self._init else [None] * 4
        rc = lib().oracle_fuse_create(f32(voxel_size), f32(truncation), f32(theta), int(capacity), int(n0), *args,
                                      C.byref(h))
        if rc != 0:
            raise ValueError(f"oracle_fuse_create failed: {rc}")
        self.h = h
        self.voxel_size, self.truncation, self.theta = voxel_size, truncation, theta

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and _lib is not None:
            _lib.oracle_fuse_destroy(h)
            self.h = None

    def fuse(self, depth, normal, color, pose, K, w_max=W_MAX, carve_weight=CARVE_WEIGHT, carve_radius=CARVE_RADIUS):
        """Allocate + fuse one frame; returns the number of new blocks (raises when full)."""
        depth = np.ascontiguousarray(depth, np.float32)
        normal = np.ascontiguousarray(normal, np.float32)
        color = None if color is None else np.ascontiguousarray(color, np.uint8)
        prm = np.array([np.float32(w_max), np.float32(carve_weight), carve_radius], np.float64)
        n = lib().oracle_fuse_frame(self.h, _ptr(depth), _ptr(normal), _ptr(color), _ptr(_pose32(pose)),
                                    _ptr(_intr32(K)), _ptr(prm))
        if n < 0:
            raise MemoryError("oracle fusion capacity exhausted")
        return int(n)

    def volume(self, with_color_weight=False):
        """The fused blocks as a scenes.BlockVolume (insertion order)."""
        from scenes import BlockVolume
        n = int(lib().oracle_fuse_count(self.h))
        keys = np.zeros((n, 4), np.int32)
        sdf = np.zeros((n, 512), np.float32)
        w = np.zeros((n, 512), np.float32)
        rgb = np.zeros((n, 512, 3), np.uint8)
        cw = np.zeros((n, 512), np.float32)
        lib().oracle_fuse_get(self.h, _ptr(keys), _ptr(sdf), _ptr(w), _ptr(rgb), _ptr(cw))
        vol = BlockVolume(self.voxel_size, self.truncation, self.theta, keys, sdf, w, rgb, 0.0)
        return (vol, cw) if with_color_weight else vol


# ------------------------------------------------------------------------------------------
# NEXT-3: weighted geometric point-to-plane ICP (icp.c, readings R47-R52)
# ------------------------------------------------------------------------------------------
ICP_MAX_ITERS, ICP_MIN_STEP, ICP_OUTLIER = 50, 1e-6, 0.005  # PAPER.md:626-628 (fine level)


def se3_exp(xi):
    xi = np.ascontiguousarray(xi, np.float64)
    T = np.zeros(16)
    lib().oracle_se3_exp(_ptr(xi), _ptr(T))
    return T.reshape(4, 4)


def _icp_inputs(depth, ref_depth, ref_normal):
    return (np.ascontiguousarray(depth, np.float32), np.ascontiguousarray(ref_depth, np.float32),
            np.ascontiguousarray(ref_normal, np.float32))


def icp_normal_equations(depth, ref_depth, ref_normal, ref_pose, K, delta=None, outlier=ICP_OUTLIER):
    """(H [6,6], g [6], inliers, sum w r^2) of eq:ICP_Hessian at DeltaT = delta."""
    d, rd, rn = _icp_inputs(depth, ref_depth, ref_normal)
    delta = np.ascontiguousarray(np.eye(4) if delta is None else delta, np.float64).reshape(16)
    H, g, st = np.zeros(36), np.zeros(6), np.zeros(2)
    lib().oracle_icp_normal_equations(_ptr(d), _ptr(rd), _ptr(rn), _ptr(_pose32(ref_pose)), _ptr(_intr32(K)),
                                      _ptr(delta), float(np.float32(outlier)), _ptr(H), _ptr(g), _ptr(st))
    return H.reshape(6, 6), g, int(st[0]), float(st[1])


def cholesky_solve6(H, b):
    x = np.zeros(6)
    rc = lib().oracle_cholesky_solve6(_ptr(np.ascontiguousarray(H, np.float64).reshape(36)),
                                      _ptr(np.ascontiguousarray(b, np.float64)), _ptr(x))
    return x if rc == 0 else None


def icp(depth, ref_depth, ref_normal, ref_pose, K, delta=None, outlier=ICP_OUTLIER, max_iters=ICP_MAX_ITERS,
        min_step=ICP_MIN_STEP):
    """Gauss-Newton ICP (eq:ICP_solution / eq:deltaT_update).  Returns (DeltaT [4,4] mapping the
    frame's camera into the rendered view's camera, dict(iterations, step, inliers, residual, ok))."""
    d, rd, rn = _icp_inputs(depth, ref_depth, ref_normal)
    delta = np.ascontiguousarray(np.eye(4) if delta is None else delta, np.float64).reshape(16).copy()
    out = np.zeros(4)
    rc = lib().oracle_icp(_ptr(d), _ptr(rd), _ptr(rn), _ptr(_pose32(ref_pose)), _ptr(_intr32(K)),
                          float(np.float32(outlier)), int(max_iters), float(min_step), _ptr(delta), _ptr(out))
    return delta.reshape(4, 4), dict(iterations=int(out[0]), step=out[1], inliers=int(out[2]), residual=out[3],
                                     ok=rc == 0)
