"""Seeded synthetic DTSDF volumes (SURVEY.md §8(d) generator rules G0 and G1).

These stand in for volumes fused from the paper's RGB-D datasets, which are
not available here.  They emulate *ideal* fusion of analytic geometry:

  * G0 (BASELINE.json configs[0]): every voxel of every direction of a dense 64^3 grid holds
    the clamped normalised distance to one sphere and the directional weight max(0, n.v^D)
    (the "old" direction factor of PAPER.md:87, which configs[0] prescribes).
  * G1 (configs[1..4]): geometry is a set of rectangular patches with outward normals and
    colours.  A patch is written into direction D iff its normal passes the angular
    threshold of eq:angular_threshold, with weight <n, v^D> (the direction
    factor of PAPER.md:87) -- a stand-in for eq:combined_fusion_weight with
    w_depth = w_angle = 1.  The signed distance is the point-to-plane distance,
    positive in front of the surface (reading R6), normalised by tau and
    clamped to [-1, 1].

Nothing here evaluates the rendering method (membership ramp, combination weights, trilinear
interpolation, gradients, march or refinement); those live separately in ``oracle/`` and in
the CUDA path.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess

import numpy as np

from .volume import BLOCK, DIRECTION_VECTORS, VOXELS_PER_BLOCK, BlockVolume

_LOCAL = np.stack(np.meshgrid(np.arange(BLOCK), np.arange(BLOCK), np.arange(BLOCK), indexing="ij"),
                  axis=-1).reshape(-1, 3)
# reorder so that flat index l = lx + 8*ly + 64*lz
_LOCAL = _LOCAL[np.lexsort((_LOCAL[:, 0], _LOCAL[:, 1], _LOCAL[:, 2]))]
assert (_LOCAL[1] == [1, 0, 0]).all() and (_LOCAL[8] == [0, 1, 0]).all()


def local_offsets() -> np.ndarray:
    """int [512, 3] voxel offsets inside a block, flat index l = lx + 8 ly + 64 lz."""
    return _LOCAL.copy()


# ----------------------------------------------------------------------------------------
# G0: dense sphere (configs[0])
# ----------------------------------------------------------------------------------------
def sphere_volume(radius=0.2, voxel_size=0.01, truncation=0.04, theta=np.deg2rad(65.0),
                  blocks_per_axis=8) -> BlockVolume:
    """configs[0]: 64^3 voxels at 1 cm, all six directions allocated everywhere.

    phi = clamp((|x| - r)/tau, -1, 1), omega_D = max(0, n.v^D) with n = x/|x| (0 at x = 0),
    rgb = 0.  The sphere centre is the world origin (half a voxel from the exact grid centre,
    readings R15/R17).
    """
    h = blocks_per_axis // 2
    rng = np.arange(-h, h)
    loc = np.stack(np.meshgrid(rng, rng, rng, indexing="ij"), -1).reshape(-1, 3)
    loc = loc[np.lexsort((loc[:, 0], loc[:, 1], loc[:, 2]))]
    keys = np.concatenate([np.concatenate([loc, np.full((len(loc), 1), d)], 1) for d in range(6)])
    vox = (keys[:, None, :3] * BLOCK + _LOCAL[None]).astype(np.float64) * voxel_size
    r = np.linalg.norm(vox, axis=-1)
    sdf = np.clip((r - radius) / truncation, -1.0, 1.0)
    with np.errstate(invalid="ignore", divide="ignore"):
        nrm = np.where(r[..., None] > 0, vox / r[..., None], 0.0)
    w = np.maximum(0.0, np.einsum("nvk,nk->nv", nrm, DIRECTION_VECTORS[keys[:, 3]]))
    rgb = np.zeros(sdf.shape + (3,), np.uint8)
    return BlockVolume(voxel_size, truncation, float(theta), keys.astype(np.int32),
                       sdf.astype(np.float32), w.astype(np.float32), rgb)


# ----------------------------------------------------------------------------------------
# G1: ideal-fusion patch fill
# ----------------------------------------------------------------------------------------
RECT, DISK, CYL = 0, 1, 2


@dataclasses.dataclass
class Patches:
    """Surface patches with outward normals (towards free space) and an RGB colour.

    kind RECT (0): centre q, unit normal n, in-plane unit axes u, v, half extents hu, hv.
    kind DISK (1): centre q, normal n, in-plane axes u, v, radius hu.
    kind CYL  (2): lateral surface of a cylinder, axis through q along n, radius hu,
                   half height hv (u, v: any orthonormal pair perpendicular to n).
    ``patch_fill`` (numpy) handles RECT only; ``patch_fill_c`` (gen.c) handles all three."""

    q: np.ndarray
    n: np.ndarray
    u: np.ndarray
    v: np.ndarray
    hu: np.ndarray
    hv: np.ndarray
    color: np.ndarray
    kind: np.ndarray = None

    def __post_init__(self):
        if self.kind is None:
            self.kind = np.zeros(len(self.hu), np.int32)

    @staticmethod
    def empty():
        z3 = np.zeros((0, 3))
        return Patches(z3, z3, z3, z3, np.zeros(0), np.zeros(0), np.zeros((0, 3), np.uint8), np.zeros(0, np.int32))

    def __len__(self):
        return len(self.hu)

    def extend(self, q, n, u, v, hu, hv, color, kind=RECT):
        self.kind = np.concatenate([self.kind, np.atleast_1d(np.int32(kind))])
        self.q = np.vstack([self.q, np.atleast_2d(q)])
        self.n = np.vstack([self.n, np.atleast_2d(n)])
        self.u = np.vstack([self.u, np.atleast_2d(u)])
        self.v = np.vstack([self.v, np.atleast_2d(v)])
        self.hu = np.concatenate([self.hu, np.atleast_1d(hu)])
        self.hv = np.concatenate([self.hv, np.atleast_1d(hv)])
        self.color = np.vstack([self.color, np.atleast_2d(color).astype(np.uint8)])

    def ray_hit(self, o, d):
        """Closed-form first intersection of rays o + t d (t > 0) with the patches seen from
        their front side.  Returns (t, patch_id) with t = inf / id = -1 on a miss.
        Test helper for closed-form pins (analytic geometry, not the method); RECT patches only."""
        if (self.kind != RECT).any():
            raise NotImplementedError("ray_hit: RECT patches only")
        o = np.asarray(o, np.float64).reshape(-1, 3)
        d = np.asarray(d, np.float64).reshape(-1, 3)
        best = np.full(len(d), np.inf)
        pid = np.full(len(d), -1)
        for p in range(len(self)):
            den = d @ self.n[p]
            with np.errstate(divide="ignore", invalid="ignore"):
                t = ((self.q[p] - o) @ self.n[p]) / den
            x = o + t[:, None] * d
            a = (x - self.q[p]) @ self.u[p]
            b = (x - self.q[p]) @ self.v[p]
            ok = (den < 0) & (t > 0) & (np.abs(a) <= self.hu[p]) & (np.abs(b) <= self.hv[p]) & (t < best)
            best = np.where(ok, t, best)
            pid = np.where(ok, p, pid)
        return best, pid


def box_patches(pat: Patches, center, size, yaw, colors, with_bottom=False):
    """Six (or five, bottom omitted when resting on a floor) faces of a yawed box."""
    c, s = np.cos(yaw), np.sin(yaw)
    ex, ey, ez = np.array([c, s, 0.0]), np.array([-s, c, 0.0]), np.array([0.0, 0.0, 1.0])
    hx, hy, hz = 0.5 * np.asarray(size, np.float64)
    center = np.asarray(center, np.float64)
    faces = [(ex, ey, ez, hx, hy, hz), (-ex, ey, ez, hx, hy, hz),
             (ey, ex, ez, hy, hx, hz), (-ey, ex, ez, hy, hx, hz),
             (ez, ex, ey, hz, hx, hy), (-ez, ex, ey, hz, hx, hy)]
    for f, (n, u, v, hn, hu, hv) in enumerate(faces):
        if f == 5 and not with_bottom:
            continue
        pat.extend(center + hn * n, n, u, v, hu, hv, colors[f])


def patch_fill(pat: Patches, voxel_size: float, truncation: float, theta: float,
               chunk_groups: int = 4096) -> BlockVolume:
    """G1 ideal-fusion fill of SURVEY.md §8(d) with the direction rule of DESIGN.md §3.

    For direction D and voxel x, candidate patches p have <n_p, v^D> > cos(theta)
    (eq:angular_threshold), x's in-plane coordinates inside the rectangle, and
    |s_p(x)| <= tau + 2 s with s_p = <x - q_p, n_p>.  The candidate with the smallest |s_p|
    (ties -> lower patch id) writes phi = clamp(s_p / tau, -1, 1), omega = <n_p, v^D>,
    rgb = colour_p; other voxels get phi = 1, omega = 0, rgb = 0.  A block (b, D) is
    allocated iff any voxel was written.
    """
    if (pat.kind != RECT).any():
        raise NotImplementedError("patch_fill (numpy): RECT patches only; use patch_fill_c")
    s = voxel_size
    band = truncation + 2.0 * s
    cos_t = np.cos(theta)
    bsz = BLOCK * s
    triples = []  # (bx, by, bz, D, patch)
    for p in range(len(pat)):
        corners = np.array([pat.q[p] + a * pat.hu[p] * pat.u[p] + b * pat.hv[p] * pat.v[p] + c * band * pat.n[p]
                            for a in (-1, 1) for b in (-1, 1) for c in (-1, 1)])
        lo = np.floor(corners.min(0) / bsz - 1e-9).astype(np.int64)
        hi = np.floor(corners.max(0) / bsz + 1e-9).astype(np.int64)
        grid = np.stack(np.meshgrid(*[np.arange(lo[k], hi[k] + 1) for k in range(3)], indexing="ij"),
                        -1).reshape(-1, 3)
        # keep only blocks whose AABB intersects the patch slab (cheap separating-axis on n)
        cen = (grid + 0.5) * bsz
        rad = 0.5 * bsz * np.abs(pat.n[p]).sum()
        keep = np.abs((cen - pat.q[p]) @ pat.n[p]) <= band + rad
        grid = grid[keep]
        for D in range(6):
            if pat.n[p] @ DIRECTION_VECTORS[D] > cos_t:
                triples.append(np.concatenate([grid, np.full((len(grid), 1), D), np.full((len(grid), 1), p)], 1))
    if not triples:
        return BlockVolume(s, truncation, theta, np.zeros((0, 4), np.int32), np.zeros((0, 512), np.float32),
                           np.zeros((0, 512), np.float32), np.zeros((0, 512, 3), np.uint8))
    tri = np.concatenate(triples).astype(np.int64)
    # group by (block, D); inside a group ascending patch id
    order = np.lexsort((tri[:, 4], tri[:, 3], tri[:, 2], tri[:, 1], tri[:, 0]))
    tri = tri[order]
    gkey = tri[:, :4]
    newg = np.ones(len(tri), bool)
    newg[1:] = (gkey[1:] != gkey[:-1]).any(1)
    gstart = np.flatnonzero(newg)
    gend = np.append(gstart[1:], len(tri))

    keys_out, sdf_out, w_out, rgb_out = [], [], [], []
    for g0 in range(0, len(gstart), chunk_groups):
        gs, ge = gstart[g0:g0 + chunk_groups], gend[g0:g0 + chunk_groups]
        t0, t1 = gs[0], ge[-1]
        sub = tri[t0:t1]
        p = sub[:, 4]
        vox = (sub[:, None, :3] * BLOCK + _LOCAL[None]).astype(np.float64) * s  # [T,512,3]
        rel = vox - pat.q[p][:, None, :]
        sp = np.einsum("tvk,tk->tv", rel, pat.n[p])
        a = np.einsum("tvk,tk->tv", rel, pat.u[p])
        b = np.einsum("tvk,tk->tv", rel, pat.v[p])
        ok = (np.abs(a) <= pat.hu[p][:, None]) & (np.abs(b) <= pat.hv[p][:, None]) & (np.abs(sp) <= band)
        score = np.where(ok, np.abs(sp), np.inf)
        seg = gs - t0
        best = np.minimum.reduceat(score, seg, axis=0)  # [G,512]
        gid = np.repeat(np.arange(len(gs)), ge - gs)
        tidx = np.arange(len(sub))[:, None].repeat(VOXELS_PER_BLOCK, 1)
        winner = np.where((score == best[gid]) & np.isfinite(score), tidx, np.iinfo(np.int64).max)
        win = np.minimum.reduceat(winner, seg, axis=0)  # first (lowest patch id) achieving the min
        written = win != np.iinfo(np.int64).max
        keep = written.any(1)
        if not keep.any():
            continue
        win_c = np.where(written, win, 0)
        vv = np.arange(VOXELS_PER_BLOCK)[None, :]
        pw = p[win_c]
        phi = np.clip(sp[win_c, vv] / truncation, -1.0, 1.0)
        Dg = sub[gs - t0, 3]
        omega = np.einsum("gvk,gk->gv", pat.n[pw], DIRECTION_VECTORS[Dg])
        phi = np.where(written, phi, 1.0)
        omega = np.where(written, omega, 0.0)
        col = np.where(written[..., None], pat.color[pw], 0)
        keys_out.append(sub[gs - t0][keep, :4])
        sdf_out.append(phi[keep].astype(np.float32))
        w_out.append(omega[keep].astype(np.float32))
        rgb_out.append(col[keep].astype(np.uint8))
    return BlockVolume(s, truncation, theta, np.concatenate(keys_out).astype(np.int32),
                       np.concatenate(sdf_out), np.concatenate(w_out), np.concatenate(rgb_out))


def cylinder_patches(pat: Patches, base, radius, height, colors):
    """Upright cylinder standing on z = base[2]: lateral surface plus the top cap (the bottom
    rests on the floor and is omitted, like a box's bottom face)."""
    base = np.asarray(base, np.float64)
    ez = np.array([0.0, 0.0, 1.0])
    pat.extend(base + 0.5 * height * ez, ez, [1.0, 0, 0], [0, 1.0, 0], radius, 0.5 * height, colors[0], kind=CYL)
    pat.extend(base + height * ez, ez, [1.0, 0, 0], [0, 1.0, 0], radius, radius, colors[1], kind=DISK)


# ----------------------------------------------------------------------------------------
# G1 in C (gen.c): same rule, multithreaded, all patch kinds -- for the large configs
# ----------------------------------------------------------------------------------------
_GEN_SRC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "gen.c")
_GEN_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libscenegen.so")
_gen = None


def build_gen(force: bool = False) -> str:
    if force or not os.path.exists(_GEN_LIB) or os.path.getmtime(_GEN_LIB) < os.path.getmtime(_GEN_SRC):
        tmp = _GEN_LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-ffp-contract=off", "-fno-fast-math",
                               "-Wall", "-shared", "-fPIC", "-pthread", _GEN_SRC, "-lm", "-o", tmp])
        os.replace(tmp, _GEN_LIB)
    return _GEN_LIB


def _genlib():
    global _gen
    if _gen is None:
        build_gen()
        L = ctypes.CDLL(_GEN_LIB)
        P, D, I = ctypes.c_void_p, ctypes.c_double, ctypes.c_int
        L.scenegen_plan.argtypes = [I, P, P, P, P, P, P, P, P, D, D, D, I, ctypes.POINTER(P),
                                    ctypes.POINTER(ctypes.c_int64)]
        L.scenegen_plan.restype = I
        L.scenegen_fill.argtypes = [P, I, P, P, P, P]
        L.scenegen_fill.restype = None
        L.scenegen_free.argtypes = [P]
        L.scenegen_free.restype = None
        _gen = L
    return _gen


def patch_fill_c(pat: Patches, voxel_size: float, truncation: float, theta: float, threads: int = 0) -> BlockVolume:
    """G1 fill by gen.c: the rule of ``patch_fill`` extended to DISK and CYL patches.
    On RECT-only scenes it writes the same bytes as ``patch_fill`` (tests/test_scenes.py)."""
    L = _genlib()
    arr = {k: np.ascontiguousarray(getattr(pat, k), np.float64) for k in ("q", "n", "u", "v", "hu", "hv")}
    kind = np.ascontiguousarray(pat.kind, np.int32)
    color = np.ascontiguousarray(pat.color, np.uint8)
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    threads = threads or os.cpu_count() or 1
    h, n = ctypes.c_void_p(), ctypes.c_int64()
    rc = L.scenegen_plan(len(pat), ptr(kind), ptr(arr["q"]), ptr(arr["n"]), ptr(arr["u"]), ptr(arr["v"]),
                         ptr(arr["hu"]), ptr(arr["hv"]), ptr(color), float(voxel_size), float(truncation),
                         float(theta), threads, ctypes.byref(h), ctypes.byref(n))
    if rc != 0:
        raise MemoryError("scenegen_plan")
    try:
        N = n.value
        keys = np.empty((N, 4), np.int32)
        sdf = np.empty((N, VOXELS_PER_BLOCK), np.float32)
        w = np.empty((N, VOXELS_PER_BLOCK), np.float32)
        rgb = np.empty((N, VOXELS_PER_BLOCK, 3), np.uint8)
        L.scenegen_fill(h, threads, ptr(keys), ptr(sdf), ptr(w), ptr(rgb))
    finally:
        L.scenegen_free(h)
    return BlockVolume(voxel_size, truncation, theta, keys, sdf, w, rgb)
