// fusion.cu -- voxel-projection fusion of depth frames into the DTSDF (
// DESIGN.md §12).
//
//   k_depth_normals  one thread per pixel: camera-frame normal from the cross product of the
//                    neighbouring back-projected pixels in x and y, facing the camera (R39)
//   k_fuse_alloc     one thread per pixel: for every direction the pixel's normal admits
//                    (eq:angular_threshold) the blocks holding the points p + t n,
//                    t = -tau + j 2tau/M (R40), computed in fp64 with the oracle's roundings so
//                    both sides allocate the same key set; a new (location, D) key claims its
//                    direction slot in the location hash (CAS) and takes the next pool index
//   k_fuse_init      new blocks: free space of weight 0
//   k_fuse           one CTA per block, 2 voxels per thread: the voxel is projected into the frame
//                    (nearest pixel, association in fp64), d = <x - p, n> / tau (eq:point-to-plane
//                    with the sign of R6), then carving (d > 1, 2-pixel depth-edge guard)
//                    or the weighted running average with w_d = w_ICP(z) <n,-ray>^+ w_dir^D(n)
//                    (eq:combined_fusion_weight) and w_c = w_d (1 - min(1, |p - x| / tau))
//                    (eq:color_weight); weights capped at w_max (R41-R45)
//
// Every voxel is updated at most once per frame and only from frame data, so the result does not
// depend on thread order; the pool order of new blocks does (keys are compared as a set).
#include <climits>

#include <math_constants.h>

#include "common.cuh"

#ifndef DTSDF_FUSE_PRETEST
#define DTSDF_FUSE_PRETEST 1  // fp32 pre-test of the association and band decisions in k_fuse (exact)
#endif

namespace dtsdf {

__device__ __forceinline__ bool depth_ok(const FuseLaunch &p, float z) {
  return z > 0.0f && (double)z >= p.z_min && (double)z <= p.z_max;
}

// camera point of pixel (u, v) at depth z, ((u - cx) / fx) z, one rounding per operation
__device__ __forceinline__ void backproject(const FuseLaunch &p, int u, int v, double z, double P[3]) {
  P[0] = __dmul_rn(__ddiv_rn(__dsub_rn((double)u, p.cx), p.fx), z);
  P[1] = __dmul_rn(__ddiv_rn(__dsub_rn((double)v, p.cy), p.fy), z);
  P[2] = z;
}

// ((R0 a0 + R1 a1) + R2 a2) (+ t): the oracle's evaluation order, no contraction
__device__ __forceinline__ void rotate(const FuseLaunch &p, const double a[3], double o[3]) {
#pragma unroll
  for (int r = 0; r < 3; ++r)
    o[r] = __dadd_rn(__dadd_rn(__dmul_rn(p.R[3 * r], a[0]), __dmul_rn(p.R[3 * r + 1], a[1])),
                     __dmul_rn(p.R[3 * r + 2], a[2]));
}

__global__ void __launch_bounds__(256) k_depth_normals(const float *__restrict__ depth, FuseLaunch p,
                                                       float *__restrict__ out) {
  const int u = blockIdx.x * 16 + (threadIdx.x & 15), v = blockIdx.y * 16 + (threadIdx.x >> 4);
  if (u >= p.width || v >= p.height) return;
  float *o = out + 3 * ((size_t)v * p.width + u);
  float n0 = 0.f, n1 = 0.f, n2 = 0.f;
  if (u >= 1 && v >= 1 && u < p.width - 1 && v < p.height - 1) {
    const size_t i = (size_t)v * p.width + u;
    const float zc = depth[i], zl = depth[i - 1], zr = depth[i + 1], zu = depth[i - p.width], zd = depth[i + p.width];
    if (depth_ok(p, zc) && depth_ok(p, zl) && depth_ok(p, zr) && depth_ok(p, zu) && depth_ok(p, zd)) {
      // fp64: the neighbour differences cancel metre-scale coordinates to centimetres
      double L[3], Rr[3], U[3], Dn[3], P[3];
      backproject(p, u - 1, v, zl, L);
      backproject(p, u + 1, v, zr, Rr);
      backproject(p, u, v - 1, zu, U);
      backproject(p, u, v + 1, zd, Dn);
      backproject(p, u, v, zc, P);
      const double ax = Rr[0] - L[0], ay = Rr[1] - L[1], az = Rr[2] - L[2];
      const double bx = Dn[0] - U[0], by = Dn[1] - U[1], bz = Dn[2] - U[2];
      const double cxn = ay * bz - az * by, cyn = az * bx - ax * bz, czn = ax * by - ay * bx;
      const double nn = sqrt(cxn * cxn + cyn * cyn + czn * czn);
      if (nn > 0.0) {
        const double sgn = (cxn * P[0] + cyn * P[1] + czn * P[2]) > 0.0 ? -1.0 : 1.0;  // face the camera
        n0 = (float)(sgn * cxn / nn); n1 = (float)(sgn * cyn / nn); n2 = (float)(sgn * czn / nn);
      }
    }
  }
  o[0] = n0; o[1] = n1; o[2] = n2;
}

__device__ __forceinline__ long long floordiv8(long long i) { return i >= 0 ? i / 8 : -((-i + 7) / 8); }

// insert (block, D): returns 0 present or inserted, 1 capacity / table exhausted
__device__ int alloc_key(const FuseLaunch &p, int bx, int by, int bz, int D) {
  const unsigned long long key = pack_key(bx, by, bz);
  unsigned int h = hash_key(key) & p.table_mask;
  for (unsigned int probe = 0; probe <= p.table_mask; ++probe) {
    unsigned long long k = p.table[h].key;
    if (k != key) {
      if (k != kEmptyKey) { h = (h + 1) & p.table_mask; continue; }
      k = atomicCAS(&p.table[h].key, kEmptyKey, key);
      if (k != kEmptyKey && k != key) { h = (h + 1) & p.table_mask; continue; }
      if (k == kEmptyKey && p.locations) {  // this thread added the location: append it
        const unsigned long long li = atomicAdd(p.n_loc, 1ull);
        p.locations[li] = make_int4(bx, by, bz, (int)h);
        if ((unsigned)(bx - p.lo[0]) >= (unsigned)p.dim[0] || (unsigned)(by - p.lo[1]) >= (unsigned)p.dim[1] ||
            (unsigned)(bz - p.lo[2]) >= (unsigned)p.dim[2])
          atomicExch(&p.flags[1], 1);  // outside the location AABB: the index needs a full rebuild
      }
    }
    int *slot = &p.table[h].slot[D];
    if (*((volatile int *)slot) != -1) return 0;
    if (atomicCAS(slot, -1, -2) != -1) return 0;  // another thread claimed it
    const unsigned long long idx = atomicAdd(p.n_blocks, 1ull);
    if ((long long)idx >= p.capacity) {
      atomicExch(slot, -1);
      atomicExch(p.flags, 1);
      return 1;
    }
    reinterpret_cast<int4 *>(p.keys)[idx] = make_int4(bx, by, bz, D);
    atomicExch(slot, (int)idx);
    return 0;
  }
  atomicExch(p.flags, 2);
  return 1;
}

// Per pixel of the frame: first its frame point (when p.pix_x is set) -- R P (the back-projected
// depth point rotated into the world, relative to the camera centre), R n (the world normal) and
// the carving guard, with the operations k_fuse would apply per voxel, once per frame -- then the
// allocation of the blocks around the depth point in every admitted direction (R40).
__global__ void __launch_bounds__(256) k_fuse_alloc(const __grid_constant__ FuseLaunch p) {
  const int u = blockIdx.x * 16 + (threadIdx.x & 15), v = blockIdx.y * 16 + (threadIdx.x >> 4);
  if (u >= p.width || v >= p.height) return;
  const size_t i = (size_t)v * p.width + u;
  const float z = p.depth[i];
  const float n0 = p.normal[3 * i], n1 = p.normal[3 * i + 1], n2 = p.normal[3 * i + 2];
  double P[3], X[3] = {0, 0, 0}, nc[3] = {n0, n1, n2}, n[3] = {0, 0, 0};
  const bool zok = depth_ok(p, z);
  if (zok) {
    backproject(p, u, v, (double)z, P);
    rotate(p, P, X);
    rotate(p, nc, n);
  }
  if (p.pix_x) {
    bool edge = false;
    if (zok) {
      // R43's carving guard of this pixel: a valid depth within carve_radius differing by more than tau
      for (int dv = -p.carve_radius; dv <= p.carve_radius && !edge; ++dv)
        for (int du = -p.carve_radius; du <= p.carve_radius; ++du) {
          const int qu = u + du, qv = v + dv;
          if (qu < 0 || qv < 0 || qu >= p.width || qv >= p.height) continue;
          const float zq = p.depth[(size_t)qv * p.width + qu];
          if (!depth_ok(p, zq)) continue;
          if (fabs((double)zq - (double)z) > p.tau) { edge = true; break; }
        }
    }
    p.pix_x[i] = make_double4(X[0], X[1], X[2], edge ? 1.0 : 0.0);
    p.pix_n[i] = make_double4(n[0], n[1], n[2], 0.0);
    const bool usable = zok && !(nc[0] == 0.0 && nc[1] == 0.0 && nc[2] == 0.0);
    p.pix_a[i] = make_float4((float)X[0], (float)X[1], (float)X[2], usable ? z : -1.0f);
    p.pix_b[i] = make_float4((float)n[0], (float)n[1], (float)n[2], edge ? 1.0f : 0.0f);
  }
  if (!zok || (n0 == 0.f && n1 == 0.f && n2 == 0.f)) return;
#pragma unroll
  for (int a = 0; a < 3; ++a) X[a] = __dadd_rn(X[a], p.t[a]);
  for (int D = 0; D < 6; ++D) {
    const double dot = (D & 1) ? -n[D >> 1] : n[D >> 1];
    if (!(dot > p.cos_theta)) continue;
    long long pb[3] = {LLONG_MIN, 0, 0};
    for (int j = 0; j <= p.M; ++j) {
      const double tj = __dadd_rn(-p.tau, __dmul_rn((double)j, p.step));
      long long b[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
#if DTSDF_FUSE_PRETEST
        // the voxel index floor((X + t n) / s) in fp32 where the fraction clears 0 and 1 by more
        // than its fp32 error (relative 2^-24 per operand and operation, in voxel units); else fp64
        const float g = ((float)X[a] + (float)tj * (float)n[a]) * p.inv_s_f;
        const float fl = floorf(g), fr = g - fl;
        const float m = 1e-4f + 5e-7f * (fabsf((float)X[a]) + (float)p.tau) * p.inv_s_f;
        if (fr > m && fr < 1.0f - m) {
          b[a] = floordiv8((long long)fl);
          continue;
        }
#endif
        b[a] = floordiv8((long long)floor(__ddiv_rn(__dadd_rn(X[a], __dmul_rn(tj, n[a])), p.s)));
      }
      if (b[0] == pb[0] && b[1] == pb[1] && b[2] == pb[2]) continue;
      pb[0] = b[0]; pb[1] = b[1]; pb[2] = b[2];
      if (p.grid) {  // already allocated at the last commit: nothing to insert
        const unsigned gx = (unsigned)(b[0] - p.lo[0]), gy = (unsigned)(b[1] - p.lo[1]), gz = (unsigned)(b[2] - p.lo[2]);
        if (gx < (unsigned)p.dim[0] && gy < (unsigned)p.dim[1] && gz < (unsigned)p.dim[2]) {
          const int gv = __ldg(&p.grid[((size_t)gz * p.dim[1] + gy) * p.dim[0] + gx]);
          if (gv >= 0 && ((gv >> kGridEntryBits) >> D) & 1) continue;
        }
      }
      if (alloc_key(p, (int)b[0], (int)b[1], (int)b[2], D)) return;
    }
  }
}

__global__ void __launch_bounds__(256) k_fuse_init(FuseLaunch p, long long n0, long long n1) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long b = n0 + (g >> 9);
  if (b >= n1) return;
  const size_t r = (size_t)b * kVoxPerBlock + (g & 511);
  if (p.dirty && (g & 511) == 0) p.dirty[b] = 1;
  p.sdf[r] = 1.0f;
  p.weight[r] = 0.0f;
  p.cweight[r] = 0.0f;
  p.rgb[3 * r] = p.rgb[3 * r + 1] = p.rgb[3 * r + 2] = 0;
}

__device__ __forceinline__ float w_dir_f(float c, const FuseLaunch &p) {
  if (c <= p.cos_theta_f) return 0.0f;
  if (c >= p.sin_theta_f) return 1.0f;
  const float a = acosf(fminf(c, 1.0f));
  return fminf(fmaxf((p.theta_f - a) * p.inv_blend, 0.0f), 1.0f);
}

// One warp per block: does any voxel of the block project into the frame?  A voxel is associated
// iff its camera z > 0 and its nearest pixel floor(u + 1/2), floor(v + 1/2) lies in the image, i.e.
// u in [-1/2, W - 1/2), v likewise -- for z > 0 linear constraints in camera coordinates
// (fx x + (cx + 1/2) z >= 0, ...).  The block's voxels are convex combinations of its 8 corner
// voxels, so when all 8 corners violate one constraint (by a margin far above fp64 rounding) no
// voxel is associated and the block is left out (exact).  Selected blocks go to list / *count.
__global__ void __launch_bounds__(256) k_fuse_select(const __grid_constant__ FuseLaunch p, long long n, int *list,
                                                     unsigned long long *count) {
  // four blocks per warp, eight lanes (the corners) each
  const long long b = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int lane = threadIdx.x & 31, grp = lane & ~7;
  const int4 key = reinterpret_cast<const int4 *>(p.keys)[b < n ? b : n - 1];
  const int q = lane & 7;
  const int i = kBlock * key.x + ((q & 1) ? kBlock - 1 : 0), j = kBlock * key.y + ((q & 2) ? kBlock - 1 : 0),
            k = kBlock * key.z + ((q & 4) ? kBlock - 1 : 0);
  const double d0 = (double)i * p.s - p.t[0], d1 = (double)j * p.s - p.t[1], d2 = (double)k * p.s - p.t[2];
  const double xc = p.R[0] * d0 + p.R[3] * d1 + p.R[6] * d2;
  const double yc = p.R[1] * d0 + p.R[4] * d1 + p.R[7] * d2;
  const double zc = p.R[2] * d0 + p.R[5] * d1 + p.R[8] * d2;
  const double tol = 1e-6;
  double g[5];
  g[0] = zc;                                                   // z > 0
  g[1] = p.fx * xc + (p.cx + 0.5) * zc;                         // u >= -1/2
  g[2] = ((double)p.width - 0.5 - p.cx) * zc - p.fx * xc;       // u < W - 1/2
  g[3] = p.fy * yc + (p.cy + 0.5) * zc;                         // v >= -1/2
  g[4] = ((double)p.height - 0.5 - p.cy) * zc - p.fy * yc;      // v < H - 1/2
  bool out = false;
#pragma unroll
  for (int c = 0; c < 5; ++c) out |= ((__ballot_sync(0xffffffffu, g[c] < -tol) >> grp) & 0xffu) == 0xffu;
  if (out || b >= n || lane != grp) return;
  list[atomicAdd(count, 1ull)] = (int)b;
}

#ifndef DTSDF_FUSE_MINB
#define DTSDF_FUSE_MINB 8  // 32 registers, full occupancy: fused frame kernels 0.348 -> 0.285 ms (profiles/r3_ab_fusion.txt)
#endif
// store v over old only if its bits differ; true when stored.  A block whose stored values did not
// change keeps its record bricks (and its neighbours'): the incremental index update skips it.
__device__ __forceinline__ bool store_changed(float *a, float old, float v) {
  if (__float_as_uint(old) == __float_as_uint(v)) return false;
  *a = v;
  return true;
}

__device__ __forceinline__ void fuse_block(const FuseLaunch &p, long long b) {
  const int4 key = reinterpret_cast<const int4 *>(p.keys)[b];
  const int D = key.w;
  const int axis = D >> 1;
  const float sgnD = (D & 1) ? -1.0f : 1.0f;
  const float tau = (float)p.tau;
  bool wrote = false;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int l = threadIdx.x + 256 * h;
    const int i = kBlock * key.x + (l & 7), j = kBlock * key.y + ((l >> 3) & 7), k = kBlock * key.z + (l >> 6);
    // association (R41): projection and nearest pixel in fp64 with the oracle's roundings
    const double x0 = __dmul_rn((double)i, p.s), x1 = __dmul_rn((double)j, p.s), x2 = __dmul_rn((double)k, p.s);
    const double d0 = __dsub_rn(x0, p.t[0]), d1 = __dsub_rn(x1, p.t[1]), d2 = __dsub_rn(x2, p.t[2]);
    int iu, iv;
    bool exact64 = true;
#if DTSDF_FUSE_PRETEST
    {
      // fp32 pre-test: the projection in fp32 from the fp64 offset; where u + 1/2 and v + 1/2 are
      // clear of an integer (and z of 0) by more than a bound on the fp32 error, the nearest
      // pixel -- or "outside the image" -- is the fp64 decision; else the fp64 path decides
      const float e0 = (float)d0, e1 = (float)d1, e2 = (float)d2;
      const float zc = p.Rf[2] * e0 + p.Rf[5] * e1 + p.Rf[8] * e2;
      if (zc > 0.05f) {
        const float xcf = p.Rf[0] * e0 + p.Rf[3] * e1 + p.Rf[6] * e2;
        const float ycf = p.Rf[1] * e0 + p.Rf[4] * e1 + p.Rf[7] * e2;
        const float dn = fabsf(e0) + fabsf(e1) + fabsf(e2);
        const float iz = 1.0f / zc;
        const float uf = p.fxf * xcf * iz + p.cxf + 0.5f, vf = p.fyf * ycf * iz + p.cyf + 0.5f;
        // |error| of u, v: relative 2.5e-7 of |d| in xc and zc (fp32 rotation of a rounded offset),
        // amplified by f (z + |x|) / z^2, plus the roundings of the division and additions
        const float eu = 2.5e-7f * p.fxf * dn * (zc + fabsf(xcf)) * iz * iz + 1e-5f * (1.0f + fabsf(uf));
        const float ev = 2.5e-7f * p.fyf * dn * (zc + fabsf(ycf)) * iz * iz + 1e-5f * (1.0f + fabsf(vf));
        const float fu = floorf(uf), fv = floorf(vf);
        if (uf - fu > eu && fu + 1.0f - uf > eu && vf - fv > ev && fv + 1.0f - vf > ev) {
          exact64 = false;
          if (!(fu >= 0.0f && fu <= (float)(p.width - 1) && fv >= 0.0f && fv <= (float)(p.height - 1))) continue;
          iu = (int)fu;
          iv = (int)fv;
        }
      } else if (zc < -0.05f) {
        continue;  // behind the camera (z < 0 with an fp32 error far below 0.05 m)
      }
    }
#endif
    if (exact64) {
      double xc[3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
        xc[a] = __dadd_rn(__dadd_rn(__dmul_rn(p.R[a], d0), __dmul_rn(p.R[3 + a], d1)), __dmul_rn(p.R[6 + a], d2));
      if (!(xc[2] > 0.0)) continue;
      const double uu = __dadd_rn(__ddiv_rn(__dmul_rn(p.fx, xc[0]), xc[2]), p.cx);
      const double vv = __dadd_rn(__ddiv_rn(__dmul_rn(p.fy, xc[1]), xc[2]), p.cy);
      const double fu = floor(__dadd_rn(uu, 0.5)), fv = floor(__dadd_rn(vv, 0.5));
      if (!(fu >= 0.0 && fu <= (double)(p.width - 1) && fv >= 0.0 && fv <= (double)(p.height - 1))) continue;
      iu = (int)fu;
      iv = (int)fv;
    }
    const size_t pi = (size_t)iv * p.width + iu;
    DTSDF_CHECK(iu >= 0 && iu < p.width && iv >= 0 && iv < p.height);
#if DTSDF_FUSE_PRETEST
    // the pixel's fp32 record: no usable depth -> untouched; a band decision clear of -1 and 1 by
    // more than its fp32 error is taken here (behind: untouched; free space: carving)
    float4 pa = make_float4(0.f, 0.f, 0.f, 0.f), pb = pa;
    if (p.pix_a) {
      pa = p.pix_a[pi];
      if (!(pa.w > 0.0f)) continue;
      pb = p.pix_b[pi];
      const float fex = (float)d0 - pa.x, fey = (float)d1 - pa.y, fez = (float)d2 - pa.z;
      const float df = (fex * pb.x + fey * pb.y + fez * pb.z) * p.inv_tau_f;
      const float m = 1e-5f + 5e-7f * (fabsf((float)d0) + fabsf((float)d1) + fabsf((float)d2) + fabsf(pa.x) +
                                        fabsf(pa.y) + fabsf(pa.z)) * p.inv_tau_f;
      if (df < -1.0f - m) continue;  // behind the surface beyond the band: untouched
      if (df > 1.0f + m) {           // R43 free space
        if (!(p.carve_weight > 0.f) || pb.w != 0.0f) continue;
        const size_t r = (size_t)b * kVoxPerBlock + l;
        const float W0 = p.weight[r], S0 = p.sdf[r];
        wrote |= store_changed(p.sdf + r, S0, (W0 * S0 + p.carve_weight) / (W0 + p.carve_weight));
        wrote |= store_changed(p.weight + r, W0, fminf(W0 + p.carve_weight, p.max_weight));
        continue;
      }
    }
#endif
    const float z = p.depth[pi];
    const float nc0 = p.normal[3 * pi], nc1 = p.normal[3 * pi + 1], nc2 = p.normal[3 * pi + 2];
    if (!depth_ok(p, z) || (nc0 == 0.f && nc1 == 0.f && nc2 == 0.f)) continue;
    // the band decisions (|d| <= 1, d > 1) sit exactly on lattice planes for axis-aligned
    // surfaces (a voxel tau from a floor at z = 0), so d is formed in fp64 with the oracle's
    // operation order -- both sides take the same decision
    double X[3], nd[3];
    if (p.pix_x) {  // the frame's per-pixel values, computed once by k_fuse_alloc (same operations)
      const double4 xx = p.pix_x[pi], nn = p.pix_n[pi];
      X[0] = xx.x; X[1] = xx.y; X[2] = xx.z;
      nd[0] = nn.x; nd[1] = nn.y; nd[2] = nn.z;
    } else {
      double P[3], ncd[3] = {nc0, nc1, nc2};
      backproject(p, iu, iv, (double)z, P);
      rotate(p, P, X);
      rotate(p, ncd, nd);
    }
    const double ex = __dsub_rn(x0, __dadd_rn(X[0], p.t[0])), ey = __dsub_rn(x1, __dadd_rn(X[1], p.t[1])),
                 ez = __dsub_rn(x2, __dadd_rn(X[2], p.t[2]));
    // the band decision: -1 behind the band (untouched), 1 free space (carving), 0 in the band
    int cls = 2;  // 2: decide from d in fp64
    double ddd = 0.0;
    if (cls == 2) {
      ddd = __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn(ex, nd[0]), __dmul_rn(ey, nd[1])), __dmul_rn(ez, nd[2])), p.tau);
      cls = ddd < -1.0 ? -1 : (ddd > 1.0 ? 1 : 0);
    }
    const float dd = (float)ddd;  // eq:point-to-plane, sign of reading R6
    const float nx = (float)nd[0], ny = (float)nd[1], nz = (float)nd[2];
    const size_t r = (size_t)b * kVoxPerBlock + l;
    if (cls < 0) continue;  // behind the surface beyond the band: untouched
    if (cls == 1) {
      // R43: free space, unless a depth within the guard radius differs by more than tau;
      // carve_weight 0 turns carving off (on a fresh voxel, W0 = 0, the update would be 0/0)
      if (!(p.carve_weight > 0.f)) continue;
      bool edge = false;
      if (p.pix_x) edge = p.pix_x[pi].w != 0.0;  // the pixel's guard, once per frame (k_fuse_alloc)
      else
      for (int dv = -p.carve_radius; dv <= p.carve_radius && !edge; ++dv)
        for (int du = -p.carve_radius; du <= p.carve_radius; ++du) {
          const int qu = iu + du, qv = iv + dv;
          if (qu < 0 || qv < 0 || qu >= p.width || qv >= p.height) continue;
          const float zq = p.depth[(size_t)qv * p.width + qu];
          if (!depth_ok(p, zq)) continue;
          if (fabs((double)zq - (double)z) > p.tau) { edge = true; break; }
        }
      if (edge) continue;
      const float W0 = p.weight[r], S0 = p.sdf[r];
      wrote |= store_changed(p.sdf + r, S0, (W0 * S0 + p.carve_weight) / (W0 + p.carve_weight));
      wrote |= store_changed(p.weight + r, W0, fminf(W0 + p.carve_weight, p.max_weight));
      continue;
    }
    const float wdir = w_dir_f(sgnD * (axis == 0 ? nx : (axis == 1 ? ny : nz)), p);
    const float rx = (float)X[0], ry = (float)X[1], rz = (float)X[2];  // ray = p - camera centre
    const float rl = sqrtf(rx * rx + ry * ry + rz * rz);
    const float ca = rl > 0.f ? -(nx * rx + ny * ry + nz * rz) / rl : 0.f;
    const float zz = z + (1.0f - (float)p.z_min);
    const float wn = (1.0f / (zz * zz)) * fmaxf(ca, 0.0f) * wdir;  // w_ICP(z) w_angle w_dir
    if (!(wn > 0.0f)) continue;
    const float W0 = p.weight[r], S0 = p.sdf[r];
    wrote |= store_changed(p.sdf + r, S0, (W0 * S0 + wn * dd) / (W0 + wn));
    wrote |= store_changed(p.weight + r, W0, fminf(W0 + wn, p.max_weight));
    if (p.color) {
      const float dist = (float)sqrt(ex * ex + ey * ey + ez * ez);
      const float wc = wn * (1.0f - fminf(1.0f, dist / tau));  // eq:color_weight
      if (wc > 0.0f) {
        const float C0 = p.cweight[r];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const unsigned char q0 = p.rgb[3 * r + a];
          const float c = (C0 * (float)q0 + wc * (float)p.color[3 * pi + a]) / (C0 + wc);
          const unsigned char q1 = (unsigned char)fminf(fmaxf(floorf(c + 0.5f), 0.f), 255.f);
          if (q1 != q0) {
            p.rgb[3 * r + a] = q1;
            wrote = true;
          }
        }
        // (the colour weight is not read by the index: no rebuild for it alone)
        store_changed(p.cweight + r, C0, fminf(C0 + wc, p.max_weight));
      }
    }
  }
  if (!p.dirty && !p.loc_mark) return;  // uniform
  if (!__syncthreads_or(wrote)) return;
  if (threadIdx.x == 0 && p.dirty) p.dirty[b] = 1;
  if (p.loc_mark && threadIdx.x < 27) {
    // the record bricks of this block's 27-neighbourhood (its direction) read its voxels: their
    // locations are rebuilt by the incremental index update (hash table: new locations included)
    const int ox = (int)threadIdx.x % 3 - 1, oy = ((int)threadIdx.x / 3) % 3 - 1, oz = (int)threadIdx.x / 9 - 1;
    const unsigned long long nkey = pack_key(key.x + ox, key.y + oy, key.z + oz);
    unsigned int h = hash_key(nkey) & p.table_mask;
    int e = -1;
    for (unsigned int probe = 0; probe <= p.table_mask; ++probe) {
      const unsigned long long kk = p.table[h].key;
      if (kk == nkey) { e = (int)h; break; }
      if (kk == kEmptyKey) break;
      h = (h + 1) & p.table_mask;
    }
    if (e >= 0 && p.table[e].slot[D] >= 0 && atomicCAS(&p.loc_mark[e], 0, 1) == 0)
      p.loc_list[atomicAdd(p.loc_ctr, 1ull)] = make_int4(key.x + ox, key.y + oy, key.z + oz, e);
  }
}

// One CTA per selected block
__global__ void __launch_bounds__(256, DTSDF_FUSE_MINB) k_fuse(const __grid_constant__ FuseLaunch p, const int *list,
                                                               const unsigned long long *count) {
  if (list && blockIdx.x >= *count) return;  // CTA-uniform
  fuse_block(p, list ? (long long)list[blockIdx.x] : (long long)blockIdx.x);
}

cudaError_t launch_depth_normals(const float *depth, const FuseLaunch &p, float *out, cudaStream_t s) {
  dim3 grid((unsigned)((p.width + 15) / 16), (unsigned)((p.height + 15) / 16));
  k_depth_normals<<<grid, 256, 0, s>>>(depth, p, out);
  return cudaGetLastError();
}

cudaError_t launch_fuse_alloc(const FuseLaunch &p, cudaStream_t s) {
  dim3 grid((unsigned)((p.width + 15) / 16), (unsigned)((p.height + 15) / 16));
  k_fuse_alloc<<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_fuse(const FuseLaunch &p, long long n_old, long long n_new, bool fuse, int *list,
                        unsigned long long *count, cudaStream_t s) {
  if (n_new > n_old) {
    k_fuse_init<<<(unsigned)(((n_new - n_old) * kVoxPerBlock + 255) / 256), 256, 0, s>>>(p, n_old, n_new);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (n_new == 0 || !fuse) return cudaSuccess;
  if (list) {  // only the blocks with a voxel in the frame's view (count zeroed by the caller)
    k_fuse_select<<<(unsigned)((n_new * 8 + 255) / 256), 256, 0, s>>>(p, n_new, list, count);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  k_fuse<<<(unsigned)n_new, 256, 0, s>>>(p, list, count);
  return cudaGetLastError();
}

}  // namespace dtsdf
