// render.cu -- the per-pixel DTSDF raycast.
//
//   k_range    (a3) block-bounds range pass: every allocated block location's AABB, clipped
//              to z >= z_min, is projected into each view; per 8x8 pixel tile the min/max
//              camera z of the covering blocks is kept with order-independent atomics.
//   k_raycast  (a2, a4-a7) one thread per pixel, 8x4-pixel warps: lattice march t_k = k*Delta
//               inside the tile's [z_near, z_far], occupancy-bitmap skipping of
//              unallocated block locations, one hash probe per block location, per-sample
//              combination of the six directions (eq:combine_weight / eq:combine_tsdf_weight,
//              PAPER.md:235-270) read from apron bricks, first +->- crossing, Illinois
//              regula-falsi refinement, and the shading epilogue (normal, colour, dirmask).
//
// Skipping and the range pass are exact accelerations: a lattice point whose base voxel lies
// in an unallocated block location has no present direction and is invalid (DESIGN.md §2 O2).
#include <math_constants.h>

#include "common.cuh"

#ifndef DTSDF_RAYCAST_MINB
#define DTSDF_RAYCAST_MINB 2
#endif

namespace dtsdf {

// ------------------------------------------------------------------------------------------
// a3: range pass
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_range(const __grid_constant__ RangeLaunch p) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int view = blockIdx.y;
  if (i >= p.n_locations) return;
  const int4 b = p.locations[i];
  const ViewPose &P = p.pose[view];
  const float bs = kBlock * p.vol.voxel_size;
  // camera coordinates of the block corners: Xc = R^T (X - t)
  const float wx = b.x * bs - P.t[0], wy = b.y * bs - P.t[1], wz = b.z * bs - P.t[2];
  float c0[3], e[3][3];
  for (int a = 0; a < 3; ++a) {
    c0[a] = P.r[0 * 3 + a] * wx + P.r[1 * 3 + a] * wy + P.r[2 * 3 + a] * wz;
    for (int ax = 0; ax < 3; ++ax) e[ax][a] = P.r[ax * 3 + a] * bs;  // camera coords of world axis ax * bs
  }
  float cx[8], cy[8], cz[8];
  float zmax = -CUDART_INF_F;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float dx = (q & 1), dy = ((q >> 1) & 1), dz = ((q >> 2) & 1);
    cx[q] = c0[0] + dx * e[0][0] + dy * e[1][0] + dz * e[2][0];
    cy[q] = c0[1] + dx * e[0][1] + dy * e[1][1] + dz * e[2][1];
    cz[q] = c0[2] + dx * e[0][2] + dy * e[1][2] + dz * e[2][2];
    zmax = fmaxf(zmax, cz[q]);
  }
  if (zmax < p.z_min) return;  // entirely in front of the near plane
  float umin = CUDART_INF_F, umax = -CUDART_INF_F, vmin = CUDART_INF_F, vmax = -CUDART_INF_F;
  float zmin = CUDART_INF_F;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (cz[q] >= p.z_min) {
      const float iz = 1.0f / cz[q];
      const float u = p.fx * cx[q] * iz + p.cx, v = p.fy * cy[q] * iz + p.cy;
      umin = fminf(umin, u); umax = fmaxf(umax, u);
      vmin = fminf(vmin, v); vmax = fmaxf(vmax, v);
      zmin = fminf(zmin, cz[q]);
    }
  }
  // edges crossing the near plane contribute their intersection point
#pragma unroll
  for (int q = 0; q < 8; ++q) {
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const int q2 = q | (1 << ax);
      if (q2 == q) continue;
      const bool in1 = cz[q] >= p.z_min, in2 = cz[q2] >= p.z_min;
      if (in1 == in2) continue;
      const float s = (p.z_min - cz[q]) / (cz[q2] - cz[q]);
      const float x = cx[q] + s * (cx[q2] - cx[q]), y = cy[q] + s * (cy[q2] - cy[q]);
      const float u = p.fx * x / p.z_min + p.cx, v = p.fy * y / p.z_min + p.cy;
      umin = fminf(umin, u); umax = fmaxf(umax, u);
      vmin = fminf(vmin, v); vmax = fmaxf(vmax, v);
      zmin = p.z_min;
    }
  }
  // conservative pixel range (+1 px), clipped to the image / row shard
  const float fu0 = fmaxf(floorf(umin) - 1.0f, 0.0f), fu1 = fminf(ceilf(umax) + 1.0f, (float)(p.width - 1));
  const float fv0 = fmaxf(floorf(vmin) - 1.0f, (float)p.row0), fv1 = fminf(ceilf(vmax) + 1.0f, (float)(p.row1 - 1));
  if (!(fu0 <= fu1) || !(fv0 <= fv1)) return;
  const int tx0 = (int)fu0 / kRangeTile, tx1 = (int)fu1 / kRangeTile;
  const int ty0 = ((int)fv0 - p.row0) / kRangeTile, ty1 = ((int)fv1 - p.row0) / kRangeTile;
  const unsigned int zn = __float_as_uint(zmin), zf = __float_as_uint(zmax);
  unsigned int *zn_v = p.z_near + (size_t)view * p.tiles_x * p.tiles_y;
  unsigned int *zf_v = p.z_far + (size_t)view * p.tiles_x * p.tiles_y;
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx) {
      atomicMin(&zn_v[ty * p.tiles_x + tx], zn);
      atomicMax(&zf_v[ty * p.tiles_x + tx], zf);
    }
}

// ------------------------------------------------------------------------------------------
// a2: index lookup
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ bool occupied(const VolumeView &V, int bx, int by, int bz, bool *surf) {
  const unsigned x = (unsigned)(bx - V.lo_x), y = (unsigned)(by - V.lo_y), z = (unsigned)(bz - V.lo_z);
  *surf = false;
  if (x >= (unsigned)V.dim_x || y >= (unsigned)V.dim_y || z >= (unsigned)V.dim_z) return false;
  const unsigned long long cell = ((unsigned long long)z * V.dim_y + y) * V.dim_x + x;
  *surf = (__ldg(&V.surface[cell >> 5]) >> (cell & 31)) & 1u;
  return (__ldg(&V.bitmap[cell >> 5]) >> (cell & 31)) & 1u;
}

__device__ __forceinline__ int lookup_slots(const VolumeView &V, int bx, int by, int bz, int slots[6]) {
  const unsigned long long key = pack_key(bx, by, bz);
  unsigned int h = hash_key(key) & V.table_mask;
  for (unsigned int probe = 0; probe <= V.table_mask; ++probe) {
    const int4 *e = reinterpret_cast<const int4 *>(&V.table[h]);
    const int4 a = __ldg(e);
    const unsigned long long k = (unsigned long long)(unsigned)a.x | ((unsigned long long)(unsigned)a.y << 32);
    if (k == key) {
      const int4 c = __ldg(e + 1);
      slots[0] = a.z; slots[1] = a.w; slots[2] = c.x; slots[3] = c.y; slots[4] = c.z; slots[5] = c.w;
      return (int)h;
    }
    if (k == kEmptyKey) break;
    h = (h + 1) & V.table_mask;
  }
#pragma unroll
  for (int d = 0; d < 6; ++d) slots[d] = -1;
  return -1;
}

// ------------------------------------------------------------------------------------------
// a5: per-sample directional combination
// ------------------------------------------------------------------------------------------
struct SampleResult {
  bool valid;
  float f;
};

struct ShadeResult {
  float n[3];
  float c[3];
  float S;
  int mask;
};

__device__ __forceinline__ float lerpf(float a, float b, float t) { return fmaf(t, b - a, a); }

#define APRON_IDX(dx, dy, dz) (((dx) + 1) + kApron * ((dy) + 1) + kApron * kApron * ((dz) + 1))
#define RGB_IDX(dx, dy, dz) ((dx) + kRgbApron * (dy) + kRgbApron * kRgbApron * (dz))

// eq:direction_weight with reading R1: clamp((theta - acos c) / (2 theta - pi/2), 0, 1)
// (outside the blend band the clamp decides: c <= cos(theta) -> 0, c >= sin(theta) -> 1)
__device__ __forceinline__ float w_dir(float c, const VolumeView &V) {
  if (c <= V.cos_theta) return 0.0f;
  if (c >= V.sin_theta) return 1.0f;
  const float a = acosf(fminf(c, 1.0f));
  return fminf(fmaxf((V.theta - a) * V.inv_blend, 0.0f), 1.0f);
}

struct Cursor {
  int bx, by, bz;
  bool occ;      // location allocated in some direction (occupancy bitmap)
  bool surf;     // some corner-range voxel has sdf <= 0 (surface bitmap)
  int present;   // bit D: direction D has a brick at this location
  int entry;     // hash entry index (row of cell_pos), -1 if unallocated
  int slots[6];
};

// cell l (= lx + 8 ly + 64 lz) of the cursor's location is certainly positive (k_cell_pos)
__device__ __forceinline__ bool cell_positive(const VolumeView &V, const Cursor &cur, int l) {
  return (__ldg(&V.cell_pos[(size_t)cur.entry * 16 + (l >> 5)]) >> (l & 31)) & 1u;
}

__device__ __forceinline__ int pick6(const int s[6], int d) {
  // register-resident select (a dynamic index would spill the array to local memory)
  int v = s[0];
  v = d == 1 ? s[1] : v;
  v = d == 2 ? s[2] : v;
  v = d == 3 ? s[3] : v;
  v = d == 4 ? s[4] : v;
  v = d == 5 ? s[5] : v;
  return v;
}

// F(x, r) of DESIGN.md §2 O3 for the sample at base voxel (block-local l, fractions f) of the
// current cursor location; with shade = true also the shading sums of O7.  One instance of this
// body is compiled (runtime direction loop) to keep the kernel inside the instruction cache.
__device__ __forceinline__ SampleResult eval_sample(const VolumeView &V, const Cursor &cur, int lx, int ly, int lz,
                                                 float fx, float fy, float fz, float rx, float ry, float rz,
                                                 bool shade, ShadeResult *sh) {
  float S1 = 0.f, F1 = 0.f, S2 = 0.f, F2 = 0.f;
  bool any_grad = false;
  float N1x = 0.f, N1y = 0.f, N1z = 0.f, N2x = 0.f, N2y = 0.f, N2z = 0.f;
  float C1r = 0.f, C1g = 0.f, C1b = 0.f, C2r = 0.f, C2g = 0.f, C2b = 0.f;
  int m1 = 0, m2 = 0;
  const float half_inv_s = 0.5f * V.inv_voxel;
  const int off = lx + kApron * ly + kApron * kApron * lz;
  int present = cur.present;
#pragma unroll 1
  while (present) {
    const int D = __ffs(present) - 1;
    present &= present - 1;
    const int slot = pick6(cur.slots, D);
    const float2 *br = V.apron + (size_t)slot * kApronStride + off;
    // O3(a) trilinear phi_D, omega_D over the 8 cell corners
    const float2 c000 = __ldg(br + APRON_IDX(0, 0, 0)), c100 = __ldg(br + APRON_IDX(1, 0, 0));
    const float2 c010 = __ldg(br + APRON_IDX(0, 1, 0)), c110 = __ldg(br + APRON_IDX(1, 1, 0));
    const float2 c001 = __ldg(br + APRON_IDX(0, 0, 1)), c101 = __ldg(br + APRON_IDX(1, 0, 1));
    const float2 c011 = __ldg(br + APRON_IDX(0, 1, 1)), c111 = __ldg(br + APRON_IDX(1, 1, 1));
    const float w00 = lerpf(c000.y, c100.y, fx), w10 = lerpf(c010.y, c110.y, fx);
    const float w01 = lerpf(c001.y, c101.y, fx), w11 = lerpf(c011.y, c111.y, fx);
    const float omega = lerpf(lerpf(w00, w10, fy), lerpf(w01, w11, fy), fz);
    // x-lerps of the four corner rows e_yz; R(dz) = bilinear over (x, y) of slab dz
    const float e00 = lerpf(c000.x, c100.x, fx), e10 = lerpf(c010.x, c110.x, fx);
    const float e01 = lerpf(c001.x, c101.x, fx), e11 = lerpf(c011.x, c111.x, fx);
    const float R0 = lerpf(e00, e10, fy), R1 = lerpf(e01, e11, fy);
    const float phi = lerpf(R0, R1, fz);
    if (isnan(phi)) continue;       // D absent: a corner lies in an unallocated block
    if (!(omega > 0.0f)) continue;  // D holds no data at x (reading R8)
    // O3(c) central differences of trilinear phi at x +- s e_a (24 further stencil voxels):
    // phi(x + s e_a) - phi(x - s e_a) = (1 - f_a)(A1 - A-1) + f_a (A2 - A0) with A(d) the
    // bilinear interpolant of the stencil layer d along axis a
    const float P0 = lerpf(lerpf(c000.x, c010.x, fy), lerpf(c001.x, c011.x, fy), fz);
    const float P1 = lerpf(lerpf(c100.x, c110.x, fy), lerpf(c101.x, c111.x, fy), fz);
    const float Q0 = lerpf(e00, e01, fz), Q1 = lerpf(e10, e11, fz);
    const float Pm = lerpf(lerpf(__ldg(&br[APRON_IDX(-1, 0, 0)].x), __ldg(&br[APRON_IDX(-1, 1, 0)].x), fy),
                           lerpf(__ldg(&br[APRON_IDX(-1, 0, 1)].x), __ldg(&br[APRON_IDX(-1, 1, 1)].x), fy), fz);
    const float Pp = lerpf(lerpf(__ldg(&br[APRON_IDX(2, 0, 0)].x), __ldg(&br[APRON_IDX(2, 1, 0)].x), fy),
                           lerpf(__ldg(&br[APRON_IDX(2, 0, 1)].x), __ldg(&br[APRON_IDX(2, 1, 1)].x), fy), fz);
    const float Qm = lerpf(lerpf(__ldg(&br[APRON_IDX(0, -1, 0)].x), __ldg(&br[APRON_IDX(1, -1, 0)].x), fx),
                           lerpf(__ldg(&br[APRON_IDX(0, -1, 1)].x), __ldg(&br[APRON_IDX(1, -1, 1)].x), fx), fz);
    const float Qp = lerpf(lerpf(__ldg(&br[APRON_IDX(0, 2, 0)].x), __ldg(&br[APRON_IDX(1, 2, 0)].x), fx),
                           lerpf(__ldg(&br[APRON_IDX(0, 2, 1)].x), __ldg(&br[APRON_IDX(1, 2, 1)].x), fx), fz);
    const float Rm = lerpf(lerpf(__ldg(&br[APRON_IDX(0, 0, -1)].x), __ldg(&br[APRON_IDX(1, 0, -1)].x), fx),
                           lerpf(__ldg(&br[APRON_IDX(0, 1, -1)].x), __ldg(&br[APRON_IDX(1, 1, -1)].x), fx), fy);
    const float Rp = lerpf(lerpf(__ldg(&br[APRON_IDX(0, 0, 2)].x), __ldg(&br[APRON_IDX(1, 0, 2)].x), fx),
                           lerpf(__ldg(&br[APRON_IDX(0, 1, 2)].x), __ldg(&br[APRON_IDX(1, 1, 2)].x), fx), fy);
    const float gx = lerpf(P1 - Pm, Pp - P0, fx) * half_inv_s;
    const float gy = lerpf(Q1 - Qm, Qp - Q0, fy) * half_inv_s;
    const float gz = lerpf(R1 - Rm, Rp - R0, fz) * half_inv_s;
    const float gn = sqrtf(gx * gx + gy * gy + gz * gz);
    // v^D = sign * e_axis
    const int axis = D >> 1;
    const float sign = (D & 1) ? -1.0f : 1.0f;
    const float r_axis = axis == 0 ? rx : (axis == 1 ? ry : rz);
    // eq:combine_tsdf_weight: omega * max(0, <v^D, -r>)
    const float W2 = omega * fmaxf(-sign * r_axis, 0.0f);
    S2 += W2;
    F2 = fmaf(W2, phi, F2);
    float W1 = 0.0f, nx = 0.f, ny = 0.f, nz = 0.f;
    if (gn > 1e-3f) {  // reading R8: gradient present (NaN stencil -> false)
      any_grad = true;
      const float ig = 1.0f / gn;
      nx = gx * ig; ny = gy * ig; nz = gz * ig;
      const float n_axis = axis == 0 ? nx : (axis == 1 ? ny : nz);
      const float nr = -(nx * rx + ny * ry + nz * rz);
      // eq:combine_weight: w_dir(<n,v>) * max(0, <n,-r>) * omega
      W1 = w_dir(sign * n_axis, V) * fmaxf(nr, 0.0f) * omega;
      S1 += W1;
      F1 = fmaf(W1, phi, F1);
    }
    if (shade) {
      const uchar4 *cb = V.rgb_apron + (size_t)slot * kRgbApronStride + (lx + kRgbApron * ly + kRgbApron * kRgbApron * lz);
      const uchar4 q000 = cb[RGB_IDX(0, 0, 0)], q100 = cb[RGB_IDX(1, 0, 0)], q010 = cb[RGB_IDX(0, 1, 0)],
                   q110 = cb[RGB_IDX(1, 1, 0)], q001 = cb[RGB_IDX(0, 0, 1)], q101 = cb[RGB_IDX(1, 0, 1)],
                   q011 = cb[RGB_IDX(0, 1, 1)], q111 = cb[RGB_IDX(1, 1, 1)];
#define TRI_CH(ch)                                                                                              \
  lerpf(lerpf(lerpf((float)q000.ch, (float)q100.ch, fx), lerpf((float)q010.ch, (float)q110.ch, fx), fy),        \
        lerpf(lerpf((float)q001.ch, (float)q101.ch, fx), lerpf((float)q011.ch, (float)q111.ch, fx), fy), fz)
      const float cr = TRI_CH(x), cg = TRI_CH(y), cbl = TRI_CH(z);
#undef TRI_CH
      if (W1 > 0.0f) {
        N1x = fmaf(W1, nx, N1x); N1y = fmaf(W1, ny, N1y); N1z = fmaf(W1, nz, N1z);
        C1r = fmaf(W1, cr, C1r); C1g = fmaf(W1, cg, C1g); C1b = fmaf(W1, cbl, C1b);
        m1 |= 1 << D;
      }
      if (W2 > 0.0f) {
        const float ws = W2 * sign;
        N2x += axis == 0 ? ws : 0.f; N2y += axis == 1 ? ws : 0.f; N2z += axis == 2 ? ws : 0.f;
        C2r = fmaf(W2, cr, C2r); C2g = fmaf(W2, cg, C2g); C2b = fmaf(W2, cbl, C2b);
        m2 |= 1 << D;
      }
    }
  }
  // O3(d)/(e): eq:combine_weight if any direction holding data has a gradient, else the fallback
  const float S = any_grad ? S1 : S2;
  const float F = any_grad ? F1 : F2;
  SampleResult res;
  res.valid = S > 0.0f;
  res.f = res.valid ? F / S : 0.0f;
  if (shade) {
    sh->S = S;
    sh->mask = any_grad ? m1 : m2;
    sh->n[0] = any_grad ? N1x : N2x; sh->n[1] = any_grad ? N1y : N2y; sh->n[2] = any_grad ? N1z : N2z;
    sh->c[0] = any_grad ? C1r : C2r; sh->c[1] = any_grad ? C1g : C2g; sh->c[2] = any_grad ? C1b : C2b;
  }
  return res;
}

// ------------------------------------------------------------------------------------------
// a4-a7: the raycast kernel, one state machine per ray so that a warp's rays -- marching,
// bisecting, regula-falsi or shading -- all run the same sample-evaluation code together
// ------------------------------------------------------------------------------------------
enum : int { kMarch = 0, kBisect = 1, kIllinois = 2, kShade = 3 };

__global__ void __launch_bounds__(256, DTSDF_RAYCAST_MINB) k_raycast(const __grid_constant__ RenderLaunch p) {
  const int view = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.x * 16 + (warp & 1) * 8 + (lane & 7);
  const int vrel = blockIdx.y * 16 + (warp >> 1) * 4 + (lane >> 3);
  const int v = p.row0 + vrel;
  if (u >= p.width || v >= p.row1) return;
  const VolumeView &V = p.vol;
  const ViewPose &P = p.pose[view];
  // O1 ray (eq:reprojection) in fp64: sample positions are formed in fp64 so that
  // refinement can locate the shading point to ~1e-9 m (reading R32); the combination itself
  // runs in fp32 on cell-local fractions
  double od[3], rd[3];
  float r[3];
  double L;
  {
    const double ddx = ((double)u - (double)p.cx) / (double)p.fx, ddy = ((double)v - (double)p.cy) / (double)p.fy;
    L = sqrt(ddx * ddx + ddy * ddy + 1.0);
    const double iLd = 1.0 / L;
    for (int q = 0; q < 3; ++q) {
      rd[q] = ((double)P.r[3 * q] * ddx + (double)P.r[3 * q + 1] * ddy + (double)P.r[3 * q + 2]) * iLd;
      od[q] = (double)P.t[q];
      r[q] = (float)rd[q];
    }
  }
  const int rows = p.row1 - p.row0;
  const size_t pix = ((size_t)view * rows + vrel) * p.width + u;
  // O2 lattice bounds, narrowed to the tile's block range (a3)
  const float Lf = (float)L;
  const size_t tile = ((size_t)view * p.tiles_y + (vrel >> 3)) * p.tiles_x + (u >> 3);
  const float zn = __uint_as_float(__ldg(&p.z_near[tile])), zf = __uint_as_float(__ldg(&p.z_far[tile]));
  const int kmin = (int)ceilf(p.z_min * Lf * V.inv_delta), kmax = (int)floorf(p.z_max * Lf * V.inv_delta);
  int k = kmin, k1 = kmax;
  if (p.use_range) {
    if (zn <= zf) {
      k = max(kmin, (int)floorf(zn * (1.0f - 1e-4f) * Lf * V.inv_delta));
      k1 = min(kmax, (int)ceilf(zf * (1.0f + 1e-4f) * Lf * V.inv_delta) + 1);
    } else {
      k1 = k - 1;  // no allocated block projects onto this tile
    }
  }
  const double dd = (double)V.delta, idd = 1.0 / dd, inv_s = 1.0 / (double)V.voxel_size;
  double ird[3];
  for (int q = 0; q < 3; ++q) ird[q] = 1.0 / rd[q];
  const double bsz = (double)kBlock * (double)V.voxel_size;
  Cursor cur;
  cur.bx = 0x7fffffff; cur.by = 0; cur.bz = 0; cur.occ = false; cur.surf = false; cur.present = 0; cur.entry = -1;
#pragma unroll
  for (int d = 0; d < 6; ++d) cur.slots[d] = -1;
  int mode = kMarch;
  bool prev_valid = false;
  float prev_f = 0.0f;
  // refinement state: bracket [a, b] with f(a) > 0 (or invalid), f(b) <= 0
  double a = 0.0, b = 0.0, t = (double)k * dd;
  float fa = 0.f, fb = 0.f;
  bool fa_valid = true;
  int it = 0, side = 0;
  bool hit = false;
  ShadeResult sh;
#ifdef DTSDF_STATS
  int st_march = 0, st_refine = 0, st_skip = 0;
#endif
  // cell of the current sample and the cursor over its block location
  double gx = 0, gy = 0, gz = 0, flx = 0, fly = 0, flz = 0;
  int ix = 0, iy = 0, iz = 0;
  auto locate = [&](double tt) {
    gx = fma(tt, rd[0], od[0]) * inv_s;
    gy = fma(tt, rd[1], od[1]) * inv_s;
    gz = fma(tt, rd[2], od[2]) * inv_s;
    flx = floor(gx); fly = floor(gy); flz = floor(gz);
    ix = (int)flx; iy = (int)fly; iz = (int)flz;
    const int bx = ix >> 3, by = iy >> 3, bz = iz >> 3;
    if (bx != cur.bx || by != cur.by || bz != cur.bz) {
      cur.bx = bx; cur.by = by; cur.bz = bz;
      cur.occ = occupied(V, bx, by, bz, &cur.surf);
      cur.present = 0;
      cur.entry = -1;
      if (cur.occ) {
        cur.entry = lookup_slots(V, bx, by, bz, cur.slots);
#pragma unroll
        for (int d = 0; d < 6; ++d) cur.present |= (cur.slots[d] >= 0) << d;
      }
    }
  };
  auto block_exit = [&]() {
    double texit = 1e300;
    const int bb[3] = {cur.bx, cur.by, cur.bz};
    for (int q = 0; q < 3; ++q) {
      if (rd[q] > 0.0) texit = fmin(texit, ((bb[q] + 1) * bsz - od[q]) * ird[q]);
      else if (rd[q] < 0.0) texit = fmin(texit, (bb[q] * bsz - od[q]) * ird[q]);
    }
    return texit;
  };
  for (;;) {
    if (mode == kMarch) {
      // a4: advance to the next lattice point that needs an evaluation.  Every step skipped here
      // is exact (DESIGN.md §2 O2): lattice points in unallocated locations are invalid; in a
      // location without an sdf <= 0 corner, and in a certainly-positive cell followed by
      // another, no crossing can end or start.  Lanes of a warp run this cheap loop, then all
      // evaluate together below.
      bool found = false;
      while (k <= k1) {
        t = (double)k * dd;
        locate(t);
        if (!cur.occ) {
          prev_valid = false;
#ifdef DTSDF_STATS
          ++st_skip;
#endif
          if (p.use_skip) {  // land on the first lattice point at or before the block exit
            const double kn = floor(block_exit() * idd);
            k = (kn > (double)k1) ? k1 + 1 : max(k + 1, (int)kn);
          } else {
            ++k;
          }
          continue;
        }
        if (p.use_skip && !cur.surf) {
          // jump to (at most) the location's second-to-last lattice point: the point evaluated
          // there becomes prev for the first point of the next location
          const double kj = ceil(block_exit() * idd) - 2.0;
          if (kj > (double)k) {
#ifdef DTSDF_STATS
            ++st_skip;
#endif
            k = (kj > (double)k1) ? k1 + 1 : (int)kj;
            prev_valid = false;
            continue;
          }
        }
        if (p.use_skip && cell_positive(V, cur, (ix & 7) + 8 * (iy & 7) + 64 * (iz & 7))) {
          const double t2 = t + dd;
          const int jx = (int)floor(fma(t2, rd[0], od[0]) * inv_s), jy = (int)floor(fma(t2, rd[1], od[1]) * inv_s),
                    jz = (int)floor(fma(t2, rd[2], od[2]) * inv_s);
          if ((jx >> 3) == cur.bx && (jy >> 3) == cur.by && (jz >> 3) == cur.bz &&
              cell_positive(V, cur, (jx & 7) + 8 * (jy & 7) + 64 * (jz & 7))) {
#ifdef DTSDF_STATS
            ++st_skip;
#endif
            prev_valid = false;
            ++k;
            continue;
          }
        }
        found = true;
        break;
      }
      if (!found) break;  // no crossing: a miss
    } else {
      locate(t);
    }
#ifdef DTSDF_STATS
    if (mode == kMarch) ++st_march;
    else ++st_refine;
#endif
    SampleResult s;
    if (cur.occ) {
      s = eval_sample(V, cur, ix & 7, iy & 7, iz & 7, (float)(gx - flx), (float)(gy - fly), (float)(gz - flz), r[0],
                      r[1], r[2], mode == kShade, &sh);
    } else {
      s.valid = false;
      s.f = 0.f;
    }
    if (mode == kMarch) {
      if (s.valid && prev_valid && prev_f > 0.0f && s.f <= 0.0f) {
        // a6: bracket [t_{k-1}, t_k].  Phase 1: bisection with the oracle's decisions (an
        // invalid midpoint counts as positive, R21) until the bracket is <= 5e-5 m, so it
        // keeps the oracle's root when F has several sign changes (reading R20).
        a = (double)(k - 1) * dd;
        b = t;
        fa = prev_f;
        fb = s.f;
        fa_valid = true;
        it = 0;
        side = 0;
        mode = p.n_bisect > 0 ? kBisect : kIllinois;
      } else {
        prev_valid = s.valid;
        prev_f = s.f;
        ++k;
        t = (double)k * dd;
        continue;
      }
    } else if (mode == kBisect) {
      if (!s.valid || s.f > 0.0f) { a = t; fa = s.f; fa_valid = s.valid; }
      else { b = t; fb = s.f; }
      if (++it >= p.n_bisect) { mode = kIllinois; it = 0; }
    } else if (mode == kIllinois) {
      // Phase 2: Illinois regula falsi inside the narrowed bracket until b sits on the root
      if (!s.valid || s.f > 0.0f) {
        a = t; fa = s.f; fa_valid = s.valid;
        if (side == 1) fb *= 0.5f;
        side = 1;
      } else {
        b = t; fb = s.f;
        if (side == -1) fa *= 0.5f;
        side = -1;
        if (s.f > -1e-7f) mode = kShade;  // b sits on the root
      }
      if (++it >= 12 || b - a <= 1e-12) mode = kShade;
    } else {  // kShade: a7 done at b, a valid sample on the surface side (reading R32)
      hit = true;
      break;
    }
    // next position
    if (mode == kBisect) t = 0.5 * (a + b);
    else if (mode == kIllinois) {
      double m = (fa_valid && fa > fb) ? a + (double)(fa / (fa - fb)) * (b - a) : 0.5 * (a + b);
      if (!(m > a && m < b)) m = 0.5 * (a + b);
      t = m;
    } else t = b;  // kShade
  }
  float depth = 0.f, nrm[3] = {0.f, 0.f, 0.f};
  int col[3] = {0, 0, 0}, mask = 0;
  if (hit) {
    depth = (float)(b / L);
    const float nn = sqrtf(sh.n[0] * sh.n[0] + sh.n[1] * sh.n[1] + sh.n[2] * sh.n[2]);
    const float inn = nn > 0.f ? 1.0f / nn : 0.f;
    for (int q = 0; q < 3; ++q) {
      nrm[q] = sh.n[q] * inn;
      const float c = sh.S > 0.f ? floorf(sh.c[q] / sh.S + 0.5f) : 0.f;  // reading R13
      col[q] = (int)fminf(fmaxf(c, 0.f), 255.f);
    }
    mask = sh.mask;
  }
#ifdef DTSDF_STATS
  nrm[0] = (float)st_march; nrm[1] = (float)st_refine; nrm[2] = (float)st_skip;
#endif
  p.out_depth[pix] = depth;
  if (p.out_normal) {
    p.out_normal[3 * pix + 0] = nrm[0];
    p.out_normal[3 * pix + 1] = nrm[1];
    p.out_normal[3 * pix + 2] = nrm[2];
  }
  if (p.out_color) {
    p.out_color[3 * pix + 0] = (unsigned char)col[0];
    p.out_color[3 * pix + 1] = (unsigned char)col[1];
    p.out_color[3 * pix + 2] = (unsigned char)col[2];
  }
  if (p.out_mask) p.out_mask[pix] = (unsigned char)mask;
}

cudaError_t launch_range(const RangeLaunch &p, cudaStream_t s) {
  if (p.n_locations == 0 || p.n_views == 0) return cudaSuccess;
  dim3 grid((unsigned)((p.n_locations + 255) / 256), (unsigned)p.n_views);
  k_range<<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_raycast(const RenderLaunch &p, cudaStream_t s) {
  if (p.n_views == 0) return cudaSuccess;
  dim3 grid((unsigned)((p.width + 15) / 16), (unsigned)((p.row1 - p.row0 + 15) / 16), (unsigned)p.n_views);
  k_raycast<<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace dtsdf
