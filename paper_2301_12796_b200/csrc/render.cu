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
__device__ __forceinline__ bool occupied(const VolumeView &V, int bx, int by, int bz) {
  const unsigned x = (unsigned)(bx - V.lo_x), y = (unsigned)(by - V.lo_y), z = (unsigned)(bz - V.lo_z);
  if (x >= (unsigned)V.dim_x || y >= (unsigned)V.dim_y || z >= (unsigned)V.dim_z) return false;
  const unsigned long long cell = ((unsigned long long)z * V.dim_y + y) * V.dim_x + x;
  return (__ldg(&V.bitmap[cell >> 5]) >> (cell & 31)) & 1u;
}

__device__ __forceinline__ void lookup_slots(const VolumeView &V, int bx, int by, int bz, int slots[6]) {
  const unsigned long long key = pack_key(bx, by, bz);
  unsigned int h = hash_key(key) & V.table_mask;
  for (unsigned int probe = 0; probe <= V.table_mask; ++probe) {
    const int4 *e = reinterpret_cast<const int4 *>(&V.table[h]);
    const int4 a = __ldg(e);
    const unsigned long long k = (unsigned long long)(unsigned)a.x | ((unsigned long long)(unsigned)a.y << 32);
    if (k == key) {
      const int4 c = __ldg(e + 1);
      slots[0] = a.z; slots[1] = a.w; slots[2] = c.x; slots[3] = c.y; slots[4] = c.z; slots[5] = c.w;
      return;
    }
    if (k == kEmptyKey) break;
    h = (h + 1) & V.table_mask;
  }
#pragma unroll
  for (int d = 0; d < 6; ++d) slots[d] = -1;
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
__device__ __forceinline__ float w_dir(float c, const VolumeView &V) {
  const float a = acosf(fminf(fmaxf(c, -1.0f), 1.0f));
  return fminf(fmaxf((V.theta - a) * V.inv_blend, 0.0f), 1.0f);
}

template <bool SHADE>
__device__ __forceinline__ SampleResult eval_sample(const VolumeView &V, const int slots[6], int lx, int ly, int lz,
                                                    float fx, float fy, float fz, float rx, float ry, float rz,
                                                    ShadeResult *sh) {
  float S1 = 0.f, F1 = 0.f, S2 = 0.f, F2 = 0.f;
  bool any_grad = false;
  float N1[3] = {0.f, 0.f, 0.f}, N2[3] = {0.f, 0.f, 0.f}, C1[3] = {0.f, 0.f, 0.f}, C2[3] = {0.f, 0.f, 0.f};
  int m1 = 0, m2 = 0;
  const float half_inv_s = 0.5f * V.inv_voxel;
  const int off = lx + kApron * ly + kApron * kApron * lz;
#pragma unroll
  for (int D = 0; D < 6; ++D) {
    const int slot = slots[D];
    if (slot < 0) continue;
    const float2 *br = V.apron + (size_t)slot * kApronStride + off;
    // O3(a) trilinear phi_D, omega_D over the 8 cell corners
    const float2 c000 = __ldg(br + APRON_IDX(0, 0, 0)), c100 = __ldg(br + APRON_IDX(1, 0, 0));
    const float2 c010 = __ldg(br + APRON_IDX(0, 1, 0)), c110 = __ldg(br + APRON_IDX(1, 1, 0));
    const float2 c001 = __ldg(br + APRON_IDX(0, 0, 1)), c101 = __ldg(br + APRON_IDX(1, 0, 1));
    const float2 c011 = __ldg(br + APRON_IDX(0, 1, 1)), c111 = __ldg(br + APRON_IDX(1, 1, 1));
    const float w00 = lerpf(c000.y, c100.y, fx), w10 = lerpf(c010.y, c110.y, fx);
    const float w01 = lerpf(c001.y, c101.y, fx), w11 = lerpf(c011.y, c111.y, fx);
    const float omega = lerpf(lerpf(w00, w10, fy), lerpf(w01, w11, fy), fz);
    // x-columns of the cell corners: P(dx) = bilinear over (y, z)
    const float P0 = lerpf(lerpf(c000.x, c010.x, fy), lerpf(c001.x, c011.x, fy), fz);
    const float P1 = lerpf(lerpf(c100.x, c110.x, fy), lerpf(c101.x, c111.x, fy), fz);
    const float phi = lerpf(P0, P1, fx);
    if (isnan(phi)) continue;       // D absent: a corner lies in an unallocated block
    if (!(omega > 0.0f)) continue;  // D holds no data at x (reading R8)
    // O3(c) central differences of trilinear phi at x +- s e_a (24 further stencil voxels)
    const float Pm = lerpf(lerpf(__ldg(&br[APRON_IDX(-1, 0, 0)].x), __ldg(&br[APRON_IDX(-1, 1, 0)].x), fy),
                           lerpf(__ldg(&br[APRON_IDX(-1, 0, 1)].x), __ldg(&br[APRON_IDX(-1, 1, 1)].x), fy), fz);
    const float Pp = lerpf(lerpf(__ldg(&br[APRON_IDX(2, 0, 0)].x), __ldg(&br[APRON_IDX(2, 1, 0)].x), fy),
                           lerpf(__ldg(&br[APRON_IDX(2, 0, 1)].x), __ldg(&br[APRON_IDX(2, 1, 1)].x), fy), fz);
    const float Q0 = lerpf(lerpf(c000.x, c100.x, fx), lerpf(c001.x, c101.x, fx), fz);
    const float Q1 = lerpf(lerpf(c010.x, c110.x, fx), lerpf(c011.x, c111.x, fx), fz);
    const float Qm = lerpf(lerpf(__ldg(&br[APRON_IDX(0, -1, 0)].x), __ldg(&br[APRON_IDX(1, -1, 0)].x), fx),
                           lerpf(__ldg(&br[APRON_IDX(0, -1, 1)].x), __ldg(&br[APRON_IDX(1, -1, 1)].x), fx), fz);
    const float Qp = lerpf(lerpf(__ldg(&br[APRON_IDX(0, 2, 0)].x), __ldg(&br[APRON_IDX(1, 2, 0)].x), fx),
                           lerpf(__ldg(&br[APRON_IDX(0, 2, 1)].x), __ldg(&br[APRON_IDX(1, 2, 1)].x), fx), fz);
    const float R0 = lerpf(lerpf(c000.x, c100.x, fx), lerpf(c010.x, c110.x, fx), fy);
    const float R1 = lerpf(lerpf(c001.x, c101.x, fx), lerpf(c011.x, c111.x, fx), fy);
    const float Rm = lerpf(lerpf(__ldg(&br[APRON_IDX(0, 0, -1)].x), __ldg(&br[APRON_IDX(1, 0, -1)].x), fx),
                           lerpf(__ldg(&br[APRON_IDX(0, 1, -1)].x), __ldg(&br[APRON_IDX(1, 1, -1)].x), fx), fy);
    const float Rp = lerpf(lerpf(__ldg(&br[APRON_IDX(0, 0, 2)].x), __ldg(&br[APRON_IDX(1, 0, 2)].x), fx),
                           lerpf(__ldg(&br[APRON_IDX(0, 1, 2)].x), __ldg(&br[APRON_IDX(1, 1, 2)].x), fx), fy);
    const float gx = (lerpf(P1, Pp, fx) - lerpf(Pm, P0, fx)) * half_inv_s;
    const float gy = (lerpf(Q1, Qp, fy) - lerpf(Qm, Q0, fy)) * half_inv_s;
    const float gz = (lerpf(R1, Rp, fz) - lerpf(Rm, R0, fz)) * half_inv_s;
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
    if (SHADE) {
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
        N1[0] = fmaf(W1, nx, N1[0]); N1[1] = fmaf(W1, ny, N1[1]); N1[2] = fmaf(W1, nz, N1[2]);
        C1[0] = fmaf(W1, cr, C1[0]); C1[1] = fmaf(W1, cg, C1[1]); C1[2] = fmaf(W1, cbl, C1[2]);
        m1 |= 1 << D;
      }
      if (W2 > 0.0f) {
        if (axis == 0) N2[0] = fmaf(W2, sign, N2[0]);
        else if (axis == 1) N2[1] = fmaf(W2, sign, N2[1]);
        else N2[2] = fmaf(W2, sign, N2[2]);
        C2[0] = fmaf(W2, cr, C2[0]); C2[1] = fmaf(W2, cg, C2[1]); C2[2] = fmaf(W2, cbl, C2[2]);
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
  if (SHADE) {
    const float *N = any_grad ? N1 : N2;
    const float *Cc = any_grad ? C1 : C2;
    sh->S = S;
    sh->mask = any_grad ? m1 : m2;
    for (int a = 0; a < 3; ++a) { sh->n[a] = N[a]; sh->c[a] = Cc[a]; }
  }
  return res;
}

// ------------------------------------------------------------------------------------------
// a4-a7: the raycast kernel
// ------------------------------------------------------------------------------------------
struct Cursor {
  int bx, by, bz;
  bool occ;
  int slots[6];
};

template <bool SHADE>
__device__ __forceinline__ SampleResult eval_at(const VolumeView &V, Cursor &cur, float t, const float o[3],
                                                const float r[3], ShadeResult *sh, bool *in_occupied) {
  const float x = fmaf(t, r[0], o[0]), y = fmaf(t, r[1], o[1]), z = fmaf(t, r[2], o[2]);
  const float gx = x * V.inv_voxel, gy = y * V.inv_voxel, gz = z * V.inv_voxel;
  const float flx = floorf(gx), fly = floorf(gy), flz = floorf(gz);
  const int ix = (int)flx, iy = (int)fly, iz = (int)flz;
  const int bx = ix >> 3, by = iy >> 3, bz = iz >> 3;
  if (bx != cur.bx || by != cur.by || bz != cur.bz) {
    cur.bx = bx; cur.by = by; cur.bz = bz;
    cur.occ = occupied(V, bx, by, bz);
    if (cur.occ) lookup_slots(V, bx, by, bz, cur.slots);
  }
  *in_occupied = cur.occ;
  if (!cur.occ) {
    SampleResult s;
    s.valid = false;
    s.f = 0.f;
    if (SHADE) { sh->S = 0.f; sh->mask = 0; }
    return s;
  }
  return eval_sample<SHADE>(V, cur.slots, ix & 7, iy & 7, iz & 7, gx - flx, gy - fly, gz - flz, r[0], r[1], r[2], sh);
}

// Same as eval_at, but the sample position x = o + t r and its cell/fractions are computed in
// fp64 (refinement and shading only): near a root the combination weights can vary on a
// sub-micrometre scale (ill-conditioned mixtures of directions, e.g. configs[2]), so the shading
// point must be located to ~1e-9 m, finer than an fp32 coordinate can resolve.
template <bool SHADE>
__device__ __forceinline__ SampleResult eval_at_d(const VolumeView &V, Cursor &cur, double t, const double o[3],
                                                  const double r[3], const float rf[3], ShadeResult *sh) {
  const double inv_s = 1.0 / (double)V.voxel_size;
  const double gx = fma(t, r[0], o[0]) * inv_s, gy = fma(t, r[1], o[1]) * inv_s, gz = fma(t, r[2], o[2]) * inv_s;
  const double flx = floor(gx), fly = floor(gy), flz = floor(gz);
  const int ix = (int)flx, iy = (int)fly, iz = (int)flz;
  const int bx = ix >> 3, by = iy >> 3, bz = iz >> 3;
  if (bx != cur.bx || by != cur.by || bz != cur.bz) {
    cur.bx = bx; cur.by = by; cur.bz = bz;
    cur.occ = occupied(V, bx, by, bz);
    if (cur.occ) lookup_slots(V, bx, by, bz, cur.slots);
  }
  if (!cur.occ) {
    SampleResult s;
    s.valid = false;
    s.f = 0.f;
    if (SHADE) { sh->S = 0.f; sh->mask = 0; }
    return s;
  }
  return eval_sample<SHADE>(V, cur.slots, ix & 7, iy & 7, iz & 7, (float)(gx - flx), (float)(gy - fly),
                            (float)(gz - flz), rf[0], rf[1], rf[2], sh);
}

__global__ void __launch_bounds__(256) k_raycast(const __grid_constant__ RenderLaunch p) {
  const int view = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.x * 16 + (warp & 1) * 8 + (lane & 7);
  const int vrel = blockIdx.y * 16 + (warp >> 1) * 4 + (lane >> 3);
  const int v = p.row0 + vrel;
  if (u >= p.width || v >= p.row1) return;
  const VolumeView &V = p.vol;
  const ViewPose &P = p.pose[view];
  // O1 ray (eq:reprojection)
  const float dx = (u - p.cx) / p.fx, dy = (v - p.cy) / p.fy;
  const float L = sqrtf(dx * dx + dy * dy + 1.0f);
  const float iL = 1.0f / L;
  float r[3], o[3];
  for (int a = 0; a < 3; ++a) {
    r[a] = (P.r[3 * a] * dx + P.r[3 * a + 1] * dy + P.r[3 * a + 2]) * iL;
    o[a] = P.t[a];
  }
  const int rows = p.row1 - p.row0;
  const size_t pix = ((size_t)view * rows + vrel) * p.width + u;
  // O2 lattice bounds, narrowed to the tile's block range (a3)
  const size_t tile = ((size_t)view * p.tiles_y + (vrel >> 3)) * p.tiles_x + (u >> 3);
  const float zn = __uint_as_float(__ldg(&p.z_near[tile])), zf = __uint_as_float(__ldg(&p.z_far[tile]));
  const int kmin = (int)ceilf(p.z_min * L * V.inv_delta), kmax = (int)floorf(p.z_max * L * V.inv_delta);
  int k = kmin, k1 = kmax;
  if (!p.use_range) {
    // march every lattice point from z_min to z_max
  } else if (zn <= zf) {
    k = max(kmin, (int)floorf(zn * (1.0f - 1e-4f) * L * V.inv_delta));
    k1 = min(kmax, (int)ceilf(zf * (1.0f + 1e-4f) * L * V.inv_delta) + 1);
  } else {
    k1 = k - 1;  // no allocated block projects onto this tile
  }
  float inv_r[3];
  for (int a = 0; a < 3; ++a) inv_r[a] = 1.0f / r[a];
  Cursor cur;
  cur.bx = 0x7fffffff; cur.by = 0; cur.bz = 0; cur.occ = false;
  bool prev_valid = false;
  float prev_f = 0.0f;
  bool hit = false;
  float depth = 0.f, nrm[3] = {0.f, 0.f, 0.f};
  int col[3] = {0, 0, 0}, mask = 0;
  const float bsz = kBlock * V.voxel_size;
  while (k <= k1) {
    const float t = (float)k * V.delta;
    bool occ;
    const SampleResult s = eval_at<false>(V, cur, t, o, r, nullptr, &occ);
    if (!occ && !p.use_skip) {
      prev_valid = false;
      ++k;
      continue;
    }
    if (!occ) {
      // a4: skip the rest of this unallocated block location (exact: every lattice point
      // there is invalid); land on the first lattice point at or before the block exit
      float texit = CUDART_INF_F;
      const int bb[3] = {cur.bx, cur.by, cur.bz};
      for (int a = 0; a < 3; ++a) {
        if (r[a] > 0.f) texit = fminf(texit, ((bb[a] + 1) * bsz - o[a]) * inv_r[a]);
        else if (r[a] < 0.f) texit = fminf(texit, (bb[a] * bsz - o[a]) * inv_r[a]);
      }
      const float kn = floorf(texit * V.inv_delta);
      k = (kn > (float)k1) ? k1 + 1 : max(k + 1, (int)kn);
      prev_valid = false;
      continue;
    }
    if (s.valid && prev_valid && prev_f > 0.0f && s.f <= 0.0f) {
      // a6: refine the root in [t_{k-1}, t_k] with fp64 ray positions.  Phase 1: bisection
      // with the oracle's decisions (an invalid midpoint counts as positive, R21) until the
      // bracket is <= 5e-5 m, so it keeps the oracle's root when F has several sign changes
      // (reading R20).  Phase 2: Illinois regula falsi inside it until b sits on the root.
      double od[3], rd[3];
      {
        const double ddx = ((double)u - (double)p.cx) / (double)p.fx, ddy = ((double)v - (double)p.cy) / (double)p.fy;
        const double iLd = 1.0 / sqrt(ddx * ddx + ddy * ddy + 1.0);
        for (int q = 0; q < 3; ++q) {
          rd[q] = ((double)P.r[3 * q] * ddx + (double)P.r[3 * q + 1] * ddy + (double)P.r[3 * q + 2]) * iLd;
          od[q] = (double)P.t[q];
        }
      }
      const double dd = (double)V.delta;
      double a = (double)(k - 1) * dd, b = (double)k * dd;
      float fa = prev_f, fb = s.f;
      bool fa_valid = true;
      for (int it = 0; it < p.n_bisect; ++it) {
        const double m = 0.5 * (a + b);
        const SampleResult sm = eval_at_d<false>(V, cur, m, od, rd, r, nullptr);
        if (!sm.valid || sm.f > 0.0f) {
          a = m;
          fa = sm.f;
          fa_valid = sm.valid;
        } else {
          b = m;
          fb = sm.f;
        }
      }
      int side = 0;
      for (int it = 0; it < 12 && b - a > 1e-12; ++it) {
        double m = (fa_valid && fa > fb) ? a + (double)(fa / (fa - fb)) * (b - a) : 0.5 * (a + b);
        if (!(m > a && m < b)) m = 0.5 * (a + b);
        const SampleResult sm = eval_at_d<false>(V, cur, m, od, rd, r, nullptr);
        if (!sm.valid || sm.f > 0.0f) {
          a = m;
          fa = sm.f;
          fa_valid = sm.valid;
          if (side == 1) fb *= 0.5f;
          side = 1;
        } else {
          b = m;
          fb = sm.f;
          if (side == -1) fa *= 0.5f;
          side = -1;
          if (sm.f > -1e-7f) break;  // b sits on the root
        }
      }
      const float tstar = (float)b;
      // a7: shading at the bracket end b, a valid sample on the surface side (reading R32)
      ShadeResult sh;
      eval_at_d<true>(V, cur, b, od, rd, r, &sh);
      hit = true;
      depth = tstar * iL;
      const float nn = sqrtf(sh.n[0] * sh.n[0] + sh.n[1] * sh.n[1] + sh.n[2] * sh.n[2]);
      const float inn = nn > 0.f ? 1.0f / nn : 0.f;
      for (int q = 0; q < 3; ++q) {
        nrm[q] = sh.n[q] * inn;
        const float c = sh.S > 0.f ? floorf(sh.c[q] / sh.S + 0.5f) : 0.f;  // reading R13
        col[q] = (int)fminf(fmaxf(c, 0.f), 255.f);
      }
      mask = sh.mask;
      break;
    }
    prev_valid = s.valid;
    prev_f = s.f;
    ++k;
  }
  p.out_depth[pix] = hit ? depth : 0.0f;
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
