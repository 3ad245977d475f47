// combine.cu -- the view-dependent combined TSDF.
//
// Lemma 1: for a fixed camera the six directional fields combine into one
// conflict-free regular TSDF.  PAPER.md:251-263 computes it "for every voxel in the view
// frustum" (widened by 1/8 of the image on every side) with the combination weights
// eq:combine_weight / eq:combine_tsdf_weight, and P:610 notes that at integer voxel positions no
// trilinear interpolation is needed and the gradient comes from the 6 neighbouring voxels.
//
//   k_comb_select    one warp per allocated block location: the block is classified against the
//                    widened frustum from its 8 corner voxels (exact by convexity); a location
//                    with any voxel inside takes a combined slot (atomic counter)
//   k_combine        one thread per voxel of a combined slot: fp64 frustum test for straddling
//                    blocks (reading R33), then combined sdf / weight / u8 colour / direction mask
//                    from the directional aprons (centre + 6 neighbours, R34-R35); invalid voxels
//                    are NaN
//   k_comb_finish    per combined slot: the 26 neighbouring slots resolved once, the apron border
//                    (voxels -1, 8, 9 per axis) and the colour brick's far faces gathered from
//                    them, then the exact skip masks of the 512 base cells (no valid corner <= 0)
//                    and the brick's surface flag
//
// The slot order depends on the atomic counter; no value does.
#include <math_constants.h>

#include "common.cuh"

namespace dtsdf {

#define CAPRON(dx, dy, dz) (((dx) + 1) + kApron * ((dy) + 1) + kApron * kApron * ((dz) + 1))

// R33: voxel (i,j,k) inside the widened frustum; one rounding per operation in the oracle's
// order (no FMA contraction), so both sides take the same decision
__device__ __forceinline__ bool in_frustum(const CombineLaunch &p, double s, int i, int j, int k, double d[3]) {
  const double x0 = __dmul_rn((double)i, s), x1 = __dmul_rn((double)j, s), x2 = __dmul_rn((double)k, s);
  d[0] = __dsub_rn(x0, p.t[0]);
  d[1] = __dsub_rn(x1, p.t[1]);
  d[2] = __dsub_rn(x2, p.t[2]);
  double xc[3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
    xc[a] = __dadd_rn(__dadd_rn(__dmul_rn(p.R[a], d[0]), __dmul_rn(p.R[3 + a], d[1])), __dmul_rn(p.R[6 + a], d[2]));
  if (!(xc[2] >= p.z_min && xc[2] <= p.z_max)) return false;
  const double u = __dadd_rn(__ddiv_rn(__dmul_rn(p.fx, xc[0]), xc[2]), p.cx);
  const double v = __dadd_rn(__ddiv_rn(__dmul_rn(p.fy, xc[1]), xc[2]), p.cy);
  return u >= -p.mu && u <= p.umax && v >= -p.mv && v <= p.vmax;
}

__device__ __forceinline__ float w_dir_c(float c, const VolumeView &V) {
  if (c <= V.cos_theta) return 0.0f;
  if (c >= V.sin_theta) return 1.0f;
  const float a = acosf(fminf(c, 1.0f));
  return fminf(fmaxf((V.theta - a) * V.inv_blend, 0.0f), 1.0f);
}

struct CombVox {
  float sdf, S;
  uchar4 c;  // rgb + mask
};

// The widened frustum is convex (camera z in [z_min, z_max] and, for z > 0, four half-spaces
// fx x + (cx + mu) z >= 0 ...), so the 8 corner voxels of a block classify it exactly: every
// corner inside all six linear constraints (by a margin far above fp64 rounding) -> every voxel
// inside; every corner outside one constraint -> every voxel outside; else each voxel is tested
// with in_frustum.  Returns 0 outside, 1 inside, 2 straddling (lanes 0..7 carry the corners).
__device__ int classify_block(const CombineLaunch &p, int bx, int by, int bz, int lane) {
  const double s = (double)p.vol.voxel_size, tol = 1e-6;
  double g[6];
  {
    const int q = lane & 7;
    const int i = kBlock * bx + ((q & 1) ? kBlock - 1 : 0), j = kBlock * by + ((q & 2) ? kBlock - 1 : 0),
              k = kBlock * bz + ((q & 4) ? kBlock - 1 : 0);
    const double d0 = (double)i * s - p.t[0], d1 = (double)j * s - p.t[1], d2 = (double)k * s - p.t[2];
    const double xc = p.R[0] * d0 + p.R[3] * d1 + p.R[6] * d2;
    const double yc = p.R[1] * d0 + p.R[4] * d1 + p.R[7] * d2;
    const double zc = p.R[2] * d0 + p.R[5] * d1 + p.R[8] * d2;
    g[0] = zc - p.z_min;
    g[1] = p.z_max - zc;
    g[2] = p.fx * xc + (p.cx + p.mu) * zc;
    g[3] = (p.umax - p.cx) * zc - p.fx * xc;
    g[4] = p.fy * yc + (p.cy + p.mv) * zc;
    g[5] = (p.vmax - p.cy) * zc - p.fy * yc;
  }
  bool inside = true, outside = false;
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    const unsigned in_c = __ballot_sync(0xffffffffu, g[c] >= tol) & 0xffu;
    const unsigned out_c = __ballot_sync(0xffffffffu, g[c] < -tol) & 0xffu;
    inside &= in_c == 0xffu;
    outside |= out_c == 0xffu;
  }
  return outside ? 0 : (inside ? 1 : 2);
}

// One warp per allocated block location: a location with any voxel in the widened frustum gets a
// combined slot (atomic counter); .w of comb_loc keeps the hash entry, cls (1 inside, 2
// straddling) goes to p.cls.  Locations that already hold a slot are skipped (an R58 update
// selects only the locations a fused frame added).
__global__ void __launch_bounds__(256) k_comb_select(const __grid_constant__ CombineLaunch p, unsigned char *cls_out) {
  const long long u = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (u >= p.n_loc) return;
  const int4 b = p.locations[u];
  if (p.slot_of_entry[b.w] >= 0) return;  // warp-uniform
  const int cls = classify_block(p, b.x, b.y, b.z, lane);
  if (cls == 0 || lane != 0) return;
  const int slot = (int)atomicAdd(p.n_sel, 1u);
  p.slot_of_entry[b.w] = slot;
  p.comb_loc[slot] = b;
  cls_out[slot] = (unsigned char)cls;
}

// R58: in a full combination every voxel is computed; in an update after a fused frame, a voxel of
// a slot that existed before the frame is recomputed only if it had no data before (had bit
// clear) and has data now (some direction's record with weight > 0); new slots are computed whole.
__device__ __forceinline__ bool first_time(const CombineLaunch &p, size_t slot, int l, const int sl[6]) {
  if (!p.had || (long long)slot >= p.n_old) return true;
  if ((__ldg(&p.had[slot * 16 + (l >> 5)]) >> (l & 31)) & 1u) return false;
  const int roff = (l & 7) + kRec * ((l >> 3) & 7) + kRec * kRec * (l >> 6);
  bool now = false;
#pragma unroll
  for (int D = 0; D < 6; ++D)
    if (sl[D] >= 0) now |= __ldg(&p.vol.brick_a[(size_t)sl[D] * kRecStride + roff].y) > 0.0f;
  return now;
}

// R34: one thread per voxel of a combined slot (4 CTAs of 128 per slot).  All loads of the
// present directions -- centre {sdf, weight}, the 6 neighbouring sdf values ("the
// gradient can be computed with just looking up the SDF values stored in the 6 neighboring
// voxels"; NaN where unallocated) and the colour -- are issued before any is used.
#ifndef DTSDF_COMB_MINB
#define DTSDF_COMB_MINB 16  // 32 registers, full occupancy: C1 combine 0.195 -> 0.165 ms (profiles/r2j_ab_combine.txt)
#endif
__global__ void __launch_bounds__(128, DTSDF_COMB_MINB) k_combine(const __grid_constant__ CombineLaunch p) {
  const VolumeView &V = p.vol;
  // the 4 CTAs of a slot are adjacent in launch order (blockIdx.x = 4 slot + quarter, so any
  // number of slots fits the grid's x extent): they share the slot's bricks in L2 while they run
  const size_t slot = blockIdx.x >> 2;
  const int l = (blockIdx.x & 3) * 128 + threadIdx.x;
  const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
  const int4 b = p.comb_loc[slot];
  DTSDF_CHECK(b.w >= 0 && (long long)b.w < V.table_cap);
  const int4 *e = reinterpret_cast<const int4 *>(&V.table[b.w]);
  const int4 ea = __ldg(e), eb = __ldg(e + 1);
  const int sl[6] = {ea.z, ea.w, eb.x, eb.y, eb.z, eb.w};
  if (!first_time(p, slot, l, sl)) return;  // R58 update: this voxel keeps its value
  const int i = kBlock * b.x + lx, j = kBlock * b.y + ly, k = kBlock * b.z + lz;
  double d[3];
  bool in = true;
  if (p.cls[slot] == 2) {
    in = in_frustum(p, (double)V.voxel_size, i, j, k, d);
  } else {
    const double s = (double)V.voxel_size;
    d[0] = __dsub_rn(__dmul_rn((double)i, s), p.t[0]);
    d[1] = __dsub_rn(__dmul_rn((double)j, s), p.t[1]);
    d[2] = __dsub_rn(__dmul_rn((double)k, s), p.t[2]);
  }
  const int off = CAPRON(lx, ly, lz), coff = lx + kRgbApron * ly + kRgbApron * kRgbApron * lz;
  const int roff = lx + kRec * ly + kRec * kRec * lz;  // the voxel's record in the directional bricks
  // r in fp32 from the fp64 offset (its rounding is far below the tolerance of the weights)
  const float dx = (float)d[0], dy = (float)d[1], dz = (float)d[2];
  const float dd = dx * dx + dy * dy + dz * dz;
  const float il = dd > 0.f ? rsqrtf(dd) : 0.f;
  const float rx = dx * il, ry = dy * il, rz = dz * il;
  const float half_inv_s = 0.5f * V.inv_voxel;
  float S1 = 0.f, F1 = 0.f, S2 = 0.f, F2 = 0.f;
  float C1[3] = {0.f, 0.f, 0.f}, C2[3] = {0.f, 0.f, 0.f};
  int m1 = 0, m2 = 0;
  bool any_grad = false;
  // present directions, two at a time: both directions' loads are in flight together
  unsigned present = 0;
#pragma unroll
  for (int D = 0; D < 6; ++D) present |= (unsigned)(sl[D] >= 0) << D;
  if (!in) present = 0;
#pragma unroll 1
  while (present) {
    int Dp[2];
    float4 ra[2];  // {sdf, weight, dsdf_x, dsdf_y}
    float2 rb[2];  // {dsdf_z, rgb}
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      Dp[h] = present ? __ffs(present) - 1 : -1;
      present &= present - 1;
      ra[h] = make_float4(0.f, 0.f, 0.f, 0.f);
      rb[h] = make_float2(0.f, 0.f);
      if (Dp[h] >= 0) {
        int slot_d = sl[0];
#pragma unroll
        for (int D = 1; D < 6; ++D) slot_d = Dp[h] == D ? sl[D] : slot_d;  // register select
        ra[h] = __ldg(V.brick_a + (size_t)slot_d * kRecStride + roff);
        rb[h] = __ldg(V.brick_b + (size_t)slot_d * kRecStride + roff);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int D = Dp[h];
      const float2 c = make_float2(ra[h].x, ra[h].y);
      if (D < 0 || !(c.y > 0.0f)) continue;  // D holds no data at the voxel (reading R8)
      // the gradient from the 6 neighbouring voxels (the record's central
      // differences, NaN where a neighbour is unallocated)
      const float gx = ra[h].z * half_inv_s;
      const float gy = ra[h].w * half_inv_s;
      const float gz = rb[h].x * half_inv_s;
      const float gn = sqrtf(gx * gx + gy * gy + gz * gz);
      const int axis = D >> 1;
      const float sign = (D & 1) ? -1.0f : 1.0f;
      const float r_axis = axis == 0 ? rx : (axis == 1 ? ry : rz);
      const unsigned int qq = rec_rgb(rb[h].y);
      const float cr = (float)(qq & 255u), cg = (float)((qq >> 8) & 255u), cb = (float)(qq >> 16);
      // eq:combine_tsdf_weight: omega <v^D, -r>^+
      const float W2 = c.y * fmaxf(-sign * r_axis, 0.0f);
      if (W2 > 0.0f) {
        S2 += W2;
        F2 = fmaf(W2, c.x, F2);
        C2[0] = fmaf(W2, cr, C2[0]); C2[1] = fmaf(W2, cg, C2[1]); C2[2] = fmaf(W2, cb, C2[2]);
        m2 |= 1 << D;
      }
      if (gn > 1e-3f) {  // reading R8 (NaN -> false)
        any_grad = true;
        const float ig = 1.0f / gn;
        const float nx = gx * ig, ny = gy * ig, nz = gz * ig;
        const float n_axis = axis == 0 ? nx : (axis == 1 ? ny : nz);
        const float nr = -(nx * rx + ny * ry + nz * rz);
        // eq:combine_weight: w_dir(<n,v>) <n,-r>^+ omega
        const float W1 = w_dir_c(sign * n_axis, V) * fmaxf(nr, 0.0f) * c.y;
        if (W1 > 0.0f) {
          S1 += W1;
          F1 = fmaf(W1, c.x, F1);
          C1[0] = fmaf(W1, cr, C1[0]); C1[1] = fmaf(W1, cg, C1[1]); C1[2] = fmaf(W1, cb, C1[2]);
          m1 |= 1 << D;
        }
      }
    }
  }
  const float S = any_grad ? S1 : S2;
  const bool valid = in && dd > 0.f && S > 0.0f;
  float sdf = CUDART_NAN_F;
  uchar4 col = make_uchar4(0, 0, 0, 0);
  if (valid) {
    const float *Cc = any_grad ? C1 : C2;
    sdf = (any_grad ? F1 : F2) / S;
    unsigned char cc[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) cc[a] = (unsigned char)fminf(fmaxf(floorf(Cc[a] / S + 0.5f), 0.f), 255.f);  // R35
    col = make_uchar4(cc[0], cc[1], cc[2], (unsigned char)(any_grad ? m1 : m2));
  }
  p.apron[slot * kApronStride + off] = sdf;
  p.rgb[slot * kRgbApronStride + coff] = col;
  p.weight[slot * kVoxPerBlock + l] = valid ? S : 0.f;
}


// ------------------------------------------------------------------------------------------
// NEXT-4: Algorithm 1 "Compute Combined TSDF", readings R53-R57 (oracle.c
// combine_voxel_alg1): per voxel, the directions taking part (valid gradient w.r.t. the
// direction, stored weight above the floor) split into free (phi > 0) and occupied; a free
// direction's free space stands unless its first zero transition towards the camera lies in the
// occupied space of another direction whose surface faces the camera; the result is the stored-
// weight average of the free directions if any free space stands, else of the occupied ones.
//
// Every quantity that feeds one of these discrete decisions -- participation, the first
// transition q, "Phi^D~(q) < 0" (taken as printed), "<n^D~(q), -r> > 0" -- is evaluated in
// fp64 with the oracle's operations in the oracle's order (explicit _rn intrinsics, so nvcc cannot
// contract them into FMAs; the oracle is compiled with -ffp-contract=off) on the same float voxel
// values.  A direction storing the same surface as D is ~0 at D's own root, so its sign there is
// decided by the last bit: both sides take that decision on identical bits.  (The acos of the
// membership test is the one libm call; a flip needs acos(c) within an ulp of theta.)
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ long long floordiv8_ll(long long i) { return i >= 0 ? i / 8 : -((-i + 7) / 8); }
__device__ __forceinline__ double m64(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double a64(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double s64(double a, double b) { return __dsub_rn(a, b); }

// record brick (A) of direction D at block location (b0, b1, b2), or null if unallocated
__device__ const float4 *dir_brick(const CombineLaunch &p, int D, long long b0, long long b1, long long b2) {
  const VolumeView &V = p.vol;
  int e = -1;
  if (V.loc_grid) {
    const long long x = b0 - V.lo_x, yy = b1 - V.lo_y, z = b2 - V.lo_z;
    if (x < 0 || yy < 0 || z < 0 || x >= V.dim_x || yy >= V.dim_y || z >= V.dim_z) return nullptr;
    const int gv = __ldg(&V.loc_grid[((size_t)z * V.dim_y + yy) * V.dim_x + x]);
    if (gv < 0) return nullptr;
    e = gv & kGridEntryMask;
  } else {
    if (b0 < -(1 << 20) || b0 >= (1 << 20) || b1 < -(1 << 20) || b1 >= (1 << 20) || b2 < -(1 << 20) || b2 >= (1 << 20))
      return nullptr;
    const unsigned long long key = pack_key((int)b0, (int)b1, (int)b2);
    unsigned int h = hash_key(key) & V.table_mask;
    for (unsigned int probe = 0; probe <= V.table_mask; ++probe) {
      const unsigned long long k = V.table[h].key;
      if (k == key) { e = (int)h; break; }
      if (k == kEmptyKey) return nullptr;
      h = (h + 1) & V.table_mask;
    }
    if (e < 0) return nullptr;
  }
  const int slot = V.table[e].slot[D];
  if (slot < 0) return nullptr;
  DTSDF_CHECK(slot < V.n_blocks);
  return V.brick_a + (size_t)slot * kRecStride;
}

// oracle record_of: the stored sdf of voxel (i, j, k) in direction D; false if its block is
// unallocated (the voxel's own record in its block's brick)
__device__ bool vox_sdf(const CombineLaunch &p, int D, long long i, long long j, long long k, double *v) {
  const long long b0 = floordiv8_ll(i), b1 = floordiv8_ll(j), b2 = floordiv8_ll(k);
  const float4 *br = dir_brick(p, D, b0, b1, b2);
  if (!br) return false;
  *v = (double)__ldg(&br[(i - 8 * b0) + kRec * (j - 8 * b1) + kRec * kRec * (k - 8 * b2)].x);
  return true;
}

// oracle cell_interp (phi only): plain trilinear over the 8 corners of cell c with fractions fr,
// corners in the oracle's order, wt = (x-factor * y-factor) * z-factor, p += wt * sdf; false
// unless every corner's block is allocated.  The base block's brick holds voxels 0..8, i.e. all 8
// corners, with NaN where a corner's block is unallocated.
__device__ bool cell_interp64(const CombineLaunch &p, int D, const long long c[3], const double fr[3], double *phi) {
  const long long b0 = floordiv8_ll(c[0]), b1 = floordiv8_ll(c[1]), b2 = floordiv8_ll(c[2]);
  const float4 *br = dir_brick(p, D, b0, b1, b2);
  if (!br) return false;
  br += (c[0] - 8 * b0) + kRec * (c[1] - 8 * b1) + kRec * kRec * (c[2] - 8 * b2);
  const double u0 = s64(1.0, fr[0]), u1 = s64(1.0, fr[1]), u2 = s64(1.0, fr[2]);
  double acc = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int dx = q & 1, dy = (q >> 1) & 1, dz = (q >> 2) & 1;
    const float v = __ldg(&br[dx + kRec * dy + kRec * kRec * dz].x);
    if (isnan(v)) return false;
    const double wt = m64(m64(dx ? fr[0] : u0, dy ? fr[1] : u1), dz ? fr[2] : u2);
    acc = a64(acc, m64(wt, (double)v));
  }
  *phi = acc;
  return true;
}

// oracle locate: g = x / s, c = floor(g), fr = g - floor(g)
__device__ __forceinline__ void locate64(double s, const double y[3], long long c[3], double fr[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double g = __ddiv_rn(y[a], s);
    const double fl = floor(g);
    c[a] = (long long)fl;
    fr[a] = s64(g, fl);
  }
}

// oracle dir_value: trilinear phi_D at y; false when D is absent there
__device__ bool dir_value(const CombineLaunch &p, int D, double s, const double y[3], double *f) {
  long long c[3];
  double fr[3];
  locate64(s, y, c, fr);
  return cell_interp64(p, D, c, fr, f);
}

// oracle dir_normal: central differences of the trilinear field at +-s (cells shifted by one
// voxel, same fractions, R7); false if the stencil is incomplete or |g| <= 1e-3
__device__ bool dir_normal(const CombineLaunch &p, int D, double s, const double y[3], double n[3]) {
  long long c[3];
  double fr[3], g[3];
  locate64(s, y, c, fr);
  for (int a = 0; a < 3; ++a) {
    long long cp[3] = {c[0], c[1], c[2]}, cm[3] = {c[0], c[1], c[2]};
    cp[a] += 1;
    cm[a] -= 1;
    double pp, pm;
    if (!cell_interp64(p, D, cp, fr, &pp) || !cell_interp64(p, D, cm, fr, &pm)) return false;
    g[a] = __ddiv_rn(s64(pp, pm), m64(2.0, s));
  }
  const double gn = __dsqrt_rn(a64(a64(m64(g[0], g[0]), m64(g[1], g[1])), m64(g[2], g[2])));
  if (!(gn > 1e-3)) return false;
#pragma unroll
  for (int a = 0; a < 3; ++a) n[a] = __ddiv_rn(g[a], gn);
  return true;
}

// y = x - t r per component (the oracle's back-march / bisection / q positions)
__device__ __forceinline__ void back_point(const double x[3], double t, const double r[3], double y[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) y[a] = s64(x[a], m64(t, r[a]));
}

__global__ void __launch_bounds__(128) k_combine_alg1(const __grid_constant__ CombineLaunch p) {
  const VolumeView &V = p.vol;
  const size_t slot = blockIdx.x >> 2;  // as k_combine: 4 adjacent CTAs per slot on grid x
  const int l = (blockIdx.x & 3) * 128 + threadIdx.x;
  const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
  const int4 b = p.comb_loc[slot];
  const int4 *ent = reinterpret_cast<const int4 *>(&V.table[b.w]);
  const int4 ea = __ldg(ent), eb = __ldg(ent + 1);
  const int sl[6] = {ea.z, ea.w, eb.x, eb.y, eb.z, eb.w};
  if (!first_time(p, slot, l, sl)) return;  // R58 update: this voxel keeps its value
  const int i = kBlock * b.x + lx, j = kBlock * b.y + ly, k = kBlock * b.z + lz;
  const double s = (double)V.voxel_size;
  double d[3];
  bool in = true;
  if (p.cls[slot] == 2) {
    in = in_frustum(p, s, i, j, k, d);
  } else {
    d[0] = s64(m64((double)i, s), p.t[0]);
    d[1] = s64(m64((double)j, s), p.t[1]);
    d[2] = s64(m64((double)k, s), p.t[2]);
  }
  const double dist = __dsqrt_rn(a64(a64(m64(d[0], d[0]), m64(d[1], d[1])), m64(d[2], d[2])));
  const double x[3] = {m64((double)i, s), m64((double)j, s), m64((double)k, s)};
  const double r[3] = {__ddiv_rn(d[0], dist), __ddiv_rn(d[1], dist), __ddiv_rn(d[2], dist)};
  const int off = CAPRON(lx, ly, lz), coff = lx + kRgbApron * ly + kRgbApron * kRgbApron * lz;
  const int roff = lx + kRec * ly + kRec * kRec * lz;
  const long long vi[3] = {i, j, k};
  float phi[6], om[6];
  unsigned part = 0, free_m = 0;
  if (in && dist > 0.0) {
    for (int D = 0; D < 6; ++D) {
      if (sl[D] < 0) continue;
      const float4 c = __ldg(V.brick_a + (size_t)sl[D] * kRecStride + roff);
      phi[D] = c.x;
      om[D] = c.y;
      if (!(c.y > p.w_floor)) continue;  // R53
      // the voxel's 6-neighbour gradient from the stored values, as the oracle
      double g[3];
      bool ok = true;
      for (int a = 0; a < 3 && ok; ++a) {
        long long pp[3] = {vi[0], vi[1], vi[2]}, mm[3] = {vi[0], vi[1], vi[2]};
        pp[a] += 1;
        mm[a] -= 1;
        double vp, vm;
        if (!vox_sdf(p, D, pp[0], pp[1], pp[2], &vp) || !vox_sdf(p, D, mm[0], mm[1], mm[2], &vm)) { ok = false; break; }
        g[a] = __ddiv_rn(s64(vp, vm), m64(2.0, s));
      }
      if (!ok) continue;
      const double gn = __dsqrt_rn(a64(a64(m64(g[0], g[0]), m64(g[1], g[1])), m64(g[2], g[2])));
      if (!(gn > 1e-3)) continue;
      // <n, v^D> = +-g_axis / gn (the other products with v^D are exact zeros)
      const double nv = __ddiv_rn((D & 1) ? -g[D >> 1] : g[D >> 1], gn);
      const double cc = nv < -1.0 ? -1.0 : (nv > 1.0 ? 1.0 : nv);
      const double w = __ddiv_rn(s64(p.theta64, acos(cc)), s64(m64(2.0, p.theta64), 1.5707963267948966));
      if (!(w > 0.0)) continue;  // w_dir > 0 (eq:direction_weight, R1)
      part |= 1u << D;
      if (c.x > 0.0f) free_m |= 1u << D;
    }
  }
  // R55-R56: does any free direction's free space stand?
  bool freespace = false;
  const long long K = (long long)floor(__ddiv_rn(dist, s));
  for (int D = 0; D < 6 && !freespace; ++D) {
    if (!((free_m >> D) & 1u)) continue;
    double prev_t = 0.0, qt = -1.0;
    for (long long kk = 1; kk <= K; ++kk) {
      const double t = m64((double)kk, s);
      double y[3], f;
      back_point(x, t, r, y);
      if (!dir_value(p, D, s, y, &f)) break;  // D absent: no transition observed
      if (f <= 0.0) {
        double a = prev_t, bb = t;
        for (int it = 0; it < 50; ++it) {
          const double m = m64(0.5, a64(a, bb));
          if (!(m > a && m < bb)) break;
          double ym[3], fm;
          back_point(x, m, r, ym);
          if (!dir_value(p, D, s, ym, &fm) || fm > 0.0) a = m; else bb = m;
        }
        qt = m64(0.5, a64(a, bb));
        break;
      }
      prev_t = t;
    }
    if (qt < 0.0) { freespace = true; break; }
    double q[3];
    back_point(x, qt, r, q);
    bool conflict = false;
    for (int E = 0; E < 6 && !conflict; ++E) {
      if (E == D) continue;
      double fe;
      if (!dir_value(p, E, s, q, &fe) || !(fe < 0.0)) continue;  // "Phi^D~(q) < 0" (R56)
      double ne[3];
      if (!dir_normal(p, E, s, q, ne)) continue;
      if (-a64(a64(m64(ne[0], r[0]), m64(ne[1], r[1])), m64(ne[2], r[2])) > 0.0) conflict = true;
    }
    if (!conflict) freespace = true;
  }
  // R57: stored-weight average of the chosen set in fp64, as the oracle: stored weights are float32
  // and colours integers, so an average that is exactly k + 1/2 (equal weights, e.g. a plate's
  // front and back directions) rounds as in the oracle.
  const unsigned use = freespace ? free_m : (part & ~free_m);
  double S = 0.0, F = 0.0, C[3] = {0.0, 0.0, 0.0};
  for (int D = 0; D < 6; ++D) {
    if (!((use >> D) & 1u)) continue;
    const unsigned int qc = rec_rgb(__ldg(&V.brick_b[(size_t)sl[D] * kRecStride + roff].y));
    S = a64(S, (double)om[D]);
    F = a64(F, m64((double)om[D], (double)phi[D]));
    C[0] = a64(C[0], m64((double)om[D], (double)(qc & 255u)));
    C[1] = a64(C[1], m64((double)om[D], (double)((qc >> 8) & 255u)));
    C[2] = a64(C[2], m64((double)om[D], (double)(qc >> 16)));
  }
  float sdf = CUDART_NAN_F;
  uchar4 col = make_uchar4(0, 0, 0, 0);
  const bool valid = use != 0 && S > 0.0;
  if (valid) {
    sdf = (float)__ddiv_rn(F, S);
    unsigned char cc[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) cc[a] = (unsigned char)fmin(fmax(floor(a64(__ddiv_rn(C[a], S), 0.5)), 0.0), 255.0);
    col = make_uchar4(cc[0], cc[1], cc[2], (unsigned char)use);
  }
  p.apron[slot * kApronStride + off] = sdf;
  p.rgb[slot * kRgbApronStride + coff] = col;
  p.weight[slot * kVoxPerBlock + l] = valid ? (float)S : 0.f;
}

// combined slot of block location (bx,by,bz), or -1
__device__ __forceinline__ int comb_slot_of(const CombineLaunch &p, int bx, int by, int bz) {
  const VolumeView &V = p.vol;
  int e = -1;
  if (V.loc_grid) {
    const unsigned x = (unsigned)(bx - V.lo_x), y = (unsigned)(by - V.lo_y), z = (unsigned)(bz - V.lo_z);
    if (x >= (unsigned)V.dim_x || y >= (unsigned)V.dim_y || z >= (unsigned)V.dim_z) return -1;
    const int gv = __ldg(&V.loc_grid[((size_t)z * V.dim_y + y) * V.dim_x + x]);
    if (gv < 0) return -1;
    e = gv & kGridEntryMask;
  } else {
    const unsigned long long key = pack_key(bx, by, bz);
    unsigned int h = hash_key(key) & V.table_mask;
    for (unsigned int probe = 0; probe <= V.table_mask; ++probe) {
      const unsigned long long k = V.table[h].key;
      if (k == key) { e = (int)h; break; }
      if (k == kEmptyKey) return -1;
      h = (h + 1) & V.table_mask;
    }
    if (e < 0) return -1;
  }
  return p.slot_of_entry[e];
}

constexpr int kFinishThreads = 256;
constexpr int kApronBorder = kApronVox - kVoxPerBlock;                          // 819: voxels -1, 8, 9
constexpr int kRgbFar = kRgbApronVox - kVoxPerBlock;                            // 217: voxels 8
constexpr int kBorderPer = (kApronBorder + kFinishThreads - 1) / kFinishThreads;  // 4

// The border of a combined brick, built at compile time (no index arithmetic in the kernel): for
// each border voxel of the sdf apron its apron index, and the neighbour (0..26) and that
// neighbour's apron index it is copied from; likewise for the colour brick's far faces.
struct FinishTable {
  unsigned short dst[kApronBorder];
  unsigned int src[kApronBorder];   // nbi << 16 | source apron index
  unsigned short rgb_dst[kRgbFar];
  unsigned int rgb_src[kRgbFar];    // nbi << 16 | source colour index
  constexpr FinishTable() : dst(), src(), rgb_dst(), rgb_src() {
    int n = 0;
    for (int a = 0; a < kApronVox; ++a) {
      const int lx = a % kApron - 1, ly = (a / kApron) % kApron - 1, lz = a / (kApron * kApron) - 1;
      const int ox = lx < 0 ? -1 : (lx >= kBlock ? 1 : 0), oy = ly < 0 ? -1 : (ly >= kBlock ? 1 : 0),
                oz = lz < 0 ? -1 : (lz >= kBlock ? 1 : 0);
      if (!(ox | oy | oz)) continue;
      dst[n] = (unsigned short)a;
      src[n] = ((unsigned)((ox + 1) + 3 * (oy + 1) + 9 * (oz + 1)) << 16) |
               (unsigned)(((lx - ox * kBlock) + 1) + kApron * ((ly - oy * kBlock) + 1) +
                          kApron * kApron * ((lz - oz * kBlock) + 1));
      ++n;
    }
    n = 0;
    for (int a = 0; a < kRgbApronVox; ++a) {
      const int lx = a % kRgbApron, ly = (a / kRgbApron) % kRgbApron, lz = a / (kRgbApron * kRgbApron);
      const int ox = lx >= kBlock, oy = ly >= kBlock, oz = lz >= kBlock;
      if (!(ox | oy | oz)) continue;
      rgb_dst[n] = (unsigned short)a;
      rgb_src[n] = ((unsigned)((ox + 1) + 3 * (oy + 1) + 9 * (oz + 1)) << 16) |
                   (unsigned)((lx - ox * kBlock) + kRgbApron * (ly - oy * kBlock) + kRgbApron * kRgbApron * (lz - oz * kBlock));
      ++n;
    }
  }
};
__device__ const FinishTable kFin = FinishTable();

// One CTA per combined slot: resolve the 26 neighbouring combined slots once, gather the apron
// border (voxels -1, 8, 9 per axis) and the colour brick's far faces from the neighbours'
// interiors (k_combine wrote them) with all loads in flight together and write them -- only
// border positions are written and only interiors read, so the slots' CTAs never race -- then the
// exact skip masks of the 512 base cells from the brick assembled in shared memory (bit set: no
// valid corner with sdf <= 0, R36) and the brick's surface flag.
__global__ void __launch_bounds__(kFinishThreads) k_comb_finish(const __grid_constant__ CombineLaunch p) {
  __shared__ float s_c[kApronStride];
  __shared__ int s_nb[27];
  const size_t slot = blockIdx.x;
  const int tid = threadIdx.x;
  const int4 b = p.comb_loc[slot];
  if (tid < 27) {
    const int ox = tid % 3 - 1, oy = (tid / 3) % 3 - 1, oz = tid / 9 - 1;
    s_nb[tid] = (ox | oy | oz) ? comb_slot_of(p, b.x + ox, b.y + oy, b.z + oz) : (int)slot;
  }
  __syncthreads();
  const float *__restrict__ apin = p.apron;
  float *ap = p.apron + slot * kApronStride;
  float vi[2];  // own interior
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int l = tid + h * kFinishThreads;
    vi[h] = __ldg(apin + slot * kApronStride + CAPRON(l & 7, (l >> 3) & 7, l >> 6));
  }
  float v[kBorderPer];
  int dst[kBorderPer];
#pragma unroll
  for (int k = 0; k < kBorderPer; ++k) {
    const int e = tid + k * kFinishThreads;
    v[k] = CUDART_NAN_F;
    dst[k] = -1;
    if (e < kApronBorder) {
      const unsigned int sr = __ldg(&kFin.src[e]);
      dst[k] = __ldg(&kFin.dst[e]);
      const int ns = s_nb[sr >> 16];
      DTSDF_CHECK(ns < (int)gridDim.x && (sr >> 16) < 27 && (sr & 0xffffu) < kApronVox && dst[k] < kApronVox);
      if (ns >= 0) v[k] = __ldg(apin + (size_t)ns * kApronStride + (sr & 0xffffu));
    }
  }
  uchar4 cv = make_uchar4(0, 0, 0, 0);
  int rdst = -1;
  if (tid < kRgbFar) {
    const unsigned int sr = __ldg(&kFin.rgb_src[tid]);
    rdst = __ldg(&kFin.rgb_dst[tid]);
    const int ns = s_nb[sr >> 16];
    DTSDF_CHECK(ns < (int)gridDim.x && (sr >> 16) < 27 && (sr & 0xffffu) < kRgbApronVox && rdst < kRgbApronVox);
    if (ns >= 0) cv = __ldg(p.rgb + (size_t)ns * kRgbApronStride + (sr & 0xffffu));
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int l = tid + h * kFinishThreads;
    s_c[CAPRON(l & 7, (l >> 3) & 7, l >> 6)] = vi[h];
  }
#pragma unroll
  for (int k = 0; k < kBorderPer; ++k) {
    if (dst[k] >= 0) {
      s_c[dst[k]] = v[k];
      ap[dst[k]] = v[k];
    }
  }
  if (rdst >= 0) p.rgb[slot * kRgbApronStride + rdst] = cv;
  __syncthreads();
  int any_neg = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int l = tid + h * kFinishThreads;
    const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
    const float *c = s_c + CAPRON(lx, ly, lz);
    bool pos = true;
#pragma unroll
    for (int q = 0; q < 8; ++q) pos &= !(c[(q & 1) + kApron * ((q >> 1) & 1) + kApron * kApron * (q >> 2)] <= 0.0f);
    const unsigned int word = __ballot_sync(0xffffffffu, pos);
    if ((l & 31) == 0) p.cell_pos[slot * 16 + (l >> 5)] = word;
    any_neg |= !pos;
  }
  any_neg = __syncthreads_or(any_neg);
  if (tid == 0) p.surf[slot] = (unsigned char)any_neg;
}

// After a re-commit (e.g. a fused frame) the hash entries move: re-point the kept combined slots
// (stale by design until the next recombination) at their locations' new entries.
__global__ void k_comb_remap(const HashEntry *__restrict__ table, unsigned int mask, int4 *comb_loc, long long n,
                             int *slot_of_entry) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int4 b = comb_loc[i];
  const unsigned long long key = pack_key(b.x, b.y, b.z);
  unsigned int h = hash_key(key) & mask;
  for (unsigned int probe = 0; probe <= mask; ++probe) {
    const unsigned long long k = table[h].key;
    if (k == key) {
      b.w = (int)h;
      comb_loc[i] = b;
      slot_of_entry[h] = (int)i;
      return;
    }
    if (k == kEmptyKey) break;
    h = (h + 1) & mask;
  }
  b.w = -1;  // the location left the volume: the slot is kept but unreachable
  comb_loc[i] = b;
}

cudaError_t launch_comb_remap(const HashEntry *table, unsigned int mask, int4 *comb_loc, long long n,
                              int *slot_of_entry, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_comb_remap<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(table, mask, comb_loc, n, slot_of_entry);
  return cudaGetLastError();
}

// R58: one thread per voxel of a combined slot: did any direction hold data there (pool weight > 0)?
__global__ void k_comb_had(const HashEntry *__restrict__ table, const int4 *__restrict__ comb_loc, long long n,
                           const float *__restrict__ w, unsigned int *had) {
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long slot = g >> 9;
  const int l = (int)(g & 511);
  bool h = false;
  if (slot < n) {
    const int e = comb_loc[slot].w;
    if (e < 0) {
      h = true;  // the location left the volume: nothing to add
    } else {
#pragma unroll
      for (int D = 0; D < 6; ++D) {
        const int b = table[e].slot[D];
        if (b >= 0) h |= w[(size_t)b * kVoxPerBlock + l] > 0.0f;
      }
    }
  }
  const unsigned int word = __ballot_sync(0xffffffffu, h);
  if (slot < n && (l & 31) == 0) had[slot * 16 + (l >> 5)] = word;
}

cudaError_t launch_comb_had(const HashEntry *table, const int4 *comb_loc, long long n, const float *pool_weight,
                            unsigned int *had, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_comb_had<<<(unsigned)((n * 512 + 255) / 256), 256, 0, s>>>(table, comb_loc, n, pool_weight, had);
  return cudaGetLastError();
}

cudaError_t launch_combine(const CombineLaunch &p, cudaStream_t s) {
  if (p.n_loc == 0) return cudaSuccess;
  k_comb_select<<<(unsigned)((p.n_loc * 32 + 255) / 256), 256, 0, s>>>(p, p.cls);
  return cudaGetLastError();
}

cudaError_t launch_combine_finish(const CombineLaunch &p, long long n_sel, cudaStream_t s) {
  if (n_sel == 0) return cudaSuccess;
  // one grid row of 4 CTAs per slot would cap n_sel at gridDim.y's 65535: the slots go on x
  const unsigned grid = (unsigned)(4 * n_sel);
  if (p.mode == 1)
    k_combine_alg1<<<grid, 128, 0, s>>>(p);
  else
    k_combine<<<grid, 128, 0, s>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_comb_finish<<<(unsigned)n_sel, kFinishThreads, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace dtsdf
