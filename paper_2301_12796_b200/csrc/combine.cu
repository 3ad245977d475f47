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
// straddling) rides in bit 30 of slot_of_entry's companion array comb_cls.
__global__ void __launch_bounds__(256) k_comb_select(const __grid_constant__ CombineLaunch p, unsigned char *cls_out) {
  const long long u = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (u >= p.n_loc) return;
  const int4 b = p.locations[u];
  const int cls = classify_block(p, b.x, b.y, b.z, lane);
  if (cls == 0 || lane != 0) return;
  const int slot = (int)atomicAdd(p.n_sel, 1u);
  p.slot_of_entry[b.w] = slot;
  p.comb_loc[slot] = b;
  cls_out[slot] = (unsigned char)cls;
}

// R34: one thread per voxel of a combined slot (4 CTAs of 128 per slot).  All loads of the
// present directions -- centre {sdf, weight}, the 6 neighbouring sdf values ("the
// gradient can be computed with just looking up the SDF values stored in the 6 neighboring
// voxels"; NaN where unallocated) and the colour -- are issued before any is used.
__global__ void __launch_bounds__(128) k_combine(const __grid_constant__ CombineLaunch p,
                                                 const unsigned char *__restrict__ cls_in) {
  const VolumeView &V = p.vol;
  const size_t slot = blockIdx.x;
  const int l = blockIdx.y * 128 + threadIdx.x;
  const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
  const int4 b = p.comb_loc[slot];
  const int4 *e = reinterpret_cast<const int4 *>(&V.table[b.w]);
  const int4 ea = __ldg(e), eb = __ldg(e + 1);
  const int sl[6] = {ea.z, ea.w, eb.x, eb.y, eb.z, eb.w};
  const int i = kBlock * b.x + lx, j = kBlock * b.y + ly, k = kBlock * b.z + lz;
  double d[3];
  bool in = true;
  if (cls_in[slot] == 2) {
    in = in_frustum(p, (double)V.voxel_size, i, j, k, d);
  } else {
    const double s = (double)V.voxel_size;
    d[0] = __dsub_rn(__dmul_rn((double)i, s), p.t[0]);
    d[1] = __dsub_rn(__dmul_rn((double)j, s), p.t[1]);
    d[2] = __dsub_rn(__dmul_rn((double)k, s), p.t[2]);
  }
  const int off = CAPRON(lx, ly, lz), coff = lx + kRgbApron * ly + kRgbApron * kRgbApron * lz;
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
    float2 c[2];
    float nb[2][6];
    uchar4 q[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      Dp[h] = present ? __ffs(present) - 1 : -1;
      present &= present - 1;
      c[h] = make_float2(0.f, 0.f);
      q[h] = make_uchar4(0, 0, 0, 0);
#pragma unroll
      for (int a = 0; a < 6; ++a) nb[h][a] = 0.f;
      if (Dp[h] >= 0) {
        int slot_d = sl[0];
#pragma unroll
        for (int D = 1; D < 6; ++D) slot_d = Dp[h] == D ? sl[D] : slot_d;  // register select
        const float2 *br = V.apron + (size_t)slot_d * kApronStride + off;
        c[h] = __ldg(br);
        nb[h][0] = __ldg(&br[1].x);
        nb[h][1] = __ldg(&br[-1].x);
        nb[h][2] = __ldg(&br[kApron].x);
        nb[h][3] = __ldg(&br[-kApron].x);
        nb[h][4] = __ldg(&br[kApron * kApron].x);
        nb[h][5] = __ldg(&br[-kApron * kApron].x);
        q[h] = __ldg(V.rgb_apron + (size_t)slot_d * kRgbApronStride + coff);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int D = Dp[h];
      if (D < 0 || !(c[h].y > 0.0f)) continue;  // D holds no data at the voxel (reading R8)
      // the gradient from the 6 neighbouring voxels (NaN where unallocated)
      const float gx = (nb[h][0] - nb[h][1]) * half_inv_s;
      const float gy = (nb[h][2] - nb[h][3]) * half_inv_s;
      const float gz = (nb[h][4] - nb[h][5]) * half_inv_s;
      const float gn = sqrtf(gx * gx + gy * gy + gz * gz);
      const int axis = D >> 1;
      const float sign = (D & 1) ? -1.0f : 1.0f;
      const float r_axis = axis == 0 ? rx : (axis == 1 ? ry : rz);
      const float cr = (float)q[h].x, cg = (float)q[h].y, cb = (float)q[h].z;
      // eq:combine_tsdf_weight: omega <v^D, -r>^+
      const float W2 = c[h].y * fmaxf(-sign * r_axis, 0.0f);
      if (W2 > 0.0f) {
        S2 += W2;
        F2 = fmaf(W2, c[h].x, F2);
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
        const float W1 = w_dir_c(sign * n_axis, V) * fmaxf(nr, 0.0f) * c[h].y;
        if (W1 > 0.0f) {
          S1 += W1;
          F1 = fmaf(W1, c[h].x, F1);
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

// combined slot of block location (bx,by,bz), or -1
__device__ __forceinline__ int comb_slot_of(const CombineLaunch &p, int bx, int by, int bz) {
  const VolumeView &V = p.vol;
  int e = -1;
  if (V.loc_grid) {
    const unsigned x = (unsigned)(bx - V.lo_x), y = (unsigned)(by - V.lo_y), z = (unsigned)(bz - V.lo_z);
    if (x >= (unsigned)V.dim_x || y >= (unsigned)V.dim_y || z >= (unsigned)V.dim_z) return -1;
    const int gv = __ldg(&V.loc_grid[((size_t)z * V.dim_y + y) * V.dim_x + x]);
    if (gv < 0) return -1;
    e = gv & 0x3fffffff;
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

// apron cell a (< kApronVox) -> (neighbour index 0..26, that neighbour's apron index)
__device__ __forceinline__ void apron_src(int a, int *nbi, int *src) {
  const int lx = a % kApron - 1, ly = (a / kApron) % kApron - 1, lz = a / (kApron * kApron) - 1;
  const int ox = lx < 0 ? -1 : (lx >= kBlock ? 1 : 0), oy = ly < 0 ? -1 : (ly >= kBlock ? 1 : 0),
            oz = lz < 0 ? -1 : (lz >= kBlock ? 1 : 0);
  *nbi = (ox + 1) + 3 * (oy + 1) + 9 * (oz + 1);
  *src = CAPRON(lx - ox * kBlock, ly - oy * kBlock, lz - oz * kBlock);
}

constexpr int kFinishThreads = 256;
constexpr int kApronPer = (kApronStride + kFinishThreads - 1) / kFinishThreads;      // 6
constexpr int kRgbPer = (kRgbApronStride + kFinishThreads - 1) / kFinishThreads;     // 3

// One CTA per combined slot: resolve the 26 neighbouring combined slots once, gather the apron
// border (voxels -1, 8, 9 per axis) and the colour brick's far faces from them with all loads in
// flight together, assemble the brick in shared memory, then write the exact skip masks of the
// 512 base cells (bit set: no valid corner with sdf <= 0, R36) and the brick's surface flag.
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
  float v[kApronPer];
#pragma unroll
  for (int k = 0; k < kApronPer; ++k) {
    const int a = tid + k * kFinishThreads;
    v[k] = CUDART_NAN_F;
    if (a < kApronVox) {
      int nbi, src;
      apron_src(a, &nbi, &src);
      const int ns = s_nb[nbi];
      if (ns >= 0) v[k] = __ldg(apin + (size_t)ns * kApronStride + src);
    }
  }
  uchar4 cv[kRgbPer];
#pragma unroll
  for (int k = 0; k < kRgbPer; ++k) {
    const int a = tid + k * kFinishThreads;
    cv[k] = make_uchar4(0, 0, 0, 0);
    if (a < kRgbApronVox) {
      const int lx = a % kRgbApron, ly = (a / kRgbApron) % kRgbApron, lz = a / (kRgbApron * kRgbApron);
      const int ox = lx >= kBlock, oy = ly >= kBlock, oz = lz >= kBlock;
      const int ns = s_nb[(ox + 1) + 3 * (oy + 1) + 9 * (oz + 1)];
      if (ns >= 0)
        cv[k] = __ldg(p.rgb + (size_t)ns * kRgbApronStride + (lx - ox * kBlock) + kRgbApron * (ly - oy * kBlock) +
                      kRgbApron * kRgbApron * (lz - oz * kBlock));
    }
  }
  __syncthreads();  // every read of this slot's interior (by this CTA) is done before any write
  float *ap = p.apron + slot * kApronStride;
#pragma unroll
  for (int k = 0; k < kApronPer; ++k) {
    const int a = tid + k * kFinishThreads;
    if (a < kApronStride) {
      s_c[a] = v[k];
      ap[a] = v[k];
    }
  }
  uchar4 *cp = p.rgb + slot * kRgbApronStride;
#pragma unroll
  for (int k = 0; k < kRgbPer; ++k) {
    const int a = tid + k * kFinishThreads;
    if (a < kRgbApronStride) cp[a] = cv[k];
  }
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

cudaError_t launch_combine(const CombineLaunch &p, cudaStream_t s) {
  if (p.n_loc == 0) return cudaSuccess;
  k_comb_select<<<(unsigned)((p.n_loc * 32 + 255) / 256), 256, 0, s>>>(p, p.surf);
  return cudaGetLastError();
}

cudaError_t launch_combine_finish(const CombineLaunch &p, long long n_sel, cudaStream_t s) {
  if (n_sel == 0) return cudaSuccess;
  k_combine<<<dim3((unsigned)n_sel, 4), 128, 0, s>>>(p, p.surf);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_comb_finish<<<(unsigned)n_sel, kFinishThreads, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace dtsdf
