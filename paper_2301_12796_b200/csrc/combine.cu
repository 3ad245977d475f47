// combine.cu -- the view-dependent combined TSDF.
//
// Lemma 1: for a fixed camera the six directional fields combine into one
// conflict-free regular TSDF.  PAPER.md:251-263 computes it "for every voxel in the view
// frustum" (widened by 1/8 of the image on every side) with the combination weights
// eq:combine_weight / eq:combine_tsdf_weight, and P:610 notes that at integer voxel positions no
// trilinear interpolation is needed and the gradient comes from the 6 neighbouring voxels.
//
//   k_combine        one CTA per allocated block location, 2 voxels per thread: frustum test
//                    (fp64, reading R33), per-direction weights from the directional apron brick
//                    (centre + 6 neighbours, NaN = unallocated), combined sdf / weight / u8 colour /
//                    direction mask (R34-R35); a location with at least one valid voxel takes a
//                    combined slot (atomic counter) and writes its brick interior
//   k_comb_border    fills each combined brick's apron border (voxels -1 and 8..9 per axis) and
//                    the colour brick's far faces from the neighbouring combined bricks
//   k_comb_cellpos   per base cell: certainly positive or invalid (no valid corner <= 0), the
//                    exact skip masks of the raycast, and the per-brick surface flag
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

// R34: combined value of the voxel (i,j,k) = block-local (lx,ly,lz) of a location with slots[6]
__device__ __forceinline__ CombVox combine_voxel(const CombineLaunch &p, const int slots[6], int i, int j, int k,
                                                 int lx, int ly, int lz) {
  const VolumeView &V = p.vol;
  CombVox out;
  out.sdf = CUDART_NAN_F;
  out.S = 0.f;
  out.c = make_uchar4(0, 0, 0, 0);
  double d[3];
  if (!in_frustum(p, (double)V.voxel_size, i, j, k, d)) return out;
  const double dl = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  if (!(dl > 0.0)) return out;
  const float rx = (float)(d[0] / dl), ry = (float)(d[1] / dl), rz = (float)(d[2] / dl);
  const float half_inv_s = 0.5f * V.inv_voxel;
  const int off = lx + kApron * ly + kApron * kApron * lz;
  float S1 = 0.f, F1 = 0.f, S2 = 0.f, F2 = 0.f;
  float C1[3] = {0.f, 0.f, 0.f}, C2[3] = {0.f, 0.f, 0.f};
  int m1 = 0, m2 = 0;
  bool any_grad = false;
#pragma unroll 1
  for (int D = 0; D < 6; ++D) {
    const int slot = slots[D];
    if (slot < 0) continue;
    const float2 *br = V.apron + (size_t)slot * kApronStride + off;
    const float2 c = __ldg(br + CAPRON(0, 0, 0));
    if (!(c.y > 0.0f)) continue;  // D holds no data at the voxel (reading R8)
    // the gradient from the 6 neighbouring voxels (NaN where unallocated)
    const float gx = (__ldg(&br[CAPRON(1, 0, 0)].x) - __ldg(&br[CAPRON(-1, 0, 0)].x)) * half_inv_s;
    const float gy = (__ldg(&br[CAPRON(0, 1, 0)].x) - __ldg(&br[CAPRON(0, -1, 0)].x)) * half_inv_s;
    const float gz = (__ldg(&br[CAPRON(0, 0, 1)].x) - __ldg(&br[CAPRON(0, 0, -1)].x)) * half_inv_s;
    const float gn = sqrtf(gx * gx + gy * gy + gz * gz);
    const int axis = D >> 1;
    const float sign = (D & 1) ? -1.0f : 1.0f;
    const float r_axis = axis == 0 ? rx : (axis == 1 ? ry : rz);
    const uchar4 q = __ldg(V.rgb_apron + (size_t)slot * kRgbApronStride + (lx + kRgbApron * ly + kRgbApron * kRgbApron * lz));
    const float cr = (float)q.x, cg = (float)q.y, cb = (float)q.z;
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
  const float S = any_grad ? S1 : S2;
  if (!(S > 0.0f)) return out;
  const float F = any_grad ? F1 : F2;
  const float *Cc = any_grad ? C1 : C2;
  out.S = S;
  out.sdf = F / S;
  unsigned char col[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) col[a] = (unsigned char)fminf(fmaxf(floorf(Cc[a] / S + 0.5f), 0.f), 255.f);  // R35
  out.c = make_uchar4(col[0], col[1], col[2], (unsigned char)(any_grad ? m1 : m2));
  return out;
}

__global__ void __launch_bounds__(256) k_combine(const __grid_constant__ CombineLaunch p) {
  const int4 b = p.locations[blockIdx.x];
  __shared__ int slots[6];
  __shared__ int s_slot;
  if (threadIdx.x < 6) slots[threadIdx.x] = p.vol.table[b.w].slot[threadIdx.x];
  __syncthreads();
  int sl[6];
#pragma unroll
  for (int D = 0; D < 6; ++D) sl[D] = slots[D];
  CombVox v[2];
  bool any = false;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int l = threadIdx.x + 256 * h;
    const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
    v[h] = combine_voxel(p, sl, kBlock * b.x + lx, kBlock * b.y + ly, kBlock * b.z + lz, lx, ly, lz);
    any |= v[h].S > 0.f;
  }
  if (!__syncthreads_or(any)) return;  // no valid voxel: the location stays uncombined
  if (threadIdx.x == 0) {
    s_slot = (int)atomicAdd(p.n_sel, 1u);
    p.slot_of_entry[b.w] = s_slot;
    p.comb_loc[s_slot] = b;
  }
  __syncthreads();
  const size_t slot = (size_t)s_slot;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int l = threadIdx.x + 256 * h;
    const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
    p.apron[slot * kApronStride + CAPRON(lx, ly, lz)] = v[h].sdf;
    p.rgb[slot * kRgbApronStride + lx + kRgbApron * ly + kRgbApron * kRgbApron * lz] = v[h].c;
    p.weight[slot * kVoxPerBlock + l] = v[h].S;
  }
}

// combined slot of block location (bx,by,bz), or -1
__device__ __forceinline__ int comb_slot_of(const CombineLaunch &p, int bx, int by, int bz) {
  const VolumeView &V = p.vol;
  int e = -1;
  if (V.loc_grid) {
    const unsigned x = (unsigned)(bx - V.lo_x), y = (unsigned)(by - V.lo_y), z = (unsigned)(bz - V.lo_z);
    if (x >= (unsigned)V.dim_x || y >= (unsigned)V.dim_y || z >= (unsigned)V.dim_z) return -1;
    const int gv = V.loc_grid[((size_t)z * V.dim_y + y) * V.dim_x + x];
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

__global__ void __launch_bounds__(256) k_comb_border(const __grid_constant__ CombineLaunch p) {
  const size_t slot = blockIdx.x;
  const int4 b = p.comb_loc[slot];
  float *ap = p.apron + slot * kApronStride;
  for (int a = threadIdx.x; a < kApronStride; a += blockDim.x) {
    if (a >= kApronVox) { ap[a] = CUDART_NAN_F; continue; }
    const int lx = a % kApron - 1, ly = (a / kApron) % kApron - 1, lz = a / (kApron * kApron) - 1;
    const int ox = lx < 0 ? -1 : (lx >= kBlock ? 1 : 0), oy = ly < 0 ? -1 : (ly >= kBlock ? 1 : 0),
              oz = lz < 0 ? -1 : (lz >= kBlock ? 1 : 0);
    if (!(ox | oy | oz)) continue;  // interior: written by k_combine
    const int ns = comb_slot_of(p, b.x + ox, b.y + oy, b.z + oz);
    ap[a] = ns >= 0 ? p.apron[(size_t)ns * kApronStride + CAPRON(lx - ox * kBlock, ly - oy * kBlock, lz - oz * kBlock)]
                    : CUDART_NAN_F;
  }
  uchar4 *cp = p.rgb + slot * kRgbApronStride;
  for (int a = threadIdx.x; a < kRgbApronStride; a += blockDim.x) {
    if (a >= kRgbApronVox) { cp[a] = make_uchar4(0, 0, 0, 0); continue; }
    const int lx = a % kRgbApron, ly = (a / kRgbApron) % kRgbApron, lz = a / (kRgbApron * kRgbApron);
    const int ox = lx >= kBlock, oy = ly >= kBlock, oz = lz >= kBlock;
    if (!(ox | oy | oz)) continue;
    const int ns = comb_slot_of(p, b.x + ox, b.y + oy, b.z + oz);
    cp[a] = ns >= 0 ? p.rgb[(size_t)ns * kRgbApronStride + (lx - ox * kBlock) + kRgbApron * (ly - oy * kBlock) +
                           kRgbApron * kRgbApron * (lz - oz * kBlock)]
                    : make_uchar4(0, 0, 0, 0);
  }
}

// bit l of slot: base cell l has no valid corner with sdf <= 0 -- a sample there is > 0 or
// invalid (R36), so it cannot end a crossing (render.cu's exact skips)
__global__ void __launch_bounds__(256) k_comb_cellpos(const __grid_constant__ CombineLaunch p) {
  const size_t slot = blockIdx.x >> 1;
  const int l = (int)((blockIdx.x & 1) * 256 + threadIdx.x);
  const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
  const float *br = p.apron + slot * kApronStride + CAPRON(lx, ly, lz);
  bool pos = true;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float v = br[(q & 1) + kApron * ((q >> 1) & 1) + kApron * kApron * (q >> 2)];
    pos &= !(v <= 0.0f);
  }
  const unsigned int word = __ballot_sync(0xffffffffu, pos);
  if ((l & 31) == 0) {
    p.cell_pos[slot * 16 + (l >> 5)] = word;
    if (word != 0xffffffffu) p.surf[slot] = 1;
  }
}

cudaError_t launch_combine(const CombineLaunch &p, cudaStream_t s) {
  if (p.n_loc == 0) return cudaSuccess;
  k_combine<<<(unsigned)p.n_loc, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_combine_finish(const CombineLaunch &p, long long n_sel, cudaStream_t s) {
  if (n_sel == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(p.surf, 0, (size_t)n_sel, s);
  if (e != cudaSuccess) return e;
  k_comb_border<<<(unsigned)n_sel, 256, 0, s>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  k_comb_cellpos<<<(unsigned)(2 * n_sel), 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace dtsdf
