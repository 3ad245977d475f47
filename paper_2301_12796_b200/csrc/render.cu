// render.cu -- the per-pixel DTSDF raycast.
//
//   k_range_*  (a3) block-bounds range pass: every allocated block location's AABB, clipped
//              to z >= z_min, is projected into each view; per 8x8 pixel tile the min/max
//              camera z of the covering blocks is kept with order-independent atomics on
//              epoch-tagged keys, and the covering locations are counted.
//   k_order    the raycast's CTA tiles of each view, longest predicted first (counting sort of
//              the per-tile location counts), so slow tiles do not start last.
//   k_raycast  (a2, a4-a7) one thread per pixel, 8x4-pixel warps, 16x8-pixel CTA tiles taken in
//              k_order's order: lattice march t_k = k*Delta inside the tile's
//              [z_near, z_far], empty-space and certainly-positive skipping, one 4-B location-grid
//              load per block location, per-sample combination of the directions live at the
//              sample's cell (eq:combine_weight / eq:combine_tsdf_weight) read
//              from apron bricks, first +->- crossing, bisection + Illinois refinement, and the
//              shading epilogue (normal, colour, dirmask) after the step loop.
//
// Every acceleration is exact: skipped lattice points cannot end or start a crossing, skipped
// directions hold no data at the sample, and the tile order changes only when a tile runs
// (DESIGN.md §2).
#include <math_constants.h>

#include <utility>

#include "common.cuh"


namespace dtsdf {

// grid schedule of the raycast: one CTA per kTileW x kTileH-pixel tile of 8x4-pixel warps
#ifndef DTSDF_CTA
#define DTSDF_CTA 128  // 128-thread CTAs: 4% faster than 256 on C1 (smaller tail, profiles/r1c_sweep_cta.txt)
#endif
// CTA pixel tile: 8x4-pixel warps, two across when the CTA has two or more warps
constexpr int kTileW = DTSDF_CTA >= 64 ? 16 : 8, kTileH = DTSDF_CTA / kTileW;
static_assert(DTSDF_CTA % 32 == 0 && DTSDF_CTA <= 256, "whole warps, at most 8 per CTA (ray_pix)");

// Programmatic dependent launch: the range pass -> tile order -> raycast chain is launched with
// programmatic stream serialisation, so each grid is set up while its predecessor runs; the
// dependent waits for the predecessor's completion (and memory) at griddepcontrol.wait.  Without
// the launch attribute both instructions are no-ops.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t s, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ------------------------------------------------------------------------------------------
// a3: range pass
// ------------------------------------------------------------------------------------------
// One thread per (block location, view): enough parallelism for view batches.
__global__ void __launch_bounds__(256) k_range_thread(const __grid_constant__ RangeLaunch p) {
  griddep_launch_dependents();
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
  const unsigned long long zn = range_key_near(p.epoch, __float_as_uint(zmin));
  const unsigned long long zf = range_key_far(p.epoch, __float_as_uint(zmax));
  unsigned long long *zn_v = p.z_near + (size_t)view * p.tiles_x * p.tiles_y;
  unsigned long long *zf_v = p.z_far + (size_t)view * p.tiles_x * p.tiles_y;
  unsigned int *cnt_v = p.count ? p.count + (size_t)view * p.tiles_x * p.tiles_y : nullptr;
  for (int ty = ty0; ty <= ty1; ++ty)
    for (int tx = tx0; tx <= tx1; ++tx) {
      atomicMin(&zn_v[ty * p.tiles_x + tx], zn);
      atomicMax(&zf_v[ty * p.tiles_x + tx], zf);
      if (cnt_v) atomicAdd(&cnt_v[ty * p.tiles_x + tx], 1u);
    }
}

// One warp per (block location, view), for small launches (a single view): lanes 0-7 project the
// 8 AABB corners, lanes 8-19 clip the 12 edges against the near plane, warp reductions give the
// pixel bbox and z-range, and the covered tiles are shared out over the lanes (with one thread per
// location, the few near blocks covering dozens of tiles serialise a one-view pass).  Both kernels
// compute the same keys with the same operations.
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void __launch_bounds__(256) k_range_warp(const __grid_constant__ RangeLaunch p) {
  griddep_launch_dependents();
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int view = blockIdx.y;
  if (i >= p.n_locations) return;  // warp-uniform
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
  // lane < 8: corner q = lane; 8 <= lane < 20: edge (q, q | 1 << ax) with bit ax of q clear
  int q = lane & 7, q2 = q;
  if (lane >= 8 && lane < 20) {
    const int ed = lane - 8, ax = ed >> 2, low = ed & 3;  // the 4 corners with bit ax clear
    q = ax == 0 ? (low << 1) : ax == 1 ? ((low & 1) | ((low & 2) << 1)) : low;
    q2 = q | (1 << ax);
  }
  auto corner = [&](int c, float &x, float &y, float &z) {
    const float dx = (c & 1), dy = ((c >> 1) & 1), dz = ((c >> 2) & 1);
    x = c0[0] + dx * e[0][0] + dy * e[1][0] + dz * e[2][0];
    y = c0[1] + dx * e[0][1] + dy * e[1][1] + dz * e[2][1];
    z = c0[2] + dx * e[0][2] + dy * e[1][2] + dz * e[2][2];
  };
  float x1, y1, z1, x2, y2, z2;
  corner(q, x1, y1, z1);
  corner(q2, x2, y2, z2);
  const float zmax = warp_max(lane < 8 ? z1 : -CUDART_INF_F);
  if (zmax < p.z_min) return;  // entirely in front of the near plane (warp-uniform)
  float umin = CUDART_INF_F, umax = -CUDART_INF_F, vmin = CUDART_INF_F, vmax = -CUDART_INF_F;
  float zmin = CUDART_INF_F;
  if (lane < 8 && z1 >= p.z_min) {
    const float iz = 1.0f / z1;
    const float u = p.fx * x1 * iz + p.cx, v = p.fy * y1 * iz + p.cy;
    umin = umax = u;
    vmin = vmax = v;
    zmin = z1;
  } else if (lane >= 8 && lane < 20 && (z1 >= p.z_min) != (z2 >= p.z_min)) {
    // an edge crossing the near plane contributes its intersection point
    const float s = (p.z_min - z1) / (z2 - z1);
    const float x = x1 + s * (x2 - x1), y = y1 + s * (y2 - y1);
    const float u = p.fx * x / p.z_min + p.cx, v = p.fy * y / p.z_min + p.cy;
    umin = umax = u;
    vmin = vmax = v;
    zmin = p.z_min;
  }
  umin = warp_min(umin); umax = warp_max(umax);
  vmin = warp_min(vmin); vmax = warp_max(vmax);
  zmin = warp_min(zmin);
  // conservative pixel range (+1 px), clipped to the image / row shard
  const float fu0 = fmaxf(floorf(umin) - 1.0f, 0.0f), fu1 = fminf(ceilf(umax) + 1.0f, (float)(p.width - 1));
  const float fv0 = fmaxf(floorf(vmin) - 1.0f, (float)p.row0), fv1 = fminf(ceilf(vmax) + 1.0f, (float)(p.row1 - 1));
  if (!(fu0 <= fu1) || !(fv0 <= fv1)) return;
  const int tx0 = (int)fu0 / kRangeTile, tx1 = (int)fu1 / kRangeTile;
  const int ty0 = ((int)fv0 - p.row0) / kRangeTile, ty1 = ((int)fv1 - p.row0) / kRangeTile;
  const unsigned long long zn = range_key_near(p.epoch, __float_as_uint(zmin));
  const unsigned long long zf = range_key_far(p.epoch, __float_as_uint(zmax));
  unsigned long long *zn_v = p.z_near + (size_t)view * p.tiles_x * p.tiles_y;
  unsigned long long *zf_v = p.z_far + (size_t)view * p.tiles_x * p.tiles_y;
  const int nx = tx1 - tx0 + 1, n = nx * (ty1 - ty0 + 1);
  unsigned int *cnt_v = p.count ? p.count + (size_t)view * p.tiles_x * p.tiles_y : nullptr;
  for (int j = lane; j < n; j += 32) {
    const int tile = (ty0 + j / nx) * p.tiles_x + tx0 + j % nx;
    atomicMin(&zn_v[tile], zn);
    atomicMax(&zf_v[tile], zf);
    if (cnt_v) atomicAdd(&cnt_v[tile], 1u);
  }
}

// Tile order (one CTA per view): the raycast's cost is dominated by a few long-running warp tiles
// (rays grazing the floor, threading between boxes), and a tile launched late stretches the end of
// the kernel while the SMs drain (profiles/r1f_timeline.txt).  Longest-predicted-first: the cost
// proxy of a CTA tile is the number of block locations whose projection covers its range tiles;
// a counting sort on a log2 key (64 buckets) orders the CTA tiles by decreasing count.  The order
// changes only when a tile runs, never what it computes.  Clears the counts for the next pass.
constexpr int kOrderKeys = 64;
struct OrderLaunch {
  unsigned int *count;  // [views][tiles] block locations covering each range tile (k_range_*)
  int *order;           // [views][ct_x * ct_y]
  int tiles_x, tiles_y, ct_x, ct_y;
};

__device__ __forceinline__ int order_key(const OrderLaunch &p, int view, int t) {
  const int tx = t % p.ct_x, ty = t / p.ct_x;
  const size_t vo = (size_t)view * p.tiles_x * p.tiles_y;
  float c = 0.f;
  // the range tiles overlapping the CTA tile (a CTA tile may be smaller than a range tile)
  for (int ry = ty * kTileH / kRangeTile; ry <= min(p.tiles_y - 1, ((ty + 1) * kTileH - 1) / kRangeTile); ++ry)
    for (int rx = tx * kTileW / kRangeTile; rx <= min(p.tiles_x - 1, ((tx + 1) * kTileW - 1) / kRangeTile); ++rx)
      c += (float)p.count[vo + ry * p.tiles_x + rx];
  // (the depth span of the covering blocks, alone or times the count, orders worse:
  // profiles/r1f_sweep_tile_order.jsonl)
  const int lg = c > 0.f ? (int)(8.0f * __log2f(c + 1.0f)) : 0;  // 8 keys per doubling
  return kOrderKeys - 1 - min(lg, kOrderKeys - 1);              // ascending key = descending cost
}

constexpr int kOrderMaxTiles = 160 * 1024;  // CTA tiles per view whose keys fit the shared bytes below

#ifndef DTSDF_ORDER_THREADS
#define DTSDF_ORDER_THREADS 1024
#endif
__global__ void __launch_bounds__(DTSDF_ORDER_THREADS) k_order(const __grid_constant__ OrderLaunch p) {
  __shared__ unsigned int hist[kOrderKeys];
  extern __shared__ unsigned char keys[];  // [n] the sort key of every CTA tile of the view
  griddep_launch_dependents();  // the raycast may be set up now; it waits for this grid to finish
  griddep_wait();               // the range pass's counts and keys
  const int view = blockIdx.x;
  unsigned int *cnt = p.count + (size_t)view * p.tiles_x * p.tiles_y;
  int *ord = p.order + (size_t)view * p.ct_x * p.ct_y;
  const int n = p.ct_x * p.ct_y;
  if (threadIdx.x < kOrderKeys) hist[threadIdx.x] = 0;
  // keys first, with independent loads (no sync intrinsics in this loop)
#pragma unroll 4
  for (int t = threadIdx.x; t < n; t += blockDim.x) keys[t] = (unsigned char)order_key(p, view, t);
  __syncthreads();
  // warp-aggregated shared atomics: the lanes of a warp holding the same key add once (most tiles
  // share a handful of keys, and per-lane atomics on one bucket serialise)
  const int n_round = (n + (int)blockDim.x - 1) / (int)blockDim.x * (int)blockDim.x;
  for (int t = threadIdx.x; t < n_round; t += blockDim.x) {
    const int key = t < n ? keys[t] : -1;
    const unsigned same = __match_any_sync(0xffffffffu, key);
    if (key >= 0 && (threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&hist[key], (unsigned)__popc(same));
  }
  // the counts are read: clear them for the next pass
  for (int i = threadIdx.x; i < p.tiles_x * p.tiles_y; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan of the 64 bucket sizes (two per lane)
    const unsigned int a = hist[2 * threadIdx.x], b = hist[2 * threadIdx.x + 1];
    unsigned int incl = a + b;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned int v = __shfl_up_sync(0xffffffffu, incl, o);
      if ((int)threadIdx.x >= o) incl += v;
    }
    const unsigned int excl = incl - a - b;
    hist[2 * threadIdx.x] = excl;
    hist[2 * threadIdx.x + 1] = excl + a;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n_round; t += blockDim.x) {
    const int key = t < n ? keys[t] : -1;
    const unsigned same = __match_any_sync(0xffffffffu, key);
    const int lane = threadIdx.x & 31, leader = __ffs(same) - 1;
    unsigned base = 0;
    if (key >= 0 && lane == leader) base = atomicAdd(&hist[key], (unsigned)__popc(same));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (key >= 0) {
      const unsigned pos = base + __popc(same & ((1u << lane) - 1u));
      DTSDF_CHECK(pos < (unsigned)n);
      ord[pos] = t;
    }
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

#ifndef DTSDF_FAST_NORM
#define DTSDF_FAST_NORM 1    // rsqrt gradient normalisation, approximate F / S and regula-falsi quotient: one
                             // MUFU op each instead of the IEEE sequences with their special-case branches
                             // (C1 -6 %, C2 -8 %; fp32 rounding differences only, profiles/r1f_sweep_fast_norm.jsonl)
#endif
#ifndef DTSDF_SLOTS_FROM_TABLE
#define DTSDF_SLOTS_FROM_TABLE 1  // direction slots re-read from the hash entry (an L1 hit) per evaluated
                                  // direction instead of six registers through the march: with them the
                                  // kernel fits 96 registers (5 CTAs / 20 warps per SM), profiles/r1f_sweep_regs.jsonl
#endif

struct ShadeResult {
  float n[3];
  float c[3];
  float S;
  int mask;
};

__device__ __forceinline__ float lerpf(float a, float b, float t) { return fmaf(t, b - a, a); }
// a + t (b - a) on a pair: two packed FFMA2 (a - t a, then + t b)
#ifndef DTSDF_FFMA2
#define DTSDF_FFMA2 1  // 0: the same two roundings per lane with scalar FFMAs
#endif
__device__ __forceinline__ float2 lerp2(float2 a, float2 b, float2 t) {
#if DTSDF_FFMA2
  return __ffma2_rn(t, b, __ffma2_rn(make_float2(-t.x, -t.y), a, a));
#else
  return make_float2(fmaf(t.x, b.x, fmaf(-t.x, a.x, a.x)), fmaf(t.y, b.y, fmaf(-t.y, a.y, a.y)));
#endif
}

#define APRON_IDX(dx, dy, dz) (((dx) + 1) + kApron * ((dy) + 1) + kApron * kApron * ((dz) + 1))
#define RGB_IDX(dx, dy, dz) ((dx) + kRgbApron * (dy) + kRgbApron * kRgbApron * (dz))
#define REC_IDX(dx, dy, dz) ((dx) + kRec * (dy) + kRec * kRec * (dz))
// the colour of a B record (u8 r, g, b in the bits of its .y)
__device__ __forceinline__ uchar4 rec_u8(float bits) {
  const unsigned int u = __float_as_uint(bits);
  return make_uchar4(u & 255u, (u >> 8) & 255u, (u >> 16) & 255u, 0);
}

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
  int dist;      // unallocated: empty-space distance in blocks (>= 1); 0 = outside the AABB
#if DTSDF_SLOTS_FROM_TABLE
  int slot0;     // combined path: the location's combined slot (the direction slots stay in the table)
#else
  int slots[6];
#endif
};

// cell l (= lx + 8 ly + 64 lz) of the cursor's location is certainly positive (combined bricks, k_comb_finish)
__device__ __forceinline__ bool cell_positive(const unsigned int *cell_pos, const Cursor &cur, int l) {
  DTSDF_CHECK(cur.entry >= 0 && l >= 0 && l < 512);
  return (__ldg(&cell_pos[(size_t)cur.entry * 16 + (l >> 5)]) >> (l & 31)) & 1u;
}

// byte l of the cursor's location in the live-direction masks (bits 0-5 live directions, bit 7
// certainly positive)
__device__ __forceinline__ int cell_byte(const VolumeView &V, const Cursor &cur, int l) {
  DTSDF_CHECK(cur.entry >= 0 && l >= 0 && l < 512);
  return __ldg(&V.cell_dirs[(size_t)cur.entry * 512 + l]);
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

// brick slot of direction D at the cursor's location: from the cursor's registers, or re-read from
// the location's hash entry (an L1 hit) so that the six slots need no registers through the march
__device__ __forceinline__ int dir_slot(const VolumeView &V, const Cursor &cur, int D) {
#if DTSDF_SLOTS_FROM_TABLE
  return __ldg(&V.table[cur.entry].slot[D]);
#else
  return pick6(cur.slots, D);
#endif
}

#ifndef DTSDF_SEL_PTX
#define DTSDF_SEL_PTX 1  // C1 -1.8 %, C2 -2.3 % (profiles/r1n_sweep_grad_sel.jsonl)
#endif
#ifndef DTSDF_LA_IDX
#define DTSDF_LA_IDX 1  // lookahead cells addressed by offsets from the block corner
#endif
#ifndef DTSDF_RSQRT_FTZ
#define DTSDF_RSQRT_FTZ 1
#endif
// 1/sqrt(x) for a normal x > 0 (the caller guarantees x > 1e-6): the MUFU approximation without
// rsqrtf's subnormal rescaling (identical result for normal inputs, three instructions fewer)
__device__ __forceinline__ float rsqrt_normal(float x) {
#if DTSDF_RSQRT_FTZ
  float r;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
#else
  return rsqrtf(x);
#endif
}
// (a, b, c)[axis] without a branch (the ternary chain compiles to a divergent branch region)
__device__ __forceinline__ float sel3(int axis, float a, float b, float c) {
#if DTSDF_SEL_PTX
  float r;
  asm("{\n\t.reg .pred p0, p1;\n\tsetp.eq.s32 p0, %1, 0;\n\tsetp.eq.s32 p1, %1, 1;\n\t"
      "selp.f32 %0, %3, %4, p1;\n\tselp.f32 %0, %2, %0, p0;\n\t}"
      : "=f"(r) : "r"(axis), "f"(a), "f"(b), "f"(c));
  return r;
#else
  return axis == 0 ? a : (axis == 1 ? b : c);
#endif
}

// F(x, r) of DESIGN.md §2 O3 for the sample at base voxel (block-local l, fractions f) of the
// current cursor location; with shade = true also the shading sums of O7.  One instance of this
// body is compiled (runtime direction loop) to keep the kernel inside the instruction cache.
template <bool shade>
__device__ __forceinline__ SampleResult eval_sample(const VolumeView &V, const Cursor &cur, int lx, int ly, int lz,
                                                 float fx, float fy, float fz, float rx, float ry, float rz,
                                                 ShadeResult *sh, int live = -1) {
  SampleResult res;
  const int off = lx + kRec * ly + kRec * kRec * lz;
  float S1 = 0.f, F1 = 0.f, S2 = 0.f, F2 = 0.f;
  bool any_grad = false;
  float N1x = 0.f, N1y = 0.f, N1z = 0.f, N2x = 0.f, N2y = 0.f, N2z = 0.f;
  float C1r = 0.f, C1g = 0.f, C1b = 0.f, C2r = 0.f, C2g = 0.f, C2b = 0.f;
  int m1 = 0, m2 = 0;
  const float half_inv_s = 0.5f * V.inv_voxel;
  const float2 fx2 = make_float2(fx, fx), fy2 = make_float2(fy, fy), fz2 = make_float2(fz, fz);
  // the directions that can hold data at this base cell (a subset of the location's, exact)
  DTSDF_CHECK(!V.cell_dirs || cur.entry >= 0);
  // (live >= 0: the advance loop already read this cell's byte)
  int present = !V.use_live ? cur.present : live >= 0 ? live : (cell_byte(V, cur, lx + 8 * ly + 64 * lz) & 63);
#pragma unroll 1
  while (present) {
    const int D = __ffs(present) - 1;
    present &= present - 1;
    const int slot = dir_slot(V, cur, D);
    DTSDF_CHECK(slot >= 0 && slot < V.n_blocks && lx >= 0 && lx < 8 && ly >= 0 && ly < 8 && lz >= 0 && lz < 8);
    const float4 *ba = V.brick_a + (size_t)slot * kRecStride + off;
    const float2 *bb = V.brick_b + (size_t)slot * kRecStride + off;
    // the 8 corner records {sdf, weight, dsdf_x, dsdf_y} + dsdf_z are issued before any test (one
    // load round per direction; the brick always holds them, NaN marking unallocated neighbours)
    const float4 a000 = __ldg(ba + REC_IDX(0, 0, 0)), a100 = __ldg(ba + REC_IDX(1, 0, 0));
    const float4 a010 = __ldg(ba + REC_IDX(0, 1, 0)), a110 = __ldg(ba + REC_IDX(1, 1, 0));
    const float4 a001 = __ldg(ba + REC_IDX(0, 0, 1)), a101 = __ldg(ba + REC_IDX(1, 0, 1));
    const float4 a011 = __ldg(ba + REC_IDX(0, 1, 1)), a111 = __ldg(ba + REC_IDX(1, 1, 1));
    const float z000 = __ldg(&bb[REC_IDX(0, 0, 0)].x), z100 = __ldg(&bb[REC_IDX(1, 0, 0)].x);
    const float z010 = __ldg(&bb[REC_IDX(0, 1, 0)].x), z110 = __ldg(&bb[REC_IDX(1, 1, 0)].x);
    const float z001 = __ldg(&bb[REC_IDX(0, 0, 1)].x), z101 = __ldg(&bb[REC_IDX(1, 0, 1)].x);
    const float z011 = __ldg(&bb[REC_IDX(0, 1, 1)].x), z111 = __ldg(&bb[REC_IDX(1, 1, 1)].x);
    // The lerps run pairwise on Blackwell's packed fp32x2 FMA (FFMA2): {sdf, weight} of the
    // corners, and pairs of corner differences.
    // O3(a) trilinear phi_D, omega_D over the 8 cell corners (x: rows e_yz, y: slabs R(dz), z)
    const float2 e00 = lerp2(make_float2(a000.x, a000.y), make_float2(a100.x, a100.y), fx2);
    const float2 e10 = lerp2(make_float2(a010.x, a010.y), make_float2(a110.x, a110.y), fx2);
    const float2 e01 = lerp2(make_float2(a001.x, a001.y), make_float2(a101.x, a101.y), fx2);
    const float2 e11 = lerp2(make_float2(a011.x, a011.y), make_float2(a111.x, a111.y), fx2);
    const float2 R0w = lerp2(e00, e10, fy2), R1w = lerp2(e01, e11, fy2);
    const float2 pw = lerp2(R0w, R1w, fz2);
    const float phi = pw.x, omega = pw.y;
    if (isnan(phi)) continue;       // D absent: a corner lies in an unallocated block
    if (!(omega > 0.0f)) continue;  // D holds no data at x (reading R8)
    // O3(c) central differences of trilinear phi at x +- s e_a: phi(x + s e_a) - phi(x - s e_a) is
    // the trilinear interpolant of the corners' differences dsdf_a = sdf(+e_a) - sdf(-e_a) -- taken
    // pairwise along a (corner 0, corner 1), bilinear over the other two axes, then along a
    const float2 Dx = lerp2(lerp2(make_float2(a000.z, a100.z), make_float2(a010.z, a110.z), fy2),
                            lerp2(make_float2(a001.z, a101.z), make_float2(a011.z, a111.z), fy2), fz2);
    const float2 Dy = lerp2(lerp2(make_float2(a000.w, a010.w), make_float2(a100.w, a110.w), fx2),
                            lerp2(make_float2(a001.w, a011.w), make_float2(a101.w, a111.w), fx2), fz2);
    const float2 Dz = lerp2(lerp2(make_float2(z000, z001), make_float2(z100, z101), fx2),
                            lerp2(make_float2(z010, z011), make_float2(z110, z111), fx2), fy2);
    const float gx = lerpf(Dx.x, Dx.y, fx) * half_inv_s;
    const float gy = lerpf(Dy.x, Dy.y, fy) * half_inv_s;
    const float gz = lerpf(Dz.x, Dz.y, fz) * half_inv_s;
#if DTSDF_FAST_NORM
    const float gn2 = gx * gx + gy * gy + gz * gz;  // |g|^2: |g| > 1e-3 <=> |g|^2 > 1e-6 (up to rounding)
#else
    const float gn = sqrtf(gx * gx + gy * gy + gz * gz);
#endif
    // v^D = sign * e_axis
    const int axis = D >> 1;
    const float sign = (D & 1) ? -1.0f : 1.0f;
    const float r_axis = sel3(axis, rx, ry, rz);
    // eq:combine_tsdf_weight: omega * max(0, <v^D, -r>)
    const float W2 = omega * fmaxf(-sign * r_axis, 0.0f);
    S2 += W2;
    F2 = fmaf(W2, phi, F2);
    float W1 = 0.0f, nx = 0.f, ny = 0.f, nz = 0.f;
#if DTSDF_FAST_NORM
    if (gn2 > 1e-6f) {  // reading R8: gradient present (NaN stencil -> false)
      any_grad = true;
      const float ig = rsqrt_normal(gn2);
#else
    if (gn > 1e-3f) {  // reading R8: gradient present (NaN stencil -> false)
      any_grad = true;
      const float ig = 1.0f / gn;
#endif
      nx = gx * ig; ny = gy * ig; nz = gz * ig;
      const float n_axis = sel3(axis, nx, ny, nz);
      const float nr = -(nx * rx + ny * ry + nz * rz);
      // eq:combine_weight: w_dir(<n,v>) * max(0, <n,-r>) * omega
      W1 = w_dir(sign * n_axis, V) * fmaxf(nr, 0.0f) * omega;
      S1 += W1;
      F1 = fmaf(W1, phi, F1);
    }
    if constexpr (shade) {
      const uchar4 q000 = rec_u8(bb[REC_IDX(0, 0, 0)].y), q100 = rec_u8(bb[REC_IDX(1, 0, 0)].y),
                   q010 = rec_u8(bb[REC_IDX(0, 1, 0)].y), q110 = rec_u8(bb[REC_IDX(1, 1, 0)].y),
                   q001 = rec_u8(bb[REC_IDX(0, 0, 1)].y), q101 = rec_u8(bb[REC_IDX(1, 0, 1)].y),
                   q011 = rec_u8(bb[REC_IDX(0, 1, 1)].y), q111 = rec_u8(bb[REC_IDX(1, 1, 1)].y);
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
  res.valid = S > 0.0f;
#if DTSDF_FAST_NORM
  res.f = res.valid ? __fdividef(F, S) : 0.0f;
#else
  res.f = res.valid ? F / S : 0.0f;
#endif
  if constexpr (shade) {
    sh->S = S;
    sh->mask = any_grad ? m1 : m2;
    sh->n[0] = any_grad ? N1x : N2x; sh->n[1] = any_grad ? N1y : N2y; sh->n[2] = any_grad ? N1z : N2z;
    sh->c[0] = any_grad ? C1r : C2r; sh->c[1] = any_grad ? C1g : C2g; sh->c[2] = any_grad ? C1b : C2b;
  }
  return res;
}

// NEXT-1: sample of the combined TSDF (readings R36-R37): plain trilinear of the combined sdf
// over the 8 cell corners, invalid if any corner is (NaN); with shade = true the normal (central
// differences of the trilinear field at +-s, else the cell's own trilinear gradient), the
// trilinear u8 colour and the OR of the direction masks of the corners with weight >= 1/8.
template <bool shade>
__device__ __forceinline__ SampleResult eval_comb(const VolumeView &V, const CombinedView &C, int slot, int lx, int ly,
                                                  int lz, float fx, float fy, float fz, ShadeResult *sh) {
  DTSDF_CHECK(slot >= 0 && slot < C.n_slots && lx >= 0 && lx < 8 && ly >= 0 && ly < 8 && lz >= 0 && lz < 8);
  const float *br = C.apron + (size_t)slot * kApronStride + (lx + kApron * ly + kApron * kApron * lz);
  const float c000 = __ldg(br + APRON_IDX(0, 0, 0)), c100 = __ldg(br + APRON_IDX(1, 0, 0));
  const float c010 = __ldg(br + APRON_IDX(0, 1, 0)), c110 = __ldg(br + APRON_IDX(1, 1, 0));
  const float c001 = __ldg(br + APRON_IDX(0, 0, 1)), c101 = __ldg(br + APRON_IDX(1, 0, 1));
  const float c011 = __ldg(br + APRON_IDX(0, 1, 1)), c111 = __ldg(br + APRON_IDX(1, 1, 1));
  const float e00 = lerpf(c000, c100, fx), e10 = lerpf(c010, c110, fx);
  const float e01 = lerpf(c001, c101, fx), e11 = lerpf(c011, c111, fx);
  const float R0 = lerpf(e00, e10, fy), R1 = lerpf(e01, e11, fy);
  const float phi = lerpf(R0, R1, fz);
  SampleResult res;
  res.valid = !isnan(phi);
  res.f = res.valid ? phi : 0.0f;
  if (shade && res.valid) {  // (compile-time shade)
    const float xm00 = __ldg(br + APRON_IDX(-1, 0, 0)), xm10 = __ldg(br + APRON_IDX(-1, 1, 0));
    const float xm01 = __ldg(br + APRON_IDX(-1, 0, 1)), xm11 = __ldg(br + APRON_IDX(-1, 1, 1));
    const float xp00 = __ldg(br + APRON_IDX(2, 0, 0)), xp10 = __ldg(br + APRON_IDX(2, 1, 0));
    const float xp01 = __ldg(br + APRON_IDX(2, 0, 1)), xp11 = __ldg(br + APRON_IDX(2, 1, 1));
    const float ym00 = __ldg(br + APRON_IDX(0, -1, 0)), ym10 = __ldg(br + APRON_IDX(1, -1, 0));
    const float ym01 = __ldg(br + APRON_IDX(0, -1, 1)), ym11 = __ldg(br + APRON_IDX(1, -1, 1));
    const float yp00 = __ldg(br + APRON_IDX(0, 2, 0)), yp10 = __ldg(br + APRON_IDX(1, 2, 0));
    const float yp01 = __ldg(br + APRON_IDX(0, 2, 1)), yp11 = __ldg(br + APRON_IDX(1, 2, 1));
    const float zm00 = __ldg(br + APRON_IDX(0, 0, -1)), zm10 = __ldg(br + APRON_IDX(1, 0, -1));
    const float zm01 = __ldg(br + APRON_IDX(0, 1, -1)), zm11 = __ldg(br + APRON_IDX(1, 1, -1));
    const float zp00 = __ldg(br + APRON_IDX(0, 0, 2)), zp10 = __ldg(br + APRON_IDX(1, 0, 2));
    const float zp01 = __ldg(br + APRON_IDX(0, 1, 2)), zp11 = __ldg(br + APRON_IDX(1, 1, 2));
    // bilinear interpolants of the stencil layers (as eval_sample): P over (y,z) at x = -1,0,1,2
    const float P0 = lerpf(lerpf(c000, c010, fy), lerpf(c001, c011, fy), fz);
    const float P1 = lerpf(lerpf(c100, c110, fy), lerpf(c101, c111, fy), fz);
    const float Pm = lerpf(lerpf(xm00, xm10, fy), lerpf(xm01, xm11, fy), fz);
    const float Pp = lerpf(lerpf(xp00, xp10, fy), lerpf(xp01, xp11, fy), fz);
    const float Q0 = lerpf(e00, e01, fz), Q1 = lerpf(e10, e11, fz);
    const float Qm = lerpf(lerpf(ym00, ym10, fx), lerpf(ym01, ym11, fx), fz);
    const float Qp = lerpf(lerpf(yp00, yp10, fx), lerpf(yp01, yp11, fx), fz);
    const float Rm = lerpf(lerpf(zm00, zm10, fx), lerpf(zm01, zm11, fx), fy);
    const float Rp = lerpf(lerpf(zp00, zp10, fx), lerpf(zp01, zp11, fx), fy);
    const float half_inv_s = 0.5f * V.inv_voxel;
    float gx = lerpf(P1 - Pm, Pp - P0, fx) * half_inv_s;
    float gy = lerpf(Q1 - Qm, Qp - Q0, fy) * half_inv_s;
    float gz = lerpf(R1 - Rm, Rp - R0, fz) * half_inv_s;
    float gn = sqrtf(gx * gx + gy * gy + gz * gz);
    if (!(gn > 1e-3f)) {  // stencil incomplete (NaN) or flat: the cell's own trilinear gradient
      gx = (P1 - P0) * V.inv_voxel;
      gy = (Q1 - Q0) * V.inv_voxel;
      gz = (R1 - R0) * V.inv_voxel;
      gn = sqrtf(gx * gx + gy * gy + gz * gz);
    }
    const float ig = gn > 1e-3f ? 1.0f / gn : 0.0f;
    sh->n[0] = gx * ig; sh->n[1] = gy * ig; sh->n[2] = gz * ig;
    const uchar4 *cb = C.rgb + (size_t)slot * kRgbApronStride + (lx + kRgbApron * ly + kRgbApron * kRgbApron * lz);
    const uchar4 q000 = cb[RGB_IDX(0, 0, 0)], q100 = cb[RGB_IDX(1, 0, 0)], q010 = cb[RGB_IDX(0, 1, 0)],
                 q110 = cb[RGB_IDX(1, 1, 0)], q001 = cb[RGB_IDX(0, 0, 1)], q101 = cb[RGB_IDX(1, 0, 1)],
                 q011 = cb[RGB_IDX(0, 1, 1)], q111 = cb[RGB_IDX(1, 1, 1)];
#define TRI_CH(ch)                                                                                              \
  lerpf(lerpf(lerpf((float)q000.ch, (float)q100.ch, fx), lerpf((float)q010.ch, (float)q110.ch, fx), fy),        \
        lerpf(lerpf((float)q001.ch, (float)q101.ch, fx), lerpf((float)q011.ch, (float)q111.ch, fx), fy), fz)
    sh->c[0] = TRI_CH(x); sh->c[1] = TRI_CH(y); sh->c[2] = TRI_CH(z);
#undef TRI_CH
    sh->S = 1.0f;
    // R37: OR of the masks of the corners with trilinear weight >= 1/8
    const float ux = 1.f - fx, uy = 1.f - fy, uz = 1.f - fz;
    int m = 0;
    m |= (ux * uy * uz >= 0.125f) ? q000.w : 0;
    m |= (fx * uy * uz >= 0.125f) ? q100.w : 0;
    m |= (ux * fy * uz >= 0.125f) ? q010.w : 0;
    m |= (fx * fy * uz >= 0.125f) ? q110.w : 0;
    m |= (ux * uy * fz >= 0.125f) ? q001.w : 0;
    m |= (fx * uy * fz >= 0.125f) ? q101.w : 0;
    m |= (ux * fy * fz >= 0.125f) ? q011.w : 0;
    m |= (fx * fy * fz >= 0.125f) ? q111.w : 0;
    sh->mask = m;
  }
  return res;
}

// ------------------------------------------------------------------------------------------
// a4-a7: the raycast kernel, one state machine per ray so that a warp's rays -- marching,
// bisecting, regula-falsi or shading -- all run the same sample-evaluation code together
// ------------------------------------------------------------------------------------------
enum : int { kMarch = 0, kBisect = 1, kIllinois = 2, kShade = 3 };
#ifndef DTSDF_PF_TABLE
#define DTSDF_PF_TABLE 0
#endif
#ifndef DTSDF_EMPTY_NEXT
#define DTSDF_EMPTY_NEXT 1  // C1 -4.2 %, C2 -2.2 %, bit-identical (profiles/r3_sweep_empty_next.jsonl)
#endif
#ifndef DTSDF_LOOKAHEAD
#define DTSDF_LOOKAHEAD 6  // with the block-offset addressing: C1 -1.9 %, C3 -0.9 %, C2 equal vs 8 (profiles/r1n_sweep_lookahead.jsonl)
#endif
constexpr int kLookahead = DTSDF_LOOKAHEAD;  // lattice points tested per certainly-positive scan

// per-thread pixel of the ray (u | vrel << 16), read back only when a bracket starts and at the end
__shared__ int ray_pix[256];
__shared__ int ray_view[256];

// One ray's complete state: the march/refinement/shading state machine of DESIGN.md §2 (a4-a7).
// step() performs the cheap advance loop plus exactly one sample evaluation, so that the lanes of
// a warp -- whatever phase each is in -- run the evaluation code together.
template <bool kComb>
struct RayT {
  // the view and the pixel (u | vrel << 16) wait in shared memory (ray_view, ray_pix): no registers
  // through the march
  __device__ __forceinline__ int pix() const { return ray_pix[threadIdx.x]; }
  __device__ __forceinline__ int view() const { return ray_view[threadIdx.x]; }
#if DTSDF_SLOTS_FROM_TABLE
  __device__ __forceinline__ int comb_slot() const { return cur.slot0; }
#else
  __device__ __forceinline__ int comb_slot() const { return cur.slots[0]; }
#endif
  float r[3];
  float o[3], ir[3];
  int k1;
  int k;
  // sample positions in voxel units g = g0 + t * rs relative to the integer cell ib of a frame:
  // the world origin during the march; re-anchored once per bracket in fp64 at x(t_{k-1}), so g
  // stays within two voxels of it and fp32 resolves the shading point to ~1e-9 m (reading R32) --
  // near a root the weights of an ill-conditioned mixture of directions change on a
  // sub-micrometre scale
  int ibx, iby, ibz;
  float g0x, g0y, g0z, rsx, rsy, rsz;
  Cursor cur;
  int mode, it, side;
  bool prev_valid, fa_valid, hit;
  float prev_f, a, b, t, fa, fb;
  ShadeResult sh;
  int ix, iy, iz;
  float frx, fry, frz;
#ifdef DTSDF_STATS
  int st_march, st_refine, st_skip, st_empty, st_jump, st_cpi, st_newblk, st_scan, st_loc;
  long long cy_adv, cy_march, cy_refine;
  unsigned long long g_start, g_end;
  unsigned smid;
#endif

  __device__ __forceinline__ void init(const RenderLaunch &p, int view_, int u_, int vrel_) {
    ray_view[threadIdx.x] = view_;
    const int view = view_;
    ray_pix[threadIdx.x] = u_ | (vrel_ << 16);
    const int u = u_, vrel = vrel_;
    const VolumeView &V = p.vol;
    const ViewPose &P = p.pose[view];
    const int v = p.row0 + vrel;
    // O1 ray (eq:reprojection)
    const float dxf = (u - p.cx) / p.fx, dyf = (v - p.cy) / p.fy;
    const float Lf = sqrtf(dxf * dxf + dyf * dyf + 1.0f);
    const float iLf = 1.0f / Lf;
    for (int q = 0; q < 3; ++q) {
      r[q] = (P.r[3 * q] * dxf + P.r[3 * q + 1] * dyf + P.r[3 * q + 2]) * iLf;
      o[q] = P.t[q];
      ir[q] = 1.0f / r[q];
    }
    // O2 lattice bounds, narrowed to the tile's block range (a3)
    const size_t tile = ((size_t)view * p.tiles_y + vrel / kRangeTile) * p.tiles_x + u / kRangeTile;
    const unsigned long long kn = __ldg(&p.z_near[tile]), kf = __ldg(&p.z_far[tile]);
    // a tile no block of this pass projected onto still holds keys of an earlier epoch: empty
    const bool covered = (kn >> 32) == (0xFFFFFFFFu - p.epoch) && (kf >> 32) == p.epoch;
    const float zn = covered ? __uint_as_float((unsigned)kn) : 1.0f, zf = covered ? __uint_as_float((unsigned)kf) : 0.0f;
    const int kmin = (int)ceilf(p.z_min * Lf * V.inv_delta), kmax = (int)floorf(p.z_max * Lf * V.inv_delta);
    k = kmin;
    int kl = kmax;
    if (p.use_range) {
      if (zn <= zf) {
        k = max(kmin, (int)floorf(zn * (1.0f - 1e-4f) * Lf * V.inv_delta));
        kl = min(kmax, (int)ceilf(zf * (1.0f + 1e-4f) * Lf * V.inv_delta) + 1);
      } else {
        kl = k - 1;  // no allocated block projects onto this tile
      }
    }
    k1 = kl;
    ibx = iby = ibz = 0;
    g0x = P.t[0] * V.inv_voxel; g0y = P.t[1] * V.inv_voxel; g0z = P.t[2] * V.inv_voxel;
    rsx = r[0] * V.inv_voxel; rsy = r[1] * V.inv_voxel; rsz = r[2] * V.inv_voxel;
    cur.bx = 0x7fffffff; cur.by = 0; cur.bz = 0; cur.occ = false; cur.surf = false; cur.present = 0; cur.entry = -1;
    cur.dist = 1;
#if DTSDF_SLOTS_FROM_TABLE
    cur.slot0 = -1;
#else
#pragma unroll
    for (int d = 0; d < 6; ++d) cur.slots[d] = -1;
#endif
    mode = kMarch;
    prev_valid = false;
    prev_f = 0.f;
    a = b = 0.f;
    t = (float)k * V.delta;
    fa = fb = 0.f;
    fa_valid = true;
    it = side = 0;
    hit = false;
#ifdef DTSDF_STATS
    st_march = st_refine = st_skip = st_empty = st_jump = st_cpi = st_newblk = st_scan = st_loc = 0;
    cy_adv = cy_march = cy_refine = 0;
#endif
  }

  __device__ __forceinline__ void locate(const VolumeView &V, const CombinedView &C, float tt) {
#ifdef DTSDF_STATS
    ++st_loc;
#endif
    const float gx = fmaf(tt, rsx, g0x), gy = fmaf(tt, rsy, g0y), gz = fmaf(tt, rsz, g0z);
    const float flx = floorf(gx), fly = floorf(gy), flz = floorf(gz);
    frx = gx - flx; fry = gy - fly; frz = gz - flz;
    ix = ibx + (int)flx; iy = iby + (int)fly; iz = ibz + (int)flz;
    const int bx = ix >> 3, by = iy >> 3, bz = iz >> 3;
    if (bx != cur.bx || by != cur.by || bz != cur.bz) {
#ifdef DTSDF_STATS
      ++st_newblk;
#endif
      cur.bx = bx; cur.by = by; cur.bz = bz;
      cur.present = 0;
      cur.entry = -1;
      if (V.loc_grid) {  // a2 via the dense location grid: one load, then the entry's slots
        const unsigned x = (unsigned)(bx - V.lo_x), y = (unsigned)(by - V.lo_y), z = (unsigned)(bz - V.lo_z);
        int gv = 0;  // outside the AABB: distance 0
        if (x < (unsigned)V.dim_x && y < (unsigned)V.dim_y && z < (unsigned)V.dim_z)
          gv = __ldg(&V.loc_grid[(z * (unsigned)V.dim_y + y) * (unsigned)V.dim_x + x]);  // < 2^28 cells: 32-bit index
        else
          gv = -0x7fffffff;
        DTSDF_CHECK(gv < 0 || (long long)(gv & kGridEntryMask) < V.table_cap);
        cur.occ = gv >= 0;
        cur.dist = gv == -0x7fffffff ? 0 : (gv < 0 ? -gv : 0);
        cur.surf = (gv >> 30) & 1;
        if (cur.occ) {
          cur.entry = gv & kGridEntryMask;
#if DTSDF_PF_TABLE
          // the entry's direction slots are read when a sample of this location is evaluated:
          // start their trip to L1 now
          asm volatile("prefetch.global.L1 [%0];" ::"l"(&V.table[cur.entry]));
#endif
#if DTSDF_SLOTS_FROM_TABLE
          cur.present = (gv >> kGridEntryBits) & 63;  // the slots themselves are read when evaluated
#else
          const int4 *e = reinterpret_cast<const int4 *>(&V.table[cur.entry]);
          const int4 ea = __ldg(e), eb = __ldg(e + 1);
          DTSDF_CHECK(ea.z < V.n_blocks && ea.w < V.n_blocks && eb.x < V.n_blocks && eb.y < V.n_blocks &&
                      eb.z < V.n_blocks && eb.w < V.n_blocks);
          cur.slots[0] = ea.z; cur.slots[1] = ea.w; cur.slots[2] = eb.x;
          cur.slots[3] = eb.y; cur.slots[4] = eb.z; cur.slots[5] = eb.w;
#endif
        }
      } else {  // a2 via occupancy bitmaps + hash probe
        cur.dist = 1;
        cur.occ = occupied(V, bx, by, bz, &cur.surf);
#if DTSDF_SLOTS_FROM_TABLE
        if (cur.occ) {
          int sl[6];
          cur.entry = lookup_slots(V, bx, by, bz, sl);
#pragma unroll
          for (int d = 0; d < 6; ++d) cur.present |= (sl[d] >= 0) << d;
        }
#else
        if (cur.occ) cur.entry = lookup_slots(V, bx, by, bz, cur.slots);
#endif
      }
#if !DTSDF_SLOTS_FROM_TABLE
      if (cur.occ) {
#pragma unroll
        for (int d = 0; d < 6; ++d) cur.present |= (cur.slots[d] >= 0) << d;
      }
#endif
      if constexpr (kComb) {  // NEXT-1: the location's combined brick (entry -> combined slot)
        if (cur.occ) {
          DTSDF_CHECK(cur.entry >= 0 && cur.entry < V.table_cap);
          const int cs = __ldg(&C.slot_of_entry[cur.entry]);
          DTSDF_CHECK(cs < C.n_slots);
          if (cs >= 0) {
            cur.entry = cs;
            cur.surf = __ldg(&C.surf[cs]) != 0;
            cur.present = 1;
#if DTSDF_SLOTS_FROM_TABLE
            cur.slot0 = cs;
#else
            cur.slots[0] = cs;
#endif
          } else {  // allocated but not combined: invalid like an unallocated location
            cur.occ = false;
            cur.dist = 1;
            cur.present = 0;
            cur.entry = -1;
          }
        }
      }
    }
  }

  // ray parameter where it leaves the cube of blocks within `rad` of the cursor's block (march frame)
  __device__ __forceinline__ float box_exit(const VolumeView &V, int rad) const {
    const float bsz = kBlock * V.voxel_size;
    float texit = 3.0e38f;
    const int bb[3] = {cur.bx, cur.by, cur.bz};
    for (int q = 0; q < 3; ++q) {
      if (r[q] > 0.f) texit = fminf(texit, ((bb[q] + 1 + rad) * bsz - o[q]) * ir[q]);
      else if (r[q] < 0.f) texit = fminf(texit, ((bb[q] - rad) * bsz - o[q]) * ir[q]);
    }
    return texit;
  }
  __device__ __forceinline__ float block_exit(const VolumeView &V) const { return box_exit(V, 0); }
  // ray parameter where it leaves an empty location's box (common.cuh: six 5-bit extents)
  __device__ __forceinline__ float packed_box_exit(const VolumeView &V, int packed) const {
    const float bsz = kBlock * V.voxel_size;
    float texit = 3.0e38f;
    const int bb[3] = {cur.bx, cur.by, cur.bz};
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (r[q] > 0.f) texit = fminf(texit, ((bb[q] + 1 + ((packed >> (kBoxBits * (2 * q + 1))) & kBoxMax)) * bsz - o[q]) * ir[q]);
      else if (r[q] < 0.f) texit = fminf(texit, ((bb[q] - ((packed >> (kBoxBits * 2 * q)) & kBoxMax)) * bsz - o[q]) * ir[q]);
    }
    return texit;
  }

  // a6: bracket [t_{k-1}, t_k] with F(t_{k-1}) = f_prev > 0 and F(t_k) = f_k <= 0
  __device__ __forceinline__ void begin_bracket(const RenderLaunch &p, float f_prev, float f_k) {
    const VolumeView &V = p.vol;
    // re-anchor the position frame at x(t_{k-1}) in fp64
    {
      const ViewPose &P = p.pose[view()];
      const int px = pix();
      const double ddx = ((double)(px & 0xffff) - (double)p.cx) / (double)p.fx;
      const double ddy = ((double)(p.row0 + (px >> 16)) - (double)p.cy) / (double)p.fy;
      const double iLd = 1.0 / sqrt(ddx * ddx + ddy * ddy + 1.0), inv_s = 1.0 / (double)V.voxel_size;
      const double t0 = (double)(k - 1) * (double)V.delta;
      double rq[3], gq[3];
      for (int q = 0; q < 3; ++q) {
        rq[q] = ((double)P.r[3 * q] * ddx + (double)P.r[3 * q + 1] * ddy + (double)P.r[3 * q + 2]) * iLd;
        gq[q] = fma(t0, rq[q], (double)P.t[q]) * inv_s;
      }
      const double fx0 = floor(gq[0]), fy0 = floor(gq[1]), fz0 = floor(gq[2]);
      ibx = (int)fx0; iby = (int)fy0; ibz = (int)fz0;
      g0x = (float)(gq[0] - fx0); g0y = (float)(gq[1] - fy0); g0z = (float)(gq[2] - fz0);
      rsx = (float)(rq[0] * inv_s); rsy = (float)(rq[1] * inv_s); rsz = (float)(rq[2] * inv_s);
    }
    // Phase 1: bisection with the oracle's decisions (an invalid midpoint counts as positive,
    // R21) until the bracket is <= 5e-5 m, so it keeps the oracle's root when F has several
    // sign changes (reading R20).  Phase 2: Illinois regula falsi inside it.
    a = 0.f;
    b = V.delta;
    fa = f_prev;
    fb = f_k;
    fa_valid = true;
    it = 0;
    side = 0;
    mode = p.n_bisect > 0 ? kBisect : kIllinois;
  }

  int live_;  // live-direction byte of the point to evaluate, if the advance loop read it (-1: not)
#ifdef DTSDF_STATS
  long long c0_;
#endif
  // One step = advance() then evaluate().  Advance (march only) to the next point to evaluate;
  // false when the ray is finished (no crossing in range: a miss).
  __device__ __forceinline__ bool advance(const RenderLaunch &p) {
    const VolumeView &V = p.vol;
#ifdef DTSDF_STATS
    c0_ = clock64();
#endif
    int &live = live_;
    live = -1;
    if (mode == kMarch) {
      // a4: advance to the next lattice point that needs an evaluation.  Every step skipped here
      // is exact (DESIGN.md §2 O2): lattice points in unallocated locations are invalid; in a
      // location without an sdf <= 0 corner, and in a certainly-positive cell followed by
      // another, no crossing can end or start.
      for (;;) {
        live = -1;
        if (k > k1) return false;  // no crossing: a miss
        t = (float)k * V.delta;
        locate(V, p.comb, t);
#ifdef DTSDF_STATS
        ++st_skip;
#endif
        if (!cur.occ) {
          prev_valid = false;
#ifdef DTSDF_STATS
          ++st_empty;
#endif
          if (p.use_skip) {
            // land on the first lattice point at or before the exit of the empty region: the
            // block itself, the cube of blocks within its empty-space distance, or -- outside the
            // volume's AABB -- straight to the AABB entry (or a miss when the ray leaves it)
            float texit;
            if (cur.dist == 0) {
              const float bsz = kBlock * V.voxel_size;
              float t0 = -3.0e38f, t1 = 3.0e38f;
              const int lo3[3] = {V.lo_x, V.lo_y, V.lo_z}, dm3[3] = {V.dim_x, V.dim_y, V.dim_z};
              for (int q = 0; q < 3; ++q) {
                const float lo = lo3[q] * bsz - o[q], hi = (lo3[q] + dm3[q]) * bsz - o[q];
                if (r[q] != 0.f) {
                  const float ta = lo * ir[q], tb = hi * ir[q];
                  t0 = fmaxf(t0, fminf(ta, tb));
                  t1 = fminf(t1, fmaxf(ta, tb));
                } else if (lo > 0.f || hi < 0.f) {
                  t0 = 3.0e38f;
                }
              }
              texit = (t0 <= t1 && t1 > t) ? fmaxf(t0, t) : 3.0e38f;
              if (texit >= 3.0e38f) { k = k1 + 1; continue; }
            } else {
#if DTSDF_EMPTY_BOX
              texit = packed_box_exit(V, cur.dist - 1);
#else
              texit = box_exit(V, cur.dist - 1);
#endif
            }
            const float kn = floorf(texit * V.inv_delta);
            k = (kn > (float)k1) ? k1 + 1 : max(k + 1, (int)kn);
#if DTSDF_EMPTY_NEXT
            // the landing point still in this empty block: the next iteration would only step on
            // to k + 1 (locate's block test, here without the loop round)
            if (cur.dist != 0 && k <= k1) {
              const float tk = (float)k * V.delta;
              const int jx = ibx + (int)floorf(fmaf(tk, rsx, g0x)), jy = iby + (int)floorf(fmaf(tk, rsy, g0y)),
                        jz = ibz + (int)floorf(fmaf(tk, rsz, g0z));
              if ((jx >> 3) == cur.bx && (jy >> 3) == cur.by && (jz >> 3) == cur.bz) ++k;
            }
#endif
          } else {
            ++k;
          }
          continue;
        }
        if (p.use_skip && !cur.surf) {
          // jump to (at most) the location's second-to-last lattice point: the point evaluated
          // there becomes prev for the first point of the next location
          const float kj = ceilf(block_exit(V) * V.inv_delta) - 2.0f;
          if (kj > (float)k) {
#ifdef DTSDF_STATS
            ++st_jump;
#endif
            k = (kj > (float)k1) ? k1 + 1 : (int)kj;
            prev_valid = false;
            continue;
          }
        }
        bool cp = false;
        if (p.use_skip) {
          const int l0 = (ix & 7) + 8 * (iy & 7) + 64 * (iz & 7);
          if constexpr (kComb) {
            cp = cell_positive(p.comb.cell_pos, cur, l0);
          } else {
            const int cb = cell_byte(V, cur, l0);
            cp = (cb & 128) != 0;
            live = cb & 63;  // handed to the evaluation of this point
          }
        }
        if (cp) {
          live = -1;
          // look ahead over the next lattice points of this location at once (independent
          // loads): in a run of certainly-positive points only the last one needs evaluating
          unsigned run = 1u;
#ifdef DTSDF_STATS
          ++st_scan;
#endif

#if DTSDF_LA_IDX
          // voxel offsets from the cursor block's corner: in the block <=> all three in [0, 8)
          const int ox = ibx - kBlock * cur.bx, oy = iby - kBlock * cur.by, oz = ibz - kBlock * cur.bz;
#endif
#pragma unroll
          for (int j = 1; j < kLookahead; ++j) {
            const float tj = (float)(k + j) * V.delta;
#if DTSDF_LA_IDX
            const int ux = ox + (int)floorf(fmaf(tj, rsx, g0x)), uy = oy + (int)floorf(fmaf(tj, rsy, g0y)),
                      uz = oz + (int)floorf(fmaf(tj, rsz, g0z));
            const int lj = ux + 8 * uy + 64 * uz;
            bool ok = ((unsigned)ux < 8u) & ((unsigned)uy < 8u) & ((unsigned)uz < 8u);
#else
            const int jx = ibx + (int)floorf(fmaf(tj, rsx, g0x)), jy = iby + (int)floorf(fmaf(tj, rsy, g0y)),
                      jz = ibz + (int)floorf(fmaf(tj, rsz, g0z));
            const int lj = (jx & 7) + 8 * (jy & 7) + 64 * (jz & 7);
            bool ok = (jx >> 3) == cur.bx && (jy >> 3) == cur.by && (jz >> 3) == cur.bz;
#endif
            if constexpr (kComb) ok = ok && cell_positive(p.comb.cell_pos, cur, lj);
            else ok = ok && (cell_byte(V, cur, lj) & 128);
            run |= (unsigned)ok << j;
          }
          const int n = __ffs(~run) - 1;  // leading certainly-positive points (>= 1)
          if (n >= 2) {
#ifdef DTSDF_STATS
            st_cpi += n - 1;
#endif
            prev_valid = false;
            k += n - 1;
            if (n == kLookahead) continue;  // the run may go on: scan again from its last point
            t = (float)k * V.delta;
            locate(V, p.comb, t);  // the run's last point: evaluate it (prev for the next point)
          }
        }
        break;
      }
    } else {
      locate(V, p.comb, t);
    }
    return true;
  }

  // Evaluate the sample advance() located and update the state; true when the ray is finished
  // (a hit, shaded after the loop).
  __device__ __forceinline__ bool evaluate(const RenderLaunch &p) {
    const VolumeView &V = p.vol;
    const int live = live_;
#ifdef DTSDF_STATS
    const long long c0 = c0_;
#endif
    SampleResult s;
#ifdef DTSDF_STATS
    if (mode == kMarch) { ++st_march; --st_skip; } else ++st_refine;
    const long long c1 = clock64();
    cy_adv += c1 - c0;
#endif
    if (cur.occ) {
      if constexpr (kComb)
        s = eval_comb<false>(V, p.comb, comb_slot(), ix & 7, iy & 7, iz & 7, frx, fry, frz, nullptr);
      else
        s = eval_sample<false>(V, cur, ix & 7, iy & 7, iz & 7, frx, fry, frz, r[0], r[1], r[2], nullptr, live);
    } else {
      s.valid = false;
      s.f = 0.f;
    }
#ifdef DTSDF_STATS
    {
      const long long c2 = clock64();
      if (mode == kMarch) cy_march += c2 - c1; else cy_refine += c2 - c1;
    }
#endif
    if (mode == kMarch) {
      if (!(s.valid && prev_valid && prev_f > 0.0f && s.f <= 0.0f)) {
        prev_valid = s.valid;
        prev_f = s.f;
        ++k;
        return false;
      }
      begin_bracket(p, prev_f, s.f);
    } else if (mode == kBisect) {
      if (!s.valid || s.f > 0.0f) { a = t; fa = s.f; fa_valid = s.valid; }
      else { b = t; fb = s.f; }
      if (++it >= p.n_bisect) { mode = kIllinois; it = 0; }
    } else if (mode == kIllinois) {
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
      if (++it >= 12 || b - a < p.refine_tol) mode = kShade;
    }
    // next position (offset from t_{k-1})
    if (mode == kBisect) {
      t = 0.5f * (a + b);
    } else if (mode == kIllinois) {
#if DTSDF_FAST_NORM
      float m = (fa_valid && fa > fb) ? fmaf(__fdividef(fa, fa - fb), b - a, a) : 0.5f * (a + b);
#else
      float m = (fa_valid && fa > fb) ? fmaf(fa / (fa - fb), b - a, a) : 0.5f * (a + b);
#endif
      if (!(m > a && m < b)) m = 0.5f * (a + b);
      if (!(m > a && m < b)) mode = kShade;  // bracket at the fp32 resolution of the offset
      t = m;
    }
    if (mode == kShade) {  // the hit is b, a valid sample on the surface side (reading R32); a7 runs
                           // after the loop (shade()), with the warp's hit lanes together
      t = b;
      hit = true;
      return true;
    }
    return false;
  }

  __device__ __forceinline__ bool step(const RenderLaunch &p) { return !advance(p) || evaluate(p); }

  // a7 at the hit t = b (refinement frame): the evaluation of the last step again, with the
  // shading sums
  __device__ __forceinline__ void shade(const RenderLaunch &p) {
    locate(p.vol, p.comb, t);
    sh.n[0] = sh.n[1] = sh.n[2] = 0.f;
    sh.c[0] = sh.c[1] = sh.c[2] = 0.f;
    sh.S = 0.f;
    sh.mask = 0;
    if (cur.occ) {
      if constexpr (kComb)
        eval_comb<true>(p.vol, p.comb, comb_slot(), ix & 7, iy & 7, iz & 7, frx, fry, frz, &sh);
      else
        eval_sample<true>(p.vol, cur, ix & 7, iy & 7, iz & 7, frx, fry, frz, r[0], r[1], r[2], &sh);
    }
  }

  // a7 outputs of this ray (zeros for a miss)
  __device__ __forceinline__ void result(const RenderLaunch &p, float &depth, float nrm[3], int col[3], int &mask) const {
    depth = 0.f;
    nrm[0] = nrm[1] = nrm[2] = 0.f;
    col[0] = col[1] = col[2] = 0;
    mask = 0;
    if (hit) {
      // 1 / |d~| of the ray, recomputed with init's operations (the same bits)
      const int u = pix() & 0xffff, v = p.row0 + (pix() >> 16);
      const float dxf = (u - p.cx) / p.fx, dyf = (v - p.cy) / p.fy;
      const float iLf = 1.0f / sqrtf(dxf * dxf + dyf * dyf + 1.0f);
      depth = ((float)(k - 1) * p.vol.delta + b) * iLf;
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
    if (p.dbg_timeline) {
      const size_t pid = ((size_t)view() * (p.row1 - p.row0) + (pix() >> 16)) * p.width + (pix() & 0xffff);
      p.dbg_timeline[3 * pid + 0] = g_start;
      p.dbg_timeline[3 * pid + 1] = g_end;
      p.dbg_timeline[3 * pid + 2] = smid;
    }
    // debug build: normal <- cycles (outside evaluations, march evaluations, refinement
    // evaluations), colour <- counts (march evaluations, refinement evaluations, advance steps)
    nrm[0] = (float)cy_adv; nrm[1] = (float)cy_march; nrm[2] = (float)cy_refine;
    col[0] = min(st_march, 255); col[1] = min(st_refine, 255); col[2] = min(st_empty, 255);
    mask = min(st_cpi, 255) | 0;  // jumps: st_jump (not stored)
#endif
  }

  // per-pixel scalar stores (device outputs)
  __device__ __forceinline__ void store(const RenderLaunch &p) const {
    float depth, nrm[3];
    int col[3], mask;
    result(p, depth, nrm, col, mask);
    const int u = pix() & 0xffff, vrel = pix() >> 16;
    const size_t px = ((size_t)view() * (p.row1 - p.row0) + vrel) * p.width + u;
    DTSDF_CHECK(view() < p.n_views && vrel >= 0 && vrel < p.row1 - p.row0 && u >= 0 && u < p.width);
    p.out_depth[px] = depth;
    if (p.out_normal) {
      p.out_normal[3 * px + 0] = nrm[0];
      p.out_normal[3 * px + 1] = nrm[1];
      p.out_normal[3 * px + 2] = nrm[2];
    }
    if (p.out_color) {
      p.out_color[3 * px + 0] = (unsigned char)col[0];
      p.out_color[3 * px + 1] = (unsigned char)col[1];
      p.out_color[3 * px + 2] = (unsigned char)col[2];
    }
    if (p.out_mask) p.out_mask[px] = (unsigned char)mask;
  }
};

cudaError_t launch_range(const RangeLaunch &p, cudaStream_t s) {
  if (p.n_locations == 0 || p.n_views == 0) return cudaSuccess;
  if (p.n_locations * p.n_views < (1 << 18)) {  // a warp per location while a thread each would fill < 1 wave
    dim3 grid((unsigned)((p.n_locations * 32 + 255) / 256), (unsigned)p.n_views);
    k_range_warp<<<grid, 256, 0, s>>>(p);
  } else {
    dim3 grid((unsigned)((p.n_locations + 255) / 256), (unsigned)p.n_views);
    k_range_thread<<<grid, 256, 0, s>>>(p);
  }
  return cudaGetLastError();
}

bool tile_order_fits(int width, int rows) {
  int cx = 0, cy = 0;
  raycast_tiles(width, rows, &cx, &cy);
  return (long long)cx * cy <= kOrderMaxTiles;
}

void raycast_tiles(int width, int rows, int *ct_x, int *ct_y) {
  *ct_x = (width + kTileW - 1) / kTileW;
  *ct_y = (rows + kTileH - 1) / kTileH;
}

cudaError_t launch_order(unsigned int *count, int *order, int tiles_x, int tiles_y, int width, int rows, int n_views,
                         cudaStream_t s) {
  if (n_views == 0) return cudaSuccess;
  OrderLaunch p;
  p.count = count; p.order = order;
  p.tiles_x = tiles_x; p.tiles_y = tiles_y;
  raycast_tiles(width, rows, &p.ct_x, &p.ct_y);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_order, cudaFuncAttributeMaxDynamicSharedMemorySize, kOrderMaxTiles);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)n_views);
  cfg.blockDim = dim3(DTSDF_ORDER_THREADS);
  cfg.dynamicSmemBytes = (size_t)p.ct_x * p.ct_y;
  cfg.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_order, p);
  return cudaGetLastError();
}

// grid schedule: one CTA per 16 x (2 * DTSDF_CTA / 64)-pixel tile of 8x4-pixel warps, one ray per thread
#ifndef DTSDF_RAYCAST_MINB
#define DTSDF_RAYCAST_MINB (640 / DTSDF_CTA)  // 96 registers per thread: 20 warps per SM (128 was 16 warps:
                                              // 4-6 % slower, profiles/r1f_sweep_regs.jsonl)
#endif
// Copy `n` bytes of one staged output row from shared memory (16-B aligned) to global (device or
// mapped pinned host) memory with the lanes of a warp, in the widest stores (16, 8, 4, 2 or 1 B) that
// the destination alignment and n allow.  Whole rows of the CTA tile leave as contiguous writes,
// which is what a PCIe write to a mapped host buffer needs (strided 4-byte stores would split into
// 4-byte TLPs).
template <typename T>
__device__ __forceinline__ void copy_row_t(unsigned char *dst, const unsigned char *src, int n, int lane) {
  for (int i = lane; i < n / (int)sizeof(T); i += 32)
    reinterpret_cast<T *>(dst)[i] = reinterpret_cast<const T *>(src)[i];
}
__device__ __forceinline__ void copy_row(unsigned char *dst, const unsigned char *src, int n, int lane) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(dst) | (uintptr_t)n;
  if ((a & 15) == 0) copy_row_t<uint4>(dst, src, n, lane);
  else if ((a & 7) == 0) copy_row_t<uint2>(dst, src, n, lane);
  else if ((a & 3) == 0) copy_row_t<unsigned int>(dst, src, n, lane);
  else copy_row_t<unsigned char>(dst, src, n, lane);
}


template <bool kComb>
__global__ void __launch_bounds__(DTSDF_CTA, DTSDF_RAYCAST_MINB) k_raycast(const __grid_constant__ RenderLaunch p) {
  // a7 outputs of the CTA's tile, laid out row by row as in the output arrays (16-B aligned rows)
  __shared__ __align__(16) float s_depth[kTileH][kTileW];
  __shared__ __align__(16) float s_normal[kTileH][3 * kTileW];
  __shared__ __align__(16) unsigned char s_color[kTileH][3 * kTileW];
  __shared__ __align__(16) unsigned char s_mask[kTileH][kTileW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tx = (kTileW == 16 ? (warp & 1) * 8 : 0) + (lane & 7);
  const int ty = (kTileW == 16 ? (warp >> 1) : warp) * 4 + (lane >> 3);
  griddep_wait();  // launched programmatically after the range pass / tile order: their outputs
  // CTA tile: in the view's tile order (longest predicted first, k_order) when there is one; its
  // origin is parked in shared memory for the epilogue instead of a register through the march
  __shared__ int s_origin[2];
  int u0, v0;
  {
    const int ct = p.order ? __ldg(&p.order[(size_t)blockIdx.z * gridDim.x + blockIdx.x]) : blockIdx.x;
    DTSDF_CHECK(ct >= 0 && ct < (int)gridDim.x);
    u0 = (ct % p.ct_x) * kTileW;
    v0 = (ct / p.ct_x) * kTileH;
    if (threadIdx.x == 0) { s_origin[0] = u0; s_origin[1] = v0; }
  }
  const int u = u0 + tx, vrel = v0 + ty;
  const int rows = p.row1 - p.row0;
  const bool inside = u < p.width && vrel < rows;
  RayT<kComb> ray;
#ifdef DTSDF_STATS
  unsigned long long g_start;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
#endif
  if (inside) ray.init(p, blockIdx.z, u, vrel);
#ifdef DTSDF_STATS
  const long long c0 = clock64();
  // per-step trace of one ray: clock at step start, cycles of the step, of its advance, mode
  // before | after << 8, k before, k after, new blocks located, lookahead scans
  // (all 32 lanes of the warp tile whose origin is dbg_trace_pix, 128 steps each)
  const int tu = p.dbg_trace_pix & 0xffff, tv = p.dbg_trace_pix >> 16;
  const bool tr = inside && p.dbg_trace && blockIdx.z == 0 && u - tu >= 0 && u - tu < 8 && vrel - tv >= 0 && vrel - tv < 4;
  long long *tb = p.dbg_trace + (tr ? 8 * 128 * ((u - tu) + 8 * (vrel - tv)) : 0);
  int n_tr = 0;
#endif
  if (inside) {
#ifdef DTSDF_STATS
    for (;;) {
      const long long s0 = clock64(), a0 = ray.cy_adv;
      const int m0 = ray.mode, k0 = ray.k, nb0 = ray.st_newblk, ns0 = ray.st_scan, nl0 = ray.st_loc,
                nj0 = ray.st_jump, ne0 = ray.st_empty;
      const bool done = ray.step(p);
      if (tr && n_tr < 127) {
        long long *e = tb + 8 * n_tr++;
        e[0] = s0; e[1] = clock64() - s0; e[2] = ray.cy_adv - a0; e[3] = m0 | (ray.mode << 8) | (ray.hit << 16);
        e[4] = k0; e[5] = ray.k; e[6] = (ray.st_newblk - nb0) | ((long long)(ray.st_loc - nl0) << 16);
        e[7] = (ray.st_scan - ns0) | ((long long)(ray.st_jump - nj0) << 16) | ((long long)(ray.st_empty - ne0) << 32);
      }
      if (done) break;
    }
#else
    while (!ray.step(p)) {
    }
#endif
  }
#ifdef DTSDF_STATS
  if (tr) tb[8 * n_tr] = -1;
#endif
  if (inside) {
    if (ray.hit) ray.shade(p);
#ifdef DTSDF_STATS
    ray.cy_adv = clock64() - c0 - ray.cy_march - ray.cy_refine;  // everything outside the evaluations
    unsigned long long g_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
    ray.g_start = g_start;
    ray.g_end = g_end;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    ray.smid = smid;
#endif
    if (!p.staged) {  // device outputs: per-pixel stores straight from the ray
      ray.store(p);
      return;
    }
    float depth, nrm[3];
    int col[3], mask;
    ray.result(p, depth, nrm, col, mask);
    s_depth[ty][tx] = depth;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      s_normal[ty][3 * tx + q] = nrm[q];
      s_color[ty][3 * tx + q] = (unsigned char)col[q];
    }
    s_mask[ty][tx] = (unsigned char)mask;
  }
  if (!p.staged) return;  // uniform per launch
  __syncthreads();
  u0 = s_origin[0];
  v0 = s_origin[1];
  // each warp writes whole rows of the tile, array by array
  const int nu = min(kTileW, p.width - u0);
  for (int row = warp; row < kTileH; row += DTSDF_CTA / 32) {
    if (v0 + row >= rows) break;
    const size_t pix = ((size_t)blockIdx.z * rows + v0 + row) * p.width + u0;
    DTSDF_CHECK(blockIdx.z < p.n_views && nu > 0);
    unsigned char *d0 = reinterpret_cast<unsigned char *>(p.out_depth + pix);
    unsigned char *d1 = p.out_normal ? reinterpret_cast<unsigned char *>(p.out_normal + 3 * pix) : nullptr;
    unsigned char *d2 = p.out_color ? p.out_color + 3 * pix : nullptr;
    unsigned char *d3 = p.out_mask ? p.out_mask + pix : nullptr;
    copy_row(d0, reinterpret_cast<const unsigned char *>(s_depth[row]), 4 * nu, lane);
    if (d1) copy_row(d1, reinterpret_cast<const unsigned char *>(s_normal[row]), 12 * nu, lane);
    if (d2) copy_row(d2, s_color[row], 3 * nu, lane);
    if (d3) copy_row(d3, s_mask[row], nu, lane);
  }
}

template <bool kComb>
static cudaError_t launch_raycast_t(const RenderLaunch &p, cudaStream_t s) {
  const int ct_y = (p.row1 - p.row0 + kTileH - 1) / kTileH;
  dim3 grid((unsigned)(p.ct_x * ct_y), 1u, (unsigned)p.n_views);
  return launch_pdl(k_raycast<kComb>, grid, dim3(DTSDF_CTA), s, p);
  return cudaGetLastError();
}

cudaError_t launch_raycast(const RenderLaunch &p, cudaStream_t s) {
  if (p.n_views == 0) return cudaSuccess;
  return p.combined ? launch_raycast_t<true>(p, s) : launch_raycast_t<false>(p, s);
}

}  // namespace dtsdf
