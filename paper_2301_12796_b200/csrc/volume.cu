// volume.cu -- index build for a committed volume.
//
//   validate + AABB     one thread per block: D in 0..5, coordinates in range, AABB min/max
//   insert              one thread per block: open-addressing insert of the location key
//                       (64-bit CAS, linear probing), then CAS of the direction slot; a slot
//                       already taken means a duplicate (x,y,z,D) key
//   bitmap              one thread per location: occupancy bit over the location AABB
//   bricks              one CTA per block: each (location, D) brick gets the records of voxels
//                       0..8 of its block per axis gathered from up to 27 neighbouring blocks of
//                       the same direction -- sdf (NaN where that neighbour is unallocated),
//                       weight, the three per-voxel central differences and the colour -- so one
//                       brick serves a whole sample (8 trilinear corners carrying the gradient
//                       stencil) with a single index lookup
//
// Slot placement in the table depends on insertion order; lookups do not.
#include "common.cuh"

namespace dtsdf {

__global__ void k_validate_aabb(const int4 *__restrict__ keys, long long n, int *flags, int *aabb) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int4 k = keys[i];
  const int lim = 1 << 20;
  if (k.w < 0 || k.w > 5 || k.x < -lim || k.x >= lim || k.y < -lim || k.y >= lim || k.z < -lim || k.z >= lim) {
    atomicExch(&flags[0], 1);
    return;
  }
  atomicMin(&aabb[0], k.x);
  atomicMin(&aabb[1], k.y);
  atomicMin(&aabb[2], k.z);
  atomicMax(&aabb[3], k.x);
  atomicMax(&aabb[4], k.y);
  atomicMax(&aabb[5], k.z);
}

// Voxel values: sdf must be finite (the apron bricks use NaN as their "unallocated" sentinel, so a
// NaN in the input would silently read as an absent direction) and weights finite and >= 0
// (eq:combine_weight and eq:combine_tsdf_weight are proportional to the weight).  flags[3] <- 1.
__global__ void __launch_bounds__(256) k_validate_values(const float4 *__restrict__ sdf, const float4 *__restrict__ w,
                                                         long long n4, int *flags) {
  bool bad = false;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    const float4 a = __ldg(sdf + i), b = __ldg(w + i);
    bad |= !isfinite(a.x) | !isfinite(a.y) | !isfinite(a.z) | !isfinite(a.w);
    bad |= !(b.x >= 0.f) | !(b.y >= 0.f) | !(b.z >= 0.f) | !(b.w >= 0.f);
    bad |= isinf(b.x) | isinf(b.y) | isinf(b.z) | isinf(b.w);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(&flags[3], 1);
}

__device__ __forceinline__ int find_entry(const HashEntry *__restrict__ table, unsigned int mask,
                                          unsigned long long key) {
  unsigned int h = hash_key(key) & mask;
  for (unsigned int probe = 0; probe <= mask; ++probe) {
    unsigned long long k = table[h].key;
    if (k == key) return (int)h;
    if (k == kEmptyKey) return -1;
    h = (h + 1) & mask;
  }
  return -1;
}

__global__ void k_insert(const int4 *__restrict__ keys, long long n, HashEntry *table, unsigned int mask,
                         int4 *locations, int *flags, unsigned long long *n_loc) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int4 k = keys[i];
  unsigned long long key = pack_key(k.x, k.y, k.z);
  unsigned int h = hash_key(key) & mask;
  for (unsigned int probe = 0; probe <= mask; ++probe) {
    unsigned long long prev = atomicCAS(&table[h].key, kEmptyKey, key);
    if (prev == kEmptyKey) {  // claimed a new location
      unsigned long long u = atomicAdd(n_loc, 1ull);
      locations[u] = make_int4(k.x, k.y, k.z, (int)h);
    }
    if (prev == kEmptyKey || prev == key) {
      int old = atomicCAS(&table[h].slot[k.w], -1, (int)i);
      if (old != -1) atomicExch(&flags[1], 1);
      return;
    }
    h = (h + 1) & mask;
  }
  atomicExch(&flags[2], 1);
}

__global__ void k_bitmap(const int4 *__restrict__ loc, long long n_loc, unsigned int *bitmap, int lo_x, int lo_y,
                         int lo_z, int dim_x, int dim_y) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_loc) return;
  int4 b = loc[i];
  long long cell = ((long long)(b.z - lo_z) * dim_y + (b.y - lo_y)) * dim_x + (b.x - lo_x);
  atomicOr(&bitmap[cell >> 5], 1u << (cell & 31));
}

// Record bricks (common.cuh kRec*): one CTA per block.  The 27 neighbour slots (same direction) are
// resolved once into shared memory -- a hash probe per neighbour instead of one per record -- the
// sdf of voxels -1..9 per axis is staged in shared memory (NaN where the neighbour block is
// unallocated), then the CTA writes the 729 records of voxels 0..8: A {sdf, weight, dsdf_x,
// dsdf_y}, B {dsdf_z, rgb} with dsdf_a = sdf(+e_a) - sdf(-e_a) (one fp32 subtraction, NaN if
// either neighbour is absent), with coalesced stores.
constexpr int kBrickThreads = 256;
constexpr int kStage = 11;  // staged sdf: voxels -1..9 per axis

// Source of a staged voxel: (neighbour index (ox+1) + 3 (oy+1) + 9 (oz+1)) << 9 | that block's
// local index l, for the 11^3 staged voxels -1..9 (kStageSrc) and the 9^3 record voxels 0..8
// (kRecSrc); built at compile time, so the staging loops do no index arithmetic.
struct SrcTable {
  unsigned short stage[kStage * kStage * kStage];
  unsigned short rec[kRecVox];
  unsigned short rec_c[kRecVox];  // staged index of record voxel a
  static constexpr unsigned short src(int lx, int ly, int lz) {
    const int ox = lx < 0 ? -1 : (lx >= kBlock ? 1 : 0), oy = ly < 0 ? -1 : (ly >= kBlock ? 1 : 0),
              oz = lz < 0 ? -1 : (lz >= kBlock ? 1 : 0);
    const int l = (lx - ox * kBlock) + kBlock * (ly - oy * kBlock) + kBlock * kBlock * (lz - oz * kBlock);
    return (unsigned short)((((ox + 1) + 3 * (oy + 1) + 9 * (oz + 1)) << 9) | l);
  }
  constexpr SrcTable() : stage(), rec(), rec_c() {
    for (int a = 0; a < kStage * kStage * kStage; ++a)
      stage[a] = src(a % kStage - 1, (a / kStage) % kStage - 1, a / (kStage * kStage) - 1);
    for (int a = 0; a < kRecVox; ++a) {
      const int lx = a % kRec, ly = (a / kRec) % kRec, lz = a / (kRec * kRec);
      rec[a] = src(lx, ly, lz);
      rec_c[a] = (unsigned short)((lx + 1) + kStage * (ly + 1) + kStage * kStage * (lz + 1));
    }
  }
};
__device__ const SrcTable kSrc = SrcTable();
#ifndef DTSDF_BRICK_MINB
#define DTSDF_BRICK_MINB 8  // 32 registers, 8 CTAs per SM: fused frame kernels -17 % (profiles/r3_ab_fusion.txt)
#endif
#ifndef DTSDF_BRICK_RES
#define DTSDF_BRICK_RES 8
#endif
__global__ void __launch_bounds__(kBrickThreads, DTSDF_BRICK_MINB) k_bricks(const int4 *__restrict__ keys, const HashEntry *__restrict__ table,
                                                         unsigned int mask, const float *__restrict__ sdf,
                                                         const float *__restrict__ weight, const unsigned char *__restrict__ rgb,
                                                         float4 *__restrict__ brick_a, float2 *__restrict__ brick_b,
                                                         unsigned int *__restrict__ cell_dirs32,
                                                         const int *__restrict__ list,
                                                         const unsigned long long *__restrict__ count,
                                                         const GridRef gr) {
  __shared__ int nb[27];  // slot of neighbour (ox, oy, oz) in -1..1, index (ox+1) + 3 (oy+1) + 9 (oz+1)
  __shared__ int self_entry;
  __shared__ float st[kStage * kStage * kStage];
  __shared__ float sw[kRecVox];
  __shared__ unsigned int sc[kRecVox];
  // blocks: one per CTA (list null or uncounted), or a grid-stride loop over a device-counted list
  const long long n_items = count ? (long long)*count : (long long)gridDim.x;
  for (long long item = blockIdx.x; item < n_items; item += count ? gridDim.x : n_items) {
  const long long b = list ? (long long)list[item] : item;
  const int4 k = keys[b];
  __syncthreads();  // the previous item's readers of nb / st / sw / sc are done
  if (threadIdx.x < 27) {
    const int ox = (int)threadIdx.x % 3 - 1, oy = ((int)threadIdx.x / 3) % 3 - 1, oz = (int)threadIdx.x / 9 - 1;
    int src = (int)b;
    const int e = gr.grid ? gr.entry(k.x + ox, k.y + oy, k.z + oz) : find_entry(table, mask, pack_key(k.x + ox, k.y + oy, k.z + oz));
    if (ox | oy | oz) src = (e >= 0) ? table[e].slot[k.w] : -1;
    else self_entry = e;
    nb[threadIdx.x] = src;
  }
  __syncthreads();
  // pool record of a table entry (neighbour << 9 | local index), or -1 when that block is unallocated
  auto rec_of = [&](unsigned int e) -> long long {
    const int src = nb[e >> 9];
    return src < 0 ? -1 : (long long)src * kVoxPerBlock + (e & 511);
  };
  // staging, unrolled so that each thread's loads are in flight together
#pragma unroll
  for (int kk = 0; kk < (kStage * kStage * kStage + kBrickThreads - 1) / kBrickThreads; ++kk) {
    const int a = threadIdx.x + kk * kBrickThreads;
    if (a < kStage * kStage * kStage) {
      const long long r = rec_of(kSrc.stage[a]);
      st[a] = r >= 0 ? __ldg(sdf + r) : __int_as_float(0x7fc00000);  // NaN sdf = unallocated
    }
  }
#pragma unroll
  for (int kk = 0; kk < (kRecVox + kBrickThreads - 1) / kBrickThreads; ++kk) {
    const int a = threadIdx.x + kk * kBrickThreads;
    if (a < kRecVox) {
      const long long r = rec_of(kSrc.rec[a]);
      sw[a] = r >= 0 ? __ldg(weight + r) : 0.0f;
      unsigned int col = 0;
      if (r >= 0 && rgb != nullptr) {
        const unsigned char *q = rgb + 3 * r;
        col = (unsigned int)__ldg(q) | ((unsigned int)__ldg(q + 1) << 8) | ((unsigned int)__ldg(q + 2) << 16);
      }
      sc[a] = col;
    }
  }
  __syncthreads();
  for (int a = threadIdx.x; a < kRecStride; a += kBrickThreads) {
    float4 ra = make_float4(__int_as_float(0x7fc00000), 0.0f, __int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
    float2 rb = make_float2(__int_as_float(0x7fc00000), 0.0f);
    if (a < kRecVox) {
      const int c = kSrc.rec_c[a];  // voxels 0..8: staged index
      ra.x = st[c];
      ra.y = sw[a];
      ra.z = st[c + 1] - st[c - 1];
      ra.w = st[c + kStage] - st[c - kStage];
      rb.x = st[c + kStage * kStage] - st[c - kStage * kStage];
      rb.y = __uint_as_float(sc[a]);
    }
    brick_a[b * kRecStride + a] = ra;
    brick_b[b * kRecStride + a] = rb;
  }
  // This direction's share of the location's live-direction byte per base cell (render.cu
  // cell_byte): bit D when no corner is unallocated and some corner weight is > 0 (the evaluation
  // drops D otherwise); bit 7, "certainly positive", cleared when all corners are allocated and
  // one has sdf <= 0.  The location's bytes start at 0x80 (k_cell_init / the commit's memset).
  if (cell_dirs32 == nullptr || self_entry < 0) continue;  // CTA-uniform
  for (int l = threadIdx.x; l < kVoxPerBlock; l += kBrickThreads) {
    const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
    bool absent = false, allpos = true, weighted = false;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int dx = q & 1, dy = (q >> 1) & 1, dz = q >> 2;
      const float v = st[(lx + dx + 1) + kStage * (ly + dy + 1) + kStage * kStage * (lz + dz + 1)];
      absent |= isnan(v);
      allpos &= v > 0.0f;
      weighted |= sw[(lx + dx) + kRec * (ly + dy) + kRec * kRec * (lz + dz)] > 0.0f;
    }
    // the 4 cells of one 32-bit word sit in 4 consecutive lanes: combine their bits first, one
    // atomic per word and only when it changes something
    const int sh = (l & 3) * 8;
    unsigned int orb = (!absent && weighted) ? (1u << k.w) << sh : 0u;
    unsigned int andb = (!absent && !allpos) ? ~(0x80u << sh) : 0xffffffffu;
    orb |= __shfl_xor_sync(0xffffffffu, orb, 1);
    andb &= __shfl_xor_sync(0xffffffffu, andb, 1);
    orb |= __shfl_xor_sync(0xffffffffu, orb, 2);
    andb &= __shfl_xor_sync(0xffffffffu, andb, 2);
    if ((l & 3) == 0) {
      unsigned int *w = cell_dirs32 + ((size_t)self_entry * kVoxPerBlock + l) / 4;
      if (orb) atomicOr(w, orb);
      if (andb != 0xffffffffu) atomicAnd(w, andb);
    }
  }
  }
}

// The live-direction bytes of the listed locations' entries set to 0x80 (no direction live,
// certainly positive) before their bricks are rebuilt (incremental commit).
// (count non-null: the number of listed locations is *count, read on the device; grid-stride)
__global__ void k_cell_init(const int4 *__restrict__ loc, long long n, unsigned int *cell_dirs32,
                            const unsigned long long *count) {
  if (count) n = (long long)*count;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < n * 128; g += (long long)gridDim.x * blockDim.x)
    cell_dirs32[(size_t)loc[g >> 7].w * (kVoxPerBlock / 4) + (g & 127)] = 0x80808080u;
}

// One warp per location: the certainly-positive masks (bit l of cell_pos[entry][l / 32]) from bit 7
// of the live-direction bytes, and the location's surface bit -- set unless every base cell is
// certainly positive (then every sample whose base voxel lies in the location has F > 0 or is
// invalid, and the march may jump to the location's last lattice points, exact).  The surface bit
// is cleared first (a re-built location may have lost its surface).
__global__ void k_cell_masks(const int4 *__restrict__ loc, long long n, const unsigned char *__restrict__ cell_dirs,
                             unsigned int *cell_pos, unsigned int *surface, int lo_x, int lo_y, int lo_z, int dim_x,
                             int dim_y, const unsigned long long *count) {
  if (count) n = (long long)*count;
  const int lane = threadIdx.x & 31;
  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((long long)gridDim.x * blockDim.x) >> 5) {  // warp-uniform
  const int4 b = loc[i];
  bool all_pos = true;
#pragma unroll
  for (int h = 0; h < 16; ++h) {
    const int l = h * 32 + lane;
    const bool cp = (cell_dirs[(size_t)b.w * kVoxPerBlock + l] & 0x80) != 0;
    const unsigned int word = __ballot_sync(0xffffffffu, cp);
    if (lane == 0) cell_pos[(size_t)b.w * 16 + h] = word;
    all_pos &= word == 0xffffffffu;
  }
  if (lane == 0) {
    const long long cell = ((long long)(b.z - lo_z) * dim_y + (b.y - lo_y)) * dim_x + (b.x - lo_x);
    if (all_pos) atomicAnd(&surface[cell >> 5], ~(1u << (cell & 31)));
    else atomicOr(&surface[cell >> 5], 1u << (cell & 31));
  }
  }
}

// Dense location grid: for each allocated location, its hash entry index, present directions and
// surface bit (kGridEntryBits layout), so the raycast resolves a location -- and knows which
// directions it holds -- with one 4-B load instead of bitmap + surface + hash probe + entry.
__global__ void k_loc_grid(const int4 *__restrict__ loc, long long n_loc, const unsigned int *__restrict__ surface,
                           const HashEntry *__restrict__ table, int *grid, int lo_x, int lo_y, int lo_z, int dim_x,
                           int dim_y, const unsigned long long *count) {
  if (count) n_loc = (long long)*count;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n_loc; i += (long long)gridDim.x * blockDim.x) {
    const int4 b = loc[i];
    const long long cell = ((long long)(b.z - lo_z) * dim_y + (b.y - lo_y)) * dim_x + (b.x - lo_x);
    const int surf = (surface[cell >> 5] >> (cell & 31)) & 1;
    int present = 0;
    for (int d = 0; d < 6; ++d) present |= (table[b.w].slot[d] >= 0) << d;
    grid[cell] = b.w | (present << kGridEntryBits) | (surf << 30);
  }
}

// Empty-space distance on the location grid (L-infinity, in blocks, capped): separable passes
// d_x(c) = min{|dx| : c + dx e_x occupied}, then d_xy(c) = min_dy max(|dy|, d_x(c + dy e_y)), then
// the same along z.  An empty location with distance d has no allocated location within d - 1
// blocks, so a ray may skip the whole (2d - 1)^3-block cube around it (render.cu, exact).
constexpr int kDistCap = 31;
__global__ void k_dist_pass(const int *__restrict__ grid, const unsigned char *__restrict__ in,
                            unsigned char *__restrict__ out, int axis, int dim_x, int dim_y, int dim_z) {
  const long long cells = (long long)dim_x * dim_y * dim_z;
  long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells) return;
  const int x = (int)(c % dim_x), y = (int)((c / dim_x) % dim_y), z = (int)(c / ((long long)dim_x * dim_y));
  const int pos = axis == 0 ? x : (axis == 1 ? y : z);
  const int n = axis == 0 ? dim_x : (axis == 1 ? dim_y : dim_z);
  const long long stride = axis == 0 ? 1 : (axis == 1 ? dim_x : (long long)dim_x * dim_y);
  int best = kDistCap;
  for (int d = -kDistCap; d <= kDistCap; ++d) {
    const int q = pos + d;
    if (q < 0 || q >= n) continue;
    const int ad = d < 0 ? -d : d;
    if (ad >= best) continue;
    const long long cq = c + d * stride;
    const int v = (axis == 0) ? (grid[cq] >= 0 ? 0 : kDistCap) : in[cq];
    const int m = ad > v ? ad : v;
    if (m < best) best = m;
  }
  out[c] = (unsigned char)best;
}

__global__ void k_dist_store(int *grid, const unsigned char *__restrict__ dist, long long cells) {
  long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells) return;
  const int d = dist[c] > 1 ? (int)dist[c] : 1;
#if DTSDF_EMPTY_BOX
  if (grid[c] < 0) grid[c] = -(1 + box_cube(d - 1));  // the cube of radius d - 1 (kDistCap = kBoxMax)
#else
  if (grid[c] < 0) grid[c] = -d;
#endif
}

// Summed-volume table of occupancy: sat[k][j][i] = allocated locations with x < i, y < j, z < k.
__global__ void k_sat_fill(const int *__restrict__ grid, int *sat, int dx, int dy, int dz) {
  const long long n = (long long)(dx + 1) * (dy + 1) * (dz + 1);
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int i = (int)(c % (dx + 1)), j = (int)((c / (dx + 1)) % (dy + 1)), k = (int)(c / ((long long)(dx + 1) * (dy + 1)));
  sat[c] = (i > 0 && j > 0 && k > 0) ? (grid[((long long)(k - 1) * dy + (j - 1)) * dx + (i - 1)] >= 0) : 0;
}
// inclusive prefix sums along one axis, one thread per line
__global__ void k_sat_scan(int *sat, int axis, int dx, int dy, int dz) {
  const int nx = dx + 1, ny = dy + 1, nz = dz + 1;
  const long long lines = axis == 0 ? (long long)ny * nz : (axis == 1 ? (long long)nx * nz : (long long)nx * ny);
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= lines) return;
  long long base, stride;
  int len;
  if (axis == 0) { base = t * nx; stride = 1; len = nx; }
  else if (axis == 1) { base = (t / nx) * (long long)nx * ny + (t % nx); stride = nx; len = ny; }
  else { base = t; stride = (long long)nx * ny; len = nz; }
  int acc = 0;
  for (int q = 0; q < len; ++q) {
    acc += sat[base + q * stride];
    sat[base + q * stride] = acc;
  }
}
// allocated locations in the box [x0, x1] x [y0, y1] x [z0, z1], clipped to the grid (outside it
// nothing is allocated)
__device__ __forceinline__ int sat_count(const int *__restrict__ sat, int dx, int dy, int dz, int x0, int x1, int y0,
                                         int y1, int z0, int z1) {
  x0 = max(x0, 0); y0 = max(y0, 0); z0 = max(z0, 0);
  x1 = min(x1, dx - 1); y1 = min(y1, dy - 1); z1 = min(z1, dz - 1);
  if (x0 > x1 || y0 > y1 || z0 > z1) return 0;
  const long long sx = 1, sy = dx + 1, sz = (long long)(dx + 1) * (dy + 1);
  auto at = [&](int i, int j, int k) {
    DTSDF_CHECK(i >= 0 && i <= dx && j >= 0 && j <= dy && k >= 0 && k <= dz);
    return __ldg(&sat[k * sz + j * sy + i * sx]);
  };
  ++x1; ++y1; ++z1;
  return at(x1, y1, z1) - at(x0, y1, z1) - at(x1, y0, z1) - at(x1, y1, z0) + at(x0, y0, z1) + at(x0, y1, z0) +
         at(x1, y0, z0) - at(x0, y0, z0);
}
// Grow each empty location's box from its distance cube: one layer at a time per face, round
// robin, while the new layer holds no allocated location (counted exactly with the table), up to
// kBoxMax blocks per face.  The box stays all-empty, so a ray inside it meets no allocated block
// before its exit (exact skipping).
__global__ void k_empty_box(int *grid, const int *__restrict__ sat, int dx, int dy, int dz) {
  const long long cells = (long long)dx * dy * dz;
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cells) return;
  const int gv = grid[c];
  if (gv >= 0) return;
  const int x = (int)(c % dx), y = (int)((c / dx) % dy), z = (int)(c / ((long long)dx * dy));
  const int packed = -gv - 1;
  int e[6];
#pragma unroll
  for (int f = 0; f < 6; ++f) e[f] = (packed >> (kBoxBits * f)) & kBoxMax;
  unsigned grow = 0x3f;
  while (grow) {
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      if (!((grow >> f) & 1)) continue;
      if (e[f] >= kBoxMax) { grow &= ~(1u << f); continue; }
      int b[6] = {x - e[0], x + e[1], y - e[2], y + e[3], z - e[4], z + e[5]};
      // the new layer beyond face f
      const int ax = f >> 1;
      if (f & 1) { b[2 * ax] = b[2 * ax + 1] + 1; b[2 * ax + 1] = b[2 * ax]; }
      else { b[2 * ax + 1] = b[2 * ax] - 1; b[2 * ax] = b[2 * ax + 1]; }
      if (sat_count(sat, dx, dy, dz, b[0], b[1], b[2], b[3], b[4], b[5]) == 0) ++e[f];
      else grow &= ~(1u << f);
    }
  }
  int np = 0;
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    DTSDF_CHECK(e[f] >= 0 && e[f] <= kBoxMax);
    np |= e[f] << (kBoxBits * f);
  }
  grid[c] = -(1 + np);
}


static inline unsigned int grid_for(long long n, int threads) { return (unsigned int)((n + threads - 1) / threads); }

cudaError_t launch_validate_aabb(const int4 *keys, long long n, CommitScratch sc, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_validate_aabb<<<grid_for(n, 256), 256, 0, s>>>(keys, n, sc.flags, sc.aabb);
  return cudaGetLastError();
}

cudaError_t launch_validate_values(const float *sdf, const float *weight, long long n, CommitScratch sc,
                                   cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const long long n4 = n * (kVoxPerBlock / 4);
  const long long blocks = std::min<long long>((n4 + 255) / 256, 148LL * 8);  // grid-stride, 8 CTAs per SM
  k_validate_values<<<(unsigned)blocks, 256, 0, s>>>(reinterpret_cast<const float4 *>(sdf),
                                                     reinterpret_cast<const float4 *>(weight), n4, sc.flags);
  return cudaGetLastError();
}

cudaError_t launch_insert(const int4 *keys, long long n, HashEntry *table, unsigned int mask, int4 *locations,
                          CommitScratch sc, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_insert<<<grid_for(n, 256), 256, 0, s>>>(keys, n, table, mask, locations, sc.flags, sc.n_loc);
  return cudaGetLastError();
}

cudaError_t launch_bitmap(const int4 *locations, long long n_loc, unsigned int *bitmap, int lo_x, int lo_y, int lo_z,
                          int dim_x, int dim_y, cudaStream_t s) {
  if (n_loc == 0) return cudaSuccess;
  k_bitmap<<<grid_for(n_loc, 256), 256, 0, s>>>(locations, n_loc, bitmap, lo_x, lo_y, lo_z, dim_x, dim_y);
  return cudaGetLastError();
}

// Launch grid for n items of `per` threads each, at most `cap` CTAs of 256 when the item count is
// read on the device (count non-null, n an upper bound): a grid-stride loop covers the rest.
static unsigned grid_counted(long long n, long long per, const unsigned long long *count, unsigned cap) {
  const unsigned g = grid_for(n * per, 256);
  return count && g > cap ? cap : g;
}

cudaError_t launch_loc_grid(const int4 *locations, long long n_loc, const unsigned int *surface, const HashEntry *table,
                            int *grid, int lo_x, int lo_y, int lo_z, int dim_x, int dim_y, cudaStream_t s,
                            const unsigned long long *count) {
  if (n_loc == 0) return cudaSuccess;
  k_loc_grid<<<grid_counted(n_loc, 1, count, 148 * 2), 256, 0, s>>>(locations, n_loc, surface, table, grid, lo_x, lo_y,
                                                                  lo_z, dim_x, dim_y, count);
  return cudaGetLastError();
}

cudaError_t launch_empty_distance(int *grid, unsigned char *tmp0, unsigned char *tmp1, int dim_x, int dim_y, int dim_z,
                                  cudaStream_t s) {
  const long long cells = (long long)dim_x * dim_y * dim_z;
  if (cells == 0) return cudaSuccess;
  k_dist_pass<<<grid_for(cells, 256), 256, 0, s>>>(grid, nullptr, tmp0, 0, dim_x, dim_y, dim_z);
  k_dist_pass<<<grid_for(cells, 256), 256, 0, s>>>(grid, tmp0, tmp1, 1, dim_x, dim_y, dim_z);
  k_dist_pass<<<grid_for(cells, 256), 256, 0, s>>>(grid, tmp1, tmp0, 2, dim_x, dim_y, dim_z);
  k_dist_store<<<grid_for(cells, 256), 256, 0, s>>>(grid, tmp0, cells);
  return cudaGetLastError();
}


cudaError_t launch_empty_box(int *grid, int *sat, int dim_x, int dim_y, int dim_z, cudaStream_t s) {
  const long long cells = (long long)dim_x * dim_y * dim_z;
  if (cells == 0) return cudaSuccess;
  const long long n = (long long)(dim_x + 1) * (dim_y + 1) * (dim_z + 1);
  k_sat_fill<<<grid_for(n, 256), 256, 0, s>>>(grid, sat, dim_x, dim_y, dim_z);
  k_sat_scan<<<grid_for((long long)(dim_y + 1) * (dim_z + 1), 128), 128, 0, s>>>(sat, 0, dim_x, dim_y, dim_z);
  k_sat_scan<<<grid_for((long long)(dim_x + 1) * (dim_z + 1), 128), 128, 0, s>>>(sat, 1, dim_x, dim_y, dim_z);
  k_sat_scan<<<grid_for((long long)(dim_x + 1) * (dim_y + 1), 128), 128, 0, s>>>(sat, 2, dim_x, dim_y, dim_z);
  k_empty_box<<<grid_for(cells, 128), 128, 0, s>>>(grid, sat, dim_x, dim_y, dim_z);
  return cudaGetLastError();
}

cudaError_t launch_bricks(const int4 *keys, long long n, const HashEntry *table, unsigned int mask, const float *sdf,
                          const float *weight, const unsigned char *rgb, float4 *brick_a, float2 *brick_b,
                          unsigned char *cell_dirs, const int *list, const GridRef &gr, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_bricks<<<(unsigned)n, kBrickThreads, 0, s>>>(keys, table, mask, sdf, weight, rgb, brick_a, brick_b,
                                                reinterpret_cast<unsigned int *>(cell_dirs), list, nullptr, gr);
  return cudaGetLastError();
}

cudaError_t launch_bricks_counted(const int4 *keys, long long grid, const unsigned long long *count,
                                  const HashEntry *table, unsigned int mask, const float *sdf, const float *weight,
                                  const unsigned char *rgb, float4 *brick_a, float2 *brick_b, unsigned char *cell_dirs,
                                  const int *list, const GridRef &gr, cudaStream_t s) {
  if (grid == 0) return cudaSuccess;
  // a grid-stride loop over the counted list: the CTAs resident at once (8 of 256 per SM, 148 SMs)
  const long long ctas = grid < 148LL * DTSDF_BRICK_RES ? grid : 148LL * DTSDF_BRICK_RES;
  k_bricks<<<(unsigned)ctas, kBrickThreads, 0, s>>>(keys, table, mask, sdf, weight, rgb, brick_a, brick_b,
                                                   reinterpret_cast<unsigned int *>(cell_dirs), list, count, gr);
  return cudaGetLastError();
}

// ---- incremental commit after a fused frame ----------------------------------------------
// A block's record brick reads voxels -1..9 of its block, i.e. all 26 neighbours in its
// direction; a location's live-direction bytes combine all its directions.  So a dirty block
// (changed voxels, or new) invalidates the bricks of its 27-neighbourhood in its direction, and
// every location holding one of those is rebuilt whole (all its directions' bricks).
__global__ void k_inc_mark(const int4 *__restrict__ keys, long long b0, long long n,
                           const unsigned char *__restrict__ dirty, const HashEntry *__restrict__ table,
                           unsigned int mask, const int *__restrict__ grid, int lo_x, int lo_y, int lo_z, int dim_x,
                           int dim_y, int dim_z, int *loc_mark, int4 *loc_list, unsigned long long *ctr) {
  // one thread per (block, neighbour q): the 27 lookups of a block run in parallel
  const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long b = b0 + g / 27;
  const int q = (int)(g % 27);
  if (b >= n || !dirty[b]) return;
  const int4 k = keys[b];
  const int ox = q % 3 - 1, oy = (q / 3) % 3 - 1, oz = q / 9 - 1;
  int e = -1;
  if (grid) {  // the dense location grid: one load instead of a hash probe
    const unsigned x = (unsigned)(k.x + ox - lo_x), y = (unsigned)(k.y + oy - lo_y), z = (unsigned)(k.z + oz - lo_z);
    if (x < (unsigned)dim_x && y < (unsigned)dim_y && z < (unsigned)dim_z) {
      const int gv = grid[((size_t)z * dim_y + y) * dim_x + x];
      e = gv >= 0 ? (gv & kGridEntryMask) : -1;
    }
    // (the locations this frame added were entered into the grid before this kernel)
  } else {
    e = find_entry(table, mask, pack_key(k.x + ox, k.y + oy, k.z + oz));
  }
  if (e < 0 || table[e].slot[k.w] < 0) return;
  if (atomicCAS(&loc_mark[e], 0, 1) != 0) return;
  const unsigned long long i = atomicAdd(&ctr[0], 1ull);
  loc_list[i] = make_int4(k.x + ox, k.y + oy, k.z + oz, e);
}

__global__ void k_inc_blocks(const int4 *__restrict__ loc_list, long long n, const HashEntry *__restrict__ table,
                             int *blk_list, unsigned long long *ctr) {
  n = (long long)ctr[0];  // the listed locations (k_fuse / k_inc_mark counted them)
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int e = loc_list[i].w;
#pragma unroll
    for (int D = 0; D < 6; ++D) {
      const int b = table[e].slot[D];
      if (b >= 0) blk_list[atomicAdd(&ctr[1], 1ull)] = b;
    }
  }
}

__global__ void k_inc_unmark(const int4 *__restrict__ loc_list, long long n, int *loc_mark,
                             const unsigned long long *count) {
  if (count) n = (long long)*count;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    loc_mark[loc_list[i].w] = 0;
}

cudaError_t launch_inc_mark(const int4 *keys, long long b0, long long n, const unsigned char *dirty,
                            const HashEntry *table, unsigned int mask, const int *grid, const int lo[3], const int dim[3],
                            int *loc_mark, int4 *loc_list, unsigned long long *ctr, cudaStream_t s) {
  if (n <= b0) return cudaSuccess;
  k_inc_mark<<<grid_for((n - b0) * 27, 256), 256, 0, s>>>(keys, b0, n, dirty, table, mask, grid, lo[0], lo[1], lo[2],
                                                          dim[0], dim[1], dim[2], loc_mark, loc_list, ctr);
  return cudaGetLastError();
}

cudaError_t launch_inc_blocks(const int4 *loc_list, long long n, const HashEntry *table, int *blk_list,
                              unsigned long long *ctr, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_inc_blocks<<<grid_counted(n, 1, ctr, 148 * 2), 256, 0, s>>>(loc_list, n, table, blk_list, ctr);
  return cudaGetLastError();
}

cudaError_t launch_inc_unmark(const int4 *loc_list, long long n, int *loc_mark, cudaStream_t s,
                              const unsigned long long *count) {
  if (n == 0) return cudaSuccess;
  k_inc_unmark<<<grid_counted(n, 1, count, 148 * 2), 256, 0, s>>>(loc_list, n, loc_mark, count);
  return cudaGetLastError();
}

cudaError_t launch_cell_init(const int4 *locations, long long n, unsigned char *cell_dirs, cudaStream_t s,
                             const unsigned long long *count) {
  if (n == 0) return cudaSuccess;
  k_cell_init<<<grid_counted(n, 128, count, 148 * 8), 256, 0, s>>>(locations, n,
                                                                   reinterpret_cast<unsigned int *>(cell_dirs), count);
  return cudaGetLastError();
}

cudaError_t launch_cell_masks(const int4 *locations, long long n, const unsigned char *cell_dirs, unsigned int *cell_pos,
                              unsigned int *surface, int lo_x, int lo_y, int lo_z, int dim_x, int dim_y,
                              cudaStream_t s, const unsigned long long *count) {
  if (n == 0) return cudaSuccess;
  k_cell_masks<<<grid_counted(n, 32, count, 148 * 8), 256, 0, s>>>(locations, n, cell_dirs, cell_pos, surface, lo_x,
                                                                   lo_y, lo_z, dim_x, dim_y, count);
  return cudaGetLastError();
}

}  // namespace dtsdf
