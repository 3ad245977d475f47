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
__global__ void __launch_bounds__(kBrickThreads) k_bricks(const int4 *__restrict__ keys, const HashEntry *__restrict__ table,
                                                         unsigned int mask, const float *__restrict__ sdf,
                                                         const float *__restrict__ weight, const unsigned char *__restrict__ rgb,
                                                         float4 *__restrict__ brick_a, float2 *__restrict__ brick_b) {
  __shared__ int nb[27];  // slot of neighbour (ox, oy, oz) in -1..1, index (ox+1) + 3 (oy+1) + 9 (oz+1)
  __shared__ float st[kStage * kStage * kStage];
  const long long b = blockIdx.x;
  const int4 k = keys[b];
  if (threadIdx.x < 27) {
    const int ox = (int)threadIdx.x % 3 - 1, oy = ((int)threadIdx.x / 3) % 3 - 1, oz = (int)threadIdx.x / 9 - 1;
    int src = (int)b;
    if (ox | oy | oz) {
      const int e = find_entry(table, mask, pack_key(k.x + ox, k.y + oy, k.z + oz));
      src = (e >= 0) ? table[e].slot[k.w] : -1;
    }
    nb[threadIdx.x] = src;
  }
  __syncthreads();
  // pool record of block-local voxel (lx, ly, lz) in -8..15, or -1 when its block is unallocated
  auto rec_of = [&](int lx, int ly, int lz) -> long long {
    const int ox = (lx < 0) ? -1 : (lx >= kBlock ? 1 : 0);
    const int oy = (ly < 0) ? -1 : (ly >= kBlock ? 1 : 0);
    const int oz = (lz < 0) ? -1 : (lz >= kBlock ? 1 : 0);
    const int src = nb[(ox + 1) + 3 * (oy + 1) + 9 * (oz + 1)];
    if (src < 0) return -1;
    const int l = (lx - ox * kBlock) + kBlock * (ly - oy * kBlock) + kBlock * kBlock * (lz - oz * kBlock);
    return (long long)src * kVoxPerBlock + l;
  };
  for (int a = threadIdx.x; a < kStage * kStage * kStage; a += kBrickThreads) {
    const long long r = rec_of(a % kStage - 1, (a / kStage) % kStage - 1, a / (kStage * kStage) - 1);
    st[a] = r >= 0 ? sdf[r] : __int_as_float(0x7fc00000);  // NaN sdf = unallocated
  }
  __syncthreads();
  for (int a = threadIdx.x; a < kRecStride; a += kBrickThreads) {
    float4 ra = make_float4(__int_as_float(0x7fc00000), 0.0f, __int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
    float2 rb = make_float2(__int_as_float(0x7fc00000), 0.0f);
    if (a < kRecVox) {
      const int lx = a % kRec, ly = (a / kRec) % kRec, lz = a / (kRec * kRec);  // 0..8
      const int c = (lx + 1) + kStage * (ly + 1) + kStage * kStage * (lz + 1);
      const long long r = rec_of(lx, ly, lz);
      ra.x = st[c];
      ra.y = r >= 0 ? weight[r] : 0.0f;
      ra.z = st[c + 1] - st[c - 1];
      ra.w = st[c + kStage] - st[c - kStage];
      rb.x = st[c + kStage * kStage] - st[c - kStage * kStage];
      unsigned int col = 0;
      if (r >= 0 && rgb != nullptr) {
        const unsigned char *q = rgb + 3 * r;
        col = (unsigned int)q[0] | ((unsigned int)q[1] << 8) | ((unsigned int)q[2] << 16);
      }
      rb.y = __uint_as_float(col);
    }
    brick_a[b * kRecStride + a] = ra;
    brick_b[b * kRecStride + a] = rb;
  }
}

// Certainly-positive base cells: bit l of location h is set iff, for every direction present
// at the cell (all 8 corners allocated), all 8 corner sdf values are > 0.  A sample in such a cell
// has F > 0 or is invalid (convex combination, O3(e)), so it can neither end a crossing nor --
// when the next lattice point is such a sample too -- start one (render.cu, exact).
// One warp per 32 consecutive cells of a location; the ballot writes one mask word.
__global__ void k_cell_pos(const int4 *__restrict__ loc, long long n_loc, const HashEntry *__restrict__ table,
                           const float4 *__restrict__ brick_a, unsigned int *cell_pos, unsigned char *cell_dirs) {
  long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long u = gid >> 9;
  int l = (int)(gid & 511);
  bool pos = false;
  int live = 0;
  if (u < n_loc) {
    const int h = loc[u].w;
    const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
    pos = true;
    for (int D = 0; D < 6; ++D) {
      const int slot = table[h].slot[D];
      if (slot < 0) continue;
      const float4 *br = brick_a + (size_t)slot * kRecStride + lx + kRec * ly + kRec * kRec * lz;
      bool absent = false, allpos = true, weighted = false;
      for (int q = 0; q < 8; ++q) {
        const float4 v = br[(q & 1) + kRec * ((q >> 1) & 1) + kRec * kRec * (q >> 2)];
        absent |= isnan(v.x);
        allpos &= v.x > 0.0f;
        weighted |= v.y > 0.0f;
      }
      if (!absent && !allpos) pos = false;
      // a NaN corner makes the trilinear phi NaN, corner weights all <= 0 make omega <= 0: either
      // way the evaluation drops D here (O3(a), reading R8), so it need not visit it
      if (!absent && weighted) live |= 1 << D;
    }
  }
  const unsigned int word = __ballot_sync(0xffffffffu, pos);
  if (u < n_loc && (l & 31) == 0) cell_pos[(size_t)loc[u].w * 16 + (l >> 5)] = word;
  if (u < n_loc && cell_dirs) cell_dirs[(size_t)loc[u].w * 512 + l] = (unsigned char)(live | (pos ? 128 : 0));
}

// Dense location grid: for each allocated location, its hash entry index, present directions and
// surface bit (kGridEntryBits layout), so the raycast resolves a location -- and knows which
// directions it holds -- with one 4-B load instead of bitmap + surface + hash probe + entry.
__global__ void k_loc_grid(const int4 *__restrict__ loc, long long n_loc, const unsigned int *__restrict__ surface,
                           const HashEntry *__restrict__ table, int *grid, int lo_x, int lo_y, int lo_z, int dim_x,
                           int dim_y) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_loc) return;
  const int4 b = loc[i];
  const long long cell = ((long long)(b.z - lo_z) * dim_y + (b.y - lo_y)) * dim_x + (b.x - lo_x);
  const int surf = (surface[cell >> 5] >> (cell & 31)) & 1;
  int present = 0;
  for (int d = 0; d < 6; ++d) present |= (table[b.w].slot[d] >= 0) << d;
  grid[cell] = b.w | (present << kGridEntryBits) | (surf << 30);
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
  if (grid[c] < 0) grid[c] = -(dist[c] > 1 ? (int)dist[c] : 1);
}

// Surface bit of a block location: set unless every base cell of the location is certainly
// positive (k_cell_pos).  Where it is clear, every sample whose base voxel lies in the location
// has F > 0 or is invalid, so the march may jump to the location's last lattice points (exact).
__global__ void k_surface(const int4 *__restrict__ loc, long long n_loc, const unsigned int *__restrict__ cell_pos,
                          unsigned int *surface, int lo_x, int lo_y, int lo_z, int dim_x, int dim_y) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_loc) return;
  const int4 b = loc[i];
  bool all_pos = true;
  for (int w = 0; w < 16; ++w) all_pos &= cell_pos[(size_t)b.w * 16 + w] == 0xffffffffu;
  if (!all_pos) {
    const long long cell = ((long long)(b.z - lo_z) * dim_y + (b.y - lo_y)) * dim_x + (b.x - lo_x);
    atomicOr(&surface[cell >> 5], 1u << (cell & 31));
  }
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

cudaError_t launch_loc_grid(const int4 *locations, long long n_loc, const unsigned int *surface, const HashEntry *table,
                            int *grid, int lo_x, int lo_y, int lo_z, int dim_x, int dim_y, cudaStream_t s) {
  if (n_loc == 0) return cudaSuccess;
  k_loc_grid<<<grid_for(n_loc, 256), 256, 0, s>>>(locations, n_loc, surface, table, grid, lo_x, lo_y, lo_z, dim_x,
                                                  dim_y);
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

cudaError_t launch_cell_pos(const int4 *locations, long long n_loc, const HashEntry *table, const float4 *brick_a,
                            unsigned int *cell_pos, unsigned char *cell_dirs, cudaStream_t s) {
  if (n_loc == 0) return cudaSuccess;
  k_cell_pos<<<grid_for(n_loc * 512, 256), 256, 0, s>>>(locations, n_loc, table, brick_a, cell_pos, cell_dirs);
  return cudaGetLastError();
}

cudaError_t launch_surface(const int4 *locations, long long n_loc, const unsigned int *cell_pos, unsigned int *surface,
                           int lo_x, int lo_y, int lo_z, int dim_x, int dim_y, cudaStream_t s) {
  if (n_loc == 0) return cudaSuccess;
  k_surface<<<grid_for(n_loc, 256), 256, 0, s>>>(locations, n_loc, cell_pos, surface, lo_x, lo_y, lo_z, dim_x, dim_y);
  return cudaGetLastError();
}

cudaError_t launch_bricks(const int4 *keys, long long n, const HashEntry *table, unsigned int mask, const float *sdf,
                          const float *weight, const unsigned char *rgb, float4 *brick_a, float2 *brick_b,
                          cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_bricks<<<(unsigned)n, kBrickThreads, 0, s>>>(keys, table, mask, sdf, weight, rgb, brick_a, brick_b);
  return cudaGetLastError();
}

}  // namespace dtsdf
