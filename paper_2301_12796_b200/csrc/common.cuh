// common.cuh -- device-side data layout shared by the index build (volume.cu) and the
// raycast (render.cu).  DESIGN.md §5 describes the layout in HBM.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dtsdf {

// Bounds checks of the debug build (-DDTSDF_CHECKS, tools/build_checked.sh): every brick, mask and
// output index is checked before it is used and a violation traps the kernel.  compute-sanitizer
// is not available on the GPU pool, so this build plus the oracle comparisons is the memory-safety
// gate.  Compiled out of the product build.
#ifdef DTSDF_CHECKS
#define DTSDF_CHECK(cond) \
  do {                    \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define DTSDF_CHECK(cond) \
  do {                    \
  } while (0)
#endif

constexpr int kBlock = 8;          // 8^3 voxel blocks
constexpr int kVoxPerBlock = 512;
// Combined-TSDF bricks (combine.cu, NEXT-1): voxels -1..9 of the block per axis
constexpr int kApron = 11;
constexpr int kApronVox = kApron * kApron * kApron;  // 1331
constexpr int kApronStride = 1344;                   // records per combined brick (128-B aligned)
constexpr int kRgbApron = 9;                         // combined colour bricks: voxels 0..8 per axis
constexpr int kRgbApronVox = kRgbApron * kRgbApron * kRgbApron;  // 729
constexpr int kRgbApronStride = 736;                 // uchar4 records per brick (2944 B)
// Directional record bricks (volume.cu k_bricks): voxels 0..8 of the block per axis -- the 8
// trilinear corners of every base cell of the block -- as two arrays of records:
//   A float4 {sdf (NaN = the voxel's block is unallocated), weight, dsdf_x, dsdf_y}
//   B float2 {dsdf_z, rgb (u8 x3 in the float's bits)}
// with dsdf_a = sdf(voxel + e_a) - sdf(voxel - e_a) (NaN if either neighbour is unallocated), the
// per-voxel central difference of reading R7: the gradient of trilinear phi at x +- s e_a is the
// trilinear interpolant of these differences / 2s, so a sample reads 8 records per direction
// (16-B + 4-B loads) instead of 8 corners + 24 stencil voxels.
constexpr int kRec = 9;
constexpr int kRecVox = kRec * kRec * kRec;          // 729
constexpr int kRecStride = 732;                      // records per brick: A 11712 B, B 5856 B (32-B aligned)
#ifndef DTSDF_RANGE_TILE
#define DTSDF_RANGE_TILE 8
#endif
constexpr int kRangeTile = DTSDF_RANGE_TILE;         // range-pass tile (pixels)
constexpr int kViewsPerLaunch = 256;
constexpr unsigned long long kEmptyKey = 0xFFFFFFFFFFFFFFFFull;
// dense location grid value of an allocated location: hash entry | present directions << 24 |
// surface bit << 30 (so a location resolves with one 4-B load); negative = empty-space distance
constexpr int kGridEntryBits = 24;
constexpr int kGridEntryMask = (1 << kGridEntryBits) - 1;
// An empty location's grid value: -(1 + box), box = six 5-bit extents (blocks, 0..31) of an
// all-empty axis-aligned box of locations around it, faces -x, +x, -y, +y, -z, +z (bits 5 f); a
// ray may skip to the box's exit (render.cu).  The distance transform alone gives the cube of
// radius d - 1 (d = L-inf distance to the nearest allocated location); k_empty_box grows it.
#ifndef DTSDF_EMPTY_BOX
#define DTSDF_EMPTY_BOX 1
#endif
constexpr int kBoxBits = 5, kBoxMax = 31;
__host__ __device__ __forceinline__ int box_cube(int r) {  // all six extents r
  return r | (r << 5) | (r << 10) | (r << 15) | (r << 20) | (r << 25);
}

// Hash-table entry: one per block location (x,y,z); the six direction slots are block ids
// (rows of the pool / apron) or -1.  32 B = one sector: one probe returns all directions.
struct __align__(16) HashEntry {
  unsigned long long key;
  int slot[6];
};

__host__ __device__ __forceinline__ unsigned long long pack_key(int bx, int by, int bz) {
  const unsigned long long m = (1ull << 21) - 1;
  return ((unsigned long long)(bx + (1 << 20)) & m) | (((unsigned long long)(by + (1 << 20)) & m) << 21) |
         (((unsigned long long)(bz + (1 << 20)) & m) << 42);
}

__host__ __device__ __forceinline__ unsigned int hash_key(unsigned long long k) {
  // splitmix64 finaliser
  k ^= k >> 30;
  k *= 0xbf58476d1ce4e5b9ull;
  k ^= k >> 27;
  k *= 0x94d049bb133111ebull;
  k ^= k >> 31;
  return (unsigned int)k;
}

// Device view of a committed volume (read-only during rendering).
struct VolumeView {
  const HashEntry *table;
  unsigned int table_mask;
  const unsigned int *bitmap;  // occupancy bit per block location over the location AABB
  const unsigned int *surface; // same layout: 1 unless every base cell of the location is certainly positive
  const int *loc_grid;         // dense location grid over the AABB (null if too large): for an
                               // allocated location its hash entry index | (surface bit << 30),
                               // else -d with d >= 1 its empty-space distance in blocks
  const unsigned int *cell_pos;  // [table_cap][16]: bit l of location entry h = base cell l is
                                 // "certainly positive": every present direction's 8 corners > 0
  const unsigned char *cell_dirs;  // [table_cap][512]: bit D (0-5) of byte l of entry h = direction D
                                   // can hold data at base cell l (present, no NaN corner, a corner
                                   // weight > 0), the directions the evaluation visits; bit 7 = the
                                   // cell is certainly positive (as cell_pos)
  int use_live;                    // 1: visit only the live directions of a cell (DTSDF_OPT_CELL_DIRS)
  int lo_x, lo_y, lo_z;        // AABB origin (block coords)
  int dim_x, dim_y, dim_z;     // AABB extent (blocks)
  const float4 *brick_a;       // [N][kRecStride] {sdf (NaN = unallocated), weight, dsdf_x, dsdf_y}
  const float2 *brick_b;       // [N][kRecStride] {dsdf_z, rgb bits}
  float voxel_size, inv_voxel;
  float theta, inv_blend;      // 1 / (2 theta - pi/2)
  float cos_theta, sin_theta;  // membership band edges: w_dir = 0 below cos(theta), 1 above sin(theta)
  float delta, inv_delta;
  long long n_blocks;          // bricks in the pool (bounds checks)
  long long table_cap;         // hash entries (bounds checks)
};

// Device view of the view-dependent combined TSDF (NEXT-1, combine.cu): one combined brick per
// selected block location, in the apron layout of the directional bricks.
struct CombinedView {
  long long n_slots;               // combined slots (bounds checks)
  const int *slot_of_entry;        // [table_cap] combined slot of a hash entry, -1 = not combined
  const float *apron;              // [cap][kApronStride] combined sdf of voxels -1..9, NaN = invalid
  const uchar4 *rgb;               // [cap][kRgbApronStride] u8 colour (xyz) + direction mask (w), voxels 0..8
  const unsigned int *cell_pos;    // [cap][16] bit l: no valid corner of base cell l has sdf <= 0
  const unsigned char *surf;       // [cap] 1 unless every base cell is certainly positive / invalid
};

// Per-view camera: world-from-camera rotation (row-major) and camera centre.
struct ViewPose {
  float r[9];
  float t[3];
};

struct RenderLaunch {
  VolumeView vol;
  float fx, fy, cx, cy, z_min, z_max;
  int width, height, row0, row1;
  int n_views;
  int tiles_x, tiles_y;            // range tiles per view
  int use_range, use_skip;         // exact accelerations (DTSDF_OPT_*)
  int n_bisect;                    // bisection steps: bracket Delta -> <= 5e-5 m
  float refine_tol;                // regula falsi also stops once the bracket is narrower (m)
  const unsigned long long *z_near;  // [n_views][tiles_y][tiles_x] range keys of k_range (epoch-tagged
  const unsigned long long *z_far;   // float bits, range_key_*)
  unsigned int epoch;                // range-pass epoch of this launch
  const int *order;                  // [n_views][ct_x * ct_y] CTA tiles, longest predicted first, or null
  int ct_x;                          // CTA tiles per image row
  float *out_depth;                // [n_views][rows][W]
  float *out_normal;               // [n_views][rows][W][3] or null
  unsigned char *out_color;        // [n_views][rows][W][3] or null
  unsigned char *out_mask;         // [n_views][rows][W] or null
  unsigned long long *dbg_timeline;  // DTSDF_STATS builds only: per-pixel start/end/smid
  long long *dbg_trace;              // DTSDF_STATS builds only: per-step trace of one ray (8 x int64 per step)
  int dbg_trace_pix;                 // its pixel u | vrel << 16 in view 0, or -1
  int staged;                      // grid schedule: outputs leave via shared memory in whole tile rows
                                   // (mapped host outputs); 0: per-pixel stores
  int combined;                    // 1: march the combined TSDF (comb) instead of the six directions
  CombinedView comb;
  ViewPose pose[kViewsPerLaunch];
};

// Combine launch (combine.cu): the source camera in fp64 (from the float32 ABI values) for the
// frustum test of reading R33, evaluated with the oracle's operation order and roundings.
struct CombineLaunch {
  VolumeView vol;
  const int4 *locations;           // [U] (bx, by, bz, hash entry)
  long long n_loc;
  double R[9], t[3];
  double fx, fy, cx, cy, z_min, z_max;
  double mu, mv, umax, vmax;       // u in [-mu, umax], v in [-mv, vmax]
  int *slot_of_entry;              // [table_cap], -1 on entry
  int4 *comb_loc;                  // [cap] location + hash entry of each combined slot
  unsigned int *n_sel;             // combined slots handed out
  float *apron;                    // [cap][kApronStride]
  uchar4 *rgb;                     // [cap][kRgbApronStride]
  float *weight;                   // [cap][512] S = sum_D W_D of each interior voxel
  unsigned int *cell_pos;          // [cap][16]
  unsigned char *surf;             // [cap]
  unsigned char *cls;              // [cap] frustum class of each slot's block: 1 inside, 2 straddling
  // R58 update after a fused frame (null had: a full combination): slots < n_old keep their
  // voxels except those without data before the frame (had bit clear) that have data now
  const unsigned int *had;         // [n_old][16] bit l: voxel l of the slot had data before the frame
  long long n_old;
  int mode;                        // 0 eq:combine_weight / eq:combine_tsdf_weight, 1 Algorithm 1
  float w_floor;                   // Algorithm 1: stored-weight floor of a taking-part direction
  double theta64;                  // Algorithm 1: theta (fp64) for the w_dir > 0 decision
};

struct RangeLaunch {
  VolumeView vol;
  const int4 *locations;  // [U] (bx,by,bz,-)
  long long n_locations;
  float fx, fy, cx, cy, z_min, z_max;
  int width, height, row0, row1;
  int n_views;
  int tiles_x, tiles_y;
  unsigned long long *z_near;      // epoch-tagged keys (range_key_near / range_key_far): entries of
  unsigned long long *z_far;       // older epochs lose every atomic and read as "no block", so the
                                   // buffers never need clearing between calls
  unsigned int epoch;              // >= 1, advanced per range pass
  unsigned int *count;             // [n_views][tiles] block locations covering each tile (cost proxy of
                                   // the tile order; zero between passes -- k_order clears it), or null
  ViewPose pose[kViewsPerLaunch];
};

// Range-pass keys: the high word tags the epoch so that atomicMin / atomicMax of the current pass
// always beat stale entries of earlier passes (z_near: smaller tag for newer epochs; z_far: larger),
// the low word holds the float bits of a positive camera z (ordered like the floats).
__host__ __device__ __forceinline__ unsigned long long range_key_near(unsigned int epoch, unsigned int zbits) {
  return ((unsigned long long)(0xFFFFFFFFu - epoch) << 32) | zbits;
}
__host__ __device__ __forceinline__ unsigned long long range_key_far(unsigned int epoch, unsigned int zbits) {
  return ((unsigned long long)epoch << 32) | zbits;
}

// host launchers (render.cu)
cudaError_t launch_range(const RangeLaunch &p, cudaStream_t s);
// raycast CTA tiles (kTileW x kTileH pixels) of a width x rows image
void raycast_tiles(int width, int rows, int *ct_x, int *ct_y);
bool tile_order_fits(int width, int rows);  // the order kernel holds one key byte per CTA tile in shared memory
// CTA tile order of each view from the range-pass counts (longest predicted first); clears the counts
cudaError_t launch_order(unsigned int *count, int *order, int tiles_x, int tiles_y, int width, int rows, int n_views,
                         cudaStream_t s);
cudaError_t launch_raycast(const RenderLaunch &p, cudaStream_t s);

// Fusion launch (fusion.cu): one depth frame against the raw block pool.  The doubles are the
// float32 ABI values, used where both sides must take the same discrete decision (R40, R41).
struct FuseLaunch {
  HashEntry *table;
  unsigned int table_mask;
  int *keys;                       // [capacity][4]
  float *sdf, *weight, *cweight;   // [capacity][512]
  unsigned char *rgb;              // [capacity][512][3]
  unsigned long long *n_blocks;    // pool size (grows during allocation)
  long long capacity;
  int *flags;                      // 1 pool full, 2 table full
  const float *depth, *normal;     // [H][W], [H][W][3] camera frame
  const unsigned char *color;      // [H][W][3] or null
  double R[9], t[3], fx, fy, cx, cy, z_min, z_max;
  int width, height;
  double s, tau, step, cos_theta;  // voxel size, truncation, allocation sample step, cos(theta)
  int M;                           // allocation samples per segment: M + 1
  float theta_f, cos_theta_f, sin_theta_f, inv_blend;
  float max_weight, carve_weight;
  int carve_radius;
  // incremental index update (dtsdf_fuse): new locations are appended to `locations` (counter
  // n_loc) and checked against the location AABB (flags[1] <- 1 when one lies outside it); blocks
  // whose voxels changed, and new blocks, get dirty[b] = 1 (null: not tracked)
  int4 *locations;
  unsigned long long *n_loc;
  int lo[3], dim[3];
  const int *grid;                 // the committed location grid (null: none): existing (location, D)
                                   // keys are recognised with one load, without a hash probe
  unsigned char *dirty;
  // per-pixel world-rotated back-projection R P and world normal R n of the frame (k_fuse_alloc,
  // once per frame instead of once per associated voxel; null: k_fuse computes them)
  double4 *pix_x, *pix_n;
  // the same in fp32 for k_fuse's pre-test: pix_a (R P, z or -1 when the pixel holds no usable
  // depth / normal), pix_b (R n, carving guard 1 / 0)
  float4 *pix_a, *pix_b;
  // fp32 copies for the pre-test of k_fuse (DTSDF_FUSE_PRETEST): rotation, intrinsics, 1 / tau
  float Rf[9], fxf, fyf, cxf, cyf, inv_tau_f, inv_s_f;
  // incremental index update: a block k_fuse changed marks the locations of its 27-neighbourhood
  // that hold a block in its direction (loc_mark dedup, appended to loc_list, counter loc_ctr);
  // null: not tracked
  int *loc_mark;
  int4 *loc_list;
  unsigned long long *loc_ctr;
};

// ICP state in device memory (icp.cu): written by k_icp_solve, read back once per call
struct IcpState {
  double delta[16];                // DeltaT: frame camera -> rendered view camera (row-major)
  double sums[29];                 // last linearisation: upper H (21), g (6), inliers, sum w r^2
  double step, residual;
  long long inliers;
  int iterations, done, status;    // status 1: singular system
  unsigned int ticket;             // k_icp_reduce CTAs done this iteration (fused solve; 0 between launches)
};

struct IcpLaunch {
  const float *depth;              // [H][W] frame camera z
  const float *ref_depth;          // [H][W] rendered view camera z
  const float *ref_normal;         // [H][W][3] rendered world normals
  double ref_R[9];                 // rendered view rotation (world-from-camera, row-major)
  double fx, fy, cx, cy, z_min, z_max, outlier, min_step;
  int width, height, max_iters;
  double *partials;                // [n_partials][29]
  IcpState *state;
  double2 *pback;                  // [H][W] ((u - cx) / fx * z, (v - cy) / fy * z) of the frame (k_icp_backproject)
  double *col_fac, *row_fac;       // [W] (u - cx) / fx, [H] (v - cy) / fy: the rendered pixels' back-projection
  int fused_solve;                 // 1: the last k_icp_reduce CTA of an iteration also solves (no k_icp_solve)
};

// host launchers (icp.cu)
int icp_partials(int width, int height);
cudaError_t launch_icp_backproject(const IcpLaunch &p, cudaStream_t s);  // once per call: pback, col/row factors
cudaError_t launch_icp_reduce(const IcpLaunch &p, cudaStream_t s);
cudaError_t launch_icp_solve(const IcpLaunch &p, cudaStream_t s);

// host launchers (fusion.cu)
cudaError_t launch_depth_normals(const float *depth, const FuseLaunch &p, float *out, cudaStream_t s);
cudaError_t launch_fuse_alloc(const FuseLaunch &p, cudaStream_t s);
// new blocks initialised; then (fuse) the frame fused into the blocks -- with list / count (count
// zeroed beforehand) only those k_fuse_select finds in the frame's view
cudaError_t launch_fuse(const FuseLaunch &p, long long n_old, long long n_new, bool fuse, int *list,
                        unsigned long long *count, cudaStream_t s);

// host launchers (combine.cu)
cudaError_t launch_combine(const CombineLaunch &p, cudaStream_t s);                  // interiors + slots
cudaError_t launch_combine_finish(const CombineLaunch &p, long long n_sel, cudaStream_t s);  // aprons, masks
cudaError_t launch_comb_remap(const HashEntry *table, unsigned int mask, int4 *comb_loc, long long n,
                              int *slot_of_entry, cudaStream_t s);
// R58: bit l of had[s] = voxel l of combined slot s has data (a direction's block with weight > 0)
// in the pool as it stands (before a fused frame); comb_loc[s].w are current hash entries
cudaError_t launch_comb_had(const HashEntry *table, const int4 *comb_loc, long long n, const float *pool_weight,
                            unsigned int *had, cudaStream_t s);

// host launchers (volume.cu); all run on stream s and return the first launch error
struct CommitScratch {
  int *flags;          // [0] bad key, [1] duplicate, [2] table full, [3] non-finite sdf / bad weight
  int *aabb;           // [6] min xyz, max xyz
  unsigned long long *n_loc;
};
cudaError_t launch_validate_aabb(const int4 *keys, long long n, CommitScratch sc, cudaStream_t s);
cudaError_t launch_validate_values(const float *sdf, const float *weight, long long n, CommitScratch sc,
                                   cudaStream_t s);
cudaError_t launch_insert(const int4 *keys, long long n, HashEntry *table, unsigned int mask, int4 *locations,
                          CommitScratch sc, cudaStream_t s);
cudaError_t launch_bitmap(const int4 *locations, long long n_loc, unsigned int *bitmap, int lo_x, int lo_y, int lo_z,
                          int dim_x, int dim_y, cudaStream_t s);
cudaError_t launch_loc_grid(const int4 *locations, long long n_loc, const unsigned int *surface, const HashEntry *table,
                            int *grid, int lo_x, int lo_y, int lo_z, int dim_x, int dim_y, cudaStream_t s,
                            const unsigned long long *count = nullptr);
cudaError_t launch_empty_distance(int *grid, unsigned char *tmp0, unsigned char *tmp1, int dim_x, int dim_y, int dim_z,
                                  cudaStream_t s);
// grows every empty location's box (after launch_empty_distance) with a summed-volume table of
// occupancy; sat: (dim_x + 1) (dim_y + 1) (dim_z + 1) ints of scratch
cudaError_t launch_empty_box(int *grid, int *sat, int dim_x, int dim_y, int dim_z, cudaStream_t s);
// The dense location grid as a lookup for index-build kernels: hash entry of a block location, or
// -1 (unallocated / outside the AABB); grid null: unavailable (use the hash table).
struct GridRef {
  const int *grid;
  int lo[3], dim[3];
  __device__ __forceinline__ int entry(int bx, int by, int bz) const {
    const unsigned x = (unsigned)(bx - lo[0]), y = (unsigned)(by - lo[1]), z = (unsigned)(bz - lo[2]);
    if (x >= (unsigned)dim[0] || y >= (unsigned)dim[1] || z >= (unsigned)dim[2]) return -1;
    const int gv = __ldg(&grid[((size_t)z * dim[1] + y) * dim[0] + x]);
    return gv >= 0 ? (gv & kGridEntryMask) : -1;
  }
};

// record bricks of n blocks (list: their pool indices, or null for blocks 0..n-1), each adding its
// direction's bits to the location's live-direction bytes (cell_dirs, which start at 0x80)
cudaError_t launch_bricks(const int4 *keys, long long n, const HashEntry *table, unsigned int mask, const float *sdf,
                          const float *weight, const unsigned char *rgb, float4 *brick_a, float2 *brick_b,
                          unsigned char *cell_dirs, const int *list, const GridRef &gr, cudaStream_t s);
// (count non-null, here and below: the item count is *count, read on the device, n an upper bound)
cudaError_t launch_cell_init(const int4 *locations, long long n, unsigned char *cell_dirs, cudaStream_t s,
                             const unsigned long long *count = nullptr);
// incremental commit after a fused frame: the locations whose record bricks must be rebuilt (the
// 27-neighbourhoods, in the dirty block's direction, of every dirty block) -> loc_list (deduplicated
// by loc_mark[entry]), then all blocks of those locations -> blk_list; counters ctr[0], ctr[1]
cudaError_t launch_inc_mark(const int4 *keys, long long b0, long long n, const unsigned char *dirty,
                            const HashEntry *table,
                            unsigned int mask, const int *grid, const int lo[3], const int dim[3], int *loc_mark,
                            int4 *loc_list, unsigned long long *ctr, cudaStream_t s);
// (the location count is read from ctr[0] on the device; n an upper bound)
cudaError_t launch_inc_blocks(const int4 *loc_list, long long n, const HashEntry *table, int *blk_list,
                              unsigned long long *ctr, cudaStream_t s);
cudaError_t launch_inc_unmark(const int4 *loc_list, long long n, int *loc_mark, cudaStream_t s,
                              const unsigned long long *count = nullptr);
// k_bricks over a device-counted list: grid = an upper bound, CTAs at or beyond *count return
cudaError_t launch_bricks_counted(const int4 *keys, long long grid, const unsigned long long *count,
                                  const HashEntry *table, unsigned int mask, const float *sdf, const float *weight,
                                  const unsigned char *rgb, float4 *brick_a, float2 *brick_b, unsigned char *cell_dirs,
                                  const int *list, const GridRef &gr, cudaStream_t s);
cudaError_t launch_cell_masks(const int4 *locations, long long n, const unsigned char *cell_dirs, unsigned int *cell_pos,
                              unsigned int *surface, int lo_x, int lo_y, int lo_z, int dim_x, int dim_y,
                              cudaStream_t s, const unsigned long long *count = nullptr);
// rgb packed into a float's bits for the B records (r | g << 8 | b << 16)
__host__ __device__ __forceinline__ unsigned int rec_rgb(float bits) {
#ifdef __CUDA_ARCH__
  return __float_as_uint(bits);
#else
  unsigned int u;
  __builtin_memcpy(&u, &bits, 4);
  return u;
#endif
}

}  // namespace dtsdf
