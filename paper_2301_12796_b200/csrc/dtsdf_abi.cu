// dtsdf_abi.cu -- host side of the C ABI declared in include/dtsdf.h.
//
// Argument checking, device memory ownership, index build orchestration (volume.cu) and
// per-batch launch packing (render.cu).  No C++ exception crosses the ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dtsdf.h"
#include "common.cuh"

using namespace dtsdf;

namespace {

thread_local std::string g_err;
thread_local std::string g_warn;  // dtsdf_last_warning: accepted-but-questionable arguments

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

struct TimedLaunch {
  cudaEvent_t start, stop;
  int kind;  // 0 range, 1 raycast, 2 other, 3 combine
};

}  // namespace

#ifdef DTSDF_STATS
extern "C" __attribute__((visibility("default"))) unsigned long long *dtsdf_debug_timeline = nullptr;
extern "C" __attribute__((visibility("default"))) long long *dtsdf_debug_trace = nullptr;  // [32 lanes][128 steps][8]
extern "C" __attribute__((visibility("default"))) int dtsdf_debug_trace_pix = -1;
#endif

struct dtsdf_ctx {
  int device = 0;
  bool sticky = false;
  // current volume
  dtsdf_volume_params params{};
  bool allocated = false, committed = false;
  bool values_trusted = false;  // set by dtsdf_fuse around its re-commit: its own kernels wrote the values
  // incremental index update after a fused frame (DTSDF_OPT_INCREMENTAL)
  int incremental = 1;
  unsigned char *blk_dirty = nullptr;  // [cap] blocks whose voxels the frame changed (or new)
  int *blk_list = nullptr;             // [cap] blocks whose record bricks are rebuilt
  int *loc_mark = nullptr;             // [table cap] 1 while the location is in loc_list (zero between frames)
  int4 *loc_list = nullptr;            // [table cap] locations whose bricks / cell bytes / grid values are rebuilt
  unsigned long long *inc_ctr = nullptr;
  size_t cap_blk_dirty = 0, cap_blk_list = 0, cap_loc_mark = 0, cap_loc_list = 0, cap_inc_ctr = 0;
  int32_t *keys = nullptr;
  float *sdf = nullptr, *weight = nullptr;
  uint8_t *rgb = nullptr;
  int64_t n = 0;
  int64_t cap = 0;            // pool capacity in blocks (>= n; fusion grows n up to it)
  float *cweight = nullptr;   // fusion: colour weights [cap][512] (eq:color_weight accumulator)
  void *fuse_stage = nullptr; // fusion / ICP: device staging of host frames
  double4 *pix_buf = nullptr;  // fusion: per-pixel world points + normals of the frame (k_fuse_alloc)
  size_t cap_pix_buf = 0;
  double *icp_partials = nullptr;
  IcpState *icp_state = nullptr;
  int *icp_done_host = nullptr;  // pinned: the done flag read back between chunks of iterations
  unsigned char *icp_pback = nullptr;  // frame back-projections + column/row factors (icp_prepare)
  size_t cap_icp_pback = 0;
  size_t cap_icp_partials = 0, cap_icp_state = 0;
  size_t fuse_stage_cap = 0;
  // index
  HashEntry *table = nullptr;
  unsigned int table_cap = 0;
  unsigned int *bitmap = nullptr, *surface = nullptr, *cell_pos = nullptr;
  unsigned char *cell_dirs = nullptr;  // [table cap][512] live directions per base cell
  size_t cap_cell_dirs = 0;
  int *loc_grid = nullptr;
  int lo[3] = {0, 0, 0}, dim[3] = {0, 0, 0};
  int4 *locations = nullptr;
  int64_t n_loc = 0;
  float4 *brick_a = nullptr;  // record bricks (common.cuh kRec*): {sdf, weight, dsdf_x, dsdf_y}
  float2 *brick_b = nullptr;  // {dsdf_z, rgb}
  size_t index_bytes = 0;
  // allocated sizes of the index buffers: a re-commit (e.g. after every fused frame) reuses them
  size_t cap_table = 0, cap_locations = 0, cap_bitmap = 0, cap_surface = 0, cap_cell_pos = 0, cap_brick_a = 0,
         cap_brick_b = 0, cap_loc_grid = 0, cap_dist = 0;
  unsigned char *dist_tmp = nullptr;
  int *box_sat = nullptr;  // summed-volume table of the location grid's occupancy (k_empty_box)
  size_t cap_box_sat = 0;
  // commit scratch
  int *scratch = nullptr;  // flags[4] + aabb[6] + n_loc(u64)
  // render scratch
  unsigned long long *z_near = nullptr, *z_far = nullptr;  // range keys (epoch-tagged)
  unsigned int range_epoch = 0;  // last epoch used; 0 = buffers need clearing
  unsigned int *tile_count = nullptr;  // range-pass block counts per tile (zero between passes)
  int *tile_order = nullptr;           // CTA tile order per view
  size_t order_cap = 0;
  int use_order = 1;                   // DTSDF_OPT_TILE_ORDER
  size_t range_cap = 0;  // tiles
  void *host_stage = nullptr;  // device scratch for host-output renders
  size_t host_stage_cap = 0;
  int use_range = 1, use_skip = 1, bisect_steps = -1, use_grid = 1, refine_tol_nm = 0;
  int host_write = 1;
  int use_live = 1;            // DTSDF_OPT_CELL_DIRS          // DTSDF_OPT_HOST_WRITE: the raycast writes mapped pinned host outputs directly
  // view-dependent combined TSDF (NEXT-1, combine.cu)
  bool combined = false;
  int64_t n_comb = 0, comb_cap = 0;
  unsigned int comb_entries = 0;  // slot_of_entry length (table capacity at allocation)
  int *comb_slot = nullptr;
  int4 *comb_loc = nullptr;
  float *comb_apron = nullptr, *comb_weight = nullptr;
  uchar4 *comb_rgb = nullptr;
  unsigned int *comb_cell_pos = nullptr, *comb_count = nullptr;
  unsigned char *comb_surf = nullptr, *comb_cls = nullptr;
  unsigned int *comb_had = nullptr;  // R58: per-slot "had data" masks captured before a fused frame
  size_t cap_comb_had = 0;
  // the camera and rule of the current combined TSDF (R58 updates after fused frames reuse them)
  float comb_pose[16] = {0};
  dtsdf_intrinsics comb_K{};
  float comb_margin = 0.f, comb_wfloor = 0.f;
  int comb_mode = 0;
  // tracing
  bool profiling = false;
  std::vector<TimedLaunch> timed;
  double times_ms[4] = {0, 0, 0, 0};
  int64_t counts[4] = {0, 0, 0, 0};
  int64_t launches = 0;
};

namespace {

int cuda_fail(dtsdf_ctx *ctx, cudaError_t e, const char *what) {
  if (ctx) ctx->sticky = true;
  return fail(DTSDF_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(ctx, expr, what)                                \
  do {                                                     \
    cudaError_t _e = (expr);                               \
    if (_e != cudaSuccess) return cuda_fail(ctx, _e, what); \
  } while (0)

template <typename T>
void dfree(T *&p) {
  if (p) cudaFree(p);
  p = nullptr;
}

void free_combined(dtsdf_ctx *c) {
  dfree(c->comb_slot);
  dfree(c->comb_loc);
  dfree(c->comb_apron);
  dfree(c->comb_weight);
  dfree(c->comb_rgb);
  dfree(c->comb_cell_pos);
  dfree(c->comb_surf);
  dfree(c->comb_cls);
  dfree(c->comb_had);
  c->cap_comb_had = 0;
  dfree(c->comb_count);
  c->combined = false;
  c->n_comb = c->comb_cap = 0;
  c->comb_entries = 0;
}

void free_volume(dtsdf_ctx *c) {
  free_combined(c);
  dfree(c->cweight);
  dfree(c->keys);
  dfree(c->sdf);
  dfree(c->weight);
  dfree(c->rgb);
  dfree(c->table);
  dfree(c->bitmap);
  dfree(c->surface);
  dfree(c->cell_pos);
  dfree(c->cell_dirs);
  dfree(c->loc_grid);
  dfree(c->locations);
  dfree(c->brick_a);
  dfree(c->brick_b);
  dfree(c->blk_dirty);
  dfree(c->blk_list);
  dfree(c->loc_mark);
  dfree(c->loc_list);
  dfree(c->inc_ctr);
  c->cap_blk_dirty = c->cap_blk_list = c->cap_loc_mark = c->cap_loc_list = c->cap_inc_ctr = 0;
  dfree(c->dist_tmp);
  dfree(c->box_sat);
  c->cap_box_sat = 0;
  c->cap_table = c->cap_locations = c->cap_bitmap = c->cap_surface = c->cap_cell_pos = c->cap_brick_a =
      c->cap_brick_b = c->cap_loc_grid = c->cap_dist = c->cap_cell_dirs = 0;
  c->allocated = c->committed = false;
  c->n = c->n_loc = c->cap = 0;
  c->index_bytes = 0;
}

bool is_device_ptr(const void *p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int check_params(const dtsdf_volume_params *p) {
  if (!p) return fail(DTSDF_ERR_INVALID_ARGUMENT, "params is NULL");
  if (!(p->voxel_size > 0.f) || !std::isfinite(p->voxel_size))
    return fail(DTSDF_ERR_INVALID_ARGUMENT, "voxel_size must be > 0");
  if (!(p->truncation >= 2.f * p->voxel_size)) return fail(DTSDF_ERR_INVALID_ARGUMENT, "truncation must be >= 2*voxel_size");
  const double pi = 3.14159265358979323846;
  if (!(p->theta > pi / 4) || !(p->theta <= pi / 2 + 1e-6))
    return fail(DTSDF_ERR_INVALID_ARGUMENT, "theta must lie in (pi/4, pi/2]");
  // reading R2: PAPER.md:84's "at least one and at most three directions" holds in 3D only for
  // theta >= arccos(1/sqrt(3)) = 54.74 deg; below it some normals get no direction (accepted)
  g_warn.clear();
  if ((double)p->theta < std::acos(1.0 / std::sqrt(3.0)))
    g_warn = "theta < 54.74 deg (arccos(1/sqrt(3))): surfaces whose normal is near a cube diagonal belong to no "
             "direction (PAPER.md:84's 1-3 directions claim fails in 3D, reading R2)";
  if (!(p->step >= 0.f) || !std::isfinite(p->step)) return fail(DTSDF_ERR_INVALID_ARGUMENT, "step must be >= 0");
  if (p->n_blocks < 0 || p->n_blocks > (int64_t)INT32_MAX) return fail(DTSDF_ERR_INVALID_ARGUMENT, "bad n_blocks");
  return DTSDF_OK;
}

int check_intr(const dtsdf_intrinsics *K) {
  if (!K) return fail(DTSDF_ERR_INVALID_ARGUMENT, "intrinsics is NULL");
  if (!(K->fx > 0.f) || !(K->fy > 0.f)) return fail(DTSDF_ERR_INVALID_ARGUMENT, "fx, fy must be > 0");
  if (K->width <= 0 || K->height <= 0) return fail(DTSDF_ERR_INVALID_ARGUMENT, "width, height must be > 0");
  // the raycast packs a pixel as u | row << 16 (render.cu ray_pix)
  if (K->width > 32768 || K->height > 32768) return fail(DTSDF_ERR_INVALID_ARGUMENT, "width, height must be <= 32768");
  if (!(K->z_min > 0.f) || !(K->z_min < K->z_max) || !std::isfinite(K->z_max))
    return fail(DTSDF_ERR_INVALID_ARGUMENT, "need 0 < z_min < z_max");
  if (!std::isfinite(K->cx) || !std::isfinite(K->cy)) return fail(DTSDF_ERR_INVALID_ARGUMENT, "cx, cy not finite");
  return DTSDF_OK;
}

template <typename T>
cudaError_t dalloc(T *&p, size_t bytes) {
  return cudaMalloc((void **)&p, std::max<size_t>(bytes, 16));
}

// grow-only device buffer: keeps the allocation when it is large enough
template <typename T>
cudaError_t ensure(T *&p, size_t &cap, size_t bytes) {
  bytes = std::max<size_t>(bytes, 16);
  if (p && cap >= bytes) return cudaSuccess;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  cudaError_t e = cudaMalloc((void **)&p, bytes);
  if (e == cudaSuccess) cap = bytes;
  return e;
}

// kernels: number of this library's kernels the bracketed region launches (memsets: 0)
void begin_timed(dtsdf_ctx *c, int kind, cudaStream_t s, TimedLaunch *tl, int kernels = 1) {
  c->launches += kernels;
  if (!c->profiling) return;
  tl->kind = kind;
  cudaEventCreate(&tl->start);
  cudaEventCreate(&tl->stop);
  cudaEventRecord(tl->start, s);
}

void end_timed(dtsdf_ctx *c, cudaStream_t s, TimedLaunch *tl) {
  if (!c->profiling) return;
  cudaEventRecord(tl->stop, s);
  c->timed.push_back(*tl);
}

}  // namespace

extern "C" {

const char *dtsdf_last_error(void) { return g_err.c_str(); }
const char *dtsdf_last_warning(void) { return g_warn.c_str(); }

int dtsdf_create(int cuda_device, dtsdf_ctx **out) {
  if (!out) return fail(DTSDF_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) return fail(DTSDF_ERR_CUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  if (cuda_device < 0 || cuda_device >= n) return fail(DTSDF_ERR_INVALID_ARGUMENT, "no such CUDA device");
  if ((e = cudaSetDevice(cuda_device)) != cudaSuccess)
    return fail(DTSDF_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  dtsdf_ctx *c = new (std::nothrow) dtsdf_ctx();
  if (!c) return fail(DTSDF_ERR_OUT_OF_MEMORY, "host allocation");
  c->device = cuda_device;
  if (dalloc(c->scratch, 64) != cudaSuccess) {
    delete c;
    return fail(DTSDF_ERR_OUT_OF_MEMORY, "scratch allocation");
  }
  *out = c;
  return DTSDF_OK;
}

int dtsdf_destroy(dtsdf_ctx *c) {
  if (!c) return DTSDF_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  free_volume(c);
  dfree(c->scratch);
  if (c->fuse_stage) cudaFree(c->fuse_stage);
  dfree(c->pix_buf);
  dfree(c->icp_partials);
  dfree(c->icp_state);
  if (c->icp_done_host) cudaFreeHost(c->icp_done_host);
  dfree(c->icp_pback);
  dfree(c->z_near);
  dfree(c->z_far);
  dfree(c->tile_count);
  dfree(c->tile_order);
  if (c->host_stage) cudaFree(c->host_stage);
  for (auto &t : c->timed) {
    cudaEventDestroy(t.start);
    cudaEventDestroy(t.stop);
  }
  delete c;
  return DTSDF_OK;
}

int dtsdf_alloc_volume(dtsdf_ctx *c, const dtsdf_volume_params *p, dtsdf_volume_buffers *out) {
  if (!c || !out) return fail(DTSDF_ERR_INVALID_ARGUMENT, "ctx/out is NULL");
  if (c->sticky) return fail(DTSDF_ERR_CUDA, "context has a sticky CUDA error");
  int rc = check_params(p);
  if (rc) return rc;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  free_volume(c);
  const size_t n = (size_t)p->n_blocks;
  if (dalloc(c->keys, n * 16) != cudaSuccess || dalloc(c->sdf, n * 512 * 4) != cudaSuccess ||
      dalloc(c->weight, n * 512 * 4) != cudaSuccess || dalloc(c->rgb, n * 512 * 3) != cudaSuccess) {
    cudaGetLastError();
    free_volume(c);
    return fail(DTSDF_ERR_OUT_OF_MEMORY, "volume buffers");
  }
  c->params = *p;
  c->n = (int64_t)n;
  c->cap = (int64_t)n;
  c->allocated = true;
  out->keys = c->keys;
  out->sdf = c->sdf;
  out->weight = c->weight;
  out->rgb = c->rgb;
  return DTSDF_OK;
}

int dtsdf_commit_volume(dtsdf_ctx *c, void *stream) {
  if (!c) return fail(DTSDF_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (c->sticky) return fail(DTSDF_ERR_CUDA, "context has a sticky CUDA error");
  if (!c->allocated) return fail(DTSDF_ERR_NO_VOLUME, "no allocated volume");
  cudaSetDevice(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  c->committed = false;
  // a combined TSDF survives a re-commit of the same volume (stale until recombined);
  // its slots are re-pointed at the rebuilt hash entries below
  const long long n = c->n;
  // scratch: flags[4] | aabb[6] | pad[2] | n_loc (8 B aligned at int offset 12)
  CommitScratch sc;
  sc.flags = c->scratch;
  sc.aabb = c->scratch + 4;
  sc.n_loc = reinterpret_cast<unsigned long long *>(c->scratch + 12);
  int init[14] = {0, 0, 0, 0, INT32_MAX, INT32_MAX, INT32_MAX, INT32_MIN, INT32_MIN, INT32_MIN, 0, 0, 0, 0};
  CK(c, cudaMemcpyAsync(c->scratch, init, sizeof(init), cudaMemcpyHostToDevice, s), "commit init");
  TimedLaunch tl{};
  begin_timed(c, 2, s, &tl);
  CK(c, launch_validate_aabb(reinterpret_cast<const int4 *>(c->keys), n, sc, s), "validate");
  end_timed(c, s, &tl);
  if (!c->values_trusted) {  // user-written values: sdf finite (NaN is the apron's sentinel), weight >= 0
    begin_timed(c, 2, s, &tl);
    CK(c, launch_validate_values(c->sdf, c->weight, n, sc, s), "validate values");
    end_timed(c, s, &tl);
  }
  int host[14];
  CK(c, cudaMemcpyAsync(host, c->scratch, sizeof(host), cudaMemcpyDeviceToHost, s), "commit readback");
  CK(c, cudaStreamSynchronize(s), "commit sync");
  if (host[0]) return fail(DTSDF_ERR_INVALID_ARGUMENT, "block key with D outside 0..5 or coordinate out of range");
  if (host[3]) return fail(DTSDF_ERR_INVALID_ARGUMENT, "sdf must be finite and weight finite and >= 0");
  // hash table: capacity = next power of two >= 2N (load factor <= 1/2 over locations)
  unsigned int cap = 64;
  while ((long long)cap < 2 * std::max<long long>(n, c->cap)) cap <<= 1;  // room for fusion to grow into
  c->table_cap = cap;
  int lo[3] = {0, 0, 0}, hi[3] = {-1, -1, -1};
  if (n > 0)
    for (int a = 0; a < 3; ++a) { lo[a] = host[4 + a]; hi[a] = host[7 + a]; }
  for (int a = 0; a < 3; ++a) { c->lo[a] = lo[a]; c->dim[a] = hi[a] - lo[a] + 1; }
  const size_t cells = (size_t)c->dim[0] * c->dim[1] * c->dim[2];
  const size_t bm_words = (cells + 31) / 32;
  // per-block buffers sized for the pool capacity, so a volume growing by fusion keeps them
  const size_t nb = (size_t)std::max<long long>(std::max<long long>(n, c->cap), 1);
  if (ensure(c->table, c->cap_table, (size_t)cap * sizeof(HashEntry)) != cudaSuccess ||
      ensure(c->locations, c->cap_locations, nb * sizeof(int4)) != cudaSuccess ||
      ensure(c->bitmap, c->cap_bitmap, (bm_words + 1) * 4) != cudaSuccess ||
      ensure(c->surface, c->cap_surface, (bm_words + 1) * 4) != cudaSuccess ||
      ensure(c->cell_pos, c->cap_cell_pos, (size_t)cap * 64) != cudaSuccess ||
      ensure(c->cell_dirs, c->cap_cell_dirs, (size_t)cap * 512) != cudaSuccess ||
      ensure(c->brick_a, c->cap_brick_a, nb * kRecStride * sizeof(float4)) != cudaSuccess ||
      ensure(c->brick_b, c->cap_brick_b, nb * kRecStride * sizeof(float2)) != cudaSuccess) {
    cudaGetLastError();
    return fail(DTSDF_ERR_OUT_OF_MEMORY, "index allocation");
  }
  c->index_bytes = (size_t)cap * (sizeof(HashEntry) + 64 + 512) + (size_t)n * sizeof(int4) + 2 * bm_words * 4 +
                   (size_t)n * kRecStride * (sizeof(float4) + sizeof(float2));
  CK(c, cudaMemsetAsync(c->table, 0xFF, (size_t)cap * sizeof(HashEntry), s), "table init");
  CK(c, cudaMemsetAsync(c->bitmap, 0, (bm_words + 1) * 4, s), "bitmap init");
  CK(c, cudaMemsetAsync(c->surface, 0, (bm_words + 1) * 4, s), "surface init");
  begin_timed(c, 2, s, &tl);
  CK(c, launch_insert(reinterpret_cast<const int4 *>(c->keys), n, c->table, cap - 1, c->locations, sc, s), "insert");
  end_timed(c, s, &tl);
  CK(c, cudaMemcpyAsync(host, c->scratch, sizeof(host), cudaMemcpyDeviceToHost, s), "commit readback");
  CK(c, cudaStreamSynchronize(s), "commit sync");
  if (host[1]) return fail(DTSDF_ERR_DUPLICATE_KEY, "duplicate (bx,by,bz,D) block key");
  if (host[2]) return fail(DTSDF_ERR_OUT_OF_MEMORY, "hash table full");
  unsigned long long nl;
  std::memcpy(&nl, &host[12], sizeof(nl));
  c->n_loc = (int64_t)nl;
  begin_timed(c, 2, s, &tl);
  CK(c, launch_bitmap(c->locations, c->n_loc, c->bitmap, lo[0], lo[1], lo[2], c->dim[0], c->dim[1], s), "bitmap");
  end_timed(c, s, &tl);
  // dense location grid when the AABB is small enough (<= 2^28 locations, 1 GiB); else the
  // raycast resolves locations through the bitmaps and the hash table.  Its entries go in first
  // (k_bricks resolves neighbours through it); the final values, with the surface bits, follow
  // the cell masks.
  const bool grid_ok = cells > 0 && cells <= (size_t(1) << 28) && c->table_cap <= (size_t(1) << kGridEntryBits);
  if (grid_ok) {
    if (ensure(c->loc_grid, c->cap_loc_grid, cells * 4) != cudaSuccess) {
      cudaGetLastError();
      c->loc_grid = nullptr;
    } else {
      c->index_bytes += cells * 4;
      CK(c, cudaMemsetAsync(c->loc_grid, 0xFF, cells * 4, s), "grid init");
      begin_timed(c, 2, s, &tl);
      CK(c, launch_loc_grid(c->locations, c->n_loc, c->surface, c->table, c->loc_grid, lo[0], lo[1], lo[2],
                            c->dim[0], c->dim[1], s),
         "loc_grid entries");
      end_timed(c, s, &tl);
    }
  } else {
    dfree(c->loc_grid);  // AABB too large for the dense grid: the hash-probe path
    c->cap_loc_grid = 0;
  }
  GridRef gr{};
  gr.grid = c->loc_grid;
  for (int a = 0; a < 3; ++a) { gr.lo[a] = lo[a]; gr.dim[a] = c->dim[a]; }
  CK(c, cudaMemsetAsync(c->cell_dirs, 0x80, (size_t)cap * 512, s), "cell bytes init");
  begin_timed(c, 2, s, &tl);
  CK(c, launch_bricks(reinterpret_cast<const int4 *>(c->keys), n, c->table, cap - 1, c->sdf, c->weight, c->rgb,
                      c->brick_a, c->brick_b, c->cell_dirs, nullptr, gr, s),
     "bricks");
  end_timed(c, s, &tl);
  begin_timed(c, 2, s, &tl);
  CK(c, launch_cell_masks(c->locations, c->n_loc, c->cell_dirs, c->cell_pos, c->surface, lo[0], lo[1], lo[2], c->dim[0],
                          c->dim[1], s),
     "cell masks");
  end_timed(c, s, &tl);
  if (c->loc_grid) {
    {
      begin_timed(c, 2, s, &tl);
      CK(c, launch_loc_grid(c->locations, c->n_loc, c->surface, c->table, c->loc_grid, lo[0], lo[1], lo[2],
                            c->dim[0], c->dim[1], s),
         "loc_grid");
      end_timed(c, s, &tl);
      if (ensure(c->dist_tmp, c->cap_dist, 2 * cells) == cudaSuccess) {
        begin_timed(c, 2, s, &tl, 4);
        CK(c, launch_empty_distance(c->loc_grid, c->dist_tmp, c->dist_tmp + cells, c->dim[0], c->dim[1], c->dim[2], s),
           "distance");
        end_timed(c, s, &tl);
#if DTSDF_EMPTY_BOX
        // the cubes grown into boxes (the incremental update after a fused frame keeps the grown
        // boxes while no location is added, and falls back to the cubes when one is)
        const size_t sat_n = (size_t)(c->dim[0] + 1) * (c->dim[1] + 1) * (c->dim[2] + 1);
        if (ensure(c->box_sat, c->cap_box_sat, sat_n * 4) == cudaSuccess) {
          begin_timed(c, 2, s, &tl, 5);
          CK(c, launch_empty_box(c->loc_grid, c->box_sat, c->dim[0], c->dim[1], c->dim[2], s), "empty boxes");
          end_timed(c, s, &tl);
        } else {
          cudaGetLastError();
        }
#endif
      } else {
        cudaGetLastError();
      }
    }
  }
  if (c->combined) {
    if (c->comb_entries != c->table_cap) {
      dfree(c->comb_slot);
      if (dalloc(c->comb_slot, (size_t)c->table_cap * 4) != cudaSuccess) {
        cudaGetLastError();
        free_combined(c);
      } else {
        c->comb_entries = c->table_cap;
      }
    }
    if (c->combined) {
      CK(c, cudaMemsetAsync(c->comb_slot, 0xFF, (size_t)c->table_cap * 4, s), "combined remap init");
      begin_timed(c, 3, s, &tl, c->n_comb > 0 ? 1 : 0);
      CK(c, launch_comb_remap(c->table, c->table_cap - 1, c->comb_loc, c->n_comb, c->comb_slot, s), "combined remap");
      end_timed(c, s, &tl);
    }
  }
  CK(c, cudaStreamSynchronize(s), "commit sync");
  c->committed = true;
  return DTSDF_OK;
}

int dtsdf_upload_volume(dtsdf_ctx *c, const dtsdf_volume_params *p, const int32_t *keys, const float *sdf,
                        const float *weight, const uint8_t *rgb) {
  if (!c) return fail(DTSDF_ERR_INVALID_ARGUMENT, "ctx is NULL");
  int rc = check_params(p);
  if (rc) return rc;
  if (p->n_blocks > 0 && (!keys || !sdf || !weight))
    return fail(DTSDF_ERR_INVALID_ARGUMENT, "keys/sdf/weight must not be NULL");
  dtsdf_volume_buffers b;
  if ((rc = dtsdf_alloc_volume(c, p, &b))) return rc;
  const size_t n = (size_t)p->n_blocks;
  auto kind = [](const void *ptr) { return is_device_ptr(ptr) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice; };
  if (n > 0) {
    CK(c, cudaMemcpy(b.keys, keys, n * 16, kind(keys)), "upload keys");
    CK(c, cudaMemcpy(b.sdf, sdf, n * 512 * 4, kind(sdf)), "upload sdf");
    CK(c, cudaMemcpy(b.weight, weight, n * 512 * 4, kind(weight)), "upload weight");
    if (rgb) CK(c, cudaMemcpy(b.rgb, rgb, n * 512 * 3, kind(rgb)), "upload rgb");
    else CK(c, cudaMemset(b.rgb, 0, n * 512 * 3), "zero rgb");
  }
  return dtsdf_commit_volume(c, nullptr);
}

constexpr long long kOrderAutoMaxCtas = 65536;  // DTSDF_OPT_TILE_ORDER 1: CTA tiles per launch up to which the order is used

static int render_impl(dtsdf_ctx *c, int32_t n_views, const float *poses, const dtsdf_intrinsics *K, int32_t row0,
                       int32_t row1, float *depth, float *normal, uint8_t *color, uint8_t *mask, cudaStream_t s,
                       bool comb, bool staged = false) {
  const int W = K->width;
  const int rows = row1 - row0;
  const int tiles_x = (W + kRangeTile - 1) / kRangeTile, tiles_y = (rows + kRangeTile - 1) / kRangeTile;
  const size_t tiles = (size_t)tiles_x * tiles_y * std::min(n_views, kViewsPerLaunch);
  if (tiles > c->range_cap) {
    dfree(c->z_near);
    dfree(c->z_far);
    dfree(c->tile_count);
    c->range_cap = 0;
    if (dalloc(c->z_near, tiles * 8) != cudaSuccess || dalloc(c->z_far, tiles * 8) != cudaSuccess ||
        dalloc(c->tile_count, tiles * 4) != cudaSuccess) {
      cudaGetLastError();
      return fail(DTSDF_ERR_OUT_OF_MEMORY, "range buffers");
    }
    CK(c, cudaMemsetAsync(c->tile_count, 0, tiles * 4, s), "tile counts");
    c->range_cap = tiles;
    c->range_epoch = 0;
  }
  int ct_x = 0, ct_y = 0;
  raycast_tiles(W, rows, &ct_x, &ct_y);
  const size_t cts = (size_t)ct_x * ct_y * std::min(n_views, kViewsPerLaunch);
  if (cts > c->order_cap) {
    dfree(c->tile_order);
    c->order_cap = 0;
    if (dalloc(c->tile_order, cts * 4) != cudaSuccess) {
      cudaGetLastError();
      return fail(DTSDF_ERR_OUT_OF_MEMORY, "tile order");
    }
    c->order_cap = cts;
  }
  // the order pays most when the launch is a few waves of CTAs (one view: C1 -12 %); by 256-view
  // batches the drain is amortised and it is neutral (profiles/r1f_sweep_tile_order.jsonl)
  const bool order = tile_order_fits(W, rows) &&
                     (c->use_order == 2 || (c->use_order == 1 && cts <= (size_t)kOrderAutoMaxCtas));
  VolumeView V;
  V.table = c->table;
  V.table_mask = c->table_cap - 1;
  V.bitmap = c->bitmap;
  V.surface = c->surface;
  V.cell_pos = c->cell_pos;
  V.cell_dirs = c->cell_dirs;
  V.use_live = c->use_live;
  V.loc_grid = c->use_grid ? c->loc_grid : nullptr;
  V.lo_x = c->lo[0]; V.lo_y = c->lo[1]; V.lo_z = c->lo[2];
  V.dim_x = c->dim[0]; V.dim_y = c->dim[1]; V.dim_z = c->dim[2];
  V.brick_a = c->brick_a;
  V.brick_b = c->brick_b;
  V.voxel_size = c->params.voxel_size;
  V.inv_voxel = 1.0f / c->params.voxel_size;
  V.theta = c->params.theta;
  V.cos_theta = cosf(c->params.theta);
  V.sin_theta = sinf(c->params.theta);
  V.inv_blend = (float)(1.0 / (2.0 * (double)c->params.theta - 3.14159265358979323846 / 2.0));
  V.delta = c->params.step > 0.f ? c->params.step : c->params.voxel_size;
  V.inv_delta = 1.0f / V.delta;
  V.n_blocks = c->n;
  V.table_cap = c->table_cap;
  static thread_local RangeLaunch rl;
  static thread_local RenderLaunch pl;
  for (int v0 = 0; v0 < n_views; v0 += kViewsPerLaunch) {
    const int nv = std::min(kViewsPerLaunch, n_views - v0);
    rl.vol = V;
    rl.locations = comb ? c->comb_loc : c->locations;  // combined: only the combined locations bound rays
    rl.n_locations = comb ? c->n_comb : c->n_loc;
    rl.fx = K->fx; rl.fy = K->fy; rl.cx = K->cx; rl.cy = K->cy; rl.z_min = K->z_min; rl.z_max = K->z_max;
    rl.width = W; rl.height = K->height; rl.row0 = row0; rl.row1 = row1;
    rl.n_views = nv; rl.tiles_x = tiles_x; rl.tiles_y = tiles_y;
    rl.z_near = c->z_near; rl.z_far = c->z_far;
    for (int i = 0; i < nv; ++i) {
      const float *T = poses + 16 * (size_t)(v0 + i);
      for (int a = 0; a < 3; ++a) {
        for (int b = 0; b < 3; ++b) rl.pose[i].r[3 * a + b] = T[4 * a + b];
        rl.pose[i].t[a] = T[4 * a + 3];
      }
    }
    TimedLaunch tl{};
    if (c->range_epoch == 0 || c->range_epoch >= 0xFFFFFFF0u) {
      // fresh buffers (or the epoch counter wrapping): keys of epoch 0, which loses every atomic
      // of an epoch >= 1 (near tag 0xFFFFFFFF, far tag 0)
      begin_timed(c, 2, s, &tl, 0);
      CK(c, cudaMemsetAsync(c->z_near, 0xFF, c->range_cap * 8, s), "range init");
      CK(c, cudaMemsetAsync(c->z_far, 0x00, c->range_cap * 8, s), "range init");
      end_timed(c, s, &tl);
      c->range_epoch = 0;
    }
    rl.epoch = ++c->range_epoch;
    rl.count = order ? c->tile_count : nullptr;
    begin_timed(c, 0, s, &tl, (rl.n_locations > 0 ? 1 : 0) + (order ? 1 : 0));
    CK(c, launch_range(rl, s), "range pass");
    if (order)
      CK(c, launch_order(c->tile_count, c->tile_order, tiles_x, tiles_y, W, rows, nv, s), "tile order");
    end_timed(c, s, &tl);
    pl.vol = V;
    pl.fx = K->fx; pl.fy = K->fy; pl.cx = K->cx; pl.cy = K->cy; pl.z_min = K->z_min; pl.z_max = K->z_max;
    pl.width = W; pl.height = K->height; pl.row0 = row0; pl.row1 = row1;
    pl.n_views = nv; pl.tiles_x = tiles_x; pl.tiles_y = tiles_y;
    pl.use_range = c->use_range; pl.use_skip = c->use_skip;
    pl.n_bisect = 0;
    while (V.delta / (float)(1 << pl.n_bisect) > 5e-5f && pl.n_bisect < 20) ++pl.n_bisect;
    if (c->bisect_steps >= 0) pl.n_bisect = c->bisect_steps;
    pl.refine_tol = 1e-9f * (float)c->refine_tol_nm;
    pl.z_near = c->z_near; pl.z_far = c->z_far;
    pl.epoch = rl.epoch;
    pl.order = order ? c->tile_order : nullptr;
    pl.ct_x = ct_x;
    const size_t px = (size_t)v0 * rows * W;
    pl.out_depth = depth + px;
    pl.out_normal = normal ? normal + 3 * px : nullptr;
    pl.out_color = color ? color + 3 * px : nullptr;
    pl.out_mask = mask ? mask + px : nullptr;
    pl.dbg_timeline = nullptr;
    pl.dbg_trace = nullptr;
    pl.dbg_trace_pix = -1;
#ifdef DTSDF_ALWAYS_STAGED
    staged = true;
#endif
    pl.staged = staged ? 1 : 0;
    pl.combined = comb ? 1 : 0;
    pl.comb.n_slots = c->n_comb;
    pl.comb.slot_of_entry = c->comb_slot;
    pl.comb.apron = c->comb_apron;
    pl.comb.rgb = c->comb_rgb;
    pl.comb.cell_pos = c->comb_cell_pos;
    pl.comb.surf = c->comb_surf;
#ifdef DTSDF_STATS
    {
      static unsigned long long *tl_buf = nullptr;
      static size_t tl_cap = 0;
      const size_t need = (size_t)nv * rows * W * 3;
      if (need > tl_cap) {
        if (tl_buf) cudaFree(tl_buf);
        cudaMalloc(&tl_buf, need * 8);
        tl_cap = need;
      }
      pl.dbg_timeline = tl_buf;
      dtsdf_debug_timeline = tl_buf;
      if (!dtsdf_debug_trace) {
        cudaMalloc(&dtsdf_debug_trace, 32 * 128 * 8 * 8);
        cudaMemset(dtsdf_debug_trace, 0, 32 * 128 * 8 * 8);
      }
      pl.dbg_trace = dtsdf_debug_trace;
      pl.dbg_trace_pix = dtsdf_debug_trace_pix;
    }
#endif

    std::memcpy(pl.pose, rl.pose, sizeof(ViewPose) * nv);
    begin_timed(c, 1, s, &tl);
    CK(c, launch_raycast(pl, s), "raycast");
    end_timed(c, s, &tl);
  }
  return DTSDF_OK;
}

static int render_batch_impl(dtsdf_ctx *c, int32_t n_views, const float *poses, const dtsdf_intrinsics *K,
                             int32_t row0, int32_t row1, float *depth, float *normal, uint8_t *color, uint8_t *mask,
                             void *stream, bool comb) {
  if (!c) return fail(DTSDF_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (c->sticky) return fail(DTSDF_ERR_CUDA, "context has a sticky CUDA error");
  int rc = check_intr(K);
  if (rc) return rc;
  if (n_views < 1) return fail(DTSDF_ERR_INVALID_ARGUMENT, "n_views must be >= 1");
  if (!poses || !depth) return fail(DTSDF_ERR_INVALID_ARGUMENT, "poses/out_depth is NULL");
  if (row0 < 0 || row1 > K->height || row0 >= row1) return fail(DTSDF_ERR_INVALID_ARGUMENT, "bad row range");
  for (int64_t i = 0; i < 16 * (int64_t)n_views; ++i)
    if (!std::isfinite(poses[i])) return fail(DTSDF_ERR_INVALID_ARGUMENT, "pose is not finite");
  if (!c->committed) return fail(DTSDF_ERR_NO_VOLUME, "no committed volume");
  if (comb && !c->combined) return fail(DTSDF_ERR_NO_COMBINED, "no combined TSDF (call dtsdf_combine)");
  cudaSetDevice(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  // classify every output once (one attribute query each): device, mapped page-locked host, pageable
  void *outs[4] = {depth, normal, color, mask};
  void *mapped_ptr[4] = {nullptr, nullptr, nullptr, nullptr};
  int n_dev = 0, n_host = 0, n_mapped = 0;
  for (int i = 0; i < 4; ++i) {
    if (!outs[i]) continue;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, outs[i]) != cudaSuccess) {
      cudaGetLastError();
      a.type = cudaMemoryTypeUnregistered;
      a.devicePointer = nullptr;
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
      ++n_dev;
    } else {
      ++n_host;
      if (a.type == cudaMemoryTypeHost && a.devicePointer) {
        ++n_mapped;
        mapped_ptr[i] = a.devicePointer;
      }
    }
  }
  if (n_dev && n_host) return fail(DTSDF_ERR_INVALID_ARGUMENT, "outputs must be all device or all host pointers");
  if (n_dev) return render_impl(c, n_views, poses, K, row0, row1, depth, normal, color, mask, s, comb);
  // host outputs in page-locked memory (mapped into the device address space under UVA, e.g.
  // torch pin_memory()): the raycast writes its staged output rows straight into them across the
  // host link while it runs, then the call synchronizes -- no staging copy after the kernel
  if (c->host_write && n_mapped == n_host) {
    rc = render_impl(c, n_views, poses, K, row0, row1, (float *)mapped_ptr[0], (float *)mapped_ptr[1],
                     (uint8_t *)mapped_ptr[2], (uint8_t *)mapped_ptr[3], s, comb, /*staged=*/true);
    if (rc) return rc;
    CK(c, cudaStreamSynchronize(s), "render sync");
    return DTSDF_OK;
  }
  // pageable host outputs: render into device scratch, copy back, synchronize
  const size_t px = (size_t)n_views * (row1 - row0) * K->width;
  const size_t need = px * (4 + 12 + 3 + 1) + 64;
  if (need > c->host_stage_cap) {
    if (c->host_stage) cudaFree(c->host_stage);
    c->host_stage = nullptr;
    c->host_stage_cap = 0;
    if (cudaMalloc(&c->host_stage, need) != cudaSuccess) {
      cudaGetLastError();
      return fail(DTSDF_ERR_OUT_OF_MEMORY, "host-output staging");
    }
    c->host_stage_cap = need;
  }
  char *base = (char *)c->host_stage;
  float *dd = (float *)base;
  float *dn = normal ? (float *)(base + px * 4) : nullptr;
  uint8_t *dc = color ? (uint8_t *)(base + px * 16) : nullptr;
  uint8_t *dm = mask ? (uint8_t *)(base + px * 19) : nullptr;
  rc = render_impl(c, n_views, poses, K, row0, row1, dd, dn, dc, dm, s, comb);
  if (rc) return rc;
  CK(c, cudaMemcpyAsync(depth, dd, px * 4, cudaMemcpyDeviceToHost, s), "d2h depth");
  if (normal) CK(c, cudaMemcpyAsync(normal, dn, px * 12, cudaMemcpyDeviceToHost, s), "d2h normal");
  if (color) CK(c, cudaMemcpyAsync(color, dc, px * 3, cudaMemcpyDeviceToHost, s), "d2h color");
  if (mask) CK(c, cudaMemcpyAsync(mask, dm, px, cudaMemcpyDeviceToHost, s), "d2h mask");
  CK(c, cudaStreamSynchronize(s), "render sync");
  return DTSDF_OK;
}

int dtsdf_render_batch(dtsdf_ctx *c, int32_t n_views, const float *poses, const dtsdf_intrinsics *K, int32_t row0,
                       int32_t row1, float *depth, float *normal, uint8_t *color, uint8_t *mask, void *stream) {
  return render_batch_impl(c, n_views, poses, K, row0, row1, depth, normal, color, mask, stream, false);
}

int dtsdf_render_combined(dtsdf_ctx *c, int32_t n_views, const float *poses, const dtsdf_intrinsics *K, int32_t row0,
                          int32_t row1, float *depth, float *normal, uint8_t *color, uint8_t *mask, void *stream) {
  return render_batch_impl(c, n_views, poses, K, row0, row1, depth, normal, color, mask, stream, true);
}

int dtsdf_combine(dtsdf_ctx *c, const float pose[16], const dtsdf_intrinsics *K, float margin, void *stream) {
  return dtsdf_combine_mode(c, pose, K, margin, DTSDF_COMBINE_WEIGHTED, 0.0f, stream);
}

}  // extern "C"

namespace {

// combined-TSDF buffers for `cap` slots (slot_of_entry sized by the hash table)
int comb_alloc(dtsdf_ctx *c, int64_t cap) {
  if (dalloc(c->comb_slot, (size_t)c->table_cap * 4) != cudaSuccess ||
      dalloc(c->comb_loc, (size_t)cap * sizeof(int4)) != cudaSuccess ||
      dalloc(c->comb_apron, (size_t)cap * kApronStride * 4) != cudaSuccess ||
      dalloc(c->comb_weight, (size_t)cap * kVoxPerBlock * 4) != cudaSuccess ||
      dalloc(c->comb_rgb, (size_t)cap * kRgbApronStride * sizeof(uchar4)) != cudaSuccess ||
      dalloc(c->comb_cell_pos, (size_t)cap * 64) != cudaSuccess || dalloc(c->comb_surf, (size_t)cap) != cudaSuccess ||
      dalloc(c->comb_cls, (size_t)cap) != cudaSuccess || dalloc(c->comb_count, 16) != cudaSuccess) {
    cudaGetLastError();
    free_combined(c);
    return fail(DTSDF_ERR_OUT_OF_MEMORY, "combined TSDF buffers");
  }
  c->comb_cap = cap;
  c->comb_entries = c->table_cap;
  return DTSDF_OK;
}

// grow the combined buffers to `cap` slots keeping the first n_comb slots (R58 updates add slots)
template <typename T>
cudaError_t grow_copy(T *&p, size_t old_bytes, size_t new_bytes, cudaStream_t s) {
  T *q = nullptr;
  cudaError_t e = cudaMalloc((void **)&q, std::max<size_t>(new_bytes, 16));
  if (e != cudaSuccess) return e;
  if (old_bytes) e = cudaMemcpyAsync(q, p, old_bytes, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) { cudaFree(q); return e; }
  cudaStreamSynchronize(s);
  cudaFree(p);
  p = q;
  return cudaSuccess;
}

int comb_grow(dtsdf_ctx *c, int64_t cap, cudaStream_t s) {
  const size_t n = (size_t)c->n_comb, m = (size_t)cap;
  if (grow_copy(c->comb_loc, n * sizeof(int4), m * sizeof(int4), s) != cudaSuccess ||
      grow_copy(c->comb_apron, n * kApronStride * 4, m * kApronStride * 4, s) != cudaSuccess ||
      grow_copy(c->comb_weight, n * kVoxPerBlock * 4, m * kVoxPerBlock * 4, s) != cudaSuccess ||
      grow_copy(c->comb_rgb, n * kRgbApronStride * sizeof(uchar4), m * kRgbApronStride * sizeof(uchar4), s) != cudaSuccess ||
      grow_copy(c->comb_cell_pos, n * 64, m * 64, s) != cudaSuccess || grow_copy(c->comb_surf, n, m, s) != cudaSuccess ||
      grow_copy(c->comb_cls, n, m, s) != cudaSuccess) {
    cudaGetLastError();
    free_combined(c);
    return fail(DTSDF_ERR_OUT_OF_MEMORY, "combined TSDF buffers (growth after fusion)");
  }
  c->comb_cap = cap;
  return DTSDF_OK;
}

// the combine launch of the current volume and the stored camera / rule of the combined TSDF
void comb_launch(dtsdf_ctx *c, CombineLaunch &L) {
  const float *pose = c->comb_pose;
  const dtsdf_intrinsics *K = &c->comb_K;
  const float margin = c->comb_margin;
  L = CombineLaunch{};
  L.vol.table = c->table;
  L.vol.table_mask = c->table_cap - 1;
  L.vol.loc_grid = c->use_grid ? c->loc_grid : nullptr;
  L.vol.lo_x = c->lo[0]; L.vol.lo_y = c->lo[1]; L.vol.lo_z = c->lo[2];
  L.vol.dim_x = c->dim[0]; L.vol.dim_y = c->dim[1]; L.vol.dim_z = c->dim[2];
  L.vol.brick_a = c->brick_a;
  L.vol.brick_b = c->brick_b;
  L.vol.voxel_size = c->params.voxel_size;
  L.vol.inv_voxel = 1.0f / c->params.voxel_size;
  L.vol.theta = c->params.theta;
  L.vol.cos_theta = cosf(c->params.theta);
  L.vol.sin_theta = sinf(c->params.theta);
  L.vol.inv_blend = (float)(1.0 / (2.0 * (double)c->params.theta - 3.14159265358979323846 / 2.0));
  L.vol.n_blocks = c->n;
  L.vol.table_cap = c->table_cap;
  L.locations = c->locations;
  L.n_loc = c->n_loc;
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) L.R[3 * a + b] = (double)pose[4 * a + b];
    L.t[a] = (double)pose[4 * a + 3];
  }
  L.fx = K->fx; L.fy = K->fy; L.cx = K->cx; L.cy = K->cy; L.z_min = K->z_min; L.z_max = K->z_max;
  L.mu = (double)margin * (double)K->width;
  L.mv = (double)margin * (double)K->height;
  L.umax = (double)(K->width - 1) + L.mu;
  L.vmax = (double)(K->height - 1) + L.mv;
  L.slot_of_entry = c->comb_slot;
  L.comb_loc = c->comb_loc;
  L.n_sel = c->comb_count;
  L.apron = c->comb_apron;
  L.rgb = c->comb_rgb;
  L.weight = c->comb_weight;
  L.cell_pos = c->comb_cell_pos;
  L.surf = c->comb_surf;
  L.cls = c->comb_cls;
  L.had = nullptr;
  L.n_old = 0;
  L.mode = c->comb_mode;
  L.w_floor = c->comb_wfloor;
  L.theta64 = (double)c->params.theta;
}

// R58: after a fused frame -- the volume re-committed, the kept slots re-pointed --
// combine the voxels that received data for the first time with the stored camera: the frame's
// new locations inside the widened frustum get slots (computed whole), the old slots only at
// voxels whose had bit (captured before the frame) is clear and that hold data now; then the
// aprons and skip masks of every slot are rebuilt.
int comb_update(dtsdf_ctx *c, cudaStream_t s) {
  const int64_t n_old = c->n_comb;
  if (c->n_loc > c->comb_cap) {
    int rc = comb_grow(c, c->n_loc, s);
    if (rc) return rc;
  }
  CombineLaunch L;
  comb_launch(c, L);
  L.had = c->comb_had;
  L.n_old = n_old;
  const unsigned int n0 = (unsigned int)n_old;
  CK(c, cudaMemcpyAsync(c->comb_count, &n0, 4, cudaMemcpyHostToDevice, s), "combine update init");
  TimedLaunch tl{};
  begin_timed(c, 3, s, &tl, c->n_loc > 0 ? 1 : 0);
  CK(c, launch_combine(L, s), "combine update select");
  end_timed(c, s, &tl);
  unsigned int nsel = 0;
  CK(c, cudaMemcpyAsync(&nsel, c->comb_count, 4, cudaMemcpyDeviceToHost, s), "combine update readback");
  CK(c, cudaStreamSynchronize(s), "combine update sync");
  begin_timed(c, 3, s, &tl, nsel > 0 ? 2 : 0);
  CK(c, launch_combine_finish(L, (long long)nsel, s), "combine update");
  end_timed(c, s, &tl);
  c->n_comb = nsel;
  return DTSDF_OK;
}

}  // namespace

extern "C" {

int dtsdf_combine_mode(dtsdf_ctx *c, const float pose[16], const dtsdf_intrinsics *K, float margin, int32_t mode,
                       float w_floor, void *stream) {
  if (!c) return fail(DTSDF_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (mode != DTSDF_COMBINE_WEIGHTED && mode != DTSDF_COMBINE_ALGORITHM1)
    return fail(DTSDF_ERR_INVALID_ARGUMENT, "unknown combination mode");
  if (!(w_floor >= 0.f) || !std::isfinite(w_floor)) return fail(DTSDF_ERR_INVALID_ARGUMENT, "w_floor must be >= 0");
  if (c->sticky) return fail(DTSDF_ERR_CUDA, "context has a sticky CUDA error");
  int rc = check_intr(K);
  if (rc) return rc;
  if (!pose) return fail(DTSDF_ERR_INVALID_ARGUMENT, "pose is NULL");
  for (int i = 0; i < 16; ++i)
    if (!std::isfinite(pose[i])) return fail(DTSDF_ERR_INVALID_ARGUMENT, "pose is not finite");
  if (!(margin >= 0.f) || !(margin <= 16.f)) return fail(DTSDF_ERR_INVALID_ARGUMENT, "margin must lie in [0, 16]");
  if (!c->committed) return fail(DTSDF_ERR_NO_VOLUME, "no committed volume");
  cudaSetDevice(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  c->combined = false;
  // capacity: every allocated location (kept across combines of the same volume)
  const int64_t cap = std::max<int64_t>(c->n_loc, 1);
  if (c->comb_cap < cap || c->comb_entries != c->table_cap) {
    free_combined(c);
    if ((rc = comb_alloc(c, cap))) return rc;
  }
  std::memcpy(c->comb_pose, pose, sizeof(c->comb_pose));
  c->comb_K = *K;
  c->comb_margin = margin;
  c->comb_mode = mode;
  c->comb_wfloor = w_floor;
  CombineLaunch L;
  comb_launch(c, L);
  TimedLaunch tl{};
  CK(c, cudaMemsetAsync(c->comb_slot, 0xFF, (size_t)c->table_cap * 4, s), "combine init");
  CK(c, cudaMemsetAsync(c->comb_count, 0, 16, s), "combine init");
  begin_timed(c, 3, s, &tl, c->n_loc > 0 ? 1 : 0);
  CK(c, launch_combine(L, s), "combine");
  end_timed(c, s, &tl);
  unsigned int nsel = 0;
  CK(c, cudaMemcpyAsync(&nsel, c->comb_count, 4, cudaMemcpyDeviceToHost, s), "combine readback");
  CK(c, cudaStreamSynchronize(s), "combine sync");
  begin_timed(c, 3, s, &tl, nsel > 0 ? 2 : 0);
  CK(c, launch_combine_finish(L, (long long)nsel, s), "combine finish");
  end_timed(c, s, &tl);
  c->n_comb = nsel;
  c->combined = true;
  return DTSDF_OK;
}

int dtsdf_combined_stats(dtsdf_ctx *c, int64_t *n_locations, int64_t *bytes) {
  if (!c) return fail(DTSDF_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (!c->combined) return fail(DTSDF_ERR_NO_COMBINED, "no combined TSDF");
  if (n_locations) *n_locations = c->n_comb;
  if (bytes)
    *bytes = (int64_t)c->comb_entries * 4 +
             c->comb_cap * (int64_t)(sizeof(int4) + kApronStride * 4 + kVoxPerBlock * 4 + kRgbApronStride * 4 + 64 + 1);
  return DTSDF_OK;
}

int dtsdf_get_combined(dtsdf_ctx *c, int64_t capacity, int32_t *locs, float *sdf, float *weight, uint8_t *rgb,
                       uint8_t *mask, int64_t *n_out) {
  if (!c || !n_out) return fail(DTSDF_ERR_INVALID_ARGUMENT, "ctx/n_out is NULL");
  if (!c->combined) return fail(DTSDF_ERR_NO_COMBINED, "no combined TSDF");
  *n_out = c->n_comb;
  if (capacity < c->n_comb) return fail(DTSDF_ERR_INVALID_ARGUMENT, "capacity smaller than the combined locations");
  if (c->n_comb == 0) return DTSDF_OK;
  if (!locs || !sdf || !weight || !rgb || !mask) return fail(DTSDF_ERR_INVALID_ARGUMENT, "NULL output");
  cudaSetDevice(c->device);
  const size_t n = (size_t)c->n_comb;
  std::vector<int4> hl(n);
  std::vector<float> ha(n * kApronStride), hw(n * kVoxPerBlock);
  std::vector<uchar4> hr(n * kRgbApronStride);
  CK(c, cudaDeviceSynchronize(), "get_combined sync");
  CK(c, cudaMemcpy(hl.data(), c->comb_loc, n * sizeof(int4), cudaMemcpyDeviceToHost), "get_combined");
  CK(c, cudaMemcpy(ha.data(), c->comb_apron, n * kApronStride * 4, cudaMemcpyDeviceToHost), "get_combined");
  CK(c, cudaMemcpy(hw.data(), c->comb_weight, n * kVoxPerBlock * 4, cudaMemcpyDeviceToHost), "get_combined");
  CK(c, cudaMemcpy(hr.data(), c->comb_rgb, n * kRgbApronStride * sizeof(uchar4), cudaMemcpyDeviceToHost), "get_combined");
  for (size_t i = 0; i < n; ++i) {
    locs[3 * i + 0] = hl[i].x;
    locs[3 * i + 1] = hl[i].y;
    locs[3 * i + 2] = hl[i].z;
    for (int l = 0; l < kVoxPerBlock; ++l) {
      const int lx = l & 7, ly = (l >> 3) & 7, lz = l >> 6;
      sdf[i * kVoxPerBlock + l] = ha[i * kApronStride + (lx + 1) + kApron * (ly + 1) + kApron * kApron * (lz + 1)];
      weight[i * kVoxPerBlock + l] = hw[i * kVoxPerBlock + l];
      const uchar4 q = hr[i * kRgbApronStride + lx + kRgbApron * ly + kRgbApron * kRgbApron * lz];
      rgb[3 * (i * kVoxPerBlock + l) + 0] = q.x;
      rgb[3 * (i * kVoxPerBlock + l) + 1] = q.y;
      rgb[3 * (i * kVoxPerBlock + l) + 2] = q.z;
      mask[i * kVoxPerBlock + l] = q.w;
    }
  }
  return DTSDF_OK;
}

void dtsdf_default_policy(dtsdf_combine_policy *p) {
  if (!p) return;
  p->boot_frames = 5;
  p->stale_frames = 50;
  p->translation = 0.05f;
  p->rotation = (float)(0.05 * 3.14159265358979323846 / 2.0);
}

int dtsdf_should_recombine(const dtsdf_combine_policy *p, int64_t frame, int64_t last, const float pose[16],
                           const float last_pose[16]) {
  if (!p || !pose || !last_pose) return fail(DTSDF_ERR_INVALID_ARGUMENT, "NULL argument");
  if (frame < 0 || last < 0 || last > frame) return fail(DTSDF_ERR_INVALID_ARGUMENT, "need 0 <= last <= frame");
  if (!(p->translation > 0.f) || !(p->rotation > 0.f) || p->boot_frames < 0 || p->stale_frames < 0)
    return fail(DTSDF_ERR_INVALID_ARGUMENT, "policy thresholds must be positive");
  if (frame < p->boot_frames) return 1;                 // eq. condition_1: boot up
  if (frame - last > p->stale_frames) return 1;         // eq. condition_2: stale state
  double d2 = 0.0, tr = 0.0;
  for (int a = 0; a < 3; ++a) {
    const double d = (double)pose[4 * a + 3] - (double)last_pose[4 * a + 3];
    d2 += d * d;
    for (int b = 0; b < 3; ++b) tr += (double)last_pose[4 * a + b] * (double)pose[4 * a + b];
  }
  if (std::sqrt(d2) > (double)p->translation) return 1;  // eq. condition_3: translation
  const double cs = std::min(1.0, std::max(-1.0, (tr - 1.0) / 2.0));
  return std::acos(cs) > (double)p->rotation ? 1 : 0;   // eq. condition_4: rotation
}

// ---- fusion (NEXT-2, fusion.cu) ----------------------------------------------------------
void dtsdf_default_fusion_params(dtsdf_fusion_params *p) {
  if (!p) return;
  p->max_weight = 128.0f;
  p->carve_weight = 1.0f;
  p->carve_radius = 2;
  p->reserved = 0;
}

int dtsdf_fusion_reserve(dtsdf_ctx *c, const dtsdf_volume_params *p, int64_t capacity) {
  if (!c) return fail(DTSDF_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (c->sticky) return fail(DTSDF_ERR_CUDA, "context has a sticky CUDA error");
  if (capacity < 1 || capacity > (int64_t)INT32_MAX / 2) return fail(DTSDF_ERR_INVALID_ARGUMENT, "bad capacity");
  cudaSetDevice(c->device);
  if (!c->allocated) {
    int rc = check_params(p);
    if (rc) return rc;
    dtsdf_volume_params q = *p;
    q.n_blocks = 0;
    dtsdf_volume_buffers b;
    if ((rc = dtsdf_alloc_volume(c, &q, &b))) return rc;
  }
  if (capacity < c->n) return fail(DTSDF_ERR_INVALID_ARGUMENT, "capacity below the current block count");
  CK(c, cudaDeviceSynchronize(), "reserve sync");
  const size_t n = (size_t)c->n, cp = (size_t)capacity;
  int32_t *keys = nullptr;
  float *sdf = nullptr, *weight = nullptr, *cw = nullptr;
  uint8_t *rgb = nullptr;
  if (dalloc(keys, cp * 16) != cudaSuccess || dalloc(sdf, cp * 512 * 4) != cudaSuccess ||
      dalloc(weight, cp * 512 * 4) != cudaSuccess || dalloc(rgb, cp * 512 * 3) != cudaSuccess ||
      dalloc(cw, cp * 512 * 4) != cudaSuccess) {
    cudaGetLastError();
    dfree(keys); dfree(sdf); dfree(weight); dfree(rgb); dfree(cw);
    return fail(DTSDF_ERR_OUT_OF_MEMORY, "fusion pool");
  }
  if (n > 0) {
    CK(c, cudaMemcpy(keys, c->keys, n * 16, cudaMemcpyDeviceToDevice), "reserve copy");
    CK(c, cudaMemcpy(sdf, c->sdf, n * 512 * 4, cudaMemcpyDeviceToDevice), "reserve copy");
    CK(c, cudaMemcpy(weight, c->weight, n * 512 * 4, cudaMemcpyDeviceToDevice), "reserve copy");
    CK(c, cudaMemcpy(rgb, c->rgb, n * 512 * 3, cudaMemcpyDeviceToDevice), "reserve copy");
    // reading R45: blocks that were not fused here count their colour as observed with the depth weight
    CK(c, cudaMemcpy(cw, c->cweight ? c->cweight : c->weight, n * 512 * 4, cudaMemcpyDeviceToDevice), "reserve copy");
  }
  dfree(c->keys); dfree(c->sdf); dfree(c->weight); dfree(c->rgb); dfree(c->cweight);
  c->keys = keys; c->sdf = sdf; c->weight = weight; c->rgb = rgb; c->cweight = cw;
  c->cap = capacity;
  c->params.n_blocks = c->n;
  return dtsdf_commit_volume(c, nullptr);
}

// Incremental index update after a fused frame (the hash table was extended in place by the
// allocation, new locations appended, dirty blocks flagged): the 27-neighbourhoods of the dirty
// blocks get their locations' record bricks, live-direction bytes, certainly-positive masks,
// surface bits and location-grid values rebuilt; new locations set their occupancy bits and, if
// any, the empty-space distances are recomputed.  Equals a full re-commit (tests: DTSDF_OPT_
// INCREMENTAL 0 vs 1 render bit-identical).
static int recommit_incremental(dtsdf_ctx *c, cudaStream_t s, int64_t n_blk_old, int64_t n_loc_old,
                                int64_t n_loc_new) {
  const unsigned int mask = c->table_cap - 1;
  const int4 *keys = reinterpret_cast<const int4 *>(c->keys);
  TimedLaunch tl{};
  // (inc_ctr[0] already counts the locations k_fuse marked; [1] is zero)
  if (n_loc_new > n_loc_old) {  // the new locations enter the grid first (their final values follow below)
    begin_timed(c, 2, s, &tl);
    CK(c, launch_loc_grid(c->locations + n_loc_old, n_loc_new - n_loc_old, c->surface, c->table, c->loc_grid, c->lo[0],
                          c->lo[1], c->lo[2], c->dim[0], c->dim[1], s),
       "incremental grid (new locations)");
    end_timed(c, s, &tl);
  }
  begin_timed(c, 2, s, &tl);
  // the frame's new blocks (k_fuse marked the neighbourhoods of the blocks it changed)
  CK(c, launch_inc_mark(keys, n_blk_old, c->n, c->blk_dirty, c->table, mask, c->loc_grid, c->lo, c->dim, c->loc_mark,
                        c->loc_list, c->inc_ctr, s),
     "incremental mark");
  end_timed(c, s, &tl);
  // the listed locations are counted on the device (inc_ctr[0]); the kernels below read the count
  // themselves (n_list: its upper bound, every location of the table), so the host does not wait
  const unsigned long long *cnt = c->inc_ctr;
  const long long n_list = (long long)c->table_cap;
  begin_timed(c, 2, s, &tl, 5);
  CK(c, launch_cell_init(c->loc_list, n_list, c->cell_dirs, s, cnt), "incremental cell init");
  CK(c, launch_inc_blocks(c->loc_list, n_list, c->table, c->blk_list, c->inc_ctr, s), "incremental blocks");
  GridRef gr{};
  gr.grid = c->loc_grid;
  for (int a = 0; a < 3; ++a) { gr.lo[a] = c->lo[a]; gr.dim[a] = c->dim[a]; }
  CK(c, launch_bricks_counted(keys, 6 * n_list, c->inc_ctr + 1, c->table, mask, c->sdf, c->weight, c->rgb, c->brick_a,
                              c->brick_b, c->cell_dirs, c->blk_list, gr, s),
     "incremental bricks");
  CK(c, launch_cell_masks(c->loc_list, n_list, c->cell_dirs, c->cell_pos, c->surface, c->lo[0], c->lo[1], c->lo[2],
                          c->dim[0], c->dim[1], s, cnt),
     "incremental cell masks");
  CK(c, launch_loc_grid(c->loc_list, n_list, c->surface, c->table, c->loc_grid, c->lo[0], c->lo[1], c->lo[2],
                        c->dim[0], c->dim[1], s, cnt),
     "incremental grid");
  end_timed(c, s, &tl);
  if (n_loc_new > n_loc_old) {
    begin_timed(c, 2, s, &tl, 1);
    CK(c, launch_bitmap(c->locations + n_loc_old, n_loc_new - n_loc_old, c->bitmap, c->lo[0], c->lo[1], c->lo[2],
                        c->dim[0], c->dim[1], s),
       "incremental bitmap");
    end_timed(c, s, &tl);
    const size_t cells = (size_t)c->dim[0] * c->dim[1] * c->dim[2];
    if (c->dist_tmp && c->cap_dist >= 2 * cells) {
      begin_timed(c, 2, s, &tl, 4);
      CK(c, launch_empty_distance(c->loc_grid, c->dist_tmp, c->dist_tmp + cells, c->dim[0], c->dim[1], c->dim[2], s),
         "incremental distance");
      end_timed(c, s, &tl);
    }
  }
  begin_timed(c, 2, s, &tl, 1);
  CK(c, launch_inc_unmark(c->loc_list, n_list, c->loc_mark, s, cnt), "incremental unmark");
  end_timed(c, s, &tl);
  CK(c, cudaStreamSynchronize(s), "incremental sync");
  c->n_loc = n_loc_new;
  c->committed = true;
  return DTSDF_OK;
}

static void fuse_launch_common(dtsdf_ctx *c, const float pose[16], const dtsdf_intrinsics *K, FuseLaunch &L) {
  std::memset(&L, 0, sizeof(L));
  for (int a = 0; a < 3; ++a) {
    for (int b = 0; b < 3; ++b) L.R[3 * a + b] = (double)pose[4 * a + b];
    L.t[a] = (double)pose[4 * a + 3];
  }
  L.fx = K->fx; L.fy = K->fy; L.cx = K->cx; L.cy = K->cy; L.z_min = K->z_min; L.z_max = K->z_max;
  L.width = K->width;
  L.height = K->height;
  for (int a = 0; a < 9; ++a) L.Rf[a] = (float)L.R[a];
  L.fxf = K->fx; L.fyf = K->fy; L.cxf = K->cx; L.cyf = K->cy;
}

static const void *to_device(dtsdf_ctx *c, const void *src, size_t bytes, size_t offset, cudaStream_t s, bool *ok) {
  *ok = true;
  if (!src || is_device_ptr(src)) return src;
  char *dst = (char *)c->fuse_stage + offset;
  if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s) != cudaSuccess) *ok = false;
  return dst;
}

static int ensure_stage(dtsdf_ctx *c, size_t need) {
  if (need <= c->fuse_stage_cap) return DTSDF_OK;
  if (c->fuse_stage) cudaFree(c->fuse_stage);
  c->fuse_stage = nullptr;
  c->fuse_stage_cap = 0;
  if (cudaMalloc(&c->fuse_stage, need) != cudaSuccess) {
    cudaGetLastError();
    return fail(DTSDF_ERR_OUT_OF_MEMORY, "frame staging");
  }
  c->fuse_stage_cap = need;
  return DTSDF_OK;
}

int dtsdf_depth_normals(dtsdf_ctx *c, const float *depth, const dtsdf_intrinsics *K, float *out_normal, void *stream) {
  if (!c || !depth || !out_normal) return fail(DTSDF_ERR_INVALID_ARGUMENT, "NULL argument");
  if (c->sticky) return fail(DTSDF_ERR_CUDA, "context has a sticky CUDA error");
  int rc = check_intr(K);
  if (rc) return rc;
  cudaSetDevice(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t px = (size_t)K->width * K->height;
  const bool host_out = !is_device_ptr(out_normal);
  if ((rc = ensure_stage(c, px * 16 + 256))) return rc;
  bool ok;
  const float *dd = (const float *)to_device(c, depth, px * 4, 0, s, &ok);
  if (!ok) return cuda_fail(c, cudaGetLastError(), "stage depth");
  float *on = host_out ? (float *)((char *)c->fuse_stage + ((px * 4 + 255) & ~size_t(255))) : out_normal;
  FuseLaunch L;
  const float I[16] = {1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};
  fuse_launch_common(c, I, K, L);
  TimedLaunch tl{};
  begin_timed(c, 2, s, &tl);
  CK(c, launch_depth_normals(dd, L, on, s), "depth normals");
  end_timed(c, s, &tl);
  if (host_out) {
    CK(c, cudaMemcpyAsync(out_normal, on, px * 12, cudaMemcpyDeviceToHost, s), "normals d2h");
    CK(c, cudaStreamSynchronize(s), "normals sync");
  }
  return DTSDF_OK;
}

int dtsdf_fuse(dtsdf_ctx *c, const float *depth, const float *normal, const uint8_t *color, const float pose[16],
               const dtsdf_intrinsics *K, const dtsdf_fusion_params *fp, int64_t *new_blocks, void *stream) {
  if (!c || !depth || !normal || !pose) return fail(DTSDF_ERR_INVALID_ARGUMENT, "NULL argument");
  if (c->sticky) return fail(DTSDF_ERR_CUDA, "context has a sticky CUDA error");
  int rc = check_intr(K);
  if (rc) return rc;
  for (int i = 0; i < 16; ++i)
    if (!std::isfinite(pose[i])) return fail(DTSDF_ERR_INVALID_ARGUMENT, "pose is not finite");
  dtsdf_fusion_params prm;
  dtsdf_default_fusion_params(&prm);
  if (fp) prm = *fp;
  if (!(prm.max_weight > 0.f) || !(prm.carve_weight >= 0.f) || prm.carve_radius < 0 || prm.carve_radius > 16)
    return fail(DTSDF_ERR_INVALID_ARGUMENT, "bad fusion parameters");
  if (!c->committed || !c->cweight) return fail(DTSDF_ERR_NO_VOLUME, "no fusion volume (call dtsdf_fusion_reserve)");
  cudaSetDevice(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  const size_t px = (size_t)K->width * K->height;
  const size_t o_n = (px * 4 + 255) & ~size_t(255), o_c = o_n + ((px * 12 + 255) & ~size_t(255));
  if ((rc = ensure_stage(c, o_c + px * 3 + 256))) return rc;
  bool ok1, ok2, ok3;
  FuseLaunch L;
  fuse_launch_common(c, pose, K, L);
  L.depth = (const float *)to_device(c, depth, px * 4, 0, s, &ok1);
  L.normal = (const float *)to_device(c, normal, px * 12, o_n, s, &ok2);
  L.color = (const unsigned char *)to_device(c, color, px * 3, o_c, s, &ok3);
  if (!ok1 || !ok2 || !ok3) return cuda_fail(c, cudaGetLastError(), "stage frame");
  L.table = c->table;
  L.table_mask = c->table_cap - 1;
  L.keys = c->keys;
  L.sdf = c->sdf;
  L.weight = c->weight;
  L.cweight = c->cweight;
  L.rgb = c->rgb;
  L.capacity = c->cap;
  L.s = (double)c->params.voxel_size;
  L.tau = (double)c->params.truncation;
  L.inv_tau_f = (float)(1.0 / L.tau);
  L.inv_s_f = (float)(1.0 / L.s);
  L.M = (int)std::ceil(4.0 * L.tau / L.s);
  L.step = 2.0 * L.tau / (double)L.M;
  L.cos_theta = std::cos((double)c->params.theta);
  L.theta_f = c->params.theta;
  L.cos_theta_f = cosf(c->params.theta);
  L.sin_theta_f = sinf(c->params.theta);
  L.inv_blend = (float)(1.0 / (2.0 * (double)c->params.theta - 3.14159265358979323846 / 2.0));
  L.max_weight = prm.max_weight;
  L.carve_weight = prm.carve_weight;
  L.carve_radius = prm.carve_radius;
  // R58: which voxels of the combined TSDF's slots hold data before this frame
  const bool comb = c->combined;
  if (comb && c->n_comb > 0) {
    if (ensure(c->comb_had, c->cap_comb_had, (size_t)c->n_comb * 64) != cudaSuccess) {
      cudaGetLastError();
      return fail(DTSDF_ERR_OUT_OF_MEMORY, "combined TSDF update masks");
    }
    TimedLaunch tlh{};
    begin_timed(c, 3, s, &tlh);
    CK(c, launch_comb_had(c->table, c->comb_loc, c->n_comb, c->weight, c->comb_had, s), "combine had");
    end_timed(c, s, &tlh);
  }
  // incremental index update: dirty blocks, appended locations (the full re-commit rebuilds both)
  const bool inc = c->incremental && c->loc_grid != nullptr;
  if (inc) {
    const size_t capb = (size_t)std::max<int64_t>(c->cap, 1), cape = (size_t)c->table_cap;
    const bool fresh_mark = c->cap_loc_mark < cape * 4;
    if (ensure(c->blk_dirty, c->cap_blk_dirty, capb) != cudaSuccess ||
        ensure(c->blk_list, c->cap_blk_list, capb * 4) != cudaSuccess ||
        ensure(c->loc_mark, c->cap_loc_mark, cape * 4) != cudaSuccess ||
        ensure(c->loc_list, c->cap_loc_list, cape * sizeof(int4)) != cudaSuccess ||
        ensure(c->inc_ctr, c->cap_inc_ctr, 32) != cudaSuccess) {
      cudaGetLastError();
      return fail(DTSDF_ERR_OUT_OF_MEMORY, "incremental fusion buffers");
    }
    if (fresh_mark) CK(c, cudaMemsetAsync(c->loc_mark, 0, cape * 4, s), "loc mark init");
    CK(c, cudaMemsetAsync(c->blk_dirty, 0, capb, s), "dirty init");
    L.dirty = c->blk_dirty;
    L.loc_mark = c->loc_mark;
    L.loc_list = c->loc_list;
    L.loc_ctr = c->inc_ctr;
    L.locations = c->locations;
    L.grid = c->loc_grid;
    L.n_loc = reinterpret_cast<unsigned long long *>(c->scratch + 4);
    for (int a = 0; a < 3; ++a) { L.lo[a] = c->lo[a]; L.dim[a] = c->dim[a]; }
  }
  // scratch: flags [0] pool / table full, [1] a new location outside the AABB; u64 location
  // counter at int 4, u64 pool counter at int 12
  L.flags = c->scratch;
  L.n_blocks = reinterpret_cast<unsigned long long *>(c->scratch + 12);
  int init[14] = {0};
  const unsigned long long n0 = (unsigned long long)c->n, nl0 = (unsigned long long)c->n_loc;
  std::memcpy(&init[12], &n0, 8);
  std::memcpy(&init[4], &nl0, 8);
  CK(c, cudaMemcpyAsync(c->scratch, init, sizeof(init), cudaMemcpyHostToDevice, s), "fuse init");
  if (ensure(c->pix_buf, c->cap_pix_buf, px * 3 * sizeof(double4)) != cudaSuccess) {
    cudaGetLastError();
    return fail(DTSDF_ERR_OUT_OF_MEMORY, "frame points");
  }
  L.pix_x = c->pix_buf;
  L.pix_n = c->pix_buf + px;
  L.pix_a = reinterpret_cast<float4 *>(c->pix_buf + 2 * px);
  L.pix_b = L.pix_a + px;
  TimedLaunch tl{};
  begin_timed(c, 2, s, &tl, 1);
  CK(c, launch_fuse_alloc(L, s), "fuse alloc");  // (with the frame points)
  end_timed(c, s, &tl);
  int host[14];
  CK(c, cudaMemcpyAsync(host, c->scratch, sizeof(host), cudaMemcpyDeviceToHost, s), "fuse readback");
  CK(c, cudaStreamSynchronize(s), "fuse sync");
  unsigned long long n1;
  std::memcpy(&n1, &host[12], 8);
  const int64_t n_new = std::min<int64_t>((int64_t)n1, c->cap);
  const bool full = host[0] != 0;
  // counters: [0] marked locations (k_fuse), [1] rebuilt blocks, [2] k_fuse's frustum selection
  // (into blk_list, free until the incremental update)
  int *fuse_list = inc ? c->blk_list : nullptr;
  if (fuse_list) CK(c, cudaMemsetAsync(c->inc_ctr, 0, 32, s), "fuse counters init");
  const int64_t n_blk_old = c->n;
  begin_timed(c, 2, s, &tl, full ? (n_new > c->n ? 1 : 0) : (fuse_list ? 3 : 2));
  CK(c, launch_fuse(L, c->n, n_new, !full, fuse_list, fuse_list ? c->inc_ctr + 2 : nullptr, s), "fuse");  // when full: new blocks initialised, not fused
  end_timed(c, s, &tl);
  if (new_blocks) *new_blocks = n_new - c->n;
  c->n = n_new;
  c->params.n_blocks = n_new;
  unsigned long long nl1;
  std::memcpy(&nl1, &host[4], 8);
  if (inc && !full && host[1] == 0) {
    rc = recommit_incremental(c, s, n_blk_old, c->n_loc, (int64_t)nl1);
  } else {
    if (inc) CK(c, cudaMemsetAsync(c->loc_mark, 0, (size_t)c->table_cap * 4, s), "loc mark reset");
    c->values_trusted = true;  // this library's fusion kernels wrote every value
    rc = dtsdf_commit_volume(c, stream);
    c->values_trusted = false;
  }
  if (rc) return rc;
  if (comb && c->combined && (rc = comb_update(c, s))) return rc;
  if (full) return fail(DTSDF_ERR_OUT_OF_MEMORY, "fusion capacity exhausted (blocks allocated so far are kept)");
  return DTSDF_OK;
}

// ---- ICP (NEXT-3, icp.cu) -----------------------------------------------------------------
void dtsdf_default_icp_params(dtsdf_icp_params *p) {
  if (!p) return;
  p->max_iters = 50;
  p->min_step = 1e-6f;
  p->outlier = 0.005f;
  p->reserved = 0;
}

// stage the three ICP inputs on the device; fills L's input pointers and geometry
static int icp_prepare(dtsdf_ctx *c, const float *depth, const float *ref_depth, const float *ref_normal,
                       const float ref_pose[16], const dtsdf_intrinsics *K, float outlier, cudaStream_t s,
                       IcpLaunch &L) {
  if (!depth || !ref_depth || !ref_normal || !ref_pose) return fail(DTSDF_ERR_INVALID_ARGUMENT, "NULL argument");
  int rc = check_intr(K);
  if (rc) return rc;
  for (int i = 0; i < 16; ++i)
    if (!std::isfinite(ref_pose[i])) return fail(DTSDF_ERR_INVALID_ARGUMENT, "pose is not finite");
  if (!(outlier > 0.f)) return fail(DTSDF_ERR_INVALID_ARGUMENT, "outlier threshold must be > 0");
  const size_t px = (size_t)K->width * K->height;
  const size_t o_r = (px * 4 + 255) & ~size_t(255), o_n = o_r + o_r;
  if ((rc = ensure_stage(c, o_n + px * 12 + 256))) return rc;
  bool ok1, ok2, ok3;
  std::memset(&L, 0, sizeof(L));
  L.depth = (const float *)to_device(c, depth, px * 4, 0, s, &ok1);
  L.ref_depth = (const float *)to_device(c, ref_depth, px * 4, o_r, s, &ok2);
  L.ref_normal = (const float *)to_device(c, ref_normal, px * 12, o_n, s, &ok3);
  if (!ok1 || !ok2 || !ok3) return cuda_fail(c, cudaGetLastError(), "stage ICP inputs");
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) L.ref_R[3 * a + b] = (double)ref_pose[4 * a + b];
  L.fx = K->fx; L.fy = K->fy; L.cx = K->cx; L.cy = K->cy; L.z_min = K->z_min; L.z_max = K->z_max;
  L.outlier = (double)outlier;
  L.width = K->width;
  L.height = K->height;
  const size_t np = (size_t)icp_partials(K->width, K->height);
  if (ensure(c->icp_partials, c->cap_icp_partials, np * 29 * sizeof(double)) != cudaSuccess ||
      ensure(c->icp_state, c->cap_icp_state, sizeof(IcpState)) != cudaSuccess) {
    cudaGetLastError();
    return fail(DTSDF_ERR_OUT_OF_MEMORY, "ICP scratch");
  }
  L.partials = c->icp_partials;
  L.state = c->icp_state;
  if (ensure(c->icp_pback, c->cap_icp_pback, px * sizeof(double2) + (K->width + K->height) * sizeof(double)) !=
      cudaSuccess) {
    cudaGetLastError();
    return fail(DTSDF_ERR_OUT_OF_MEMORY, "ICP back-projections");
  }
  L.pback = reinterpret_cast<double2 *>(c->icp_pback);
  L.col_fac = reinterpret_cast<double *>(c->icp_pback + px * sizeof(double2));
  L.row_fac = L.col_fac + K->width;
  TimedLaunch tl{};
  begin_timed(c, 2, s, &tl);
  CK(c, launch_icp_backproject(L, s), "ICP back-projection");
  end_timed(c, s, &tl);
  return DTSDF_OK;
}

constexpr int kIcpChunk = 4;  // iterations enqueued before the first convergence poll (then 8, 16, ...)

int dtsdf_icp(dtsdf_ctx *c, const float *depth, const float *ref_depth, const float *ref_normal,
              const float ref_pose[16], const dtsdf_intrinsics *K, const float init_delta[16],
              const dtsdf_icp_params *params, dtsdf_icp_result *out, void *stream) {
  if (!c || !out) return fail(DTSDF_ERR_INVALID_ARGUMENT, "ctx/out is NULL");
  if (c->sticky) return fail(DTSDF_ERR_CUDA, "context has a sticky CUDA error");
  dtsdf_icp_params prm;
  dtsdf_default_icp_params(&prm);
  if (params) prm = *params;
  if (prm.max_iters < 1 || prm.max_iters > 1000 || !(prm.min_step >= 0.f))
    return fail(DTSDF_ERR_INVALID_ARGUMENT, "bad ICP parameters");
  cudaSetDevice(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  IcpLaunch L;
  int rc = icp_prepare(c, depth, ref_depth, ref_normal, ref_pose, K, prm.outlier, s, L);
  if (rc) return rc;
  L.min_step = prm.min_step;
  L.max_iters = prm.max_iters;
  L.fused_solve = 1;
  IcpState init;
  std::memset(&init, 0, sizeof(init));
  for (int i = 0; i < 16; ++i) init.delta[i] = init_delta ? (double)init_delta[i] : ((i % 5) == 0 ? 1.0 : 0.0);
  CK(c, cudaMemcpyAsync(c->icp_state, &init, sizeof(init), cudaMemcpyHostToDevice, s), "ICP init");
  if (!c->icp_done_host && cudaMallocHost((void **)&c->icp_done_host, sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    return fail(DTSDF_ERR_OUT_OF_MEMORY, "ICP host flag");
  }
  // Iterations are enqueued in chunks; between chunks the device's done flag (set by k_icp_solve
  // on convergence or the cap) is read back, so a converged call does not pay for up to max_iters
  // no-op launches (a launch after convergence returns at once but still costs a few us).
  TimedLaunch tl{};
  int launched = 0;
  for (int chunk = kIcpChunk; launched < prm.max_iters; chunk *= 2) {
    const int n = std::min(chunk, prm.max_iters - launched);
    begin_timed(c, 2, s, &tl, n);
    for (int it = 0; it < n; ++it) CK(c, launch_icp_reduce(L, s), "ICP reduce + solve");
    end_timed(c, s, &tl);
    launched += n;
    if (launched >= prm.max_iters) break;
    CK(c, cudaMemcpyAsync(c->icp_done_host, &c->icp_state->done, sizeof(int), cudaMemcpyDeviceToHost, s), "ICP poll");
    CK(c, cudaStreamSynchronize(s), "ICP poll sync");
    if (*c->icp_done_host) break;
  }
  IcpState fin;
  CK(c, cudaMemcpyAsync(&fin, c->icp_state, sizeof(fin), cudaMemcpyDeviceToHost, s), "ICP readback");
  CK(c, cudaStreamSynchronize(s), "ICP sync");
  for (int i = 0; i < 16; ++i) out->delta[i] = (float)fin.delta[i];
  for (int i = 0; i < 16; ++i) out->delta64[i] = fin.delta[i];
  out->iterations = fin.iterations;
  out->inliers = fin.inliers;
  out->step = fin.step;
  out->residual = fin.residual;
  out->status = fin.status;
  return fin.status ? fail(DTSDF_ERR_SINGULAR, "singular ICP system (no or degenerate inliers)") : DTSDF_OK;
}

int dtsdf_icp_normal_equations(dtsdf_ctx *c, const float *depth, const float *ref_depth, const float *ref_normal,
                               const float ref_pose[16], const dtsdf_intrinsics *K, const double delta[16],
                               float outlier, double H[36], double g[6], int64_t *inliers, double *residual,
                               void *stream) {
  if (!c || !delta || !H || !g) return fail(DTSDF_ERR_INVALID_ARGUMENT, "NULL argument");
  if (c->sticky) return fail(DTSDF_ERR_CUDA, "context has a sticky CUDA error");
  cudaSetDevice(c->device);
  cudaStream_t s = (cudaStream_t)stream;
  IcpLaunch L;
  int rc = icp_prepare(c, depth, ref_depth, ref_normal, ref_pose, K, outlier, s, L);
  if (rc) return rc;
  L.min_step = 0.0;
  L.max_iters = 1;
  L.fused_solve = 0;
  IcpState init;
  std::memset(&init, 0, sizeof(init));
  for (int i = 0; i < 16; ++i) init.delta[i] = delta[i];
  CK(c, cudaMemcpyAsync(c->icp_state, &init, sizeof(init), cudaMemcpyHostToDevice, s), "ICP init");
  TimedLaunch tl{};
  begin_timed(c, 2, s, &tl, 2);
  CK(c, launch_icp_reduce(L, s), "ICP reduce");
  CK(c, launch_icp_solve(L, s), "ICP solve");
  end_timed(c, s, &tl);
  IcpState fin;
  CK(c, cudaMemcpyAsync(&fin, c->icp_state, sizeof(fin), cudaMemcpyDeviceToHost, s), "ICP readback");
  CK(c, cudaStreamSynchronize(s), "ICP sync");
  int k = 0;
  for (int a = 0; a < 6; ++a)
    for (int b = a; b < 6; ++b) { H[6 * a + b] = H[6 * b + a] = fin.sums[k]; ++k; }
  for (int a = 0; a < 6; ++a) g[a] = fin.sums[21 + a];
  if (inliers) *inliers = (int64_t)fin.sums[27];
  if (residual) *residual = fin.sums[28];
  return DTSDF_OK;
}

int dtsdf_get_volume(dtsdf_ctx *c, int64_t capacity, int32_t *keys, float *sdf, float *weight, uint8_t *rgb,
                     int64_t *n_out) {
  if (!c || !n_out) return fail(DTSDF_ERR_INVALID_ARGUMENT, "ctx/n_out is NULL");
  if (!c->allocated) return fail(DTSDF_ERR_NO_VOLUME, "no volume");
  *n_out = c->n;
  if (capacity < c->n) return fail(DTSDF_ERR_INVALID_ARGUMENT, "capacity smaller than the block count");
  if (c->n == 0) return DTSDF_OK;
  if (!keys || !sdf || !weight || !rgb) return fail(DTSDF_ERR_INVALID_ARGUMENT, "NULL output");
  cudaSetDevice(c->device);
  const size_t n = (size_t)c->n;
  CK(c, cudaDeviceSynchronize(), "get_volume sync");
  CK(c, cudaMemcpy(keys, c->keys, n * 16, cudaMemcpyDeviceToHost), "get_volume");
  CK(c, cudaMemcpy(sdf, c->sdf, n * 512 * 4, cudaMemcpyDeviceToHost), "get_volume");
  CK(c, cudaMemcpy(weight, c->weight, n * 512 * 4, cudaMemcpyDeviceToHost), "get_volume");
  CK(c, cudaMemcpy(rgb, c->rgb, n * 512 * 3, cudaMemcpyDeviceToHost), "get_volume");
  return DTSDF_OK;
}

int dtsdf_render(dtsdf_ctx *c, const float pose[16], const dtsdf_intrinsics *K, float *depth, float *normal,
                 uint8_t *color, uint8_t *mask, void *stream) {
  if (!K) return fail(DTSDF_ERR_INVALID_ARGUMENT, "intrinsics is NULL");
  return dtsdf_render_batch(c, 1, pose, K, 0, K->height, depth, normal, color, mask, stream);
}

int dtsdf_volume_stats(dtsdf_ctx *c, int64_t *n_blocks, int64_t *n_locations, int64_t *bytes) {
  if (!c) return fail(DTSDF_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (n_blocks) *n_blocks = c->n;
  if (n_locations) *n_locations = c->n_loc;
  if (bytes) *bytes = (int64_t)(c->n * (16 + 512 * 11) + c->index_bytes);
  return DTSDF_OK;
}

int dtsdf_set_profiling(dtsdf_ctx *c, int enable) {
  if (!c) return fail(DTSDF_ERR_INVALID_ARGUMENT, "ctx is NULL");
  c->profiling = enable != 0;
  return DTSDF_OK;
}

int dtsdf_kernel_times(dtsdf_ctx *c, double times_ms[4], int64_t counts[4]) {
  if (!c || !times_ms || !counts) return fail(DTSDF_ERR_INVALID_ARGUMENT, "NULL argument");
  for (auto &t : c->timed) {
    cudaError_t e = cudaEventSynchronize(t.stop);
    if (e != cudaSuccess) return cuda_fail(c, e, "event sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t.start, t.stop);
    c->times_ms[t.kind] += ms;
    c->counts[t.kind] += 1;
    cudaEventDestroy(t.start);
    cudaEventDestroy(t.stop);
  }
  c->timed.clear();
  for (int i = 0; i < 4; ++i) {
    times_ms[i] = c->times_ms[i];
    counts[i] = c->counts[i];
  }
  return DTSDF_OK;
}

int dtsdf_reset_kernel_times(dtsdf_ctx *c) {
  if (!c) return fail(DTSDF_ERR_INVALID_ARGUMENT, "ctx is NULL");
  double t[4];
  int64_t n[4];
  int rc = dtsdf_kernel_times(c, t, n);
  for (int i = 0; i < 4; ++i) {
    c->times_ms[i] = 0;
    c->counts[i] = 0;
  }
  return rc;
}

int dtsdf_set_option(dtsdf_ctx *c, int option, int value) {
  if (!c) return fail(DTSDF_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (option == DTSDF_OPT_RANGE_PASS) c->use_range = value ? 1 : 0;
  else if (option == DTSDF_OPT_BLOCK_SKIP) c->use_skip = value ? 1 : 0;
  else if (option == DTSDF_OPT_LOCATION_GRID) c->use_grid = value ? 1 : 0;
  else if (option == DTSDF_OPT_BISECT_STEPS && value >= -1 && value <= 30) c->bisect_steps = value;
  else if (option == DTSDF_OPT_REFINE_TOL_NM && value >= 0 && value <= 100000) c->refine_tol_nm = value;
  else if (option == DTSDF_OPT_HOST_WRITE) c->host_write = value ? 1 : 0;
  else if (option == DTSDF_OPT_CELL_DIRS) c->use_live = value ? 1 : 0;
  else if (option == DTSDF_OPT_TILE_ORDER && value >= 0 && value <= 2) c->use_order = value;
  else if (option == DTSDF_OPT_INCREMENTAL) c->incremental = value ? 1 : 0;
  else if (option == DTSDF_OPT_RANGE_EPOCH && value != 0) {  // value: the epoch's 32 bits
    if (c->range_epoch != 0) c->range_epoch = (unsigned int)value;  // testing: next pass uses value + 1
  }
  else return fail(DTSDF_ERR_INVALID_ARGUMENT, "unknown option");
  return DTSDF_OK;
}

int64_t dtsdf_launch_count(dtsdf_ctx *c) { return c ? c->launches : 0; }

}  // extern "C"
