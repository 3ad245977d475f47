/*
 * dtsdf.h -- C ABI of libdtsdf.so, the B200 (sm_100a) DTSDF raycast renderer.
 *
 * The library renders depth, normal, colour and direction-mask images from a six-direction
 * Directional TSDF ("one for each direction {X+, X-, Y+, Y-, Z+, Z-}") stored as
 * 8x8x8 voxel blocks keyed by (x, y, z, D).  Each ray probes the field at
 * regular intervals until the first positive -> negative transition and refines the root
 * (PAPER.md:178); every probe combines the directions on the fly with the
 * combination weight eq:combine_weight or, when no direction has a
 * gradient, eq:combine_tsdf_weight.  DESIGN.md §2 states the exact
 * definition the results follow and §4 the readings of the paper it rests on.
 *
 * Conventions (DESIGN.md §4 readings R14-R17):
 *   - voxel (i,j,k) sits at world (i,j,k) * voxel_size; block = floor(i/8) per axis;
 *     local voxel index l = lx + 8*ly + 64*lz;
 *   - direction D in 0..5 = X+, X-, Y+, Y-, Z+, Z-;
 *   - sdf is normalised (units of truncation), positive in front of the surface;
 *   - camera frame x right, y down, z forward; pixel (u, v) at integer coordinates;
 *     ray direction ((u-cx)/fx, (v-cy)/fy, 1) (eq:reprojection);
 *   - output depth is camera-frame z (0 = miss), normals are unit world-frame vectors facing
 *     the camera (0 = miss), colour is u8 RGB, dirmask bit D set iff direction D contributed.
 *
 * Memory: "device" pointers are CUDA device memory of the context's device (e.g. a torch
 * tensor's data_ptr()); the library auto-detects host vs device where stated.  Small structs
 * (pose, intrinsics, params) are always host memory.
 *
 * Errors: every call returns DTSDF_OK (0) or a negative code; arguments are checked before
 * any launch; no C++ exception crosses the ABI; dtsdf_last_error() returns a thread-local
 * message for the last failing call on this thread.  DTSDF_ERR_CUDA is sticky: destroy the
 * context.  A ray that finds no surface is not an error (it yields a zero pixel).
 *
 * Threading: one host thread per context at a time; one context per GPU.  The volume is
 * immutable between commits; do not commit while a render is in flight on another stream.
 */
#ifndef DTSDF_H_
#define DTSDF_H_

#include <stdint.h>

#if defined(__GNUC__)
#define DTSDF_API __attribute__((visibility("default")))
#else
#define DTSDF_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define DTSDF_OK 0
#define DTSDF_ERR_INVALID_ARGUMENT (-1) /* null pointer, bad size/intrinsics/params, D not in 0..5, coords out of range */
#define DTSDF_ERR_DUPLICATE_KEY (-2)    /* two blocks with the same (bx,by,bz,D) */
#define DTSDF_ERR_NO_VOLUME (-3)        /* render before a successful commit */
#define DTSDF_ERR_OUT_OF_MEMORY (-4)    /* device allocation failed */
#define DTSDF_ERR_CUDA (-5)             /* CUDA runtime error (sticky) */
#define DTSDF_ERR_NO_COMBINED (-6)      /* render_combined / combined query before dtsdf_combine */
#define DTSDF_ERR_SINGULAR (-7)         /* ICP normal equations not positive definite (tracking failure) */

/* block coordinates must lie in [-2^20, 2^20) (21-bit packed index key) */
#define DTSDF_MAX_BLOCK_COORD (1 << 20)
/* views rendered per kernel launch; larger batches are split into several launches */
#define DTSDF_VIEWS_PER_LAUNCH 256

typedef struct dtsdf_ctx dtsdf_ctx; /* opaque, one per device */

/* Pinhole intrinsics and the march depth range.  fx, fy > 0; 0 < width, height <= 32768;
 * 0 < z_min < z_max (camera-frame z, metres; reading R24). */
typedef struct {
  float fx, fy, cx, cy;
  int32_t width, height;
  float z_min, z_max;
} dtsdf_intrinsics;

/* Volume parameters.
 *   voxel_size  > 0 (metres)
 *   truncation  >= 2 * voxel_size (metres) -- metadata: stored sdf is normalised
 *   theta       angular threshold in (pi/4, pi/2]; used by eq:direction_weight
 *   step        lattice step Delta (metres); 0 -> voxel_size (reading R4)
 *   n_blocks    N >= 0 */
typedef struct {
  float voxel_size, truncation, theta, step;
  int64_t n_blocks;
} dtsdf_volume_params;

/* Library-owned device buffers of the current volume (filled by dtsdf_alloc_volume).
 *   keys    int32 [N][4] = (bx, by, bz, D)
 *   sdf     f32   [N][512] normalised signed distance, positive in front; must be finite
 *   weight  f32   [N][512] distance weight w_d, finite and >= 0
 * dtsdf_commit_volume rejects a non-finite sdf or a negative / non-finite weight with
 * DTSDF_ERR_INVALID_ARGUMENT (NaN is the apron bricks' "unallocated" sentinel).
 *   rgb     u8    [N][512][3] */
typedef struct {
  int32_t *keys;
  float *sdf;
  float *weight;
  uint8_t *rgb;
} dtsdf_volume_buffers;

/* Create a context on CUDA device `cuda_device`.  *out receives the handle. */
DTSDF_API int dtsdf_create(int cuda_device, dtsdf_ctx **out);
/* Destroy the context and free all device memory it owns.  NULL is a no-op. */
DTSDF_API int dtsdf_destroy(dtsdf_ctx *ctx);

/* Allocate library-owned device buffers for N blocks (dropping any previous volume) and return
 * their pointers in *out; the caller fills them (cudaMemcpy, NCCL broadcast, a kernel) and then
 * calls dtsdf_commit_volume.  Validates params (see dtsdf_volume_params). */
DTSDF_API int dtsdf_alloc_volume(dtsdf_ctx *ctx, const dtsdf_volume_params *params, dtsdf_volume_buffers *out);

/* Validate the filled buffers and build the device index on `cuda_stream` (a cudaStream_t, or
 * NULL for the legacy default stream): the (x,y,z) -> six direction slots hash table, the
 * block-occupancy bitmap, the location list and the apron bricks the raycast kernel reads
 * (DESIGN.md §5).  Synchronous: returns after the index is built.  Errors: INVALID_ARGUMENT
 * (D not in 0..5 or a coordinate out of range), DUPLICATE_KEY, OUT_OF_MEMORY, CUDA. */
DTSDF_API int dtsdf_commit_volume(dtsdf_ctx *ctx, void *cuda_stream);

/* Convenience: alloc + copy + commit.  keys/sdf/weight/rgb may be host or device pointers (auto
 * detected per pointer); rgb may be NULL (all zero).  Synchronous; the caller may free its
 * inputs on return. */
DTSDF_API int dtsdf_upload_volume(dtsdf_ctx *ctx, const dtsdf_volume_params *params, const int32_t *keys, const float *sdf,
                        const float *weight, const uint8_t *rgb);

/* Render one view.  pose_w_c: world-from-camera 4x4 row-major (host; the bottom row is ignored).
 * Outputs (all [H][W] row-major, caller-owned):
 *   out_depth   f32 [H][W]      camera z of the surface, 0 = miss
 *   out_normal  f32 [H][W][3]   unit world normal, 0 = miss        (may be NULL)
 *   out_color   u8  [H][W][3]   RGB, 0 = miss                      (may be NULL)
 *   out_dirmask u8  [H][W]      bit D set iff W_D > 0 at the hit    (may be NULL)
 * If all non-NULL outputs are device pointers the call is asynchronous on cuda_stream; if they
 * are host pointers the call synchronizes: page-locked (pinned) host outputs are written by the
 * kernel directly (DTSDF_OPT_HOST_WRITE), pageable ones via device scratch and a copy back. */
DTSDF_API int dtsdf_render(dtsdf_ctx *ctx, const float pose_w_c[16], const dtsdf_intrinsics *intr, float *out_depth,
                 float *out_normal, uint8_t *out_color, uint8_t *out_dirmask, void *cuda_stream);

/* Render n_views views with shared intrinsics.  poses_w_c: host [n_views][16].  Only image rows
 * [row0, row1) are rendered (0 <= row0 < row1 <= height), so one large view can be sharded by
 * rows across GPUs; outputs are contiguous [n_views][row1-row0][W][...] with the layouts of
 * dtsdf_render.  Host/device output handling as in dtsdf_render. */
DTSDF_API int dtsdf_render_batch(dtsdf_ctx *ctx, int32_t n_views, const float *poses_w_c, const dtsdf_intrinsics *intr,
                       int32_t row0, int32_t row1, float *out_depth, float *out_normal, uint8_t *out_color,
                       uint8_t *out_dirmask, void *cuda_stream);

/* Current volume: N blocks, U distinct block locations, device bytes held by the context. */
DTSDF_API int dtsdf_volume_stats(dtsdf_ctx *ctx, int64_t *n_blocks, int64_t *n_locations, int64_t *bytes);

/* ---- view-dependent combined TSDF --------------------
 * Lemma 1: for a fixed camera the six directions combine into one conflict-free
 * regular TSDF.  dtsdf_combine computes it "for every voxel in the view frustum",
 * widened by margin x image size on every side (1/8), at integer voxel positions
 * with the 6-neighbour gradient and the weights eq:combine_weight /
 * eq:combine_tsdf_weight; readings R33-R35.  A voxel with no positive
 * combination weight, or outside the widened frustum, is invalid.
 *   pose_w_c, intr: the source camera (host); margin in [0, 16] (0.125 in the paper).
 * Replaces the previous combined TSDF.  Runs on cuda_stream and synchronizes it (the number of
 * combined block locations is read back).  Errors: INVALID_ARGUMENT, NO_VOLUME, OUT_OF_MEMORY, CUDA. */
DTSDF_API int dtsdf_combine(dtsdf_ctx *ctx, const float pose_w_c[16], const dtsdf_intrinsics *intr, float margin,
                            void *cuda_stream);

/* Same with a choice of combination rule:
 *   DTSDF_COMBINE_WEIGHTED    eq:combine_weight / eq:combine_tsdf_weight (the paper's method; dtsdf_combine)
 *   DTSDF_COMBINE_ALGORITHM1  Algorithm 1 "Compute Combined TSDF" (readings R53-R57): a
 *                             direction takes part iff its stored weight exceeds w_floor and its gradient is
 *                             valid for it; a free direction's free space stands unless its first zero
 *                             transition towards the camera lies in another direction's visible occupied
 *                             space; stored-weight average of the free (else occupied) directions.  The paper
 *                             reports it underperforms on real data; w_floor >= 0 (0 in the paper). */
#define DTSDF_COMBINE_WEIGHTED 0
#define DTSDF_COMBINE_ALGORITHM1 1
DTSDF_API int dtsdf_combine_mode(dtsdf_ctx *ctx, const float pose_w_c[16], const dtsdf_intrinsics *intr, float margin,
                                 int32_t mode, float w_floor, void *cuda_stream);

/* Raycast the current combined TSDF "like a regular TSDF" (readings R36-R37) from
 * n_views poses: same lattice, crossing rule, refinement, argument layout, host/device output
 * handling and errors as dtsdf_render_batch, plus NO_COMBINED.  Valid for poses near the source
 * pose (the recombination conditions below keep them near). */
DTSDF_API int dtsdf_render_combined(dtsdf_ctx *ctx, int32_t n_views, const float *poses_w_c,
                                    const dtsdf_intrinsics *intr, int32_t row0, int32_t row1, float *out_depth,
                                    float *out_normal, uint8_t *out_color, uint8_t *out_dirmask, void *cuda_stream);

/* Combined block locations (those with at least one voxel in the widened frustum) and device bytes held. */
DTSDF_API int dtsdf_combined_stats(dtsdf_ctx *ctx, int64_t *n_locations, int64_t *bytes);

/* Export the combined TSDF to HOST buffers (synchronous; for checks and external consumers):
 * locs int32 [n][3] block coordinates, sdf f32 [n][512] (NaN = invalid voxel), weight f32 [n][512]
 * (sum of the combination weights, 0 = invalid), rgb u8 [n][512][3], mask u8 [n][512] (bit D:
 * direction D contributed).  *n_out = n always; INVALID_ARGUMENT if capacity < n.  Location order
 * is unspecified. */
DTSDF_API int dtsdf_get_combined(dtsdf_ctx *ctx, int64_t capacity, int32_t *locs, float *sdf, float *weight,
                                 uint8_t *rgb, uint8_t *mask, int64_t *n_out);

/* Conditional combination (eqs. condition_1-4; reading R38): recombine iff
 * frame < boot_frames OR frame - last > stale_frames OR |t - t_last| > translation (metres) OR
 * angle(R_last^T R) > rotation (radians).  Frames count from 0; last = frame of the last combine.
 * Returns 1 (recombine), 0, or INVALID_ARGUMENT (NULL, last > frame, non-positive thresholds). */
typedef struct {
  int32_t boot_frames, stale_frames; /* 5, 50 */
  float translation, rotation;       /* 0.05 m, 0.05 * pi / 2 */
} dtsdf_combine_policy;
DTSDF_API void dtsdf_default_policy(dtsdf_combine_policy *policy);
DTSDF_API int dtsdf_should_recombine(const dtsdf_combine_policy *policy, int64_t frame, int64_t last,
                                     const float pose_w_c[16], const float last_pose_w_c[16]);

/* ---- voxel-projection fusion --------------------------
 * every allocated voxel in the frame's view is projected into the depth frame,
 * associated with the nearest pixel and updated as a weighted running average with the
 * point-to-plane distance d = <x - p, n>/tau (positive in front, reading R6), the weight
 * w_d = w_ICP(z) <n,-ray>^+ w_dir^D(n) (eq:combined_fusion_weight; w_ICP eq:ICP_weight) and the
 * colour weight w_c = w_d (1 - min(1, |p - x|/tau)) (eq:color_weight); d > 1 carves towards +1 with
 * a constant weight unless a depth within carve_radius pixels differs by more than tau; weights are
 * capped at max_weight.  Blocks are allocated first: for every valid pixel and every direction its
 * normal admits (eq:angular_threshold), the blocks holding p + t n, t in [-tau, tau] sampled at
 * <= voxel/2 (readings R39-R45). */
typedef struct {
  float max_weight;     /* 128 */
  float carve_weight;   /* 1; 0 = no carving; negative -> DTSDF_ERR_INVALID_ARGUMENT */
  int32_t carve_radius; /* 2 pixels */
  int32_t reserved;     /* 0 */
} dtsdf_fusion_params;
DTSDF_API void dtsdf_default_fusion_params(dtsdf_fusion_params *params);

/* Make room for `capacity` blocks (keeping the current ones; with no volume yet, create an empty
 * one with `params`, which is otherwise ignored) and commit.  The library-owned buffers move
 * (pointers from dtsdf_alloc_volume become invalid).  Colour weights of existing blocks start at
 * their depth weights (R45).  Synchronous.  Errors: INVALID_ARGUMENT (capacity < current blocks),
 * OUT_OF_MEMORY, CUDA. */
DTSDF_API int dtsdf_fusion_reserve(dtsdf_ctx *ctx, const dtsdf_volume_params *params, int64_t capacity);

/* Camera-frame normals of a depth map ("cross product of neighboring pixels in x- and
 * y direction"; no bilateral filter, R39): depth f32 [H][W] camera z (0 = missing), out f32
 * [H][W][3] unit normals facing the camera, 0 on the border and next to missing depth.  Host or
 * device pointers (host output -> synchronous). */
DTSDF_API int dtsdf_depth_normals(dtsdf_ctx *ctx, const float *depth, const dtsdf_intrinsics *intr, float *out_normal,
                                  void *cuda_stream);

/* Allocate and fuse one frame: depth f32 [H][W] (camera z, 0 = missing; valid in [z_min, z_max]),
 * normal f32 [H][W][3] (camera frame, facing the camera, 0 = invalid), color u8 [H][W][3] or NULL,
 * pose world-from-camera (host), params NULL -> defaults.  Frames may be host or device memory.
 * Re-commits the volume; a combined TSDF is kept, stale, until the next dtsdf_combine (the paper's
 * conditional recombination: blocks allocated since are invalid in it).  *new_blocks
 * (may be NULL) receives the
 * number of blocks allocated.  Synchronous.  Errors: INVALID_ARGUMENT, NO_VOLUME (no
 * dtsdf_fusion_reserve), OUT_OF_MEMORY (capacity reached: the blocks allocated so far are kept and
 * initialised, the frame is not fused), CUDA. */
DTSDF_API int dtsdf_fuse(dtsdf_ctx *ctx, const float *depth, const float *normal, const uint8_t *color,
                         const float pose_w_c[16], const dtsdf_intrinsics *intr, const dtsdf_fusion_params *params,
                         int64_t *new_blocks, void *cuda_stream);

/* Copy the current blocks to HOST buffers (synchronous): keys int32 [n][4], sdf/weight f32
 * [n][512], rgb u8 [n][512][3]; *n_out = n always; INVALID_ARGUMENT if capacity < n.  Block order
 * is the pool order (fusion appends in allocation order). */
DTSDF_API int dtsdf_get_volume(dtsdf_ctx *ctx, int64_t capacity, int32_t *keys, float *sdf, float *weight, uint8_t *rgb,
                               int64_t *n_out);

/* ---- geometric point-to-plane ICP against a rendered view
 * the frame's points p_i (depth back-projected) are mapped by DeltaT into the
 * camera of a view rendered at ref_pose and associated projectively with the nearest rendered pixel
 * (q_i, n_i); E = sum w_i <q_i - exp(xi) DeltaT p_i, n_i>^2 with w_i = w_ICP(z_i) =
 * 1/(z + 1 - z_min)^2; H = 2 sum w J J^T, g = 2 sum w J r with J = (-n, -DeltaT p x n), summed by a
 * fixed-topology (deterministic) tree; H xi = -g by Cholesky; DeltaT <- exp(xi) DeltaT
 * until |xi| < min_step or max_iters; residuals above `outlier` metres are rejected. */
typedef struct {
  int32_t max_iters; /* 50 (fine level) */
  float min_step;    /* 1e-6 */
  float outlier;     /* 0.005 m (fine level; 0.05 coarse) */
  int32_t reserved;
} dtsdf_icp_params;
typedef struct {
  float delta[16];       /* DeltaT, row-major: frame camera -> rendered view camera; new pose = ref_pose DeltaT */
  double delta64[16];    /* the same in fp64 */
  int32_t iterations;    /* Gauss-Newton steps taken */
  int32_t status;        /* 0 ok, 1 singular */
  int64_t inliers;       /* associated, non-outlier pixels of the last linearisation */
  double step;           /* |xi| of the last step */
  double residual;       /* sum w r^2 of the last linearisation */
} dtsdf_icp_result;
DTSDF_API void dtsdf_default_icp_params(dtsdf_icp_params *params);

/* Register a depth frame against a rendered view.  depth f32 [H][W] (camera z, 0 = missing),
 * ref_depth f32 [H][W] and ref_normal f32 [H][W][3] (world frame) as dtsdf_render outputs at
 * ref_pose; shared intrinsics; init_delta (NULL = identity).  Host or device buffers.  All
 * iterations are enqueued on cuda_stream in chunks of 4, 8, 16, ...; after each chunk the call reads the
 * device's convergence flag back (one synchronization per chunk).  Errors: INVALID_ARGUMENT,
 * SINGULAR (the result holds the last DeltaT), OUT_OF_MEMORY, CUDA. */
DTSDF_API int dtsdf_icp(dtsdf_ctx *ctx, const float *depth, const float *ref_depth, const float *ref_normal,
                        const float ref_pose[16], const dtsdf_intrinsics *intr, const float init_delta[16],
                        const dtsdf_icp_params *params, dtsdf_icp_result *out, void *cuda_stream);

/* One linearisation at DeltaT = delta (fp64, row-major): H [36] (full symmetric), g [6], inliers,
 * sum w r^2 -- the deterministic reduction exposed for checks.  Synchronous. */
DTSDF_API int dtsdf_icp_normal_equations(dtsdf_ctx *ctx, const float *depth, const float *ref_depth,
                                         const float *ref_normal, const float ref_pose[16],
                                         const dtsdf_intrinsics *intr, const double delta[16], float outlier,
                                         double H[36], double g[6], int64_t *inliers, double *residual,
                                         void *cuda_stream);

/* Kernel timing (tracing).  While enabled, every range-pass, raycast and combine
 * launch is bracketed by CUDA events on its stream.  dtsdf_kernel_times synchronizes those events
 * and returns the summed milliseconds and launch counts since the last reset: times_ms[0] range
 * pass, [1] raycast, [2] other (index build, memsets), [3] combine; counts[0..3] likewise. */
DTSDF_API int dtsdf_set_profiling(dtsdf_ctx *ctx, int enable);
DTSDF_API int dtsdf_kernel_times(dtsdf_ctx *ctx, double times_ms[4], int64_t counts[4]);
DTSDF_API int dtsdf_reset_kernel_times(dtsdf_ctx *ctx);

/* Exact accelerations that can be switched off to check they are result-invisible:
 *   DTSDF_OPT_RANGE_PASS  1 (default) narrow each ray to its tile's [z_near, z_far] from the
 *                         block-bounds range pass; 0 march every lattice point from z_min to z_max
 *   DTSDF_OPT_BLOCK_SKIP  1 (default) jump over unallocated block locations; 0 step every point */
#define DTSDF_OPT_RANGE_PASS 1
#define DTSDF_OPT_BLOCK_SKIP 2
/*   DTSDF_OPT_CELL_DIRS   1 (default) a sample visits only the directions that can hold data at its base
 *                         cell (present, no NaN corner, a corner weight > 0; built at commit); 0 visits
 *                         every direction present at the block location */
#define DTSDF_OPT_CELL_DIRS 8
/* Tuning (results unchanged):
 *   (option 3, a persistent warp schedule, was measured slower and removed in round 2)
 *   DTSDF_OPT_LOCATION_GRID 1 (default) resolve block locations through the dense location grid
 *                         (built when the location AABB has <= 2^28 cells); 0 through the
 *                         occupancy bitmaps and the hash table
 * Testing only (changes which root a multi-root lattice interval yields):
 *   DTSDF_OPT_BISECT_STEPS  -1 (default) enough bisection steps to narrow the bracket to
 *                           <= 5e-5 m before regula falsi; n >= 0 forces n steps */
#define DTSDF_OPT_BISECT_STEPS 4
#define DTSDF_OPT_LOCATION_GRID 5
/*   DTSDF_OPT_REFINE_TOL_NM  0 (default) regula falsi stops when f(b) is within 1e-7 of the root or after
 *                            12 steps; n > 0 also stops it once the bracket is narrower than n nanometres */
#define DTSDF_OPT_REFINE_TOL_NM 6
/*   DTSDF_OPT_HOST_WRITE  1 (default) when every non-NULL output of a render call is page-locked host
 *                         memory mapped into the device address space (cudaHostAlloc / cudaMallocHost /
 *                         torch pin_memory() under unified addressing) the raycast kernel writes the
 *                         outputs there directly, in whole 16-byte-aligned tile rows, overlapping the
 *                         host-link transfer with the ray march; 0 renders into device scratch and
 *                         copies back after the kernel.  Pageable host outputs always take the copy path. */
#define DTSDF_OPT_HOST_WRITE 7
/*   DTSDF_OPT_TILE_ORDER  1 (default) automatic: for launches of up to 65536 CTA tiles (one 640x480 view is
 *                         2400) the raycast runs its 16x8-pixel CTA tiles longest-predicted-first (the
 *                         range pass counts the block locations covering each tile; a counting sort
 *                         orders them), so the slow tiles do not start last and stretch the kernel's
 *                         drain; longer batches stay row-major.  2 always, 0 never.  Changes only when a
 *                         tile runs, never what it computes. */
#define DTSDF_OPT_TILE_ORDER 9
/*   DTSDF_OPT_INCREMENTAL  1 (default) dtsdf_fuse updates the index incrementally: the allocation
 *                          extends the hash table in place, and only the locations within one block
 *                          of a block the frame changed get their record bricks, cell masks and
 *                          location-grid values rebuilt (a full re-commit when a new location falls
 *                          outside the location AABB or the pool fills); 0 re-commits the whole
 *                          volume after every frame.  Same results either way. */
#define DTSDF_OPT_INCREMENTAL 11
/* Testing only:
 *   DTSDF_OPT_RANGE_EPOCH  n != 0 (read as uint32): the next range pass uses epoch n + 1 (the range keys carry a per-pass
 *                          epoch; passes at or above 0xFFFFFFF0 clear the buffers and restart at 1), to
 *                          exercise the wrap.  No effect before the first render of the context. */
#define DTSDF_OPT_RANGE_EPOCH 10
DTSDF_API int dtsdf_set_option(dtsdf_ctx *ctx, int option, int value);

/* Kernel launches issued by this context since creation (all kinds). */
DTSDF_API int64_t dtsdf_launch_count(dtsdf_ctx *ctx);

/* Thread-local message describing the last error on this thread ("" if none). */
DTSDF_API const char *dtsdf_last_error(void);

/* Thread-local warning left by the last call on this thread that checked volume parameters
 * (dtsdf_alloc_volume / dtsdf_upload_volume / dtsdf_fusion_reserve): "" when none.  Set when
 * theta < arccos(1/sqrt(3)) = 54.74 deg, which is accepted but breaks PAPER.md:84's "at least one
 * direction" claim in 3D (reading R2). */
DTSDF_API const char *dtsdf_last_warning(void);

#ifdef __cplusplus
}
#endif
#endif /* DTSDF_H_ */
