/*
 * lodge.h -- C ABI of the B200-native LODGE per-frame renderer (liblodge.so).
 *
 * Drop-in boundary for the reference `splatlod` render path.
 * The reference is pure Python; its "FFI" is the Python API re-exported by
 * src/__init__.py:3-21.  Each entry point below replaces one group of those
 * functions; paper_2505_23158_b200/ binds them with ctypes.
 *
 * Conventions
 *   - Every pointer argument named *_dev is a CUDA device pointer on the
 *     context's device.  The library never frees caller memory.
 *   - All work is asynchronous on the context stream (lodge_set_stream);
 *     entry points that return a host-visible size say so explicitly.
 *   - Status: 0 ok, <0 one of LODGE_ERR_*; lodge_last_error() returns a
 *     thread-local message.  A context is not thread-safe; use one per GPU.
 *   - Results are deterministic bit-for-bit run to run: ordered compaction,
 *     stable radix sorts, order-independent atomicMax on float bits.
 */
#ifndef LODGE_H
#define LODGE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LODGE_OK 0
#define LODGE_ERR_BAD_ARG (-1)
#define LODGE_ERR_CUDA (-2)
#define LODGE_ERR_OOM (-3)
#define LODGE_ERR_CAPACITY (-4)

#define LODGE_MAX_LEVELS 8

typedef struct lodge_ctx lodge_ctx;

/* Camera (src/scene.py:80-121).  R is Camera.rotation_matrix (world ->
 * camera, row-major), computed on the host exactly as the reference does. */
typedef struct {
  double R[9];
  double pos[3];
  double fx, fy, cx, cy;
  int32_t w, h;
  double near_plane;
} lodge_camera;

/* RasterConfig (src/raster.py:39-56); `threads` has no device meaning. */
typedef struct {
  double alpha_clamp, alpha_min, t_min, dilation2d;
} lodge_raster_params;

/* One LOD level resident on the device (src/scene.py:124-226).
 * geom: n records of 12 values [mean xyz, scale xyz, rot wxyz, opacity,
 *       filter_variance], fp64 (96 B) or fp32 (48 B) per LODGE_GEOM_FP32.
 * sh:   (n, 3, (deg+1)^2) coefficients, fp64 or fp32 per LODGE_SH_FP32.
 * Arithmetic is fp64 either way (fp32 storage is the asset's native
 * precision, src/assets.py:240-254).  LODGE_GEOM_QNORM: the stored rotations
 * are the asset's raw values, normalised in fp64 when read, exactly as
 * read_asset does at load time (src/assets.py:275-278). */
#define LODGE_GEOM_FP32 1
#define LODGE_SH_FP32 2
#define LODGE_GEOM_QNORM 4
typedef struct {
  int64_t n;
  int32_t sh_degree;
  int32_t flags;
  const void *geom_dev;
  const void *sh_dev;
} lodge_level;

/* Chunk plan (src/scene.py:229-272): K centres (fp64, K x 3) and K*L sorted
 * uint32 index sets, set (j, l) = data[offsets[j*L+l] .. offsets[j*L+l+1]). */
typedef struct {
  int32_t K, L;
  const double *centers_dev;
  const int64_t *offsets_dev;
  const uint32_t *data_dev;
  int64_t max_set[LODGE_MAX_LEVELS]; /* host-side: max_j |set(j,l)| */
  /* Residency-bounded store (the background chunk
   * reload of src/blending.py:140-194): when non-NULL, device tables of K*L
   * pointers, entry j*L+l = the records of set (j, l) in set order (geometry
   * n x 12 and SH n x 3T in the levels' storage precision), resident at
   * least for the frame's chunk pair; lodge_render_frame then reads
   * Gaussians from the pair's chunk slabs instead of the level stores
   * (whose geom_dev / sh_dev may be NULL). */
  const void *const *slab_geom_dev;
  const void *const *slab_sh_dev;
  /* Identity of the plan's contents (any value unique to this plan for its
   * lifetime; 0: none).  A context whose previous frame used the same plan
   * uid and chunk pair reuses that frame's union (the sets, their tags and
   * sizes depend only on the pair; t enters at the projection), skipping
   * compose_active's merge -- consecutive views of a path share the pair. */
  uint64_t uid;
} lodge_chunks;

/* Compositing precision.  FAST: fp32 FMA/MUFU compositing with an fp64
 * guard band that re-decides the q<=9 and alpha>=alpha_min cut-offs exactly;
 * EXACT: fp64 compositing that reproduces the reference's blocked
 * transmittance product (src/raster.py:346-373). Projection is fp64 in both. */
#define LODGE_PREC_FAST 0
#define LODGE_PREC_EXACT 1

/* Render flags */
#define LODGE_NEED_IMAGE 1
#define LODGE_RECORD_MAX 2
/* With LODGE_RECORD_MAX: maxw is not zeroed first, the frame's per-input
 * max weights are max-ed into it on the device -- the max over views of
 * score_active_selection (src/lod.py:95-131) without a host round trip. */
#define LODGE_ACCUMULATE_MAX 4
/* Composite every tile's full sorted list in one pass, so the lists stay
 * inspectable with lodge_frame_lists.  Without it FAST frames composite in
 * two depth phases (lodge_set_phase_budget): identical outputs, but the
 * lists left after the frame are only the second phase's. */
#define LODGE_FULL_LISTS 8

/* Device outputs of one frame (src/raster.py:119-127).  image is float
 * (FAST) or double (EXACT), (h, w, 3); tile_count (tiles_y*tiles_x) int32;
 * visible (h*w) int32; maxw (n_inputs) float (FAST) or double (EXACT),
 * zeroed by the library.  Any pointer may be NULL if its flag is off. */
typedef struct {
  void *image_dev;
  int32_t *tile_count_dev;
  int32_t *visible_dev;
  void *maxw_dev;
  /* optional (FAST only): the 8-bit sRGB image (h, w, 3) the compositor
   * writes as it finishes each tile -- byte for byte lodge_to_srgb8 of the
   * float image, which image_dev may then leave out (NULL).  Device memory
   * or pinned (mapped) host memory: zero-copy read-back, in 16-byte row
   * segments when w is a multiple of 16 and the pointer 16-byte aligned */
  uint8_t *srgb8_dev;
} lodge_frame_out;

/* Per-frame scalars written by the device (lodge_render_frame /
 * lodge_rasterize): read back after the stream completes. */
typedef struct {
  int32_t f, o;          /* chunk pair (o = -1: single chunk) */
  double t_bar, t;       /* blend factor */
  uint32_t U;            /* active inputs (n_inputs of the batch) */
  uint32_t U_level[LODGE_MAX_LEVELS];
  uint32_t M;            /* survivors after culling */
  uint32_t P;            /* tile-splat pairs */
  uint32_t overflow;     /* 1 if P exceeded the pair capacity */
  uint32_t guard_hits;   /* FAST: pixel-splat decisions re-checked in fp64 */
  uint32_t P_first;      /* pairs of the first (or only) depth phase's lists */
  uint32_t P_second;     /* pairs of the second phase's lists (two-phase frames) */
  uint32_t fault;        /* nonzero: a device-side bounds check fired (one bit per
                            site, internal.cuh FAULT_*); the frame's outputs are invalid */
  uint32_t M_first;      /* two-phase frames: splats of the first phase */
  uint32_t M_second;     /* two-phase frames: later splats that meet an unfinished tile */
  uint32_t comp_members; /* compositing work: sum over tiles (and phases) of the list
                            members a tile iterates before all its pixels have
                            T < t_min, or its whole list (SURVEY.md 8d m_t) */
  uint32_t block_lists;  /* two-phase frames: bit 0 (1) the first phase, bit 1 (2) the
                            second kept block lists instead of sorted per-tile lists */
  uint32_t sorted_first; /* survivors depth-sorted for the first (or only) phase: M in
                            one pass, the first-phase candidates in two phases (the
                            second phase sorts its M_second owners) */
} lodge_frame_stats;

/* ---- context ---------------------------------------------------------- */
int lodge_create(int32_t device, lodge_ctx **out);
void lodge_destroy(lodge_ctx *ctx);
const char *lodge_last_error(void);
int lodge_set_stream(lodge_ctx *ctx, void *cuda_stream);
/* Reserve workspace: survivors M and pairs P.  Grown automatically by the
 * synchronous entry points; the async frame path reports overflow. */
int lodge_reserve(lodge_ctx *ctx, int64_t max_splats, int64_t max_pairs);
/* Two-phase FAST frames: the depth-ordered splats whose pairs
 * start within pairs_per_tile * T of the pair sequence are binned, sorted and
 * composited first; only the tiles left with live pixels receive, sort and
 * composite the rest of their pairs.  Outputs are bitwise those of one pass.
 * 0 disables (every frame one pass); default 1536. */
int lodge_set_phase_budget(lodge_ctx *ctx, int32_t pairs_per_tile);
/* Frames in flight on several contexts: the projection's and
 * the record gather's persistent grids use at most ctas_per_sm CTAs per SM
 * (0: their single-frame default, 3 and 4), leaving room on every SM for the
 * other contexts' kernels.  Outputs are the same for every value. */
int lodge_set_grid_share(lodge_ctx *ctx, int32_t ctas_per_sm);
/* Block lists: a depth phase of few large splats keeps, per
 * block of 8 x 4 tiles, its depth-ordered splats with tile masks instead of
 * emitting and sorting its pairs.  AUTO decides per frame on the device
 * (<= 128k splats averaging >= 64 tiles); FORCE uses them whenever the phase
 * has <= 128k splats (second phase: owners); OFF never.  Outputs are the same
 * in every mode; lodge_frame_stats.block_lists reports the choice. */
#define LODGE_BLOCK_LISTS_AUTO 0
#define LODGE_BLOCK_LISTS_OFF 1
#define LODGE_BLOCK_LISTS_FORCE 2
int lodge_set_block_lists(lodge_ctx *ctx, int32_t mode);
int lodge_set_precision(lodge_ctx *ctx, int32_t precision);

/* ---- chunk selection: nearest_two_chunks + blend_factor ---------------
 * replaces src/blending.py:77-99.  n positions (fp64 x3) -> f, o, t_bar, t.
 * Bit-exact with the reference's fp64 arithmetic. */
int lodge_select(lodge_ctx *ctx, const double *centers_dev, int32_t K,
                 const double *positions_dev, int32_t n, int32_t *f_dev, int32_t *o_dev,
                 double *t_bar_dev, double *t_dev);

/* blend_factor for explicit centres (src/blending.py:87-99): in_dev holds n
 * rows [position xyz, m_f xyz, m_o xyz]; out_dev n rows [|m_f-m_o|^2, t_bar,
 * t].  The caller raises when the first column is <= 0. */
int lodge_blend_factor(lodge_ctx *ctx, const double *in_dev, int32_t n, double *out_dev);

/* ---- compose_active: union of two chunks' sets with modulation ---------
 * replaces src/blending.py:102-129.  Synchronous (returns sizes).
 * out_idx_dev[l] / out_tag_dev[l] need |A_l|+|B_l| slots; tag 3 = both,
 * 1 = primary only (mod t), 2 = other only (mod 1-t).  o = -1: single chunk. */
int lodge_compose(lodge_ctx *ctx, const lodge_chunks *chunks, int32_t f, int32_t o,
                  uint32_t **out_idx_dev, uint8_t **out_tag_dev, int64_t *out_sizes);

/* ---- project_scene for one level (compat path) ------------------------
 * replaces src/raster.py:188-291.  idx_dev: n int64 indices (NULL = all);
 * mod_dev: n fp64 modulation (NULL = none).  Writes the survivors in input
 * order as the reference's Splat2DBatch fields (fp64, int64 source index).
 * Synchronous; returns M in *out_m. */
typedef struct {
  int64_t *src_dev;     /* (M,) */
  double *mean2d_dev;   /* (M,2) */
  double *cov2d_dev;    /* (M,2,2) */
  double *conic_dev;    /* (M,3) */
  double *extent_dev;   /* (M,2) */
  double *depth_dev;    /* (M,) */
  double *opacity_dev;  /* (M,) */
  double *color_dev;    /* (M,3) */
} lodge_batch;
int lodge_project(lodge_ctx *ctx, const lodge_level *level, const int64_t *idx_dev, int64_t n,
                  const double *mod_dev, const lodge_camera *cam,
                  const lodge_raster_params *rp, int32_t shade, lodge_batch *out,
                  int64_t *out_m);

/* ---- rasterize a Splat2DBatch (compat path) ----------------------------
 * replaces src/raster.py:380-449.  batch fields as above (cov2d unused),
 * M rows, n_inputs for the max-weight output.  Synchronous; *stats filled.
 * Optionally returns the sorted per-tile lists: tile_offsets_dev (T+1
 * int64) and tile_src_dev (source indices, capacity list_cap). */
int lodge_rasterize(lodge_ctx *ctx, const lodge_batch *batch, int64_t M, int64_t n_inputs,
                    const lodge_camera *cam, const lodge_raster_params *rp, int32_t flags,
                    const lodge_frame_out *out, int64_t *tile_offsets_dev,
                    int64_t *tile_src_dev, int64_t list_cap, lodge_frame_stats *stats);

/* ---- fused per-frame path ------------------------------------------------
 * One camera view rendered end to end on the device: (select ->) union +
 * modulation -> projection -> depth sort -> binning -> tile sort ->
 * compositing.  No host synchronisation.  pair: if NULL, the nearest two
 * chunks are selected on the device for cam->pos (stateless CLI blend mode,
 * src/cli.py:236-242); else {f, o} with t = *t_override (render_blend_state).
 * cam_dev is a device copy of the camera (its w,h must equal width,height,
 * which size the grids); out->maxw_dev must hold the chunk plan's maximum
 * union size (sum over levels of 2 * max_set).
 * stats_dev: device lodge_frame_stats (may be NULL). */
int lodge_render_frame(lodge_ctx *ctx, const lodge_level *levels, int32_t n_levels,
                       const lodge_chunks *chunks, const lodge_camera *cam_dev, int32_t width,
                       int32_t height, const lodge_raster_params *rp, const int32_t *pair,
                       const double *t_override, int32_t flags, const lodge_frame_out *out,
                       lodge_frame_stats *stats_dev);

/* Inspection of the last frame (async, on the context stream).
 * lodge_frame_lists: the sorted per-tile lists as source indices (T+1 int64
 * offsets, up to cap int64 sources; T = tiles of the frame).
 * lodge_frame_union: level l's union (uint32 indices, uint8 tags), up to cap. */
int lodge_frame_lists(lodge_ctx *ctx, int32_t T, int64_t *tile_offsets_dev,
                      int64_t *tile_src_dev, int64_t cap);
int lodge_frame_union(lodge_ctx *ctx, int32_t level, uint32_t *idx_dev, uint8_t *tag_dev,
                      int64_t cap);

/* Stage profiling: when enabled, lodge_render_frame records CUDA events on
 * the context stream at the boundaries of its LODGE_N_STAGES stages (select,
 * union, project, depth sort, tile setup, duplicate, tile sort, composite,
 * second phase, second-phase composite; two-phase frames count the counting
 * pass under tile setup, the first phase's emission / sort / compositing
 * under the next three, and the second phase's enumeration, emission and
 * sort under "second phase")
 * for up to `max_frames` frames.  lodge_profile_read synchronises those
 * events and returns the summed milliseconds per stage and the frame count,
 * then clears the record. */
#define LODGE_N_STAGES 10
int lodge_profile(lodge_ctx *ctx, int32_t enable, int32_t max_frames);
int lodge_profile_read(lodge_ctx *ctx, double *stage_ms, int32_t *frames);

/* Linear [0,1] RGB (fp32, n pixels) -> 8-bit sRGB, round(srgb(x) * 255)
 * (reference src/images.py:10-17).  Async. */
int lodge_to_srgb8(lodge_ctx *ctx, const float *image_dev, int64_t n_pixels, uint8_t *out_dev);

/* ---- frame report (the reference bench's per-frame fields) -------------
 * replaces visibility_histogram (src/raster.py:464-479) and the per-mode
 * metrics of cmd_bench (src/cli.py:283-320) on the device.  out_dev
 * (n_edges + 1 uint64) receives the histogram of visible (n_pixels int32)
 * over the n_edges - 1 bins [e_i, e_{i+1}) -- the last absorbs values
 * >= e_{n-1}, values below e_0 go to the first (np.searchsorted side=right,
 * clipped) --, then the sum of tile_count (n_tiles int32; mean_per_tile =
 * sum / n_tiles) and the number of nonzero max weights among n_inputs
 * (visible_gaussians; maxw may be NULL).  edges_host: 2 <= n_edges <= 257,
 * strictly increasing, else BAD_ARG with the reference's messages.  Async. */
int lodge_frame_report(lodge_ctx *ctx, const int32_t *visible_dev, int64_t n_pixels,
                       const double *edges_host, int32_t n_edges,
                       const int32_t *tile_count_dev, int64_t n_tiles, const void *maxw_dev,
                       int32_t maxw_fp64, int64_t n_inputs, uint64_t *out_dev);
/* Sum of squared differences of two fp32 images of n values into *out_dev
 * (fp64): psnr_vs_full = -10 log10(sum / n) (src/cli.py:293-294).  Async. */
int lodge_sq_err(lodge_ctx *ctx, const float *a_dev, const float *b_dev, int64_t n,
                 double *out_dev);

/* Number of kernels the last lodge_render_frame enqueued. */
int32_t lodge_last_launch_count(lodge_ctx *ctx);

/* OR of the stats.fault bits of every frame this context rendered
 * (synchronous): 0 unless a device-side bounds check ever fired. */
int lodge_fault_flags(lodge_ctx *ctx, uint32_t *flags);

/* Compositing work counters of the last frame (synchronous; all zero unless
 * liblodge was built with -DLODGE_COUNTERS): [0] per-warp list entries,
 * [1] warp iterations, [2] iterations with a pixel inside the cut-off,
 * [3] pixel evaluations inside the cut-off, [4] warp-batches. */
int lodge_debug_counters(lodge_ctx *ctx, uint64_t *out8);

/* Diagnostic: the frame depth sort alone (the onesweep passes of
 * np.lexsort((index, depth)), src/raster.py:401) over n caller keys; keys
 * equal to ~0 are dropped as culled inputs are.  Writes the surviving keys
 * sorted and their input indices; out_m_dev (device, 2 x uint32) receives
 * the survivor count and the frame's fault bits.  Async on the context
 * stream. */
int lodge_debug_depth_sort(lodge_ctx *ctx, const uint64_t *keys_dev, int64_t n,
                           uint64_t *sorted_keys_dev, uint32_t *sorted_idx_dev,
                           uint32_t *out_m_dev);

/* ---- LOD-mode and full-mode frames --------------
 * replaces render_lod (src/lod.py:230-237) and the "full" / "lod" branches
 * of _mode_selection + _render_mode (src/cli.py:219-243): the active sets
 * are chosen on the device -- lod: level l keeps the Gaussians with
 * bounds[l] <= ||mean - camera position|| < bounds[l+1] (select_active,
 * src/lod.py:192-211; bounds host, n_levels+1 values, the caller folds the
 * depth offsets in); full: every Gaussian of level 0, the other levels
 * empty -- then the fused path of lodge_render_frame.  maxw has one entry
 * per selected input, level-major.  Async on the context stream. */
int lodge_render_lod(lodge_ctx *ctx, const lodge_level *levels, int32_t n_levels,
                     const double *bounds, int32_t full, const lodge_camera *cam_dev, int32_t w,
                     int32_t h, const lodge_raster_params *rp, int32_t flags,
                     const lodge_frame_out *out, lodge_frame_stats *stats_dev);

/* The band selection alone: replaces select_active (src/lod.py:192-211) and,
 * called once per chunk centre with the radius folded into bounds,
 * build_chunk_active_sets (src/chunks.py:122-135).  Level l keeps the
 * Gaussians with bounds[l] <= ||mean - pos|| < bounds[l+1] (bounds host,
 * n_levels+1 values), in ascending index order.  pos_dev: device double[3].
 * idx_dev: uint32, capacity sum of levels[].n; level l's members start at
 * sum_{k<l} levels[k].n.  sizes_dev: uint32 per level.  Async on the context
 * stream. */
int lodge_select_active(lodge_ctx *ctx, const lodge_level *levels, int32_t n_levels,
                        const double *bounds, const double *pos_dev, uint32_t *idx_dev,
                        uint32_t *sizes_dev);

/* ---- threshold-search cost table ----------------
 * replaces ThresholdSearcher._table, src/thresholds.py:80-90: project the
 * level's inputs (idx_dev, or all n when NULL) with shade=False; for the M
 * survivors, in input order, the tile cover count (tile_cover_counts,
 * src/raster.py:316-324) and the fp64 camera distance ||mean - position||;
 * stable sort by distance.  Writes dist_dev[0..M) (sorted distances) and
 * prefix_dev[0..M] (0 then the running sum of the covers in that order,
 * int64).  Capacities n and n+1.  Synchronous; *out_m = M. */
int lodge_cover_table(lodge_ctx *ctx, const lodge_level *level, const int64_t *idx_dev,
                      int64_t n, const lodge_camera *cam, const lodge_raster_params *rp,
                      double *dist_dev, int64_t *prefix_dev, int64_t *out_m);

/* ---- asset upload -------------------------------
 * replaces the decode + value checks of _parse_level_blob, src/assets.py:
 * 257-282, on the device.  blob_dev: one level's data.bin blob already in
 * device memory, n little-endian fp32 records [mean3, scale3, rot4, opacity,
 * fv, sh 3*(deg+1)^2] (src/assets.py:240-254).  Splits them into the
 * level store (geom_dev: n x 12 fp32, raw rotations -- render the level with
 * LODGE_GEOM_QNORM; sh_dev: n x 3 x (deg+1)^2 fp32) and checks every record.
 * Synchronous; *violations gets the checks that failed, in the reference's
 * order of raising: */
#define LODGE_ASSET_NONFINITE 1 /* "level blob contains non-finite values" */
#define LODGE_ASSET_SCALE 2     /* "... non-positive scales" */
#define LODGE_ASSET_OPACITY 4   /* "... out-of-range opacity" */
#define LODGE_ASSET_FV 8        /* "... negative filter variance" */
#define LODGE_ASSET_ROTATION 16 /* "... non-unit rotations" (| |q| - 1 | > 1e-3) */
int lodge_asset_split(lodge_ctx *ctx, const void *blob_dev, int64_t n, int32_t sh_degree,
                      float *geom_dev, float *sh_dev, int32_t *violations);

/* Index-set checks of read_asset (src/assets.py:448-453) for every set of
 * a chunk plan: set_flags (K*L, host) gets bit 0 if set (j, l) is not
 * strictly increasing, bit 1 if an index is >= level_sizes[l] (host, L). */
int lodge_asset_check_sets(lodge_ctx *ctx, const lodge_chunks *chunks,
                           const int64_t *level_sizes, int32_t *set_flags);

#ifdef __cplusplus
}
#endif
#endif
