// C ABI of liblodge (include/lodge.h): context, workspace, entry points.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstddef>
#include <cmath>
#include <string>
#include <vector>

#include "internal.cuh"

using namespace lodge;

static thread_local std::string g_err;

static int set_err(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                  \
  do {                                                                            \
    cudaError_t _e = (call);                                                      \
    if (_e != cudaSuccess)                                                        \
      return set_err(_e == cudaErrorMemoryAllocation ? LODGE_ERR_OOM : LODGE_ERR_CUDA, \
                     std::string(#call) + ": " + cudaGetErrorString(_e));         \
  } while (0)

namespace {
// 8-bit sRGB (the reference's to_uint8, src/images.py:10-17: clip, the
// piecewise curve in fp64, np.round) is a non-decreasing step function of
// the fp32 input with 255 steps.  Its thresholds -- the smallest fp32 x with
// to_uint8(x) >= k, k = 1..255 -- are found once per process by bisection
// over fp32 bit patterns with the reference's own fp64 formula on the host
// (libm pow, as NumPy's power), and each pixel is a binary search over them:
// no fp64 pow per channel.  NaN and x <= 0 give 0, x >= 1 gives 255, as
// clip does.
static int srgb_level(float xf) {
  const double x = std::fmin(std::fmax((double)xf, 0.0), 1.0);
  double e;
  if (x <= 0.0031308) {
    e = 12.92 * x;
  } else {
    volatile double a = 1.055 * std::pow(x, 1.0 / 2.4);  // no contraction with the - 0.055
    e = a - 0.055;
  }
  volatile double y = e * 255.0;
  return (int)std::nearbyint(y);  // round half to even, as np.round
}

static std::vector<float> make_srgb_thresholds() {
  std::vector<float> t(256);
  {
    t[0] = -INFINITY;
    for (int k = 1; k < 256; ++k) {
      uint32_t lo = 0u, hi = 0x3f800000u;  // f(+0) = 0 < k <= 255 = f(1)
      while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        float xm;
        std::memcpy(&xm, &mid, 4);
        if (srgb_level(xm) >= k) hi = mid;
        else lo = mid + 1;
      }
      std::memcpy(&t[k], &lo, 4);
    }
  }
  return t;
}
static const float *srgb_thresholds() {
  static const std::vector<float> t = make_srgb_thresholds();  // thread-safe, once
  return t.data();
}

}  // namespace

struct lodge_ctx {
  int device = 0;
  cudaStream_t stream = 0;
  int32_t precision = LODGE_PREC_FAST;
  FrameState *fs = nullptr;
  lodge_camera *cam_dev = nullptr;   // scratch for the synchronous entry points
  lodge_camera *cam_host = nullptr;  // pinned staging
  lodge_frame_stats *stats_host = nullptr;  // pinned
  Work w{};
  int64_t tiles_cap = 0;  // capacity of tile_start (T+1) and diff
  int64_t pixels_cap = 0;  // capacity of the two-phase pixel state
  int32_t phase_budget = 1536;  // first-phase pairs per tile of two-phase frames (0: one pass)
  int32_t block_lists = LODGE_BLOCK_LISTS_AUTO;  // lodge_set_block_lists
  int debug_sync = 0;  // LODGE_DEBUG_SYNC=1: check after every stage; 2: after each segment
  int32_t launches = 0;
  LevelSlots last_slots{};  // slot layout of the last union
  double *edges_dev = nullptr;  // lodge_frame_report's bin edges (257)
  // stage profiling
  bool prof = false;
  int32_t prof_cap = 0, prof_frames = 0;
  cudaEvent_t *prof_ev = nullptr;  // prof_cap * (LODGE_N_STAGES + 1)
  void mark(int k) {
    if (prof && prof_frames < prof_cap)
      cudaEventRecord(prof_ev[prof_frames * (LODGE_N_STAGES + 1) + k], stream);
  }
};

// LODGE_DEBUG_ALLOC=1: log every workspace allocation (pointer, bytes) to stderr
static void log_alloc(const lodge_ctx *c, const char *what, const void *p, int64_t bytes) {
  static const bool on = getenv("LODGE_DEBUG_ALLOC") != nullptr;
  if (on) fprintf(stderr, "[lodge alloc] ctx %p %s %p %lld\n", (const void *)c, what, p,
                  (long long)bytes);
}

static int ensure_M(lodge_ctx *c, int64_t need) {
  Work &w = c->w;
  if (need <= w.M_cap && w.payload) return 0;
  int64_t ncap = std::max<int64_t>(std::max<int64_t>(need, w.M_cap + w.M_cap / 2), 4096);
  cudaFree(w.key_depth[0]); cudaFree(w.key_depth[1]);
  cudaFree(w.val_depth[0]); cudaFree(w.val_depth[1]);
  cudaFree(w.sel_keys); cudaFree(w.sel_vals);
  for (int q = 0; q < 4; ++q) cudaFree(w.sort_scr[q]);
  w.sel_keys = w.sel_vals = nullptr;
  for (int q = 0; q < 4; ++q) w.sort_scr[q] = nullptr;
  cudaFree(w.rect); cudaFree(w.payload); cudaFree(w.precise);
  cudaFree(w.rect_sorted); cudaFree(w.splat_off); cudaFree(w.vrank);
  w.vrank = nullptr;
  w.M_cap = 0;
  CK(cudaMalloc(&w.rect_sorted, 8 * ncap));
  CK(cudaMalloc(&w.splat_off, 4 * (ncap + 1)));
  CK(cudaMalloc(&w.key_depth[0], 8 * ncap));
  CK(cudaMalloc(&w.key_depth[1], 8 * ncap));
  CK(cudaMalloc(&w.val_depth[0], 4 * ncap));
  CK(cudaMalloc(&w.val_depth[1], 4 * ncap));
  CK(cudaMalloc(&w.sel_keys, 4 * ncap));
  CK(cudaMalloc(&w.sel_vals, 4 * ncap));
  for (int q = 0; q < 4; ++q) CK(cudaMalloc(&w.sort_scr[q], 4 * ncap));
  if (!w.sel_hist) {
    CK(cudaMalloc(&w.sel_hist, 4 * (size_t)SEL_BINS));
    CK(cudaMemset(w.sel_hist, 0, 4 * (size_t)SEL_BINS));  // re-zeroed by k_sel_scan
  }
  CK(cudaMalloc(&w.rect, 8 * ncap));
  CK(cudaMalloc(&w.payload, sizeof(Payload) * ncap));
  CK(cudaMalloc(&w.precise, sizeof(Precise) * ncap));
#ifdef LODGE_VERIFY
  CK(cudaMalloc(&w.vrank, 4 * ncap));
#endif
  w.M_cap = ncap;
  log_alloc(c, "key_depth0", w.key_depth[0], 8 * ncap);
  log_alloc(c, "key_depth1", w.key_depth[1], 8 * ncap);
  log_alloc(c, "val_depth0", w.val_depth[0], 4 * ncap);
  log_alloc(c, "val_depth1", w.val_depth[1], 4 * ncap);
  return 0;
}

static int ensure_status(lodge_ctx *c, int64_t words) {
  Work &w = c->w;
  if (words <= w.status_cap && w.status) return 0;
  int64_t ncap = std::max<int64_t>(words, w.status_cap + w.status_cap / 2);
  ncap = std::max<int64_t>(ncap, 1 << 16);
  if (w.status) cudaFree(w.status);
  w.status = nullptr;
  w.status_cap = 0;
  CK(cudaMalloc(&w.status, 8 * ncap));
  CK(cudaMemset(w.status, 0, 8 * ncap));  // epoch 0 is never used
  w.status_cap = ncap;
  log_alloc(c, "status", w.status, 8 * ncap);
  return 0;
}

static int ensure_P(lodge_ctx *c, int64_t need) {
  Work &w = c->w;
  if (need <= w.P_cap && w.pairs[0]) return 0;
  int64_t ncap = std::max<int64_t>(std::max<int64_t>(need, w.P_cap + w.P_cap / 2), 1 << 16);
  cudaFree(w.pairs[0]); cudaFree(w.pairs[1]); cudaFree(w.chunk_first);
  w.pairs[0] = w.pairs[1] = nullptr;
  w.list = nullptr;
  w.P_cap = 0;
  CK(cudaMalloc(&w.pairs[0], 8 * ncap));
  CK(cudaMalloc(&w.pairs[1], 8 * ncap));
  CK(cudaMalloc(&w.chunk_first, 4 * (ncap / 2048 + 4)));
  w.P_cap = ncap;
  return ensure_status(c, (ncap + 4095) / 4096 * 256);
}

static int ensure_tiles(lodge_ctx *c, int32_t W, int32_t H) {
  const int64_t tx = (W + 15) / 16, ty = (H + 15) / 16;
  const int64_t need = (tx + 1) * (ty + 1) + 1;
  Work &w = c->w;
  if (need > c->tiles_cap || !w.tile_diff) {
    void *old[] = {w.tile_diff, w.tile_start, w.tile_order, w.tile_diff_a, w.count_all,
                   w.tile_start_b, w.tile_order_b, w.alive, w.sat, w.bl_start, w.bl_len,
                   w.bl_live};
    for (void *p : old) cudaFree(p);
    c->tiles_cap = 0;
    CK(cudaMalloc(&w.tile_diff, 4 * need));
    CK(cudaMemset(w.tile_diff, 0, 4 * need));
    CK(cudaMalloc(&w.tile_diff_a, 4 * need));
    CK(cudaMemset(w.tile_diff_a, 0, 4 * need));
    CK(cudaMalloc(&w.tile_start, 4 * need));
    CK(cudaMalloc(&w.tile_order, 4 * need));
    CK(cudaMalloc(&w.count_all, 4 * need));
    CK(cudaMalloc(&w.tile_start_b, 4 * need));
    CK(cudaMalloc(&w.tile_order_b, 4 * need));
    CK(cudaMalloc(&w.alive, 4 * (need / 32 + 1)));
    CK(cudaMalloc(&w.sat, 4 * need));
    // block lists: capacity offsets and lengths per phase (blocks <= tiles)
    CK(cudaMalloc(&w.bl_start, 4 * 2 * need));
    CK(cudaMalloc(&w.bl_len, 4 * 2 * need));
    CK(cudaMalloc(&w.bl_live, 4 * 2 * need));
    c->tiles_cap = need;
  }
  {  // block-list look-back: BL_CHMAX status words per block
    const int rc = ensure_status(c, (int64_t)block_count((int32_t)tx, (int32_t)ty) * BL_CHMAX + 64);
    if (rc) return rc;
  }
  const int64_t px = (int64_t)W * H;
  if (px > c->pixels_cap || !w.state) {
    cudaFree(w.state);
    c->pixels_cap = 0;
    CK(cudaMalloc(&w.state, sizeof(float4) * px));
    c->pixels_cap = px;
  }
  return 0;
}

// the per-device copy of the sRGB level thresholds, once per context
static int ensure_srgb(lodge_ctx *c) {
  if (c->w.srgb_thr) return 0;
  CK(cudaMalloc(&c->w.srgb_thr, 256 * sizeof(float)));
  CK(cudaMemcpy(c->w.srgb_thr, srgb_thresholds(), 256 * sizeof(float), cudaMemcpyHostToDevice));
  return 0;
}

// a frame's optional 8-bit sRGB output: FAST frames with the image flag
static int check_srgb_out(lodge_ctx *c, int32_t flags, const lodge_frame_out *out) {
  if (!out->srgb8_dev) return 0;
  if (c->precision != LODGE_PREC_FAST)
    return set_err(LODGE_ERR_BAD_ARG, "8-bit sRGB output needs FAST precision");
  if (!(flags & LODGE_NEED_IMAGE))
    return set_err(LODGE_ERR_BAD_ARG, "8-bit sRGB output needs LODGE_NEED_IMAGE");
  return ensure_srgb(c);
}

static int ensure_slots(lodge_ctx *c, int64_t need) {
  Work &w = c->w;
  if (need <= w.slot_cap && w.union_idx) return 0;
  int64_t ncap = std::max<int64_t>(need, 4096);
  cudaFree(w.union_idx); cudaFree(w.union_tag);
  w.slot_cap = 0;
  // the cached union lived in the freed buffers
  CK(cudaMemset(reinterpret_cast<char *>(c->fs) + offsetof(FrameState, uc_uid), 0,
                sizeof(uint64_t)));
  CK(cudaMalloc(&w.union_idx, 4 * ncap));
  CK(cudaMalloc(&w.union_tag, ncap));
  w.slot_cap = ncap;
  return 0;
}

static int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return set_err(LODGE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return 0;
}

// LODGE_DEBUG_SYNC builds of a frame: a device fault is reported with the
// stage that raised it
#define DSYNC(what) DSYNC_L(1, what)
#define DSYNC_L(level, what)                                                          \
  do {                                                                                \
    if (c->debug_sync == (level) || (c->debug_sync == 1 && (level) == 2)) {           \
      cudaError_t _e = cudaStreamSynchronize(s);                                      \
      if (_e == cudaSuccess) _e = cudaGetLastError();                                 \
      if (_e != cudaSuccess)                                                          \
        return set_err(LODGE_ERR_CUDA, std::string("after ") + (what) + ": " +        \
                                           cudaGetErrorString(_e));                   \
    }                                                                                 \
  } while (0)

static int check_cam(const lodge_camera *cam) {
  if (!cam) return set_err(LODGE_ERR_BAD_ARG, "camera is NULL");
  if (cam->w <= 0 || cam->h <= 0) return set_err(LODGE_ERR_BAD_ARG, "camera resolution must be positive");
  if (cam->w > 16 * 65535 || cam->h > 16 * 65535) return set_err(LODGE_ERR_BAD_ARG, "resolution too large");
  if (!(cam->fx > 0) || !(cam->fy > 0)) return set_err(LODGE_ERR_BAD_ARG, "focal must be positive");
  return 0;
}

static int check_tile_smem(int32_t W, int32_t H) {
  const int64_t tx = (W + 15) / 16, ty = (H + 15) / 16;
  if ((tx + 1) * (ty + 1) * 4 > 200 * 1024)
    return set_err(LODGE_ERR_BAD_ARG, "resolution exceeds the tile-count table (max ~4K)");
  return 0;
}

extern "C" {

const char *lodge_last_error(void) { return g_err.c_str(); }

int lodge_create(int32_t device, lodge_ctx **out) {
  if (!out) return set_err(LODGE_ERR_BAD_ARG, "out is NULL");
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return set_err(LODGE_ERR_BAD_ARG, "no such CUDA device");
  CK(cudaSetDevice(device));
  lodge_ctx *c = new lodge_ctx();
  c->device = device;
  {
    const char *d = getenv("LODGE_DEBUG_SYNC");
    c->debug_sync = d ? atoi(d) : 0;
  }
  CK(cudaMalloc(&c->fs, sizeof(FrameState)));
  CK(cudaMemset(c->fs, 0, sizeof(FrameState)));
  log_alloc(c, "fs", c->fs, sizeof(FrameState));
  CK(cudaMalloc(&c->cam_dev, sizeof(lodge_camera)));
  CK(cudaMallocHost(&c->cam_host, sizeof(lodge_camera)));
  CK(cudaMallocHost(&c->stats_host, sizeof(lodge_frame_stats)));
  int rc = ensure_status(c, 1 << 16);
  if (rc) return rc;
  *out = c;
  return 0;
}

void lodge_destroy(lodge_ctx *c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  Work &w = c->w;
  void *ptrs[] = {w.key_depth[0], w.key_depth[1], w.val_depth[0], w.val_depth[1], w.rect,
                  w.payload, w.precise, w.pairs[0], w.pairs[1], w.tile_diff, w.tile_start,
                  w.status, w.union_idx, w.union_tag, c->fs, c->cam_dev, w.rect_sorted,
                  w.splat_off, w.chunk_first, w.tile_order, w.tile_diff_a, w.count_all,
                  w.tile_start_b, w.tile_order_b, w.alive, w.sat, w.state, w.vrank,
                  w.bl_start, w.bl_len, w.bl_live, w.srgb_thr, w.sel_hist, w.sel_keys,
                  w.sel_vals, w.sort_scr[0], w.sort_scr[1], w.sort_scr[2], w.sort_scr[3],
                  c->edges_dev};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  if (c->cam_host) cudaFreeHost(c->cam_host);
  if (c->stats_host) cudaFreeHost(c->stats_host);
  delete c;
}

int lodge_set_stream(lodge_ctx *c, void *stream) {
  if (!c) return set_err(LODGE_ERR_BAD_ARG, "ctx is NULL");
  c->stream = (cudaStream_t)stream;
  return 0;
}

int lodge_set_phase_budget(lodge_ctx *c, int32_t pairs_per_tile) {
  if (!c) return set_err(LODGE_ERR_BAD_ARG, "ctx is NULL");
  if (pairs_per_tile < 0) return set_err(LODGE_ERR_BAD_ARG, "phase budget must be >= 0");
  c->phase_budget = pairs_per_tile;
  return 0;
}

int lodge_set_grid_share(lodge_ctx *c, int32_t ctas_per_sm) {
  if (!c) return set_err(LODGE_ERR_BAD_ARG, "ctx is NULL");
  if (ctas_per_sm < 0) return set_err(LODGE_ERR_BAD_ARG, "CTAs per SM must be >= 0");
  c->w.grid_share = ctas_per_sm;
  return 0;
}

int lodge_set_block_lists(lodge_ctx *c, int32_t mode) {
  if (!c) return set_err(LODGE_ERR_BAD_ARG, "ctx is NULL");
  if (mode < LODGE_BLOCK_LISTS_AUTO || mode > LODGE_BLOCK_LISTS_FORCE)
    return set_err(LODGE_ERR_BAD_ARG, "block-list mode must be AUTO, OFF or FORCE");
  c->block_lists = mode;
  return 0;
}

int lodge_set_precision(lodge_ctx *c, int32_t p) {
  if (!c) return set_err(LODGE_ERR_BAD_ARG, "ctx is NULL");
  if (p != LODGE_PREC_FAST && p != LODGE_PREC_EXACT)
    return set_err(LODGE_ERR_BAD_ARG, "precision must be LODGE_PREC_FAST or LODGE_PREC_EXACT");
  c->precision = p;
  return 0;
}

int lodge_reserve(lodge_ctx *c, int64_t max_splats, int64_t max_pairs) {
  if (!c) return set_err(LODGE_ERR_BAD_ARG, "ctx is NULL");
  CK(cudaSetDevice(c->device));
  int rc = ensure_M(c, max_splats);
  if (rc) return rc;
  rc = ensure_P(c, max_pairs);
  if (rc) return rc;
  return ensure_status(c, std::max<int64_t>((max_splats + 4095) / 4096 * 256,
                                            (max_splats + 255) / 256 * 2));
}

int lodge_select(lodge_ctx *c, const double *centers, int32_t K, const double *pos, int32_t n,
                 int32_t *f, int32_t *o, double *tb, double *t) {
  if (!c || !centers || !pos || !f || !o || !tb || !t)
    return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  if (K < 1) return set_err(LODGE_ERR_BAD_ARG, "a chunk plan needs at least one chunk");
  launch_select(centers, K, pos, n, f, o, tb, t, c->stream);
  return check_launch("lodge_select");
}

int lodge_blend_factor(lodge_ctx *c, const double *in, int32_t n, double *out) {
  if (!c || !in || !out) return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  launch_blend_factor(in, n, out, c->stream);
  return check_launch("lodge_blend_factor");
}

int lodge_compose(lodge_ctx *c, const lodge_chunks *ch, int32_t f, int32_t o,
                  uint32_t **out_idx, uint8_t **out_tag, int64_t *out_sizes) {
  if (!c || !ch || !out_idx || !out_tag || !out_sizes) return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  if (f < 0 || f >= ch->K) return set_err(LODGE_ERR_BAD_ARG, "chunk " + std::to_string(f) + " is not in the plan");
  if (o >= ch->K || o < -1) return set_err(LODGE_ERR_BAD_ARG, "chunk " + std::to_string(o) + " is not in the plan");
  if (o == f) return set_err(LODGE_ERR_BAD_ARG, "blending needs two distinct chunks");
  if (ch->L < 1 || ch->L > LODGE_MAX_LEVELS) return set_err(LODGE_ERR_BAD_ARG, "bad level count");
  CK(cudaSetDevice(c->device));
  LevelSlots ls;
  ls.n_levels = ch->L;
  ls.slot_base[0] = 0;
  for (int l = 0; l < ch->L; ++l) ls.slot_base[l + 1] = ls.slot_base[l] + (uint32_t)(2 * ch->max_set[l]);
  int rc = ensure_slots(c, ls.slot_base[ch->L]);
  if (rc) return rc;
  rc = ensure_status(c, (int64_t)ch->L * union_status_stride(ls.slot_base[ch->L]));
  if (rc) return rc;
  launch_begin_frame(c->fs, c->stream);
  launch_select_frame(ch->centers_dev, ch->K, c->cam_dev, nullptr, nullptr, 1, f, o, 1.0, c->fs,
                      c->stream);
  launch_union(*ch, ls, c->fs, c->w.status, c->w.union_idx, c->w.union_tag, c->stream);
  rc = check_launch("lodge_compose");
  if (rc) return rc;
  CK(cudaMemcpyAsync(c->stats_host, &c->fs->stats, sizeof(lodge_frame_stats),
                     cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (int l = 0; l < ch->L; ++l) {
    out_sizes[l] = c->stats_host->U_level[l];
    if (out_idx[l] && out_sizes[l])
      CK(cudaMemcpyAsync(out_idx[l], c->w.union_idx + ls.slot_base[l], 4 * out_sizes[l],
                         cudaMemcpyDeviceToDevice, c->stream));
    if (out_tag[l] && out_sizes[l])
      CK(cudaMemcpyAsync(out_tag[l], c->w.union_tag + ls.slot_base[l], out_sizes[l],
                         cudaMemcpyDeviceToDevice, c->stream));
  }
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int lodge_project(lodge_ctx *c, const lodge_level *level, const int64_t *idx, int64_t n,
                  const double *mod, const lodge_camera *cam, const lodge_raster_params *rp,
                  int32_t shade, lodge_batch *out, int64_t *out_m) {
  if (!c || !level || !rp || !out || !out_m) return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  int rc = check_cam(cam);
  if (rc) return rc;
  if (level->sh_degree < 0 || level->sh_degree > 3)
    return set_err(LODGE_ERR_BAD_ARG, "sh degree must be in 0..3, got " + std::to_string(level->sh_degree));
  if (n > 0x3fffffff) return set_err(LODGE_ERR_BAD_ARG, "too many inputs");
  *out_m = 0;
  if (n <= 0) return 0;
  CK(cudaSetDevice(c->device));
  rc = ensure_status(c, (n + 255) / 256 + 1);
  if (rc) return rc;
  *c->cam_host = *cam;
  CK(cudaMemcpyAsync(c->cam_dev, c->cam_host, sizeof(lodge_camera), cudaMemcpyHostToDevice, c->stream));
  launch_begin_frame(c->fs, c->stream);
  launch_project_compat(*level, idx, n, mod, c->w, c->fs, c->cam_dev, *rp, shade, out, c->stream);
  rc = check_launch("lodge_project");
  if (rc) return rc;
  CK(cudaMemcpyAsync(c->stats_host, &c->fs->stats, sizeof(lodge_frame_stats),
                     cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *out_m = c->stats_host->M;
  return 0;
}

int lodge_rasterize(lodge_ctx *c, const lodge_batch *b, int64_t M, int64_t n_inputs,
                    const lodge_camera *cam, const lodge_raster_params *rp, int32_t flags,
                    const lodge_frame_out *out, int64_t *tile_offsets, int64_t *tile_src,
                    int64_t list_cap, lodge_frame_stats *stats) {
  if (!c || !b || !rp || !out) return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  int rc = check_cam(cam);
  if (rc) return rc;
  rc = check_tile_smem(cam->w, cam->h);
  if (rc) return rc;
  if (M < 0 || M > 0x3fffffff || n_inputs < M) return set_err(LODGE_ERR_BAD_ARG, "bad batch size");
  CK(cudaSetDevice(c->device));
  if ((rc = check_srgb_out(c, flags, out))) return rc;
  cudaStream_t s = c->stream;
  const int32_t tiles_x = (cam->w + 15) / 16, tiles_y = (cam->h + 15) / 16;
  const int32_t T = tiles_x * tiles_y;
  if ((rc = ensure_M(c, std::max<int64_t>(M, 1))) || (rc = ensure_tiles(c, cam->w, cam->h)) ||
      (rc = ensure_status(c, (M + 4095) / 4096 * 256 + (M + 255) / 256 + 256)) ||
      (rc = ensure_P(c, 1)))
    return rc;
  *c->cam_host = *cam;
  CK(cudaMemcpyAsync(c->cam_dev, c->cam_host, sizeof(lodge_camera), cudaMemcpyHostToDevice, s));
  const bool exact = c->precision == LODGE_PREC_EXACT;
  if ((flags & LODGE_RECORD_MAX) && !(flags & LODGE_ACCUMULATE_MAX) && out->maxw_dev &&
      n_inputs > 0)
    CK(cudaMemsetAsync(out->maxw_dev, 0, (exact ? 8 : 4) * (size_t)n_inputs, s));
  int32_t nl = 0;
  launch_begin_frame(c->fs, s);
  launch_import_batch(*b, M, c->w, c->fs, c->cam_dev, *rp, exact, s);
  launch_depth_sort(c->w, c->fs, M, &nl, s);
  launch_tile_setup(c->w, c->fs, out->tile_count_dev, tiles_x, tiles_y, s);
  rc = check_launch("lodge_rasterize: setup");
  if (rc) return rc;
  CK(cudaMemcpyAsync(c->stats_host, &c->fs->stats, sizeof(lodge_frame_stats), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const uint32_t P = c->stats_host->P;
  if ((int64_t)P > c->w.P_cap) {  // grow, then clear the overflow the setup recorded
    rc = ensure_P(c, P);
    if (rc) return rc;
    const uint32_t fix[2] = {P, 0u};
    CK(cudaMemcpy(&c->fs->n_pairs, &fix[0], 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(&c->fs->stats.overflow, &fix[1], 4, cudaMemcpyHostToDevice));
  }
  Work &w = c->w;
  launch_duplicate(w, c->fs, tiles_x, M, s);
  launch_tile_sort(w, c->fs, tiles_x, tiles_y, &nl, s);
  launch_composite(w, c->fs, c->cam_dev, cam->w, cam->h, *rp, flags, exact, *out,
                   (uint32_t)n_inputs, s);
  if (tile_offsets && tile_src) launch_export_lists(w, c->fs, T, tile_offsets, tile_src, list_cap, s);
  rc = check_launch("lodge_rasterize");
  if (rc) return rc;
  CK(cudaMemcpyAsync(c->stats_host, &c->fs->stats, sizeof(lodge_frame_stats), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (stats) *stats = *c->stats_host;
  return 0;
}

static int render_tail(lodge_ctx *c, const lodge_level *levels, const LevelSlots &ls,
                       const lodge_camera *cam_dev, int32_t W, int32_t H,
                       const lodge_raster_params &rp, int32_t flags, const lodge_frame_out *out,
                       lodge_frame_stats *stats_dev, int32_t nl, const char *name,
                       const lodge_chunks *ch);

int lodge_render_frame(lodge_ctx *c, const lodge_level *levels, int32_t n_levels,
                       const lodge_chunks *ch, const lodge_camera *cam_dev, int32_t W, int32_t H,
                       const lodge_raster_params *rp, const int32_t *pair,
                       const double *t_override, int32_t flags, const lodge_frame_out *out,
                       lodge_frame_stats *stats_dev) {
  if (!c || !levels || !ch || !cam_dev || !rp || !out) return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  if (n_levels != ch->L || n_levels < 1 || n_levels > LODGE_MAX_LEVELS)
    return set_err(LODGE_ERR_BAD_ARG, "level count does not match the chunk plan");
  if (W <= 0 || H <= 0) return set_err(LODGE_ERR_BAD_ARG, "camera resolution must be positive");
  int rc = check_tile_smem(W, H);
  if (rc) return rc;
  int32_t pf = 0, po = -1;
  double tv = 1.0;
  if (pair) {
    pf = pair[0];
    po = pair[1];
    if (pf < 0 || pf >= ch->K) return set_err(LODGE_ERR_BAD_ARG, "chunk " + std::to_string(pf) + " is not in the plan");
    if (po < -1 || po >= ch->K) return set_err(LODGE_ERR_BAD_ARG, "chunk " + std::to_string(po) + " is not in the plan");
    if (po == pf) return set_err(LODGE_ERR_BAD_ARG, "blending needs two distinct chunks");
    tv = t_override ? *t_override : 1.0;
  }
  for (int l = 0; l < n_levels; ++l)
    if (levels[l].sh_degree < 0 || levels[l].sh_degree > 3)
      return set_err(LODGE_ERR_BAD_ARG, "sh degree must be in 0..3");
  CK(cudaSetDevice(c->device));
  cudaStream_t s = c->stream;
  LevelSlots ls;
  ls.n_levels = n_levels;
  ls.slot_base[0] = 0;
  for (int l = 0; l < n_levels; ++l) ls.slot_base[l + 1] = ls.slot_base[l] + (uint32_t)(2 * ch->max_set[l]);
  const int64_t U_cap = ls.slot_base[n_levels];
  const int32_t tiles_x = (W + 15) / 16, tiles_y = (H + 15) / 16;
  if ((rc = ensure_slots(c, U_cap)) || (rc = ensure_M(c, std::max<int64_t>(U_cap, 1))) ||
      (rc = ensure_tiles(c, W, H)) || (rc = ensure_P(c, 1)) ||
      (rc = ensure_status(c, (c->w.M_cap + 4095) / 4096 * 256 + (U_cap + 255) / 256 + 256)))
    return rc;
  const bool exact = c->precision == LODGE_PREC_EXACT;
  Work &w = c->w;
  c->last_slots = ls;
  int32_t nl = 0;
  c->mark(0);
  launch_begin_frame(c->fs, s); ++nl;
  launch_select_frame(ch->centers_dev, ch->K, cam_dev, nullptr, nullptr, pair != nullptr, pf, po,
                      tv, c->fs, s); ++nl;
  c->mark(1);
  nl += launch_union(*ch, ls, c->fs, w.status, w.union_idx, w.union_tag, s);
  return render_tail(c, levels, ls, cam_dev, W, H, *rp, flags, out, stats_dev, nl,
                     "lodge_render_frame", ch);
}

// Two depth phases: FAST compositing, lists not needed for inspection, a
// visible buffer, and both tile difference arrays fit the setup kernel's
// shared memory.
static bool two_phase(const lodge_ctx *c, int32_t W, int32_t H, int32_t flags,
                      const lodge_frame_out *out) {
  const int64_t tx = (W + 15) / 16, ty = (H + 15) / 16;
  // the visible counts of unfinished tiles carry over in the visible buffer
  return c->precision == LODGE_PREC_FAST && c->phase_budget > 0 && out->visible_dev &&
         !(flags & LODGE_FULL_LISTS) && 2 * (tx + 1) * (ty + 1) * 4 <= 200 * 1024;
}

// Everything after the active-set stage, shared by the chunk and LOD paths:
// projection -> depth sort -> tile setup -> duplication -> tile sort ->
// compositing, on the context stream, stage marks 2..8.
static int render_tail(lodge_ctx *c, const lodge_level *levels, const LevelSlots &ls,
                       const lodge_camera *cam_dev, int32_t W, int32_t H,
                       const lodge_raster_params &rp, int32_t flags, const lodge_frame_out *out,
                       lodge_frame_stats *stats_dev, int32_t nl, const char *name,
                       const lodge_chunks *ch) {
  cudaStream_t s = c->stream;
  Work &w = c->w;
  const bool exact = c->precision == LODGE_PREC_EXACT;
  const int64_t U_cap = ls.slot_base[ls.n_levels];
  const int32_t tiles_x = (W + 15) / 16, tiles_y = (H + 15) / 16;
  {
    const int rc0 = check_srgb_out(c, flags, out);
    if (rc0) return rc0;
  }
  c->mark(2);
  if ((flags & LODGE_RECORD_MAX) && !(flags & LODGE_ACCUMULATE_MAX) && out->maxw_dev)
    CK(cudaMemsetAsync(out->maxw_dev, 0, (exact ? 8 : 4) * (size_t)U_cap, s));
  const int32_t shade = (flags & LODGE_NEED_IMAGE) ? 1 : 0;
  const void *const *slab_geom = ch ? ch->slab_geom_dev : nullptr;
  const void *const *slab_sh = ch ? ch->slab_sh_dev : nullptr;
  int rc = launch_project_frame(levels, ls, w, c->fs, cam_dev, rp, W, H, s, slab_geom, slab_sh);
  if (rc) return set_err(LODGE_ERR_BAD_ARG, "all levels must share one storage precision");
  ++nl;
  DSYNC("launch_project_frame");
  c->mark(3);
  const bool two = two_phase(c, W, H, flags, out);
  const uint32_t budget =
      (uint32_t)std::min<int64_t>((int64_t)c->phase_budget * tiles_x * tiles_y, 0x7fffffff);
  if (two) {
    // two-phase frames sort only the first phase's candidates
    launch_depth_select(w, c->fs, U_cap, budget, s);
    launch_subset_sort(w, c->fs, U_cap, &c->fs->n_cand, w.sel_keys, w.sel_vals, w.sort_scr[0],
                       w.sort_scr[1], w.sort_scr[2], w.sort_scr[3], w.val_depth[0], TK_DEPTH0,
                       &nl, s);
    nl += 3;
  } else {
    launch_depth_sort(w, c->fs, U_cap, &nl, s, true);
  }
  DSYNC("launch_depth_sort");
  DSYNC_L(2, "segment: select .. depth sort");
  c->mark(4);
  if (two) {
    // FAST frames in two depth phases: the splats whose pairs
    // start within the budget are binned, sorted and composited first; the
    // tiles that still have live pixels then receive the rest of their pairs
    launch_dup_count(w, c->fs, tiles_x, tiles_y, U_cap, budget, s, &c->fs->n_cand);
    DSYNC("launch_dup_count");
    // compositing records of the first phase's splats only
    launch_payload(levels, ls, w, c->fs, cam_dev, rp, shade, w.val_depth[0], &c->fs->split_S,
                   U_cap, s, slab_geom, slab_sh); ++nl;
    DSYNC("launch_payload");
    launch_tile_setup(w, c->fs, out->tile_count_dev, tiles_x, tiles_y, s, true, c->block_lists);
    DSYNC("launch_tile_setup");
    nl += 2;
    c->mark(5);
    launch_dup_emit(w, c->fs, tiles_x, s, true); ++nl;
    DSYNC("launch_dup_emit");
    c->mark(6);
    // per-tile lists from the sorted pairs (n_sort_a of them), or -- a first
    // phase of few large splats -- block lists (k_block_lists); each launch
    // does nothing in the other mode
    launch_tile_sort(w, c->fs, tiles_x, tiles_y, &nl, s, TK_TILE0, &c->fs->n_sort_a);
    launch_block_lists(w, c->fs, tiles_x, tiles_y, 1, s); ++nl;
#ifdef LODGE_VERIFY
    launch_list_verify(w, c->fs, (uint32_t)(tiles_x * tiles_y), false, s, tiles_x, tiles_y);
#endif
    DSYNC("launch_tile_sort");
    c->mark(7);
#ifndef LODGE_DEBUG_SKIP_COMPOSITE  // diagnostic builds: the frame without its compositing
    launch_composite(w, c->fs, cam_dev, W, H, rp, flags, exact, *out, (uint32_t)U_cap, s, 1);
#endif
    ++nl;
    DSYNC("launch_composite");
    DSYNC_L(2, "segment: count .. first-phase composite");
    c->mark(8);
#ifndef LODGE_DEBUG_SKIP_PHASE2  // diagnostic builds: the frame without its second phase
    launch_setup_b(w, c->fs, tiles_x, tiles_y, s);
    DSYNC("launch_setup_b");
    // the later splats that meet an alive tile, in depth order
    launch_owner_filter(w, c->fs, tiles_x, U_cap, s);
    launch_subset_sort(w, c->fs, U_cap, &c->fs->n_ocand, w.sel_keys, w.sel_vals, w.sort_scr[0],
                       w.sort_scr[1], w.sort_scr[2], w.sort_scr[3], w.val_depth[1], TK_OSORT0,
                       &nl, s);
    ++nl;
    DSYNC("launch_owner_filter + sort");
    launch_enum_b(w, c->fs, tiles_x, tiles_y, U_cap, s);
    DSYNC("launch_enum_b");
    // ... and of the later splats that meet an unfinished tile
    launch_payload(levels, ls, w, c->fs, cam_dev, rp, shade, w.val_depth[1], &c->fs->n_owners_b,
                   U_cap, s, slab_geom, slab_sh);
    DSYNC("launch_payload (second phase)");
    nl += 4;
    launch_tile_sort(w, c->fs, tiles_x, tiles_y, &nl, s, TK_TILEB0, &c->fs->n_sort_b);
    launch_block_lists(w, c->fs, tiles_x, tiles_y, 2, s); ++nl;
#ifdef LODGE_VERIFY
    launch_list_verify(w, c->fs, (uint32_t)(tiles_x * tiles_y), true, s, tiles_x, tiles_y);
#endif
    DSYNC("launch_tile_sort (second phase)");
    c->mark(9);
#if !defined(LODGE_DEBUG_SKIP_COMPOSITE) && !defined(LODGE_DEBUG_SKIP_COMPOSITE_B)
    launch_composite(w, c->fs, cam_dev, W, H, rp, flags, exact, *out, (uint32_t)U_cap, s, 2);
#endif
    ++nl;
#else
    c->mark(9);
#endif
    DSYNC("launch_composite (second phase)");
    DSYNC_L(2, "segment: second phase");
    c->mark(10);
  } else {
    launch_payload(levels, ls, w, c->fs, cam_dev, rp, shade, w.val_depth[0], &c->fs->stats.M,
                   U_cap, s, slab_geom, slab_sh); ++nl;
    DSYNC("launch_payload");
    launch_tile_setup(w, c->fs, out->tile_count_dev, tiles_x, tiles_y, s); ++nl;
    DSYNC("launch_tile_setup");
    c->mark(5);
    launch_duplicate(w, c->fs, tiles_x, U_cap, s); nl += 2;  // count, emit
    DSYNC("launch_duplicate");
    c->mark(6);
    launch_tile_sort(w, c->fs, tiles_x, tiles_y, &nl, s);
#ifdef LODGE_VERIFY
    launch_list_verify(w, c->fs, (uint32_t)(tiles_x * tiles_y), false, s);
#endif
    DSYNC("launch_tile_sort");
    c->mark(7);
    launch_composite(w, c->fs, cam_dev, W, H, rp, flags, exact, *out, (uint32_t)U_cap, s);
    ++nl;
    DSYNC("launch_composite");
    c->mark(8);
    c->mark(9);
    c->mark(10);
  }
  if (c->prof && c->prof_frames < c->prof_cap) ++c->prof_frames;
  if (stats_dev)
    CK(cudaMemcpyAsync(stats_dev, &c->fs->stats, sizeof(lodge_frame_stats), cudaMemcpyDeviceToDevice, s));
  c->launches = nl;
  return check_launch(name);
}

// device address of a device camera's position (address arithmetic only)
static const double *cam_pos(const lodge_camera *cam_dev) {
  return reinterpret_cast<const double *>(reinterpret_cast<const char *>(cam_dev) +
                                          offsetof(lodge_camera, pos));
}

int lodge_render_lod(lodge_ctx *c, const lodge_level *levels, int32_t n_levels,
                     const double *bounds, int32_t full, const lodge_camera *cam_dev, int32_t W,
                     int32_t H, const lodge_raster_params *rp, int32_t flags,
                     const lodge_frame_out *out, lodge_frame_stats *stats_dev) {
  if (!c || !levels || !cam_dev || !rp || !out || (!full && !bounds))
    return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  if (n_levels < 1 || n_levels > LODGE_MAX_LEVELS)
    return set_err(LODGE_ERR_BAD_ARG, "level count must be in 1.." + std::to_string(LODGE_MAX_LEVELS));
  if (W <= 0 || H <= 0) return set_err(LODGE_ERR_BAD_ARG, "camera resolution must be positive");
  int rc = check_tile_smem(W, H);
  if (rc) return rc;
  for (int l = 0; l < n_levels; ++l) {
    if (levels[l].sh_degree < 0 || levels[l].sh_degree > 3)
      return set_err(LODGE_ERR_BAD_ARG, "sh degree must be in 0..3");
    if (levels[l].n > 0x3fffffff) return set_err(LODGE_ERR_BAD_ARG, "level too large");
  }
  CK(cudaSetDevice(c->device));
  LevelSlots ls;
  ls.n_levels = n_levels;
  ls.slot_base[0] = 0;
  for (int l = 0; l < n_levels; ++l)
    ls.slot_base[l + 1] = ls.slot_base[l] + ((full && l > 0) ? 0u : (uint32_t)levels[l].n);
  const int64_t U_cap = ls.slot_base[n_levels];
  if (U_cap > 0x3fffffff) return set_err(LODGE_ERR_BAD_ARG, "too many inputs");
  if ((rc = ensure_slots(c, U_cap)) || (rc = ensure_M(c, std::max<int64_t>(U_cap, 1))) ||
      (rc = ensure_tiles(c, W, H)) || (rc = ensure_P(c, 1)) ||
      (rc = ensure_status(c, (c->w.M_cap + 4095) / 4096 * 256 + (U_cap + 255) / 256 + 256)))
    return rc;
  c->last_slots = ls;
  int32_t nl = 0;
  c->mark(0);
  launch_begin_frame(c->fs, c->stream); ++nl;
  c->mark(1);
  launch_band_select(levels, n_levels, bounds, full, ls, c->fs, cam_pos(cam_dev), c->w.status,
                     c->w.union_idx, c->w.union_tag, c->stream);
  nl += 2;
  return render_tail(c, levels, ls, cam_dev, W, H, *rp, flags, out, stats_dev, nl,
                     "lodge_render_lod", nullptr);
}

int lodge_select_active(lodge_ctx *c, const lodge_level *levels, int32_t n_levels,
                        const double *bounds, const double *pos_dev, uint32_t *idx_dev,
                        uint32_t *sizes_dev) {
  if (!c || !levels || !bounds || !pos_dev || !idx_dev || !sizes_dev)
    return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  if (n_levels < 1 || n_levels > LODGE_MAX_LEVELS)
    return set_err(LODGE_ERR_BAD_ARG, "level count must be in 1.." + std::to_string(LODGE_MAX_LEVELS));
  for (int l = 0; l < n_levels; ++l) {
    if (levels[l].n > 0x3fffffff) return set_err(LODGE_ERR_BAD_ARG, "level too large");
    if (levels[l].n > 0 && !levels[l].geom_dev) return set_err(LODGE_ERR_BAD_ARG, "NULL level geometry");
  }
  CK(cudaSetDevice(c->device));
  LevelSlots ls;
  ls.n_levels = n_levels;
  ls.slot_base[0] = 0;
  for (int l = 0; l < n_levels; ++l) ls.slot_base[l + 1] = ls.slot_base[l] + (uint32_t)levels[l].n;
  const int64_t U_cap = ls.slot_base[n_levels];
  if (U_cap > 0x3fffffff) return set_err(LODGE_ERR_BAD_ARG, "too many inputs");
  int rc;
  if ((rc = ensure_slots(c, std::max<int64_t>(U_cap, 1))) ||
      (rc = ensure_status(c, (U_cap + 255) / 256 + 256)))
    return rc;
  // the band kernel compacts straight into the caller's buffer (level l at
  // slot_base[l]); its tags go to the context's scratch
  launch_begin_frame(c->fs, c->stream);
  launch_band_select(levels, n_levels, bounds, 0, ls, c->fs, pos_dev, c->w.status, idx_dev,
                     c->w.union_tag, c->stream);
  CK(cudaMemcpyAsync(sizes_dev,
                     reinterpret_cast<const char *>(c->fs) + offsetof(FrameState, stats) +
                         offsetof(lodge_frame_stats, U_level),
                     4 * (size_t)n_levels, cudaMemcpyDeviceToDevice, c->stream));
  return check_launch("lodge_select_active");
}

int lodge_frame_lists(lodge_ctx *c, int32_t T, int64_t *tile_offsets, int64_t *tile_src,
                      int64_t cap) {
  if (!c || !tile_offsets || !tile_src) return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  if (!c->w.list || T + 1 > c->tiles_cap) return set_err(LODGE_ERR_BAD_ARG, "no frame rendered at this size");
  launch_export_lists(c->w, c->fs, T, tile_offsets, tile_src, cap, c->stream);
  return check_launch("lodge_frame_lists");
}

int lodge_frame_union(lodge_ctx *c, int32_t level, uint32_t *idx, uint8_t *tag, int64_t cap) {
  if (!c || !idx || !tag) return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  if (level < 0 || level >= c->last_slots.n_levels) return set_err(LODGE_ERR_BAD_ARG, "bad level");
  const int64_t n = std::min<int64_t>(cap, c->last_slots.slot_base[level + 1] - c->last_slots.slot_base[level]);
  if (n > 0) {
    CK(cudaMemcpyAsync(idx, c->w.union_idx + c->last_slots.slot_base[level], 4 * n,
                       cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(tag, c->w.union_tag + c->last_slots.slot_base[level], n,
                       cudaMemcpyDeviceToDevice, c->stream));
  }
  return 0;
}

int lodge_profile(lodge_ctx *c, int32_t enable, int32_t max_frames) {
  if (!c) return set_err(LODGE_ERR_BAD_ARG, "ctx is NULL");
  CK(cudaSetDevice(c->device));
  if (enable && max_frames > c->prof_cap) {
    if (c->prof_ev) {
      for (int i = 0; i < c->prof_cap * (LODGE_N_STAGES + 1); ++i) cudaEventDestroy(c->prof_ev[i]);
      delete[] c->prof_ev;
    }
    c->prof_ev = new cudaEvent_t[(size_t)max_frames * (LODGE_N_STAGES + 1)];
    for (int i = 0; i < max_frames * (LODGE_N_STAGES + 1); ++i) CK(cudaEventCreate(&c->prof_ev[i]));
    c->prof_cap = max_frames;
  }
  c->prof = enable != 0;
  c->prof_frames = 0;
  return 0;
}

int lodge_profile_read(lodge_ctx *c, double *stage_ms, int32_t *frames) {
  if (!c || !stage_ms || !frames) return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  for (int k = 0; k < LODGE_N_STAGES; ++k) stage_ms[k] = 0.0;
  for (int f = 0; f < c->prof_frames; ++f) {
    cudaEvent_t *e = c->prof_ev + f * (LODGE_N_STAGES + 1);
    CK(cudaEventSynchronize(e[LODGE_N_STAGES]));
    for (int k = 0; k < LODGE_N_STAGES; ++k) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e[k], e[k + 1]));
      stage_ms[k] += ms;
    }
  }
  *frames = c->prof_frames;
  c->prof_frames = 0;
  return 0;
}

__global__ void __launch_bounds__(256) k_srgb8(const float *__restrict__ img, int64_t n,
                                               const float *__restrict__ thr,
                                               uint8_t *__restrict__ out) {
  __shared__ float t[256];
  t[threadIdx.x] = thr[threadIdx.x];
  __syncthreads();
  const int64_t total = 3 * n;
  for (int64_t i0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); i0 < total;
       i0 += 4 * (int64_t)gridDim.x * blockDim.x) {
    float x[4];
    const bool full = i0 + 4 <= total && (reinterpret_cast<uintptr_t>(img + i0) & 15) == 0;
    if (full) {
      const float4 v = *reinterpret_cast<const float4 *>(img + i0);
      x[0] = v.x; x[1] = v.y; x[2] = v.z; x[3] = v.w;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) x[q] = i0 + q < total ? img[i0 + q] : 0.f;
    }
    uint32_t packed = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int k = 0;  // the number of thresholds <= x
#pragma unroll
      for (int st = 128; st >= 1; st >>= 1) k += (x[q] >= t[k + st]) ? st : 0;
      packed |= (uint32_t)k << (8 * q);
    }
    if (full && (reinterpret_cast<uintptr_t>(out + i0) & 3) == 0) {
      *reinterpret_cast<uint32_t *>(out + i0) = packed;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (i0 + q < total) out[i0 + q] = (uint8_t)(packed >> (8 * q));
    }
  }
}

int lodge_to_srgb8(lodge_ctx *c, const float *img, int64_t n, uint8_t *out) {
  if (!c || !img || !out) return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  if (n <= 0) return 0;
  int rc = ensure_srgb(c);
  if (rc) return rc;
  const int64_t quads = (3 * n + 3) / 4;
  const unsigned grid = (unsigned)std::min<int64_t>((quads + 255) / 256, 148 * 16);
  k_srgb8<<<grid, 256, 0, c->stream>>>(img, n, c->w.srgb_thr, out);
  return check_launch("lodge_to_srgb8");
}

int32_t lodge_last_launch_count(lodge_ctx *c) { return c ? c->launches : 0; }

int lodge_fault_flags(lodge_ctx *c, uint32_t *flags) {
  if (!c || !flags) return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(flags, reinterpret_cast<const char *>(c->fs) + offsetof(FrameState, fault_sticky),
                sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return 0;
}

int lodge_debug_counters(lodge_ctx *c, uint64_t *out8) {
  if (!c || !out8) return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(out8, c->fs->counters, 8 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return 0;
}

int lodge_frame_report(lodge_ctx *c, const int32_t *visible_dev, int64_t n_pixels,
                       const double *edges_host, int32_t n_edges,
                       const int32_t *tile_count_dev, int64_t n_tiles, const void *maxw_dev,
                       int32_t maxw_fp64, int64_t n_inputs, uint64_t *out_dev) {
  if (!c || !edges_host || !out_dev || (n_pixels > 0 && !visible_dev) ||
      (n_tiles > 0 && !tile_count_dev))
    return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  if (n_edges < 2) return set_err(LODGE_ERR_BAD_ARG, "need at least two bin edges");
  if (n_edges > 257) return set_err(LODGE_ERR_BAD_ARG, "at most 256 histogram bins");
  for (int i = 0; i + 1 < n_edges; ++i)
    if (!(edges_host[i + 1] > edges_host[i]))
      return set_err(LODGE_ERR_BAD_ARG, "bin edges must be strictly increasing");
  if (n_pixels < 0 || n_tiles < 0 || n_inputs < 0) return set_err(LODGE_ERR_BAD_ARG, "negative size");
  CK(cudaSetDevice(c->device));
  if (!c->edges_dev) CK(cudaMalloc(&c->edges_dev, 257 * sizeof(double)));
  CK(cudaMemcpyAsync(c->edges_dev, edges_host, sizeof(double) * n_edges, cudaMemcpyHostToDevice,
                     c->stream));
  launch_frame_report(visible_dev, n_pixels, c->edges_dev, n_edges, tile_count_dev, n_tiles,
                      maxw_dev, maxw_fp64, maxw_dev ? n_inputs : 0,
                      reinterpret_cast<unsigned long long *>(out_dev), c->stream);
  // (a pageable-memory copy is staged before cudaMemcpyAsync returns, so the
  // caller may reuse edges_host at once)
  return check_launch("lodge_frame_report");
}

int lodge_sq_err(lodge_ctx *c, const float *a_dev, const float *b_dev, int64_t n,
                 double *out_dev) {
  if (!c || !out_dev || (n > 0 && (!a_dev || !b_dev)))
    return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  if (n < 0) return set_err(LODGE_ERR_BAD_ARG, "negative size");
  CK(cudaSetDevice(c->device));
  launch_sq_err(a_dev, b_dev, n, out_dev, c->stream);
  return check_launch("lodge_sq_err");
}

int lodge_debug_depth_sort(lodge_ctx *c, const uint64_t *keys_dev, int64_t n,
                           uint64_t *sorted_keys_dev, uint32_t *sorted_idx_dev,
                           uint32_t *out_m_dev) {
  if (!c || (n > 0 && (!keys_dev || !sorted_keys_dev || !sorted_idx_dev)) || !out_m_dev)
    return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  if (n < 0 || n > 0x3fffffff) return set_err(LODGE_ERR_BAD_ARG, "bad key count");
  CK(cudaSetDevice(c->device));
  int rc;
  if ((rc = ensure_M(c, std::max<int64_t>(n, 1))) ||
      (rc = ensure_status(c, (c->w.M_cap + 4095) / 4096 * 256 + 256)))
    return rc;
  launch_begin_frame(c->fs, c->stream);
  launch_debug_depth_sort(c->w, c->fs, keys_dev, (uint32_t)n, sorted_keys_dev, sorted_idx_dev,
                          out_m_dev, c->stream);
  return check_launch("lodge_debug_depth_sort");
}

int lodge_asset_split(lodge_ctx *c, const void *blob_dev, int64_t n, int32_t sh_degree,
                      float *geom_dev, float *sh_dev, int32_t *violations) {
  if (!c || !violations || (n > 0 && (!blob_dev || !geom_dev || !sh_dev)))
    return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  if (n < 0) return set_err(LODGE_ERR_BAD_ARG, "negative record count");
  if (sh_degree < 0 || sh_degree > 3) return set_err(LODGE_ERR_BAD_ARG, "sh degree must be in 0..3");
  *violations = 0;
  if (n == 0) return 0;
  CK(cudaSetDevice(c->device));
  const int32_t width = 12 + 3 * (sh_degree + 1) * (sh_degree + 1);
  int32_t *flags = nullptr;
  CK(cudaMallocAsync(&flags, sizeof(int32_t), c->stream));
  CK(cudaMemsetAsync(flags, 0, sizeof(int32_t), c->stream));
  launch_asset_split(reinterpret_cast<const float *>(blob_dev), n, width, geom_dev, sh_dev,
                     flags, c->stream);
  const int rc = check_launch("lodge_asset_split");
  CK(cudaMemcpyAsync(violations, flags, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaFreeAsync(flags, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return rc;
}

int lodge_cover_table(lodge_ctx *c, const lodge_level *level, const int64_t *idx_dev, int64_t n,
                      const lodge_camera *cam, const lodge_raster_params *rp, double *dist_dev,
                      int64_t *prefix_dev, int64_t *out_m) {
  if (!c || !level || !rp || !out_m || (n > 0 && (!dist_dev || !prefix_dev)))
    return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  int rc = check_cam(cam);
  if (rc) return rc;
  if (n < 0 || n > 0x3fffffff) return set_err(LODGE_ERR_BAD_ARG, "bad input count");
  *out_m = 0;
  CK(cudaSetDevice(c->device));
  if (n == 0) {
    const int64_t zero = 0;
    if (prefix_dev) CK(cudaMemcpy(prefix_dev, &zero, sizeof(zero), cudaMemcpyHostToDevice));
    return 0;
  }
  if ((rc = ensure_M(c, n)) ||
      (rc = ensure_status(c, (n + 4095) / 4096 * 256 + (n + 255) / 256 + 256)))
    return rc;
  cudaStream_t s = c->stream;
  *c->cam_host = *cam;
  CK(cudaMemcpyAsync(c->cam_dev, c->cam_host, sizeof(lodge_camera), cudaMemcpyHostToDevice, s));
  int32_t nl = 0;
  launch_begin_frame(c->fs, s);
  launch_cover_keys(*level, idx_dev, n, c->w, c->fs, c->cam_dev, *rp, s);
  launch_cover_table(c->w, c->fs, n, dist_dev, prefix_dev, &nl, s);
  rc = check_launch("lodge_cover_table");
  if (rc) return rc;
  CK(cudaMemcpyAsync(c->stats_host, &c->fs->stats, sizeof(lodge_frame_stats),
                     cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *out_m = c->stats_host->M;
  return 0;
}

int lodge_asset_check_sets(lodge_ctx *c, const lodge_chunks *ch, const int64_t *level_sizes,
                           int32_t *set_flags) {
  if (!c || !ch || !level_sizes || !set_flags) return set_err(LODGE_ERR_BAD_ARG, "NULL argument");
  if (ch->K < 0 || ch->L < 1 || ch->L > LODGE_MAX_LEVELS)
    return set_err(LODGE_ERR_BAD_ARG, "bad chunk plan shape");
  const int32_t nsets = ch->K * ch->L;
  if (nsets == 0) return 0;
  CK(cudaSetDevice(c->device));
  int64_t *lsz = nullptr;
  int32_t *flags = nullptr;
  CK(cudaMallocAsync(&lsz, sizeof(int64_t) * ch->L, c->stream));
  CK(cudaMallocAsync(&flags, sizeof(int32_t) * nsets, c->stream));
  CK(cudaMemcpyAsync(lsz, level_sizes, sizeof(int64_t) * ch->L, cudaMemcpyHostToDevice,
                     c->stream));
  CK(cudaMemsetAsync(flags, 0, sizeof(int32_t) * nsets, c->stream));
  launch_asset_sets(*ch, lsz, flags, c->stream);
  const int rc = check_launch("lodge_asset_check_sets");
  CK(cudaMemcpyAsync(set_flags, flags, sizeof(int32_t) * nsets, cudaMemcpyDeviceToHost,
                     c->stream));
  CK(cudaFreeAsync(lsz, c->stream));
  CK(cudaFreeAsync(flags, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return rc;
}

}  // extern "C"
