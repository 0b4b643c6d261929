// Internal device-side definitions shared by the liblodge kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lodge.h"

#define LODGE_TILE 16
#define LODGE_SUPPORT_Q 9.0
#define FULL_MASK 0xffffffffu

namespace lodge {

// ---------------------------------------------------------------------------
// Per-frame device state (one per in-flight frame).
// ---------------------------------------------------------------------------
struct FrameState {
  lodge_frame_stats stats;            // f, o, t_bar, t, U, M, P, overflow ...
  uint32_t epoch;                     // look-back epoch base for this frame
  uint32_t n_pairs;                   // P, or 0 on overflow: pairs actually stored
  uint32_t n_sort;                    // keys in the depth sort (U fused, M compat)
  uint32_t tickets[32];               // virtual block-id tickets, zeroed per frame
  uint32_t hist_depth[8][256];        // onesweep digit histograms (depth keys)
  uint32_t off_depth[8][256];         // their exclusive scans
  uint32_t off_tile[2][256];          // digit offsets for the two tile passes
  // two-phase frames: the depth-order splat split, and the
  // second phase's tile count and pair total
  uint32_t split_S;                   // splats [0, S) form the first phase
  uint32_t P_A;                       // their pairs (a prefix of the pair sequence)
  uint32_t n_alive;                   // tiles the second phase composites
  uint32_t n_owners_b;                // second-phase splats that meet an alive tile
  uint32_t alive_box[4];              // x0, x1, y0, y1: bounding box of the alive tiles
  // block lists: a phase whose splats are few and large keeps,
  // per block of BLK_W x BLK_H tiles, its splats that meet the block in depth
  // order with their tile masks; the compositor walks them instead of sorted
  // per-tile lists
  uint32_t scan_a, scan_b;            // phase 1 / phase 2 uses block lists
  uint32_t bl_nlive[2];               // per phase: blocks with pairs (entries of bl_live)
  // two-phase frames sort only what they composite: the
  // candidates of the first phase and the owners of the second
  uint32_t n_cand;                    // first-phase candidates (depth bins <= sel_B)
  uint32_t sel_B;                     // last candidate depth bin
  uint32_t n_ocand;                   // second-phase owners found by the filter
  uint32_t p1_g;                      // the last first-phase splat (input index) ...
  uint32_t p1_k32;                    // ... its 32-bit depth key ...
  uint64_t p1_key;                    // ... and its fp64 depth key
  uint32_t n_sort_a, n_sort_b;        // pairs emitted and sorted per phase (0 with block lists)
  uint32_t fault_sticky;              // OR of every frame's stats.fault (lodge_fault_flags)
  // union reuse (lodge_chunks.uid): the pair and sizes of the union held in
  // the context's union buffers
  uint64_t uc_uid;                    // 0: nothing cached
  int32_t uc_f, uc_o;
  uint32_t uc_U[LODGE_MAX_LEVELS];
  uint32_t uc_hit;                    // this frame reuses the cached union
  unsigned long long counters[8];     // LODGE_COUNTERS builds: compositing work counters
};

enum Ticket {
  TK_COMPACT = 0,
  TK_DUP = 1,
  TK_DEPTH0 = 2,   // .. TK_DEPTH0 + 7
  TK_TILE0 = 10,   // .. TK_TILE0 + 1
  TK_UNION0 = 12,  // .. TK_UNION0 + LODGE_MAX_LEVELS - 1
  TK_DUPB = 20,    // second phase: enumeration scan
  TK_EMITB = 21,   //               ordered pair compaction
  TK_TILEB0 = 22,  //               tile passes (.. TK_TILEB0 + 1)
  TK_BLA = 24,     // block lists, phase 1
  TK_BLB = 25,     // block lists, phase 2
  TK_OSORT0 = 26,  // second-phase owner sort passes (.. TK_OSORT0 + 3)
};

// Persistent (ticketed) grids: at most this many CTAs per SM, below the
// occupancy limit, so the frames in flight on other streams keep room on
// every SM
#ifndef LODGE_PERSIST_PER
#define LODGE_PERSIST_PER 64
#endif

// Block lists: blocks of BLK_W x BLK_H tiles (tile bit (y % BLK_H) * BLK_W +
// x % BLK_W of an entry's mask), scanned in chunks of BL_CHUNK splats, at
// most BL_CHMAX chunks (a phase uses block lists only below that many splats).
#ifndef LODGE_BLK_W
#define LODGE_BLK_W 8
#endif
#ifndef LODGE_BLK_H
#define LODGE_BLK_H 4
#endif
constexpr int BLK_W = LODGE_BLK_W, BLK_H = LODGE_BLK_H;
static_assert(BLK_W * BLK_H <= 32 && BLK_W <= 16, "tile masks fit 32 bits");
constexpr int BL_CHUNK = 1024;
#ifndef LODGE_BL_CHMAX
#define LODGE_BL_CHMAX 128
#endif
constexpr int BL_CHMAX = LODGE_BL_CHMAX;
__host__ __device__ inline int32_t block_count(int32_t tiles_x, int32_t tiles_y) {
  return ((tiles_x + BLK_W - 1) / BLK_W) * ((tiles_y + BLK_H - 1) / BLK_H);
}

// Splat payload for compositing (64 B, one per survivor).  mean2d is kept in
// fp64 so the tile-local fp32 offset is exact to fp32 rounding.  The fp32
// conic is stored in exponent units: qs = KQ * q with KQ = -log2(e)/2, so a
// pixel's alpha is exp2(qs + log2 o) with no per-pixel scaling.  q_eff, the
// per-splat cut-off on q that encodes both q > 9 and alpha < alpha_min, and
// tol, the fp32 error bound of q near it, become the guard band [lo, hi] on
// qs: qs > hi keeps for certain, lo <= qs <= hi is re-decided in fp64.
constexpr double KQ = -0.72134752044448170;  // -0.5 / ln 2
struct __align__(16) Payload {
  double mx, my;
  float As, B2s, Cs, lo2;  // KQ * (A, 2B, C), log2 of the effective opacity
  float r, g, b;           // colour
  uint32_t src;            // concatenated input index
  float hi, lo;            // guard band on qs (hi rounded up, lo rounded down)
  float bx, by;            // half-widths of a box containing every pixel that can be non-skipped
};
static_assert(sizeof(Payload) == 64, "payload must be 64 B");

// fp64 copy of the compositing inputs (guard band and EXACT mode).
struct __align__(16) Precise {
  double A, B, C, o;
  double r, g, b, pad;
};
static_assert(sizeof(Precise) == 64, "precise record must be 64 B");

// Workspace pointers handed to kernels.
struct Work {
  int32_t grid_share = 0;   // lodge_set_grid_share: persistent CTAs per SM (0: default)
  uint64_t *key_depth[2];   // M_cap each (ping-pong)
  uint32_t *val_depth[2];   // M_cap each
  uint64_t *rect;           // M_cap packed x0|x1<<16|y0<<32|y1<<48
  Payload *payload;         // M_cap
  Precise *precise;         // M_cap
  uint64_t *pairs[2];       // P_cap each
  const uint32_t *list;     // per-tile lists (splat ids) of the last tile sort, in pairs[0|1]
  uint64_t *rect_sorted;    // M_cap: rectangles in depth order
  uint32_t *splat_off;      // M_cap + 1: pair offset of each depth-ordered splat
  uint32_t *chunk_first;    // P_cap / EMIT_CHUNK + 2: owner of each emission chunk
  uint32_t *tile_order;     // T: tiles, heaviest first (composite schedule)
  int32_t *tile_diff;       // (tiles_x+1)*(tiles_y+1) 2-D difference array
  uint32_t *tile_start;     // T+1
  // two-phase frames
  int32_t *tile_diff_a;     // (tiles_x+1)*(tiles_y+1): first-phase splats only
  uint32_t *count_all;      // T: pairs per tile over all splats
  uint32_t *tile_start_b;   // T+1: second-phase list ranges
  uint32_t *tile_order_b;   // T: second-phase tiles, heaviest first
  uint32_t *alive;          // ceil(T/32) bitmap: tiles the second phase composites
  uint32_t *sat;            // (tiles_y+1)*(tiles_x+1) summed-area table of alive tiles
  float4 *state;            // W*H: (T, r, g, b) of pixels of alive tiles after phase one
  uint64_t *status;         // look-back status words (epoch | flags | value)
  uint32_t *union_idx;      // slots
  uint8_t *union_tag;       // slots
  uint32_t *vrank;          // LODGE_VERIFY builds: depth rank of each input (M_cap)
  float *srgb_thr;          // 256 level thresholds of the reference's to_uint8 (lodge_to_srgb8)
  uint32_t *bl_start;       // 2 x (blocks + 1): per phase, block-list capacity offsets
  uint32_t *bl_len;         // 2 x blocks: per phase, block-list lengths
  uint32_t *bl_live;        // 2 x blocks: per phase, the blocks with pairs (any order)
  uint32_t *sel_hist;       // SEL_BINS: pair counts per depth bin (zero between frames)
  uint32_t *sel_keys, *sel_vals;  // M_cap each: candidates / owners to sort (any order)
  uint32_t *sort_scr[4];    // M_cap each: subset-sort ping-pong (keys 0, 1; values 0, 1)
  int64_t M_cap, P_cap, status_cap, slot_cap;
};

// The 32-bit depth keys ping-pong in the two halves of key_depth[1]; the
// projection's compacted survivor keys start in the second half (the first
// pass reads them and writes the first half).
__host__ __device__ inline uint32_t *depth_keys32(const Work &w, int half) {
  return reinterpret_cast<uint32_t *>(w.key_depth[1]) + (half ? w.M_cap : 0);
}
__host__ __device__ inline uint32_t *depth_keys_compact(const Work &w) {
  return depth_keys32(w, 1);
}

// Device-side bounds checks: a violated invariant sets its bit in
// stats.fault and the offending access is skipped (the frame is reported
// invalid instead of faulting the context).
enum : uint32_t {
  FAULT_OWNERS = 1,   // an emission CTA's owner range exceeds its staging
  FAULT_COMPACT = 2,  // second-phase compaction beyond the pair count
  FAULT_SCATTER = 4,  // a onesweep scatter beyond the key count
  FAULT_LIST = 8,     // a compositor tile list range beyond the list buffer
  FAULT_TILE = 16,    // an emitted pair's tile beyond the frame
  FAULT_PAYLOAD = 32, // a compositing record requested for a non-input
  FAULT_DEPTH = 64,   // LODGE_VERIFY builds: the depth order failed its check
  FAULT_MEMBER = 128, // a compositor list member beyond the payload buffer
  FAULT_SRC = 256,    // a staged record whose input index is beyond the caller's max-weight buffer
  FAULT_LISTORD = 512, // LODGE_VERIFY builds: a per-tile list failed its order check
  FAULT_STAGE = 1024,  // LODGE_VERIFY builds: a onesweep partition staged a key outside its digit run
};
__device__ __forceinline__ void raise_fault(FrameState *fs, uint32_t bit) {
  atomicOr(&fs->stats.fault, bit);
  atomicOr(&fs->fault_sticky, bit);
}

// Status word: [63:32] epoch, [31:30] flag, [29:0] value.
enum : uint32_t { ST_EMPTY = 0, ST_AGG = 1, ST_PREFIX = 2 };
__device__ __forceinline__ uint64_t st_pack(uint32_t epoch, uint32_t flag, uint32_t v) {
  return ((uint64_t)epoch << 32) | ((uint64_t)flag << 30) | (uint64_t)(v & 0x3fffffffu);
}
// Look-back status cells: one 64-bit word per (partition, digit) holding
// epoch, flag and value together, so a reader needs no ordering beyond the
// single-copy atomicity of the word: relaxed loads and stores at gpu scope.
// (The intermittent wrong orders of round 1 were a warp left diverged by the
// per-lane spin below reaching an aligned CTA barrier, not a memory-order
// issue: see onesweep.cuh and DESIGN.md "Diverged warps at aligned barriers".)
__device__ __forceinline__ void st_store(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t st_load(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Single-counter decoupled look-back (one warp).  Returns the exclusive
// prefix of partition `part`.  `agg` must be warp-uniform; lane 0 publishes.
__device__ __forceinline__ uint32_t lookback_warp(uint64_t *status, uint32_t part, uint32_t agg,
                                                  uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  if (part == 0) {
    if (lane == 0) st_store(status, st_pack(epoch, ST_PREFIX, agg));
    __syncwarp();
    return 0;
  }
  if (lane == 0) st_store(status + part, st_pack(epoch, ST_AGG, agg));
  uint32_t prefix = 0;
  int64_t window_end = (int64_t)part - 1;  // inclusive, walk backwards
  while (true) {
    int64_t q = window_end - lane;
    uint32_t flag = ST_PREFIX, val = 0;
    if (q >= 0) {
      uint64_t s;
      do {
        s = st_load(status + q);
        flag = ((uint32_t)(s >> 32) == epoch) ? (uint32_t)((s >> 30) & 3u) : ST_EMPTY;
      } while (flag == ST_EMPTY);
      val = (uint32_t)(s & 0x3fffffffu);
    }
    __syncwarp();  // the lanes' spins end at different times: reconverge
    // lanes beyond q<0 act as an implicit zero prefix
    uint32_t pmask = __ballot_sync(FULL_MASK, flag == ST_PREFIX);
    int first = __ffs(pmask) - 1;  // nearest partition holding a prefix
    // no prefix in the window: every lane holds an aggregate, take all 32
    uint32_t contrib = (pmask == 0u || lane <= first) ? val : 0u;
    for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(FULL_MASK, contrib, o);
    prefix += contrib;
    if (pmask) break;
    window_end -= 32;
  }
  if (lane == 0) st_store(status + part, st_pack(epoch, ST_PREFIX, prefix + agg));
  __syncwarp();  // callers continue into aligned barriers with the warp converged
  return prefix;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Virtual block id from an atomic ticket: partitions are processed in the
// order blocks start, so a block only ever waits on running blocks.
__device__ __forceinline__ uint32_t take_ticket(uint32_t *ticket, uint32_t *s_tmp) {
  if (threadIdx.x == 0) *s_tmp = atomicAdd(ticket, 1u);
  __syncthreads();
  return *s_tmp;
}

// Block-ordered compaction of partition `part`: returns this thread's output
// slot (or -1); one look-back per block.
__device__ __forceinline__ int64_t compact_slot(bool keep, uint64_t *status, uint32_t epoch,
                                                uint32_t part, uint32_t *s_warp,
                                                uint32_t *s_base) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const uint32_t bal = __ballot_sync(FULL_MASK, keep);
  if (lane == 0) s_warp[warp] = __popc(bal);
  __syncthreads();
  if (warp == 0) {
    uint32_t v = lane < nwarps ? s_warp[lane] : 0;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(FULL_MASK, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t total = __shfl_sync(FULL_MASK, inc, 31);
    const uint32_t pre = lookback_warp(status, part, total, epoch);
    if (lane < nwarps) s_warp[lane] = inc - v;
    if (lane == 0) *s_base = pre;
  }
  __syncthreads();
  if (!keep) return -1;
  return (int64_t)(*s_base) + s_warp[warp] + __popc(bal & lanemask_lt());
}

// Warp-aggregated atomic: lanes hitting the same counter combine first (the
// corners of border-clipped splats are shared by many splats).  Called by
// the whole warp; inactive lanes pass idx = -1.
__device__ __forceinline__ void warp_add(int32_t *base, int32_t idx, int32_t v) {
  const uint32_t peers = __match_any_sync(FULL_MASK, idx);
  if (idx >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1)
    atomicAdd(base + idx, v * __popc(peers));
}

// Warp-aggregated add into a shared-memory counter array (the CTA-private
// difference array of the projection).
__device__ __forceinline__ void warp_add_shared(int32_t *base, int32_t idx, int32_t v) {
  const uint32_t peers = __match_any_sync(FULL_MASK, idx);
  if (idx >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(base + idx, v * __popc(peers));
}

// The same update into a CTA-private difference array in shared memory.
// Corners in the last column or row (x1 + 1 == tiles_x, y1 + 1 == tiles_y)
// only feed cells beyond the tile grid, which the integration never reads:
// they are skipped (the right and bottom border clips are the frequent
// shared corners).  Per-lane shared atomics: the hardware resolves the
// lanes that meet on a corner cheaper than a __match_any_sync aggregation
// (projection 0.123 -> 0.117 ms at config 3); LODGE_DIFF_MATCH keeps that.
__device__ __forceinline__ void add_tile_diff_shared(int32_t *diff, uint64_t rc, int32_t tiles_x,
                                                     int32_t tiles_y, bool valid) {
  const int32_t x0 = (int32_t)(rc & 0xffff), x1 = (int32_t)((rc >> 16) & 0xffff);
  const int32_t y0 = (int32_t)((rc >> 32) & 0xffff), y1 = (int32_t)(rc >> 48);
  const int32_t stride = tiles_x + 1;
  const bool xr = x1 + 1 < tiles_x, yb = y1 + 1 < tiles_y;
#ifndef LODGE_DIFF_MATCH
  if (valid) {
    atomicAdd(diff + y0 * stride + x0, 1);
    if (xr) atomicAdd(diff + y0 * stride + x1 + 1, -1);
    if (yb) atomicAdd(diff + (y1 + 1) * stride + x0, -1);
    if (xr && yb) atomicAdd(diff + (y1 + 1) * stride + x1 + 1, 1);
  }
#else
  warp_add_shared(diff, valid ? y0 * stride + x0 : -1, 1);
  warp_add_shared(diff, valid && xr ? y0 * stride + x1 + 1 : -1, -1);
  warp_add_shared(diff, valid && yb ? (y1 + 1) * stride + x0 : -1, -1);
  warp_add_shared(diff, valid && xr && yb ? (y1 + 1) * stride + x1 + 1 : -1, 1);
#endif
}

// 2-D difference-array update for a tile rectangle (whole warp; valid flag).
__device__ __forceinline__ void add_tile_diff(int32_t *diff, uint64_t rc, int32_t tiles_x,
                                              bool valid) {
  const int32_t x0 = (int32_t)(rc & 0xffff), x1 = (int32_t)((rc >> 16) & 0xffff);
  const int32_t y0 = (int32_t)((rc >> 32) & 0xffff), y1 = (int32_t)(rc >> 48);
  const int32_t stride = tiles_x + 1;
  warp_add(diff, valid ? y0 * stride + x0 : -1, 1);
  warp_add(diff, valid ? y0 * stride + x1 + 1 : -1, -1);
  warp_add(diff, valid ? (y1 + 1) * stride + x0 : -1, -1);
  warp_add(diff, valid ? (y1 + 1) * stride + x1 + 1 : -1, 1);
}

__host__ __device__ __forceinline__ uint32_t union_status_stride(uint32_t max_slots) {
  return (max_slots + 255u) / 256u + 1u;
}

// Per-device launch-configuration cache (opt-in shared-memory sizes, resident
// CTA counts): both are properties of a (kernel, device), and one process can
// hold contexts on several devices.
constexpr int LODGE_MAX_DEVICES = 64;
struct PerDevice {
  int64_t v[LODGE_MAX_DEVICES] = {};
  int64_t &operator()() {
    int d = 0;
    cudaGetDevice(&d);
    return v[(d >= 0 && d < LODGE_MAX_DEVICES) ? d : 0];
  }
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

}  // namespace lodge

// ---------------------------------------------------------------------------
// Host-side launchers (implemented in the k_*.cu files)
// ---------------------------------------------------------------------------
namespace lodge {
struct LevelSlots {
  int32_t n_levels;
  uint32_t slot_base[LODGE_MAX_LEVELS + 1];  // slots per level = 2*max_set
};

void launch_begin_frame(FrameState *fs, cudaStream_t s);
void launch_select(const double *centers, int32_t K, const double *pos, int32_t n, int32_t *f,
                   int32_t *o, double *tb, double *t, cudaStream_t s);
void launch_blend_factor(const double *in, int32_t n, double *out, cudaStream_t s);
void launch_select_frame(const double *centers, int32_t K, const lodge_camera *cam,
                         const int32_t *pair, const double *t_override, int32_t have_pair,
                         int32_t pair_f, int32_t pair_o, double t_val, FrameState *fs,
                         cudaStream_t s);
int launch_union(const lodge_chunks &ch, const LevelSlots &ls, FrameState *fs, uint64_t *status,
                  uint32_t *union_idx, uint8_t *union_tag, cudaStream_t s);
// W, H: the frame's size (its tile grid bounds the difference-array updates)
int launch_project_frame(const lodge_level *levels, const LevelSlots &ls, const Work &w,
                         FrameState *fs, const lodge_camera *cam_dev,
                         const lodge_raster_params &rp, int32_t W, int32_t H,
                         cudaStream_t s,
                         const void *const *slab_geom = nullptr,
                         const void *const *slab_sh = nullptr);
// Compositing records of the splats ids[0 .. *n_ptr) (concatenated indices
// g), n_cap an upper bound of *n_ptr for the grid.
int launch_payload(const lodge_level *levels, const LevelSlots &ls, const Work &w,
                   FrameState *fs, const lodge_camera *cam_dev, const lodge_raster_params &rp,
                   int32_t shade, const uint32_t *ids, const uint32_t *n_ptr, int64_t n_cap,
                   cudaStream_t s, const void *const *slab_geom = nullptr,
                   const void *const *slab_sh = nullptr);
int launch_project_compat(const lodge_level &level, const int64_t *idx, int64_t n,
                          const double *mod, const Work &w, FrameState *fs,
                          const lodge_camera *cam_dev, const lodge_raster_params &rp,
                          int32_t shade, const lodge_batch *out, cudaStream_t s);
void launch_import_batch(const lodge_batch &b, int64_t M, const Work &w, FrameState *fs,
                         const lodge_camera *cam_dev, const lodge_raster_params &rp,
                         int32_t exact, cudaStream_t s);
// Depth sort of the frame's inputs into val_depth[0] (input indices in depth
// order).  compacted: the projection left the M survivors as (32-bit key,
// input index) in depth_keys_compact(w) and val_depth[1] (any order);
// otherwise key_depth[0] holds fs->n_sort u64 keys by position (~0: culled,
// dropped by the first pass) and val_depth[1] the positions.
void launch_depth_sort(const Work &w, FrameState *fs, int64_t M_cap, int32_t *launches,
                       cudaStream_t s, bool compacted = false);
// The same sort of *n_ptr (32-bit key, input index) pairs from kin / vin
// (any order) into vout (input indices in (fp64 depth, index) order), with
// explicit ping-pong buffers and ticket slots tk0 .. tk0 + 3.
void launch_subset_sort(const Work &w, FrameState *fs, int64_t cap, const uint32_t *n_ptr,
                        const uint32_t *kin, const uint32_t *vin, uint32_t *ks0, uint32_t *ks1,
                        uint32_t *vs0, uint32_t *vs1, uint32_t *vout, int tk0,
                        int32_t *launches, cudaStream_t s);
// Two-phase frames: the first-phase candidates -- the survivors in the depth
// bins whose preceding bins hold fewer than `budget` pairs -- into sel_keys /
// sel_vals (n_cand of them); and, after the first phase, the second-phase
// owners (survivors after the first phase that meet an alive tile).
constexpr int SEL_SHIFT = 20;                // depth bins: the top 12 bits of the 32-bit key
constexpr int SEL_BINS = 1 << (32 - SEL_SHIFT);  // (an eighth of an octave each)
void launch_depth_select(const Work &w, FrameState *fs, int64_t M_cap, uint32_t budget,
                         cudaStream_t s);
void launch_owner_filter(const Work &w, FrameState *fs, int32_t tiles_x, int64_t M_cap,
                         cudaStream_t s);
void launch_depth_sort64(const Work &w, FrameState *fs, int64_t M_cap, int32_t *launches,
                         cudaStream_t s);
void launch_debug_depth_sort(const Work &w, FrameState *fs, const uint64_t *keys, uint32_t n,
                             uint64_t *ko, uint32_t *vo, uint32_t *m_out, cudaStream_t s);
void launch_tile_setup(const Work &w, FrameState *fs, int32_t *tile_count, int32_t tiles_x,
                       int32_t tiles_y, cudaStream_t s, bool two_phase = false,
                       int32_t bl_mode = LODGE_BLOCK_LISTS_AUTO);
// two-phase frames: first-phase pair budget of the counting pass
void launch_dup_count(const Work &w, FrameState *fs, int32_t tiles_x, int32_t tiles_y,
                      int64_t M_cap, uint32_t budget, cudaStream_t s,
                      const uint32_t *n_ptr = nullptr /* &fs->stats.M */);
void launch_dup_emit(const Work &w, FrameState *fs, int32_t tiles_x, cudaStream_t s,
                     bool first_phase);
void launch_setup_b(const Work &w, FrameState *fs, int32_t tiles_x, int32_t tiles_y,
                    cudaStream_t s);
void launch_enum_b(const Work &w, FrameState *fs, int32_t tiles_x, int32_t tiles_y,
                   int64_t M_cap, cudaStream_t s);
void launch_duplicate(const Work &w, FrameState *fs, int32_t tiles_x, int64_t M_cap,
                      cudaStream_t s);
void launch_tile_sort(Work &w, FrameState *fs, int32_t tiles_x, int32_t tiles_y,
                      int32_t *launches, cudaStream_t s, int tk0 = 10 /* TK_TILE0 */,
                      const uint32_t *n_keys = nullptr /* &fs->n_pairs */);
// two-phase frames whose phase `phase` (1, 2) has few large splats
// (fs->scan_a / scan_b): its block lists, into pairs[phase - 1]
void launch_block_lists(const Work &w, FrameState *fs, int32_t tiles_x, int32_t tiles_y,
                        int phase, cudaStream_t s);
#ifdef LODGE_VERIFY
// debug builds: order check of the per-tile lists of the last tile sort
void launch_list_verify(const Work &w, FrameState *fs, uint32_t T, bool second, cudaStream_t s,
                        int32_t tiles_x = 0, int32_t tiles_y = 0);
#endif
// phase 0: one pass over the full lists; 1 / 2: the two depth phases of a
// FAST frame (1 saves the state of unfinished tiles, 2 resumes them).
// n_maxw: entries of out.maxw_dev (inputs of the batch / slots of the frame)
void launch_composite(const Work &w, FrameState *fs, const lodge_camera *cam_dev, int32_t W,
                      int32_t H, const lodge_raster_params &rp, int32_t flags, int32_t exact,
                      const lodge_frame_out &out, uint32_t n_maxw, cudaStream_t s,
                      int phase = 0);
void launch_export_lists(const Work &w, FrameState *fs, int32_t T, int64_t *tile_offsets,
                         int64_t *tile_src, int64_t cap, cudaStream_t s);
void launch_frame_report(const int32_t *visible, int64_t n_px, const double *edges_dev,
                         int32_t n_edges, const int32_t *tile_count, int64_t n_tiles,
                         const void *maxw, int32_t maxw_fp64, int64_t n_inputs,
                         unsigned long long *out, cudaStream_t s);
void launch_sq_err(const float *a, const float *b, int64_t n, double *out, cudaStream_t s);
void launch_asset_split(const float *blob, int64_t n, int32_t width, float *geom, float *sh,
                        int32_t *flags_dev, cudaStream_t s);
void launch_asset_sets(const lodge_chunks &ch, const int64_t *level_size_dev, int32_t *flags_dev,
                       cudaStream_t s);
void launch_band_select(const lodge_level *levels, int32_t L, const double *bounds, int32_t full,
                        const LevelSlots &ls, FrameState *fs, const double *pos_dev,
                        uint64_t *status, uint32_t *union_idx, uint8_t *union_tag,
                        cudaStream_t s);
int launch_cover_keys(const lodge_level &level, const int64_t *idx, int64_t n, const Work &w,
                      FrameState *fs, const lodge_camera *cam_dev, const lodge_raster_params &rp,
                      cudaStream_t s);
void launch_cover_table(const Work &w, FrameState *fs, int64_t n_cap, double *dist,
                        int64_t *prefix, int32_t *launches, cudaStream_t s);
}  // namespace lodge
