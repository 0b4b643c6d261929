// K3/K5: tile binning.  Restates reference src/raster.py:409-425:
//   per_tile_count = bincount(tile ids)           (k_tile_setup)
//   duplication of each depth-sorted splat over its tile rectangle,
//   row-major, pairs in global depth order       (k_duplicate)
//   run starts of each tile in the sorted pairs  (tile_start, from counts)
// Counts come from a 2-D difference array filled by K2 (four atomics per
// splat instead of one per pair), integrated here; the duplication kernel
// uses a single-pass look-back scan and block-cooperative emission so one
// huge splat (all 8160 tiles at 1080p) does not serialise a thread.  A
// depth phase of few large splats keeps per-block lists instead of pairs
// (k_block_lists).
#include <algorithm>

#include "emit.cuh"
#include "internal.cuh"

namespace lodge {

#ifndef LODGE_SCAN_MIN_TILES
#define LODGE_SCAN_MIN_TILES 64  // block lists for a first phase whose splats average this many tiles
#endif

// Per-tile list layout from per-tile list counts (one block of 1024
// threads): tile_start (T+1), the two onesweep tile-digit offset tables, the
// heavy-first tile order (tiles with an empty list last; *s_nz = the
// others).  Returns the list total in *s_tot.
template <typename CountFn>
__device__ __forceinline__ void lists_from_counts(CountFn count, int T, uint32_t *tile_start,
                                                  uint32_t *tile_order, FrameState *fs,
                                                  uint32_t *s_sum, uint32_t *h0, uint32_t *h1,
                                                  uint32_t *s_bk, uint32_t *s_tot,
                                                  uint32_t *s_nz) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < 256; i += nt) h0[i] = h1[i] = 0;
  if (tid < 33) s_bk[tid] = 0;
  __syncthreads();
  const int per = (T + nt - 1) / nt;
  const int b = tid * per, e = min(T, b + per);
  uint32_t loc = 0;
  for (int t = b; t < e; ++t) {
    const uint32_t c = count(t);
    loc += c;
    atomicAdd(&h0[t & 255], c);
    atomicAdd(&h1[(t >> 8) & 255], c);
    atomicAdd(&s_bk[c ? 32 - __clz(c) : 0], 1u);
  }
  s_sum[tid] = loc;
  __syncthreads();
  // exclusive scan over threads (Hillis-Steele on 1024 entries)
  for (int o = 1; o < nt; o <<= 1) {
    uint32_t v = (tid >= o) ? s_sum[tid - o] : 0u;
    __syncthreads();
    s_sum[tid] += v;
    __syncthreads();
  }
  uint32_t run = s_sum[tid] - loc;
  for (int t = b; t < e; ++t) {
    tile_start[t] = run;
    run += count(t);
  }
  // composite schedule: tiles by descending log2(count) so the longest lists
  // start first (order affects scheduling only, never results)
  if (tid == 0) {
    uint32_t acc = 0;
    for (int k = 32; k >= 0; --k) {
      const uint32_t v = s_bk[k];
      s_bk[k] = acc;
      if (k == 0) *s_nz = acc;  // tiles with a non-empty list
      acc += v;
    }
  }
  __syncthreads();
  if (tid == nt - 1) {
    *s_tot = s_sum[nt - 1];
    tile_start[T] = s_sum[nt - 1];
  }
  for (int t = b; t < e; ++t) {
    const uint32_t c = count(t);
    tile_order[atomicAdd(&s_bk[c ? 32 - __clz(c) : 0], 1u)] = (uint32_t)t;
  }
  if (tid < 32) {  // digit offsets for the two onesweep passes over tile ids
    for (int p = 0; p < 2; ++p) {
      uint32_t *h = p ? h1 : h0;
      uint32_t acc = 0;
      for (int c = 0; c < 256; c += 32) {
        const uint32_t v = h[c + tid];
        uint32_t inc = v;
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(FULL_MASK, inc, o);
          if (tid >= o) inc += t;
        }
        fs->off_tile[p][c + tid] = acc + inc - v;
        acc += __shfl_sync(FULL_MASK, inc, 31);
      }
    }
  }
  __syncthreads();
}

// 2-D prefix (in place) of an (ty+1) x (tx+1) difference array in shared
// memory: entry (y, x) becomes the count of tile (y, x).
__device__ __forceinline__ void integrate_diff(int32_t *sd, int32_t tiles_x, int32_t tiles_y) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int stride = tiles_x + 1;
  for (int y = tid; y < tiles_y; y += nt) {  // prefix along x
    int32_t run = 0;
    for (int x = 0; x < tiles_x; ++x) {
      run += sd[y * stride + x];
      sd[y * stride + x] = run;
    }
  }
  __syncthreads();
  for (int x = tid; x < tiles_x; x += nt) {  // prefix along y
    int32_t run = 0;
    for (int y = 0; y < tiles_y; ++y) {
      run += sd[y * stride + x];
      sd[y * stride + x] = run;
    }
  }
  __syncthreads();
}

// Block-list capacities (single CTA, after lists_from_counts, which leaves
// s_sum free): out[b] = the exclusive prefix over blocks of the summed
// per-tile counts cnt(t) of block b's tiles, out[nb] = the total.  A block's
// list holds the splats that meet it, each covering >= 1 of its tiles, so its
// length is at most its tiles' count sum.
// The blocks with pairs go to live[] (any order), their number to *nlive:
// the block-list kernel takes work items over those only.
template <typename CountFn>
__device__ void block_offsets(CountFn cnt, int32_t tiles_x, int32_t tiles_y, uint32_t *out,
                              uint32_t *s_sum, uint32_t *live, uint32_t *nlive) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int nbx = (tiles_x + BLK_W - 1) / BLK_W, nb = block_count(tiles_x, tiles_y);
  const int per = (nb + nt - 1) / nt, b0 = tid * per, b1 = min(nb, b0 + per);
  __shared__ uint32_t s_nlive;
  if (tid == 0) s_nlive = 0;
  __syncthreads();
  uint32_t loc = 0;
  for (int b = b0; b < b1; ++b) {
    const int x0 = (b % nbx) * BLK_W, y0 = (b / nbx) * BLK_H;
    uint32_t sum = 0;
    for (int y = y0; y < min(y0 + BLK_H, tiles_y); ++y)
      for (int x = x0; x < min(x0 + BLK_W, tiles_x); ++x) sum += cnt(y * tiles_x + x);
    out[b] = loc;
    loc += sum;
    if (sum) live[atomicAdd(&s_nlive, 1u)] = (uint32_t)b;
  }
  __syncthreads();
  s_sum[tid] = loc;
  __syncthreads();
  for (int o = 1; o < nt; o <<= 1) {
    const uint32_t v = tid >= o ? s_sum[tid - o] : 0u;
    __syncthreads();
    s_sum[tid] += v;
    __syncthreads();
  }
  const uint32_t base = tid ? s_sum[tid - 1] : 0u;
  for (int b = b0; b < b1; ++b) out[b] += base;
  if (tid == nt - 1) out[nb] = s_sum[nt - 1];
  if (tid == 0) *nlive = s_nlive;
  __syncthreads();
}

// Single block.  diff: (ty+1) x (tx+1) over all survivors -> tile_count
// (int32, may be NULL) = per_tile_count, P.  One-phase frames lay the lists
// out from the same counts; two-phase frames (diff_a != NULL) from diff_a,
// the first-phase splats, keeping the full counts in count_all.  Both
// difference arrays are re-zeroed for the next frame; the alive bitmap is
// cleared for the first phase's compositor.
__global__ void __launch_bounds__(1024) k_tile_setup(int32_t *diff, int32_t *diff_a,
                                                     int32_t tiles_x, int32_t tiles_y,
                                                     int32_t *tile_count, uint32_t *count_all,
                                                     uint32_t *alive, uint32_t *tile_start,
                                                     uint32_t *tile_order, FrameState *fs,
                                                     int64_t P_cap, uint32_t *bl_start,
                                                     int32_t bl_mode, uint32_t *bl_live) {
  extern __shared__ int32_t sd[];  // (tx+1)*(ty+1), twice with diff_a
  __shared__ uint32_t h0[256], h1[256];
  __shared__ uint32_t s_sum[1024];
  __shared__ uint32_t s_bk[33];
  __shared__ uint32_t s_tot, s_all, s_nz;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int stride = tiles_x + 1;
  const int nd = stride * (tiles_y + 1);
  int32_t *sa = sd + nd;
  for (int i = tid; i < nd; i += nt) {
    sd[i] = diff[i];
    diff[i] = 0;
    if (diff_a) {
      sa[i] = diff_a[i];
      diff_a[i] = 0;
    }
  }
  const int T = tiles_x * tiles_y;
  if (alive)
    for (int i = tid; i < (T + 31) / 32; i += nt) alive[i] = 0u;
  if (tid == 0) s_all = 0;
  __syncthreads();
  integrate_diff(sd, tiles_x, tiles_y);
  if (diff_a) integrate_diff(sa, tiles_x, tiles_y);
  auto at = [&](const int32_t *a, int t) {
    return (uint32_t)a[(t / tiles_x) * stride + (t % tiles_x)];
  };
  uint32_t all = 0;
  for (int t = tid; t < T; t += nt) {
    const uint32_t c = at(sd, t);
    all += c;
    if (tile_count) tile_count[t] = (int32_t)c;
    if (count_all) count_all[t] = c;
  }
  atomicAdd(&s_all, all);
  const int32_t *lc = diff_a ? sa : sd;
  lists_from_counts([&](int t) { return at(lc, t); }, T, tile_start, tile_order, fs, s_sum, h0,
                    h1, s_bk, &s_tot, &s_nz);
  __syncthreads();
  const uint32_t P = s_all;
  const uint32_t n_pairs = (int64_t)P <= P_cap ? s_tot : 0u;
  // a first phase of few splats with many tiles each (near, large splats)
  // keeps block lists (k_block_lists) instead of emitting and sorting P_A pairs
  const uint32_t S = fs->split_S;
#ifdef LODGE_NO_BLOCK_LISTS
  const bool scan = false;
#else
  const bool scan = diff_a && n_pairs > 0 && S <= (uint32_t)(BL_CHUNK * BL_CHMAX) &&
                    bl_mode != LODGE_BLOCK_LISTS_OFF &&
                    (bl_mode == LODGE_BLOCK_LISTS_FORCE ||
                     (uint64_t)s_tot >= (uint64_t)LODGE_SCAN_MIN_TILES * S);
#endif
  if (scan)
    block_offsets([&](int t) { return at(lc, t); }, tiles_x, tiles_y, bl_start, s_sum, bl_live,
                  &fs->bl_nlive[0]);
  if (tid == 0) {
    fs->stats.P = P;
    fs->stats.overflow = (int64_t)P > P_cap ? 1u : 0u;
    // on overflow nothing is duplicated or sorted (the digit offsets assume
    // all listed pairs); the host grows the buffers and renders the frame again
    fs->n_pairs = n_pairs;
    fs->stats.P_first = s_tot;
    fs->scan_a = scan ? 1u : 0u;
    fs->n_sort_a = scan ? 0u : n_pairs;
    fs->stats.block_lists = scan ? 1u : 0u;
  }
}

// Block lists of a phase with few large splats (fs->scan_a / scan_b): for
// each block of BLK_W x BLK_H tiles, the phase's splats that meet it, in
// depth order, as (tile mask << 32 | splat id) -- bit (y % BLK_H) * BLK_W +
// x % BLK_W set for every tile of the block the splat's rectangle covers.
// A tile's members are exactly the entries with its bit set, in list order:
// the tile's list of the emission + stable tile sort (reference
// src/raster.py:401-425), which the compositor extracts as it goes.
// Phase 1: the depth-ordered splats [0, split_S) (rect_sorted, val_depth[0]);
// phase 2: the owners of k_dup_count<true> (rect_sorted, val_depth[1]), their
// rectangles clipped to the alive tiles (the phase-2 members of an alive
// tile are unchanged by the clip).  Work items are (chunk of BL_CHUNK
// splats, block) in ticket order, chunk-major; a chunk's offset in its
// block's list comes from a decoupled look-back over the block's chunks.
// Blocks without pairs in the phase (zero capacity) are skipped.
constexpr int BL_THREADS = 256;
constexpr int BL_WARPS = BL_THREADS / 32;
constexpr int BL_R = BL_CHUNK / BL_THREADS;
static_assert(BL_R * BL_WARPS == 32, "one warp scans the chunk's (item, warp) counts");
// mask of column 0 in every row of a block (a row's column bits times this
// replicate it down the rows)
__host__ __device__ constexpr uint32_t blk_rep() {
  uint32_t r = 0;
  for (int y = 0; y < BLK_H; ++y) r |= 1u << (BLK_W * y);
  return r;
}

template <int PH>
__global__ void __launch_bounds__(BL_THREADS) k_block_lists(const Work w, FrameState *fs,
                                                            int32_t tiles_x, int32_t tiles_y) {
  __shared__ uint32_t s_cnt[32];
  __shared__ uint32_t s_tk, s_base;
  if (!(PH == 1 ? fs->scan_a : fs->scan_b) || fs->stats.overflow) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t nbx = (tiles_x + BLK_W - 1) / BLK_W, nb = block_count(tiles_x, tiles_y);
  const uint32_t nlive = fs->bl_nlive[PH - 1];  // blocks with pairs in this phase
  const uint32_t *live = w.bl_live + (PH == 1 ? 0 : nb);
  if (nlive == 0) return;
  const uint32_t n = PH == 1 ? fs->split_S : fs->n_owners_b;
  const uint32_t nch = (n + BL_CHUNK - 1) / BL_CHUNK;
  const uint64_t *__restrict__ rect = w.rect_sorted;  // depth order (phase 2: the owners, clipped)
  const uint32_t *__restrict__ ids = PH == 1 ? w.val_depth[0] : w.val_depth[1];
  const uint32_t *bl_start = w.bl_start + (PH == 1 ? 0 : nb + 1);
  uint32_t *bl_len = w.bl_len + (PH == 1 ? 0 : nb);
  uint64_t *blist = w.pairs[PH - 1];
  const int tk = PH == 1 ? TK_BLA : TK_BLB;
  for (;;) {
    if (tid == 0) s_tk = atomicAdd(&fs->tickets[tk], 1u);
    __syncthreads();
    const uint32_t item = s_tk;
    __syncthreads();  // every thread has the ticket before the next is drawn
    const uint32_t c = item / nlive, b = live[item % nlive];
    if (c >= nch || c >= (uint32_t)BL_CHMAX) break;
    const uint32_t cap0 = bl_start[b], cap1 = bl_start[b + 1];
    const uint32_t bx0 = (b % nbx) * BLK_W, by0 = (b / nbx) * BLK_H;
    const uint32_t bx1 = min(bx0 + BLK_W, (uint32_t)tiles_x) - 1,
                   by1 = min(by0 + BLK_H, (uint32_t)tiles_y) - 1;
    // phase 2 counts only the alive tiles: an owner joins a block's list when
    // it covers one of the block's alive tiles (so a list never outgrows its
    // capacity) and carries only those bits
    uint32_t keep = 0xffffffffu;
    if (PH == 2) {
      const uint32_t bx = bx0 + (lane % BLK_W), by = by0 + (lane / BLK_W);
      const uint32_t t = by * tiles_x + bx;
      const bool a = bx <= bx1 && by <= by1 && ((w.alive[t >> 5] >> (t & 31)) & 1u);
      keep = __ballot_sync(FULL_MASK, a);
    }
    uint32_t mask[BL_R];
#pragma unroll
    for (int i = 0; i < BL_R; ++i) {
      const uint32_t r = c * BL_CHUNK + i * BL_THREADS + tid;
      const uint64_t rc = r < n ? rect[r] : 0xffffull;  // x0 = 0xffff: meets nothing
      const uint32_t x0 = rc & 0xffff, x1 = (rc >> 16) & 0xffff, y0 = (rc >> 32) & 0xffff,
                     y1 = rc >> 48;
      uint32_t m = 0;
      if (x0 <= bx1 && x1 >= bx0 && y0 <= by1 && y1 >= by0) {
        const uint32_t cx0 = max(x0, bx0) - bx0, cx1 = min(x1, bx1) - bx0;
        const uint32_t cy0 = max(y0, by0) - by0, cy1 = min(y1, by1) - by0;
        const uint32_t row = (2u << cx1) - (1u << cx0);  // columns cx0..cx1
        const uint32_t rows = (uint32_t)((2ull << (BLK_W * cy1 + BLK_W - 1)) -
                                         (1ull << (BLK_W * cy0)));  // rows cy0..cy1
        m = (row * blk_rep()) & rows & keep;
      }
      mask[i] = m;
      const uint32_t bal = __ballot_sync(FULL_MASK, m != 0u);
      if (lane == 0) s_cnt[i * BL_WARPS + warp] = __popc(bal);
    }
    __syncthreads();
    // exclusive offsets over (item, warp): the depth order within the chunk
    const uint32_t v = s_cnt[lane];
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL_MASK, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t total = __shfl_sync(FULL_MASK, inc, 31);
    const uint32_t ex = inc - v;
    if (warp == 0) {
      const uint32_t pre = lookback_warp(w.status + (size_t)b * BL_CHMAX, c, total,
                                         fs->epoch + tk);
      if (lane == 0) s_base = pre;
    }
    __syncthreads();
    const uint32_t base = cap0 + s_base;
#pragma unroll
    for (int i = 0; i < BL_R; ++i) {
      const bool h = mask[i] != 0u;
      const uint32_t bal = __ballot_sync(FULL_MASK, h);
      const uint32_t off = __shfl_sync(FULL_MASK, ex, i * BL_WARPS + warp);
      if (h) {
        const uint32_t pos = base + off + __popc(bal & lt);
        if (pos < cap1)
          blist[pos] = ((uint64_t)mask[i] << 32) | ids[c * BL_CHUNK + i * BL_THREADS + tid];
        else
          raise_fault(fs, FAULT_LIST);
      }
    }
    if (tid == 0 && c == nch - 1) bl_len[b] = s_base + total;
    __syncthreads();  // s_cnt / s_base reused by the next item
  }
}

// Second phase of a two-phase frame (one block of 1024 threads): list
// counts of the tiles the first phase left unfinished (alive bitmap, written
// by k_composite<phase 1>) = their pairs not in the first phase; their list
// layout and order (tiles without a second-phase list last, n_alive = the
// others), and the summed-area table of the alive tiles the enumeration
// pass queries per splat rectangle.
__global__ void __launch_bounds__(1024) k_setup_b(const uint32_t *__restrict__ alive,
                                                  const uint32_t *__restrict__ count_all,
                                                  const uint32_t *__restrict__ start_a,
                                                  int32_t tiles_x, int32_t tiles_y,
                                                  uint32_t *tile_start, uint32_t *tile_order,
                                                  uint32_t *sat, FrameState *fs,
                                                  uint32_t *bl_start, uint32_t *bl_live) {
  extern __shared__ int32_t ss[];  // (tx+1)*(ty+1) summed-area table
  __shared__ uint32_t h0[256], h1[256];
  __shared__ uint32_t s_sum[1024];
  __shared__ uint32_t s_bk[33];
  __shared__ uint32_t s_tot, s_nz, s_box[4];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int stride = tiles_x + 1;
  const int nd = stride * (tiles_y + 1);
  const int T = tiles_x * tiles_y;
  if (tid == 0) {
    s_box[0] = s_box[2] = 0xffffffffu;
    s_box[1] = s_box[3] = 0u;
  }
  auto live = [&](int t) { return (alive[t >> 5] >> (t & 31)) & 1u; };
  auto cnt = [&](int t) {
    return live(t) ? count_all[t] - (start_a[t + 1] - start_a[t]) : 0u;
  };
  // sat[(y+1)*stride + (x+1)] = alive(y, x), row 0 / column 0 zero, then a
  // 2-D prefix over the whole table
  __syncthreads();
  for (int i = tid; i < nd; i += nt) {
    const int y = i / stride, x = i % stride;
    const bool a = y > 0 && x > 0 && live((y - 1) * tiles_x + (x - 1));
    ss[i] = a ? 1 : 0;
    if (a) {  // bounding box of the alive tiles
      atomicMin(&s_box[0], (uint32_t)(x - 1));
      atomicMax(&s_box[1], (uint32_t)(x - 1));
      atomicMin(&s_box[2], (uint32_t)(y - 1));
      atomicMax(&s_box[3], (uint32_t)(y - 1));
    }
  }
  __syncthreads();
  if (tid < 4) fs->alive_box[tid] = s_box[tid];
  for (int y = tid; y <= tiles_y; y += nt) {
    int32_t run = 0;
    for (int x = 0; x <= tiles_x; ++x) {
      run += ss[y * stride + x];
      ss[y * stride + x] = run;
    }
  }
  __syncthreads();
  for (int x = tid; x <= tiles_x; x += nt) {
    int32_t run = 0;
    for (int y = 0; y <= tiles_y; ++y) {
      run += ss[y * stride + x];
      ss[y * stride + x] = run;
    }
  }
  __syncthreads();
  for (int i = tid; i < nd; i += nt) sat[i] = (uint32_t)ss[i];
#ifdef LODGE_COUNTERS
  {  // counters[7]: alive tiles | blocks of 8 x 4 tiles holding one << 32
    const int bxn = (tiles_x + 7) / 8, byn = (tiles_y + 3) / 4;
    for (int b = tid; b < bxn * byn; b += nt) {
      const int x0 = (b % bxn) * 8, y0 = (b / bxn) * 4;
      const int x1 = min(x0 + 8, tiles_x), y1 = min(y0 + 4, tiles_y);
      const int v = ss[y1 * stride + x1] - ss[y0 * stride + x1] - ss[y1 * stride + x0] +
                    ss[y0 * stride + x0];
      if (v) atomicAdd(&fs->counters[7], (1ull << 32) + (unsigned long long)v);
    }
  }
#endif
  lists_from_counts(cnt, T, tile_start, tile_order, fs, s_sum, h0, h1, s_bk, &s_tot, &s_nz);
  __syncthreads();
  // phase-2 block lists follow the first phase's choice (k_dup_count<true>
  // confirms it once the owners are counted)
  if (fs->scan_a) block_offsets(cnt, tiles_x, tiles_y, bl_start, s_sum, bl_live, &fs->bl_nlive[1]);
  if (tid == 0) {
    fs->n_alive = s_nz;
    fs->n_pairs = fs->stats.overflow ? 0u : s_tot;
    fs->stats.P_second = s_tot;
    fs->scan_b = 0u;
    fs->n_sort_b = fs->n_pairs;
  }
}

constexpr int EMIT_ITEMS = EMIT_CHUNK / DUP_THREADS;
constexpr int COUNT_ITEMS = 8;                        // splats per thread in k_dup_count

// Any alive tile in the rectangle (summed-area table of k_setup_b)?
__device__ __forceinline__ bool rect_alive(const uint32_t *__restrict__ sat, uint64_t rc,
                                           int32_t tiles_x) {
  const uint32_t x0 = rc & 0xffff, x1 = (rc >> 16) & 0xffff, y0 = (rc >> 32) & 0xffff,
                 y1 = rc >> 48;
  const uint32_t st = tiles_x + 1;
  return sat[(y1 + 1) * st + x1 + 1] - sat[y0 * st + x1 + 1] - sat[(y1 + 1) * st + x0] +
             sat[y0 * st + x0] != 0u;
}

// Pass 1, one thread per depth-sorted splat: tile count, exclusive scan of
// the counts in depth order (single-pass look-back), the splat's rectangle
// and id in depth order, and for every EMIT_CHUNK boundary inside the
// splat's pair range the splat that owns it (the emission CTAs' splitters).
// Two-phase frames: budget > 0 makes the splats whose pairs start before it
// the first phase (their rectangles go to the tile_diff_a difference array;
// split_S and P_A record the split; the splats are the depth-sorted
// first-phase candidates, *n_ptr of them).  SECOND: the second phase's
// owners -- the depth-sorted output of launch_owner_filter, which kept the
// later splats that meet an alive tile -- with their rectangles clipped to
// the alive tiles' bounding box (into rect_sorted), pair offsets and
// splitters over that list (the same clip and alive test re-run: every
// owner passes, so the compaction is the identity).
template <bool SECOND>
__global__ void __launch_bounds__(DUP_THREADS) k_dup_count(const uint32_t *__restrict__ order,
                                                           const uint64_t *__restrict__ rect,
                                                           Work w, FrameState *fs,
                                                           uint32_t budget, int32_t tiles_x,
                                                           uint32_t chunk_cap, int32_t tiles_y,
                                                           int32_t diff_smem,
                                                           const uint32_t *n_ptr) {
  // first phase: the CTAs holding first-phase splats add their rectangles to
  // a CTA-private difference array (dynamic shared memory, when it fits),
  // flushed once -- the few CTAs at the front of the depth order otherwise
  // serialise on global atomics at the shared border corners
  extern __shared__ int32_t s_da[];
  constexpr int IT = COUNT_ITEMS;  // consecutive depth-order splats per thread
  constexpr int TK = SECOND ? TK_DUPB : TK_DUP;
  __shared__ uint32_t s_w[DUP_THREADS / 32], s_z[DUP_THREADS / 32];
  __shared__ uint32_t s_part, s_base, s_zbase;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t n = SECOND ? (fs->stats.overflow ? 0u : fs->n_ocand) : *n_ptr;
  // the grid is sized for the capacity: CTAs beyond the partitions leave
  // before drawing a ticket (the others draw 0 .. partitions - 1)
  if ((uint64_t)blockIdx.x * (DUP_THREADS * IT) >= n) return;
  if (tid == 0) s_part = atomicAdd(&fs->tickets[TK], 1u);
  __syncthreads();
  const uint32_t part = s_part;
  const uint32_t r0 = part * (DUP_THREADS * IT) + tid * IT;
  if (part * (DUP_THREADS * IT) >= n) return;
  uint32_t c[IT];
  uint64_t rc[IT];
  {
    uint32_t m[IT];
    if (r0 + IT <= n) {  // order is 16-byte aligned and r0 a multiple of IT
#pragma unroll
      for (int q = 0; q < IT / 4; ++q) {
        const uint4 o4 = *reinterpret_cast<const uint4 *>(order + r0 + 4 * q);
        m[4 * q] = o4.x; m[4 * q + 1] = o4.y; m[4 * q + 2] = o4.z; m[4 * q + 3] = o4.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < IT; ++i) m[i] = (r0 + i < n) ? order[r0 + i] : 0u;
    }
#pragma unroll
    for (int i = 0; i < IT; ++i) rc[i] = (r0 + i < n) ? rect[m[i]] : 0ull;
  }
  uint32_t cnt = 0, nz = 0;
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const uint32_t x0 = rc[i] & 0xffff, x1 = (rc[i] >> 16) & 0xffff, y0 = (rc[i] >> 32) & 0xffff,
                   y1 = rc[i] >> 48;
    c[i] = (r0 + i < n) ? (x1 - x0 + 1) * (y1 - y0 + 1) : 0u;
    if (SECOND && c[i]) {  // clip to the alive tiles' bounding box (all else is dead)
      const uint32_t cx0 = max(x0, fs->alive_box[0]), cx1 = min(x1, fs->alive_box[1]);
      const uint32_t cy0 = max(y0, fs->alive_box[2]), cy1 = min(y1, fs->alive_box[3]);
      rc[i] = (uint64_t)cx0 | ((uint64_t)cx1 << 16) | ((uint64_t)cy0 << 32) |
              ((uint64_t)cy1 << 48);
      c[i] = (cx0 <= cx1 && cy0 <= cy1 && rect_alive(w.sat, rc[i], tiles_x))
                 ? (cx1 - cx0 + 1) * (cy1 - cy0 + 1)
                 : 0u;
    }
    cnt += c[i];
    nz += c[i] ? 1u : 0u;
    if (!SECOND && r0 + i < n) w.rect_sorted[r0 + i] = rc[i];
  }
  uint32_t inc = cnt, zinc = nz;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(FULL_MASK, inc, o);
    if (lane >= o) inc += t;
    if (SECOND) {
      const uint32_t tz = __shfl_up_sync(FULL_MASK, zinc, o);
      if (lane >= o) zinc += tz;
    }
  }
  if (lane == 31) {
    s_w[warp] = inc;
    s_z[warp] = zinc;
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t wv = lane < DUP_THREADS / 32 ? s_w[lane] : 0u;
    uint32_t winc = wv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL_MASK, winc, o);
      if (lane >= o) winc += t;
    }
    const uint32_t total = __shfl_sync(FULL_MASK, winc, 31);
    if (lane < DUP_THREADS / 32) s_w[lane] = winc - wv;
    const uint32_t pre = lookback_warp(w.status, part, total, fs->epoch + TK);
    if (lane == 0) s_base = pre;
  } else if (SECOND && warp == 1) {  // the owner compaction's look-back
    const uint32_t zv = lane < DUP_THREADS / 32 ? s_z[lane] : 0u;
    uint32_t zi = zv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL_MASK, zi, o);
      if (lane >= o) zi += t;
    }
    const uint32_t total = __shfl_sync(FULL_MASK, zi, 31);
    if (lane < DUP_THREADS / 32) s_z[lane] = zi - zv;
    const uint32_t pre =
        lookback_warp(w.status + (w.status_cap >> 1), part, total, fs->epoch + TK);
    if (lane == 0) s_zbase = pre;
  }
  __syncthreads();
  const int32_t nd = (tiles_x + 1) * (tiles_y + 1);
  const bool fa = !SECOND && budget && diff_smem && s_base < budget;  // CTA-uniform
  if (fa) {
    for (int32_t q = tid; q < nd; q += DUP_THREADS) s_da[q] = 0;
    __syncthreads();
  }
  uint32_t off = s_base + s_w[warp] + inc - cnt;
  uint32_t k = SECOND ? s_zbase + s_z[warp] + zinc - nz : 0u;  // owner index
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const uint32_t r = r0 + i;
    const bool valid = r < n;
    // first phase: every splat owns its pairs; second: the splats with pairs
    const bool own = valid && (!SECOND || c[i] > 0);
    const uint32_t q = SECOND ? k : r;
    if (own) {
      w.splat_off[q] = off;
      if (SECOND) w.rect_sorted[q] = rc[i];  // (order is already the owner list)
      for (uint32_t kk = (off + EMIT_CHUNK - 1) / EMIT_CHUNK;
           kk * EMIT_CHUNK < off + c[i] && kk < chunk_cap; ++kk)
        w.chunk_first[kk] = q;
    }
    if (valid && r == n - 1) {  // totals: owners and pairs
      const uint32_t nq = SECOND ? k + (c[i] ? 1u : 0u) : n;
      w.splat_off[nq] = off + c[i];
      if (!SECOND) fs->stats.sorted_first = n;
      if (SECOND) {
        fs->n_owners_b = nq;
        fs->stats.M_second = nq;
        // block lists for the second phase too when its owners fit the chunk
        // table (else its pairs are emitted and sorted)
        const bool sb = fs->scan_a && nq <= (uint32_t)(BL_CHUNK * BL_CHMAX);
        fs->scan_b = sb ? 1u : 0u;
        fs->n_sort_b = sb ? 0u : fs->n_pairs;
        if (sb) fs->stats.block_lists |= 2u;
      }
    }
    if (!SECOND && budget) {  // whole warp: the difference-array update is collective
      const bool first = valid && off < budget;
      if (fa) add_tile_diff_shared(s_da, rc[i], tiles_x, tiles_y, first);
      else add_tile_diff(w.tile_diff_a, rc[i], tiles_x, first);
      if (first && (off + c[i] >= budget || r == n - 1)) {
        fs->split_S = r + 1;
        fs->stats.M_first = r + 1;
        fs->P_A = off + c[i];
        const uint32_t g = order[r];  // the last first-phase splat (launch_owner_filter)
        const uint64_t fk = w.key_depth[0][g];
        fs->p1_g = g;
        fs->p1_key = fk;
        fs->p1_k32 = __float_as_uint(__double2float_rz(__longlong_as_double((long long)fk)));
      }
    }
    if (valid) {
      off += c[i];
      if (SECOND && c[i]) ++k;
    }
  }
  if (fa) {
    __syncthreads();
    for (int32_t q = tid; q < nd; q += DUP_THREADS) {
      const int32_t v = s_da[q];
      if (v) atomicAdd(w.tile_diff_a + q, v);
    }
  }
}

// Pass 2, EMIT_CHUNK pairs per CTA regardless of splat sizes (emit.cuh),
// written (tile << 32 | splat) coalesced, in depth order (the tile passes in
// k_sort.cu then sort them stably by tile).
// first_phase: the pairs [0, P_A) of a two-phase frame, owned by the
// splats [0, split_S).
__global__ void __launch_bounds__(DUP_THREADS) k_dup_emit(const uint32_t *__restrict__ order,
                                                          int32_t tiles_x, Work w,
                                                          FrameState *fs, int32_t first_phase) {
  __shared__ EmitSmem<EMIT_CHUNK> E;
  const uint32_t P = first_phase ? fs->n_sort_a : fs->n_pairs;
  const uint32_t n_own = first_phase ? fs->split_S : fs->stats.M;
  // persistent CTAs, grid-stride over the chunks
  for (uint32_t c = blockIdx.x; c * EMIT_CHUNK < P; c += gridDim.x) {
    const uint32_t j0 = c * EMIT_CHUNK;
    const uint32_t j1 = min(j0 + (uint32_t)EMIT_CHUNK, P);
    uint32_t r0, r1;
    emit_owners(w, j0, j1, P, n_own, r0, r1);
    emit_stage(E, order, w, j0, j1, r0, r1, fs);
#pragma unroll
    for (int it = 0; it < EMIT_ITEMS; ++it) {
      const uint32_t j = j0 + it * DUP_THREADS + threadIdx.x;
      if (j >= j1) break;
      w.pairs[0][j] = emit_pair(E, j, j0, tiles_x);
    }
    __syncthreads();  // the next chunk restages E
  }
}

// Second phase of a two-phase frame: the enumerated pairs of the owner list
// of k_dup_count<true> (EB_CHUNK per CTA step, as k_dup_emit), keeping those whose tile
// is alive, compacted in order (block scan + decoupled look-back over CTAs
// taken in ticket order), so each alive tile receives, in depth order, its
// pairs beyond the first phase.
#ifndef LODGE_EMITB_CHUNK
#define LODGE_EMITB_CHUNK 4096  // enumerated pairs per CTA step (a multiple of EMIT_CHUNK)
#endif
constexpr int EB_CHUNK = LODGE_EMITB_CHUNK;
constexpr int EB_ITEMS = EB_CHUNK / DUP_THREADS;
static_assert(EB_CHUNK % EMIT_CHUNK == 0 && EB_ITEMS <= 32, "whole splitter chunks, <= 32 rounds");

__global__ void __launch_bounds__(DUP_THREADS) k_emit_b(const uint32_t *__restrict__ order,
                                                        int32_t tiles_x, int32_t n_tiles,
                                                        Work w, FrameState *fs) {
  extern __shared__ __align__(16) uint8_t eb_smem[];
  EmitSmem<EB_CHUNK> &E = *reinterpret_cast<EmitSmem<EB_CHUNK> *>(eb_smem);
  __shared__ uint32_t s_alive[2048];  // T <= 65536 (check_tile_smem)
  __shared__ uint32_t s_cnt[EB_ITEMS][DUP_THREADS / 32];
  __shared__ uint32_t s_part, s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t n = (fs->stats.overflow || fs->scan_b) ? 0u : fs->n_owners_b;
  const uint32_t Pe = n ? w.splat_off[n] : 0u;  // enumerated pairs
  if (Pe == 0) return;  // (block lists: no pairs)
  for (int i = tid; i < (n_tiles + 31) / 32; i += DUP_THREADS) s_alive[i] = w.alive[i];
  // persistent CTAs: chunks in ticket order (the compaction's look-back)
  for (;;) {
  if (tid == 0) s_part = atomicAdd(&fs->tickets[TK_EMITB], 1u);
  __syncthreads();
  const uint32_t part = s_part;
  const uint32_t j0 = part * EB_CHUNK;
  if (j0 >= Pe) break;
  const uint32_t j1 = min(j0 + (uint32_t)EB_CHUNK, Pe);
  uint32_t r0, r1;
  emit_owners(w, j0, j1, Pe, n, r0, r1);
  // the owner list of k_dup_count<true>: ids in val_depth[1], clipped
  // rectangles in rect_sorted
  emit_stage(E, w.val_depth[1], w, j0, j1, r0, r1, fs);  // ends with a barrier
  uint64_t key[EB_ITEMS];
  uint32_t keep = 0;
#pragma unroll
  for (int it = 0; it < EB_ITEMS; ++it) {
    const uint32_t j = j0 + it * DUP_THREADS + tid;
    key[it] = j < j1 ? emit_pair(E, j, j0, tiles_x) : 0ull;
    uint32_t t = (uint32_t)(key[it] >> 32);
    if (t >= (uint32_t)n_tiles) {
      raise_fault(fs, FAULT_TILE);
      t = 0;
    }
    const bool k = j < j1 && ((s_alive[t >> 5] >> (t & 31)) & 1u);
    keep |= k ? (1u << it) : 0u;
    const uint32_t bal = __ballot_sync(FULL_MASK, k);
    if (lane == 0) s_cnt[it][warp] = __popc(bal);
  }
  __syncthreads();
  if (warp == 0) {  // exclusive offsets over (round, warp), then the look-back
    uint32_t v[EB_ITEMS], tot = 0;
#pragma unroll
    for (int it = 0; it < EB_ITEMS; ++it) {
      v[it] = lane < DUP_THREADS / 32 ? s_cnt[it][lane] : 0u;
      uint32_t inc = v[it];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL_MASK, inc, o);
        if (lane >= o) inc += t;
      }
      if (lane < DUP_THREADS / 32) s_cnt[it][lane] = tot + inc - v[it];
      tot += __shfl_sync(FULL_MASK, inc, 31);
    }
    const uint32_t pre = lookback_warp(w.status, part, tot, fs->epoch + TK_EMITB);
    if (lane == 0) s_base = pre;
  }
  __syncthreads();
  const uint32_t base = s_base;
  const uint32_t limit = fs->n_pairs;  // the second phase's pair total (k_setup_b)
#pragma unroll
  for (int it = 0; it < EB_ITEMS; ++it) {
    const uint32_t bal = __ballot_sync(FULL_MASK, (keep >> it) & 1u);
    if ((keep >> it) & 1u) {
      const uint32_t o = base + s_cnt[it][warp] + __popc(bal & lanemask_lt());
      if (o < limit) w.pairs[0][o] = key[it];
      else raise_fault(fs, FAULT_COMPACT);
    }
  }
  __syncthreads();  // the next chunk restages E and the counters
  }
}

// ---- two-phase frames: sort only what is composited ------
// The first phase is the depth-order prefix of the survivors whose pair
// ranges start before `budget`; a survivor in depth bin b (the top 16 bits of
// its 32-bit key, monotone in the depth) starts at or after the pairs of all
// earlier bins, so only the bins whose preceding bins hold fewer than
// `budget` pairs can contribute: those survivors are the candidates, sorted
// and counted instead of all M.  The second phase's owners are found among
// the survivors after the first phase's last splat directly (the alive-tile
// test of k_dup_count<true>), then sorted.
constexpr int SEL_ITEMS = 8;  // survivors per thread and CTA step (compaction kernels)

// pairs per depth bin: a CTA-private histogram in shared memory, flushed
// once (global atomics on the few bins that hold most survivors serialised)
__global__ void __launch_bounds__(256) k_sel_hist(const Work w, const FrameState *fs) {
  __shared__ uint32_t h[SEL_BINS];
  for (int i = threadIdx.x; i < SEL_BINS; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint32_t M = fs->stats.M;
  const uint32_t *__restrict__ keys = depth_keys_compact(w);
  const uint32_t *__restrict__ ids = w.val_depth[1];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
    const uint64_t rc = w.rect[ids[i]];
    const uint32_t x0 = rc & 0xffff, x1 = (rc >> 16) & 0xffff, y0 = (rc >> 32) & 0xffff,
                   y1 = rc >> 48;
    atomicAdd(&h[keys[i] >> SEL_SHIFT], (x1 - x0 + 1) * (y1 - y0 + 1));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < SEL_BINS; i += blockDim.x)
    if (h[i]) atomicAdd(&w.sel_hist[i], h[i]);
}

// one CTA: the last bin whose preceding bins hold fewer than `budget` pairs
// (every bin when the total stays below it); the bins are re-zeroed
__global__ void __launch_bounds__(1024) k_sel_scan(const Work w, FrameState *fs,
                                                   uint32_t budget) {
  constexpr int PER = SEL_BINS / 1024;
  static_assert(PER % 4 == 0, "vector loads of the bins");
  __shared__ uint32_t s_sum[1024];
  __shared__ uint32_t s_B;
  const int tid = threadIdx.x;
  uint32_t *h = w.sel_hist + tid * PER;
  uint32_t v[PER];
  uint32_t loc = 0;
#pragma unroll
  for (int q = 0; q < PER / 4; ++q) {
    const uint4 u = reinterpret_cast<const uint4 *>(h)[q];
    v[4 * q] = u.x; v[4 * q + 1] = u.y; v[4 * q + 2] = u.z; v[4 * q + 3] = u.w;
    loc += (u.x + u.y) + (u.z + u.w);
    reinterpret_cast<uint4 *>(h)[q] = make_uint4(0u, 0u, 0u, 0u);
  }
  if (tid == 0) s_B = 0;
  s_sum[tid] = loc;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const uint32_t t = tid >= o ? s_sum[tid - o] : 0u;
    __syncthreads();
    s_sum[tid] += t;
    __syncthreads();
  }
  uint32_t cum = tid ? s_sum[tid - 1] : 0u;  // pairs of the bins before this thread's
  int last = -1;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    if (cum < budget) last = tid * PER + q;
    cum += v[q];
  }
  if (last >= 0) atomicMax(&s_B, (uint32_t)last);
  __syncthreads();
  if (tid == 0) fs->sel_B = s_B;
}

// CTA-aggregated append of the flagged survivors (32-bit key, input index)
// into sel_keys / sel_vals at *count (the order is free: they are sorted)
template <typename Keep>
__device__ __forceinline__ void sel_compact(const Work &w, uint32_t M, uint32_t *count,
                                            Keep keep) {
  __shared__ uint32_t s_w[8], s_base;
  const uint32_t *__restrict__ keys = depth_keys_compact(w);
  const uint32_t *__restrict__ ids = w.val_depth[1];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr uint32_t STEP = 256 * SEL_ITEMS;
  for (uint32_t b = blockIdx.x * STEP; b < M; b += gridDim.x * STEP) {
    uint32_t k[SEL_ITEMS], g[SEL_ITEMS], m = 0;
#pragma unroll
    for (int it = 0; it < SEL_ITEMS; ++it) {
      const uint32_t i = b + it * 256 + tid;
      k[it] = i < M ? keys[i] : 0u;
      g[it] = i < M ? ids[i] : 0u;
      if (i < M && keep(k[it], g[it])) m |= 1u << it;
    }
    const uint32_t cnt = __popc(m);
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL_MASK, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (tid == 0) {
      uint32_t tot = 0;
      for (int q = 0; q < 8; ++q) {
        const uint32_t v = s_w[q];
        s_w[q] = tot;
        tot += v;
      }
      s_base = tot ? atomicAdd(count, tot) : 0u;
    }
    __syncthreads();
    uint32_t at = s_base + s_w[warp] + inc - cnt;
#pragma unroll
    for (int it = 0; it < SEL_ITEMS; ++it)
      if ((m >> it) & 1u) {
        if (at < (uint32_t)w.M_cap) {
          w.sel_keys[at] = k[it];
          w.sel_vals[at] = g[it];
        }
        ++at;
      }
    __syncthreads();  // s_w / s_base reused
  }
}

__global__ void __launch_bounds__(256) k_sel_compact(const Work w, FrameState *fs) {
  const uint32_t B = fs->sel_B;
  sel_compact(w, fs->stats.M, &fs->n_cand,
              [&](uint32_t k, uint32_t) { return (k >> SEL_SHIFT) <= B; });
}

// the second phase's owners: survivors after the first phase's last splat in
// (fp64 depth, index) order whose rectangle, clipped to the alive tiles'
// bounding box, contains an alive tile
__global__ void __launch_bounds__(256) k_owner_filter(const Work w, FrameState *fs,
                                                      int32_t tiles_x) {
  if (fs->stats.overflow) return;
  const uint32_t S = fs->split_S;
  const uint64_t bkey = fs->p1_key;
  const uint32_t bg = fs->p1_g, bk32 = fs->p1_k32;
  const uint32_t ax0 = fs->alive_box[0], ax1 = fs->alive_box[1], ay0 = fs->alive_box[2],
                 ay1 = fs->alive_box[3];
  sel_compact(w, fs->stats.M, &fs->n_ocand, [&](uint32_t k32, uint32_t g) {
    if (S > 0) {  // the 32-bit key is monotone in the fp64 one: the full key only on a tie
      if (k32 < bk32) return false;  // a first-phase splat
      if (k32 == bk32) {
        const uint64_t fk = w.key_depth[0][g];
        if (fk < bkey || (fk == bkey && g <= bg)) return false;
      }
    }
    const uint64_t rc = w.rect[g];
    const uint32_t x0 = max((uint32_t)(rc & 0xffff), ax0), x1 = min((uint32_t)((rc >> 16) & 0xffff), ax1);
    const uint32_t y0 = max((uint32_t)((rc >> 32) & 0xffff), ay0), y1 = min((uint32_t)(rc >> 48), ay1);
    if (x0 > x1 || y0 > y1) return false;
    const uint64_t cr = (uint64_t)x0 | ((uint64_t)x1 << 16) | ((uint64_t)y0 << 32) |
                        ((uint64_t)y1 << 48);
    return rect_alive(w.sat, cr, tiles_x);
  });
}

static unsigned sel_grid(int64_t M_cap) {
  return (unsigned)std::max<int64_t>(
      1, std::min<int64_t>((M_cap + 256 * SEL_ITEMS - 1) / (256 * SEL_ITEMS), 148 * 8));
}

void launch_depth_select(const Work &w, FrameState *fs, int64_t M_cap, uint32_t budget,
                         cudaStream_t s) {
  if (M_cap <= 0) return;
  const unsigned hgrid = (unsigned)std::min<int64_t>((M_cap + 4095) / 4096, 148 * 2);
  k_sel_hist<<<hgrid, 256, 0, s>>>(w, fs);
  k_sel_scan<<<1, 1024, 0, s>>>(w, fs, budget);
  k_sel_compact<<<sel_grid(M_cap), 256, 0, s>>>(w, fs);
}

void launch_owner_filter(const Work &w, FrameState *fs, int32_t tiles_x, int64_t M_cap,
                         cudaStream_t s) {
  if (M_cap <= 0) return;
  k_owner_filter<<<sel_grid(M_cap), 256, 0, s>>>(w, fs, tiles_x);
}

void launch_tile_setup(const Work &w, FrameState *fs, int32_t *tile_count, int32_t tiles_x,
                       int32_t tiles_y, cudaStream_t s, bool two_phase, int32_t bl_mode) {
  const size_t nd = (size_t)(tiles_x + 1) * (tiles_y + 1) * 4;
  const size_t sm = two_phase ? 2 * nd : nd;
  static PerDevice attr;
  if (sm > 48 * 1024 && (int64_t)sm > attr()) {
    cudaFuncSetAttribute(k_tile_setup, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr() = (int64_t)sm;
  }
  k_tile_setup<<<1, 1024, sm, s>>>(w.tile_diff, two_phase ? w.tile_diff_a : nullptr, tiles_x,
                                   tiles_y, tile_count, two_phase ? w.count_all : nullptr,
                                   two_phase ? w.alive : nullptr, w.tile_start, w.tile_order, fs,
                                   w.P_cap, w.bl_start, bl_mode, w.bl_live);
}

static uint32_t chunk_cap(const Work &w) { return (uint32_t)(w.P_cap / EMIT_CHUNK + 4); }

constexpr size_t DUP_DIFF_SMEM_MAX = 64 * 1024;  // CTA-private first-phase difference array
void launch_dup_count(const Work &w, FrameState *fs, int32_t tiles_x, int32_t tiles_y,
                      int64_t M_cap, uint32_t budget, cudaStream_t s, const uint32_t *n_ptr) {
  if (M_cap <= 0) return;
  const unsigned grid =
      (unsigned)((M_cap + DUP_THREADS * COUNT_ITEMS - 1) / (DUP_THREADS * COUNT_ITEMS));
  const size_t sm = (size_t)(tiles_x + 1) * (tiles_y + 1) * 4;
  const bool priv = budget && sm <= DUP_DIFF_SMEM_MAX;
  static PerDevice attr;
  if (priv && sm > 48 * 1024 && (int64_t)sm > attr()) {
    cudaFuncSetAttribute(k_dup_count<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr() = (int64_t)sm;
  }
  k_dup_count<false><<<grid, DUP_THREADS, priv ? sm : 0, s>>>(
      w.val_depth[0], w.rect, w, fs, budget, tiles_x, chunk_cap(w), tiles_y, priv ? 1 : 0,
      n_ptr ? n_ptr : &fs->stats.M);
}

// Resident CTAs of a kernel on this device (persistent grids).
template <typename K>
static int64_t resident_ctas(K kernel, int threads) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, 0);
  per = std::min(per, LODGE_PERSIST_PER);
  return (int64_t)std::max(per, 1) * std::max(sms, 1);
}

void launch_dup_emit(const Work &w, FrameState *fs, int32_t tiles_x, cudaStream_t s,
                     bool first_phase) {
  static PerDevice res;
  if (!res()) res() = resident_ctas(k_dup_emit, DUP_THREADS);
  const int64_t resident = res();
#ifndef LODGE_PERSIST
#define LODGE_PERSIST 1
#endif
  const unsigned egrid = (unsigned)std::min<int64_t>((w.P_cap + EMIT_CHUNK - 1) / EMIT_CHUNK,
                                                     LODGE_PERSIST ? resident : 0x7fffffff);
  k_dup_emit<<<egrid, DUP_THREADS, 0, s>>>(w.val_depth[0], tiles_x, w, fs, first_phase ? 1 : 0);
}

void launch_duplicate(const Work &w, FrameState *fs, int32_t tiles_x, int64_t M_cap,
                      cudaStream_t s) {
  if (M_cap <= 0) return;
  launch_dup_count(w, fs, tiles_x, 0, M_cap, 0u, s);  // one pass: no first-phase array
  launch_dup_emit(w, fs, tiles_x, s, false);
}

void launch_block_lists(const Work &w, FrameState *fs, int32_t tiles_x, int32_t tiles_y,
                        int phase, cudaStream_t s) {
  static PerDevice res;
  if (!res()) res() = resident_ctas(k_block_lists<1>, BL_THREADS);
  const int64_t items = (int64_t)block_count(tiles_x, tiles_y) * BL_CHMAX;
  const unsigned grid = (unsigned)std::min<int64_t>(items, res());
  if (phase == 1) k_block_lists<1><<<grid, BL_THREADS, 0, s>>>(w, fs, tiles_x, tiles_y);
  else k_block_lists<2><<<grid, BL_THREADS, 0, s>>>(w, fs, tiles_x, tiles_y);
}

void launch_setup_b(const Work &w, FrameState *fs, int32_t tiles_x, int32_t tiles_y,
                    cudaStream_t s) {
  const size_t sm = (size_t)(tiles_x + 1) * (tiles_y + 1) * 4;
  static PerDevice attr;
  if (sm > 48 * 1024 && (int64_t)sm > attr()) {
    cudaFuncSetAttribute(k_setup_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr() = (int64_t)sm;
  }
  k_setup_b<<<1, 1024, sm, s>>>(w.alive, w.count_all, w.tile_start, tiles_x, tiles_y,
                                w.tile_start_b, w.tile_order_b, w.sat, fs,
                                w.bl_start + block_count(tiles_x, tiles_y) + 1,
                                w.bl_live + block_count(tiles_x, tiles_y));
}

void launch_enum_b(const Work &w, FrameState *fs, int32_t tiles_x, int32_t tiles_y,
                   int64_t M_cap, cudaStream_t s) {
  if (M_cap <= 0) return;
  const unsigned grid =
      (unsigned)((M_cap + DUP_THREADS * COUNT_ITEMS - 1) / (DUP_THREADS * COUNT_ITEMS));
  // the owners, depth-sorted by launch_owner_filter + launch_subset_sort
  k_dup_count<true><<<grid, DUP_THREADS, 0, s>>>(w.val_depth[1], w.rect, w, fs, 0u, tiles_x,
                                                 chunk_cap(w), tiles_y, 0, nullptr);
  static PerDevice res;
  constexpr size_t sm = sizeof(EmitSmem<EB_CHUNK>);
  if (!res()) {
    cudaFuncSetAttribute(k_emit_b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_emit_b, DUP_THREADS, sm);
    per = std::min(per, LODGE_PERSIST_PER);
    res() = (int64_t)std::max(per, 1) * std::max(sms, 1);
  }
  const int64_t resident = res();
  const unsigned egrid =
      (unsigned)std::min<int64_t>((w.P_cap + EB_CHUNK - 1) / EB_CHUNK, resident);
  k_emit_b<<<egrid, DUP_THREADS, sm, s>>>(w.val_depth[0], tiles_x, tiles_x * tiles_y, w, fs);
}

}  // namespace lodge
