// K3/K5: tile binning.  Restates reference src/raster.py:409-425:
//   per_tile_count = bincount(tile ids)           (k_tile_setup)
//   duplication of each depth-sorted splat over its tile rectangle,
//   row-major, pairs in global depth order       (k_duplicate)
//   run starts of each tile in the sorted pairs  (tile_start, from counts)
// Counts come from a 2-D difference array filled by K2 (four atomics per
// splat instead of one per pair), integrated here; the duplication kernel
// uses a single-pass look-back scan and block-cooperative emission so one
// huge splat (all 8160 tiles at 1080p) does not serialise a thread.
#include "emit.cuh"
#include "internal.cuh"

namespace lodge {

// Single block.  diff: (ty+1) x (tx+1).  Produces tile_count (int32, may be
// NULL), tile_start (T+1), the two tile-digit offset tables, P, n_pairs, and
// re-zeroes diff for the next frame.
__global__ void __launch_bounds__(1024) k_tile_setup(int32_t *diff, int32_t tiles_x,
                                                     int32_t tiles_y, int32_t *tile_count,
                                                     uint32_t *tile_start, uint32_t *tile_order,
                                                     FrameState *fs, int64_t P_cap) {
  extern __shared__ int32_t sd[];  // (tx+1)*(ty+1)
  __shared__ uint32_t h0[256], h1[256];
  __shared__ uint32_t s_sum[1024];
  __shared__ uint32_t s_bk[33];
  const int tid = threadIdx.x, nt = blockDim.x;
  const int stride = tiles_x + 1;
  const int nd = stride * (tiles_y + 1);
  for (int i = tid; i < nd; i += nt) {
    sd[i] = diff[i];
    diff[i] = 0;
  }
  for (int i = tid; i < 256; i += nt) h0[i] = h1[i] = 0;
  __syncthreads();
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
  const int T = tiles_x * tiles_y;
  const int per = (T + nt - 1) / nt;
  const int b = tid * per, e = min(T, b + per);
  uint32_t loc = 0;
  for (int t = b; t < e; ++t) {
    const uint32_t c = (uint32_t)sd[(t / tiles_x) * stride + (t % tiles_x)];
    loc += c;
    if (tile_count) tile_count[t] = (int32_t)c;
    atomicAdd(&h0[t & 255], c);
    atomicAdd(&h1[(t >> 8) & 255], c);
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
    run += (uint32_t)sd[(t / tiles_x) * stride + (t % tiles_x)];
  }
  // composite schedule: tiles by descending log2(count) so the longest lists
  // start first (order affects scheduling only, never results)
  if (tid < 33) s_bk[tid] = 0;
  __syncthreads();
  for (int t = b; t < e; ++t) {
    const uint32_t c = (uint32_t)sd[(t / tiles_x) * stride + (t % tiles_x)];
    atomicAdd(&s_bk[c ? 32 - __clz(c) : 0], 1u);
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t acc = 0;
    for (int k = 32; k >= 0; --k) {
      const uint32_t v = s_bk[k];
      s_bk[k] = acc;
      acc += v;
    }
  }
  __syncthreads();
  for (int t = b; t < e; ++t) {
    const uint32_t c = (uint32_t)sd[(t / tiles_x) * stride + (t % tiles_x)];
    tile_order[atomicAdd(&s_bk[c ? 32 - __clz(c) : 0], 1u)] = (uint32_t)t;
  }
  if (tid == nt - 1) {
    const uint32_t P = s_sum[nt - 1];
    tile_start[T] = P;
    fs->stats.P = P;
    fs->stats.overflow = (int64_t)P > P_cap ? 1u : 0u;
    // on overflow nothing is duplicated or sorted (the digit offsets assume
    // all P pairs); the host grows the buffers and renders the frame again
    fs->n_pairs = (int64_t)P <= P_cap ? P : 0u;
  }
  __syncthreads();
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
}

constexpr int EMIT_ITEMS = EMIT_CHUNK / DUP_THREADS;
constexpr int COUNT_ITEMS = 8;                        // splats per thread in k_dup_count

// Pass 1, one thread per depth-sorted splat: tile count, exclusive scan of
// the counts in depth order (single-pass look-back), the splat's rectangle
// and id in depth order, and for every EMIT_CHUNK boundary inside the
// splat's pair range the splat that owns it (the emission CTAs' splitters).
__global__ void __launch_bounds__(DUP_THREADS) k_dup_count(const uint32_t *__restrict__ order,
                                                           const uint64_t *__restrict__ rect,
                                                           Work w, FrameState *fs) {
  constexpr int IT = COUNT_ITEMS;  // consecutive depth-order splats per thread
  __shared__ uint32_t s_w[DUP_THREADS / 32];
  __shared__ uint32_t s_part, s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_part = atomicAdd(&fs->tickets[TK_DUP], 1u);
  __syncthreads();
  const uint32_t part = s_part;
  const uint32_t M = fs->stats.overflow ? 0u : fs->stats.M;
  const uint32_t r0 = part * (DUP_THREADS * IT) + tid * IT;
  if (part * (DUP_THREADS * IT) >= M) return;
  uint32_t m[IT], c[IT];
  uint64_t rc[IT];
  if (r0 + IT <= M) {  // order is 16-byte aligned and r0 a multiple of IT
#pragma unroll
    for (int q = 0; q < IT / 4; ++q) {
      const uint4 o4 = *reinterpret_cast<const uint4 *>(order + r0 + 4 * q);
      m[4 * q] = o4.x; m[4 * q + 1] = o4.y; m[4 * q + 2] = o4.z; m[4 * q + 3] = o4.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < IT; ++i) m[i] = (r0 + i < M) ? order[r0 + i] : 0u;
  }
  uint32_t cnt = 0;
#pragma unroll
  for (int i = 0; i < IT; ++i) rc[i] = (r0 + i < M) ? rect[m[i]] : 0ull;
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const uint32_t x0 = rc[i] & 0xffff, x1 = (rc[i] >> 16) & 0xffff, y0 = (rc[i] >> 32) & 0xffff,
                   y1 = rc[i] >> 48;
    c[i] = (r0 + i < M) ? (x1 - x0 + 1) * (y1 - y0 + 1) : 0u;
    cnt += c[i];
    if (r0 + i < M) w.rect_sorted[r0 + i] = rc[i];
  }
  uint32_t inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(FULL_MASK, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) s_w[warp] = inc;
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
    const uint32_t pre = lookback_warp(w.status, part, total, fs->epoch + TK_DUP);
    if (lane == 0) s_base = pre;
  }
  __syncthreads();
  if (r0 >= M) return;
  uint32_t off = s_base + s_w[warp] + inc - cnt;
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const uint32_t r = r0 + i;
    if (r < M) {
      w.splat_off[r] = off;
      if (r == M - 1) w.splat_off[M] = off + c[i];
      for (uint32_t k = (off + EMIT_CHUNK - 1) / EMIT_CHUNK; k * EMIT_CHUNK < off + c[i]; ++k)
        w.chunk_first[k] = r;
      off += c[i];
    }
  }
}

// Pass 2, EMIT_CHUNK pairs per CTA regardless of splat sizes (emit.cuh),
// written (tile << 32 | splat) coalesced, in depth order (the tile passes in
// k_sort.cu then sort them stably by tile).
__global__ void __launch_bounds__(DUP_THREADS) k_dup_emit(const uint32_t *__restrict__ order,
                                                          int32_t tiles_x, Work w,
                                                          FrameState *fs) {
  __shared__ EmitSmem<EMIT_CHUNK> E;
  const uint32_t P = fs->n_pairs;
  const uint32_t j0 = blockIdx.x * EMIT_CHUNK;
  if (j0 >= P) return;
  const uint32_t j1 = min(j0 + (uint32_t)EMIT_CHUNK, P);
  uint32_t r0, r1;
  emit_owners(w, j0, j1, P, fs->stats.M, r0, r1);
  emit_stage(E, order, w, j0, j1, r0, r1);
#pragma unroll
  for (int it = 0; it < EMIT_ITEMS; ++it) {
    const uint32_t j = j0 + it * DUP_THREADS + threadIdx.x;
    if (j >= j1) break;
    w.pairs[0][j] = emit_pair(E, j, j0, tiles_x);
  }
}

void launch_tile_setup(const Work &w, FrameState *fs, int32_t *tile_count, int32_t tiles_x,
                       int32_t tiles_y, cudaStream_t s) {
  const size_t sm = (size_t)(tiles_x + 1) * (tiles_y + 1) * 4;
  static size_t attr = 0;
  if (sm > 48 * 1024 && sm > attr) {
    cudaFuncSetAttribute(k_tile_setup, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = sm;
  }
  k_tile_setup<<<1, 1024, sm, s>>>(w.tile_diff, tiles_x, tiles_y, tile_count, w.tile_start,
                                   w.tile_order, fs, w.P_cap);
}

void launch_duplicate(const Work &w, FrameState *fs, int32_t tiles_x, int64_t M_cap,
                      cudaStream_t s) {
  if (M_cap <= 0) return;
  const unsigned grid =
      (unsigned)((M_cap + DUP_THREADS * COUNT_ITEMS - 1) / (DUP_THREADS * COUNT_ITEMS));
  k_dup_count<<<grid, DUP_THREADS, 0, s>>>(w.val_depth[0], w.rect, w, fs);
  const unsigned egrid = (unsigned)((w.P_cap + EMIT_CHUNK - 1) / EMIT_CHUNK);
  k_dup_emit<<<egrid, DUP_THREADS, 0, s>>>(w.val_depth[0], tiles_x, w, fs);
}

}  // namespace lodge
