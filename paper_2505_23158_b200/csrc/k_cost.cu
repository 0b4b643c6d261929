// Threshold-search cost table, second half (
// ThresholdSearcher._table, reference src/thresholds.py:80-90): after the
// stable sort of (distance key, cover count) pairs, the distances in sorted
// order and prefix = concatenate([[0], cumsum(cover[order])]) as int64.
// Three kernels: per-2048 block sums, one CTA scanning the block sums, then
// each block's local scan plus its offset.
#include "internal.cuh"

namespace lodge {

constexpr int SC_THREADS = 256, SC_ITEMS = 8;
constexpr int SC_TILE = SC_THREADS * SC_ITEMS;

__device__ __forceinline__ uint64_t block_exclusive_scan(uint64_t v, uint64_t *s_w,
                                                         uint64_t &total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t t = __shfl_up_sync(FULL_MASK, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  uint64_t pre = 0;
  total = 0;
#pragma unroll
  for (int i = 0; i < SC_THREADS / 32; ++i) {
    pre += (i < warp) ? s_w[i] : 0ull;
    total += s_w[i];
  }
  __syncthreads();
  return pre + inc - v;
}

__global__ void __launch_bounds__(SC_THREADS) k_cover_sums(const uint32_t *__restrict__ cover,
                                                           const FrameState *fs,
                                                           uint64_t *__restrict__ sums) {
  __shared__ uint64_t s_w[SC_THREADS / 32];
  const uint32_t M = fs->stats.M;
  const int64_t b0 = (int64_t)blockIdx.x * SC_TILE;
  if (b0 >= M) return;
  uint64_t loc = 0;
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) {
    const int64_t k = b0 + (int64_t)threadIdx.x * SC_ITEMS + i;
    loc += (k < M) ? cover[k] : 0u;
  }
  uint64_t tot;
  block_exclusive_scan(loc, s_w, tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// One CTA: exclusive scan of the nb block sums in place.
__global__ void __launch_bounds__(1024) k_cover_top(const FrameState *fs, uint64_t *sums) {
  __shared__ uint64_t s_w[32];
  const uint32_t M = fs->stats.M;
  const int64_t nb = ((int64_t)M + SC_TILE - 1) / SC_TILE;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t carry = 0;
  for (int64_t base = 0; base < nb; base += 1024) {
    const int64_t k = base + threadIdx.x;
    const uint64_t v = k < nb ? sums[k] : 0ull;
    uint64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t t = __shfl_up_sync(FULL_MASK, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    uint64_t pre = 0, tot = 0;
    for (int i = 0; i < 32; ++i) {
      pre += (i < warp) ? s_w[i] : 0ull;
      tot += s_w[i];
    }
    if (k < nb) sums[k] = carry + pre + inc - v;
    carry += tot;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(SC_THREADS) k_cover_write(
    const uint64_t *__restrict__ keys, const uint32_t *__restrict__ cover, const FrameState *fs,
    const uint64_t *__restrict__ offs, double *__restrict__ dist, int64_t *__restrict__ prefix) {
  __shared__ uint64_t s_w[SC_THREADS / 32];
  const uint32_t M = fs->stats.M;
  const int64_t b0 = (int64_t)blockIdx.x * SC_TILE;
  if (b0 >= M) return;
  uint32_t c[SC_ITEMS];
  uint64_t loc = 0;
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) {
    const int64_t k = b0 + (int64_t)threadIdx.x * SC_ITEMS + i;
    c[i] = (k < M) ? cover[k] : 0u;
    loc += c[i];
  }
  uint64_t tot;
  uint64_t run = offs[blockIdx.x] + block_exclusive_scan(loc, s_w, tot);
  if (blockIdx.x == 0 && threadIdx.x == 0) prefix[0] = 0;
#pragma unroll
  for (int i = 0; i < SC_ITEMS; ++i) {
    const int64_t k = b0 + (int64_t)threadIdx.x * SC_ITEMS + i;
    if (k < M) {
      run += c[i];
      prefix[k + 1] = (int64_t)run;
      dist[k] = __longlong_as_double((long long)keys[k]);
    }
  }
}

__global__ void k_cover_nsort(FrameState *fs) { fs->n_sort = fs->stats.M; }

void launch_cover_table(const Work &w, FrameState *fs, int64_t n_cap, double *dist,
                        int64_t *prefix, int32_t *launches, cudaStream_t s) {
  k_cover_nsort<<<1, 1, 0, s>>>(fs);
  ++*launches;
  launch_depth_sort64(w, fs, n_cap, launches, s);
  const unsigned nb = (unsigned)((n_cap + SC_TILE - 1) / SC_TILE);
  uint64_t *sums = w.rect;  // scratch: the rectangles are not used on this path
  k_cover_sums<<<nb, SC_THREADS, 0, s>>>(w.val_depth[0], fs, sums);
  k_cover_top<<<1, 1024, 0, s>>>(fs, sums);
  k_cover_write<<<nb, SC_THREADS, 0, s>>>(w.key_depth[0], w.val_depth[0], fs, sums, dist, prefix);
  *launches += 3;
}

}  // namespace lodge
