// K4: onesweep LSD radix sort (Adinets & Merrill 2022) for the two global
// orderings of rasterize (reference src/raster.py:401 and :421-423):
//   1. survivors by fp64 depth, stable over input order, which is exactly
//      np.lexsort((source_index, depth)) because compaction keeps the
//      concatenated input order (the key is the IEEE bit pattern; z > near
//      > 0 so it is monotone as an unsigned integer);
//   2. duplicated (tile<<32 | splat) pairs by tile id only, stable, which is
//      np.argsort(tile_ids, kind="stable") over pairs emitted in depth order.
// One kernel per 8-bit digit: warp-level __match_any_sync ranking, per-digit
// decoupled look-back across partitions (virtual partition ids from an
// atomic ticket for forward progress), then a shared-memory staged scatter.
#include "internal.cuh"

namespace lodge {

constexpr int OS_THREADS = 256;
constexpr int OS_ITEMS = 16;
constexpr int OS_TILE = OS_THREADS * OS_ITEMS;  // 4096 keys per partition
constexpr int OS_WSTRIDE = 257;                 // per-warp digit counters (+1 pad bucket)

static size_t onesweep_smem(bool vals) {
  return (size_t)OS_TILE * 8 + (vals ? (size_t)OS_TILE * 4 : 0) +
         (size_t)(8 * OS_WSTRIDE + 256 + 256 + 32) * 4 + (size_t)OS_TILE * 2;
}

template <bool VALS>
__global__ void __launch_bounds__(OS_THREADS, VALS ? 2 : 3) k_onesweep(
    const uint64_t *__restrict__ kin, uint64_t *__restrict__ kout,
    const uint32_t *__restrict__ vin, uint32_t *__restrict__ vout, const uint32_t *n_ptr,
    int shift, const uint32_t *__restrict__ digit_off, uint64_t *status, FrameState *fs,
    int tk) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t *s_keys = reinterpret_cast<uint64_t *>(smem);
  uint32_t *s_vals = reinterpret_cast<uint32_t *>(s_keys + OS_TILE);
  uint32_t *s_whist = VALS ? s_vals + OS_TILE : reinterpret_cast<uint32_t *>(s_keys + OS_TILE);
  uint32_t *s_dstart = s_whist + 8 * OS_WSTRIDE;
  uint32_t *s_gbase = s_dstart + 256;
  uint32_t *s_misc = s_gbase + 256;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  if (tid == 0) s_misc[0] = atomicAdd(&fs->tickets[tk], 1u);
  for (int i = tid; i < 8 * OS_WSTRIDE; i += OS_THREADS) s_whist[i] = 0;
  __syncthreads();
  const uint32_t part = s_misc[0];
  const uint32_t n = *n_ptr;
  const uint32_t base = part * OS_TILE;
  if (base >= n) return;

  // keys live in registers; ranks go to shared memory and digits are
  // recomputed from the keys, keeping the kernel at >= 2-3 CTAs per SM
  uint16_t *s_rank = reinterpret_cast<uint16_t *>(s_misc + 32);
  uint64_t k[OS_ITEMS];
  uint32_t vmask = 0;
#pragma unroll
  for (int i = 0; i < OS_ITEMS; ++i) {
    const uint32_t idx = base + warp * (OS_ITEMS * 32) + i * 32 + lane;
    const bool valid = idx < n;
    vmask |= valid ? (1u << i) : 0u;
    k[i] = valid ? kin[idx] : ~0ull;
  }
  uint32_t *wh = s_whist + warp * OS_WSTRIDE;
#pragma unroll
  for (int i = 0; i < OS_ITEMS; ++i) {
    const uint32_t di = ((vmask >> i) & 1u) ? (uint32_t)((k[i] >> shift) & 255u) : 256u;
    const uint32_t peers = __match_any_sync(FULL_MASK, di);
    const uint32_t cnt = wh[di];
    __syncwarp();
    if (lane == __ffs(peers) - 1) wh[di] = cnt + __popc(peers);
    __syncwarp();
    s_rank[warp * (OS_ITEMS * 32) + i * 32 + lane] = (uint16_t)(cnt + __popc(peers & lanemask_lt()));
  }
  __syncthreads();

  // per digit: warp-exclusive offsets and block total
  const uint32_t dg = tid;  // 256 threads == 256 digits
  uint32_t tot = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) {
    const uint32_t c = s_whist[w * OS_WSTRIDE + dg];
    s_whist[w * OS_WSTRIDE + dg] = tot;
    tot += c;
  }
  // publish aggregate, then look back for this digit's exclusive prefix
  const uint32_t epoch = fs->epoch + tk;
  uint64_t *st = status + (size_t)part * 256;
  uint32_t excl = 0;
  if (part == 0) {
    st_store(st + dg, st_pack(epoch, ST_PREFIX, tot));
  } else {
    st_store(st + dg, st_pack(epoch, ST_AGG, tot));
    // look back LB partitions per round trip (independent loads), consuming
    // aggregates from the nearest until an inclusive prefix; an empty slot
    // restarts the window at that partition
    constexpr int LB = 8;
    int64_t q = (int64_t)part - 1;
    bool done = false;
    while (!done) {
      uint64_t sv[LB];
#pragma unroll
      for (int i = 0; i < LB; ++i)
        sv[i] = (q - i >= 0) ? st_load(status + (size_t)(q - i) * 256 + dg)
                             : st_pack(epoch, ST_PREFIX, 0u);
#pragma unroll
      for (int i = 0; i < LB; ++i) {
        if (done) break;
        const uint32_t flag =
            ((uint32_t)(sv[i] >> 32) == epoch) ? (uint32_t)((sv[i] >> 30) & 3u) : 0u;
        if (flag == ST_EMPTY) break;  // retry from partition q
        excl += (uint32_t)(sv[i] & 0x3fffffffu);
        --q;
        if (flag == ST_PREFIX) done = true;
      }
    }
    st_store(st + dg, st_pack(epoch, ST_PREFIX, excl + tot));
  }
  s_gbase[dg] = digit_off[dg] + excl;
  // block-local exclusive scan of the digit totals
  uint32_t inc = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(FULL_MASK, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) s_misc[1 + warp] = inc;
  __syncthreads();
  uint32_t wpre = 0;
#pragma unroll
  for (int w = 0; w < 8; ++w) wpre += (w < warp) ? s_misc[1 + w] : 0u;
  s_dstart[dg] = wpre + inc - tot;
  __syncthreads();

#pragma unroll
  for (int i = 0; i < OS_ITEMS; ++i) {
    if ((vmask >> i) & 1u) {
      const uint32_t li = warp * (OS_ITEMS * 32) + i * 32 + lane;
      const uint32_t di = (uint32_t)((k[i] >> shift) & 255u);
      const uint32_t lp = s_dstart[di] + wh[di] + s_rank[li];
      s_keys[lp] = k[i];
      if (VALS) s_vals[lp] = vin[base + li];
    }
  }
  __syncthreads();
  const uint32_t cnt_valid = min((uint32_t)OS_TILE, n - base);
  for (uint32_t j = tid; j < cnt_valid; j += OS_THREADS) {
    const uint64_t key = s_keys[j];
    const uint32_t dd = (uint32_t)((key >> shift) & 255u);
    const uint32_t out = s_gbase[dd] + (j - s_dstart[dd]);
    kout[out] = key;
    if (VALS) vout[out] = s_vals[j];
  }
}

// Upfront histogram of all eight 8-bit digits of the depth keys.
__global__ void __launch_bounds__(256) k_depth_hist(const uint64_t *__restrict__ keys,
                                                    FrameState *fs) {
  __shared__ uint32_t h[8][256];
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint32_t n = fs->n_sort;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
#pragma unroll
    for (int p = 0; p < 8; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) {
    const uint32_t c = (&h[0][0])[i];
    if (c) atomicAdd(&fs->hist_depth[0][0] + i, c);
  }
}

// Exclusive scans of the 8 digit histograms (one warp per pass).
__global__ void k_depth_scan(FrameState *fs) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= 8) return;
  uint32_t run = 0;
  for (int c = 0; c < 256; c += 32) {
    const uint32_t v = fs->hist_depth[warp][c + lane];
    uint32_t inc = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL_MASK, inc, o);
      if (lane >= o) inc += t;
    }
    fs->off_depth[warp][c + lane] = run + inc - v;
    run += __shfl_sync(FULL_MASK, inc, 31);
  }
}

static void set_smem_once() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(k_onesweep<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)onesweep_smem(true));
  cudaFuncSetAttribute(k_onesweep<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)onesweep_smem(false));
  done = true;
}

void launch_depth_sort(const Work &w, FrameState *fs, int64_t M_cap, int32_t *launches,
                       cudaStream_t s) {
  set_smem_once();
  if (M_cap <= 0) return;
  int hist_blocks = (int)((M_cap + 1023) / 1024);
  if (hist_blocks > 148 * 4) hist_blocks = 148 * 4;
  k_depth_hist<<<hist_blocks, 256, 0, s>>>(w.key_depth[0], fs);
  k_depth_scan<<<1, 256, 0, s>>>(fs);
  *launches += 2;
  const unsigned grid = (unsigned)((M_cap + OS_TILE - 1) / OS_TILE);
  const size_t sm = onesweep_smem(true);
  for (int p = 0; p < 8; ++p) {
    const int a = p & 1;
    k_onesweep<true><<<grid, OS_THREADS, sm, s>>>(w.key_depth[a], w.key_depth[a ^ 1],
                                                  w.val_depth[a], w.val_depth[a ^ 1],
                                                  &fs->n_sort, 8 * p, fs->off_depth[p],
                                                  w.status, fs, TK_DEPTH0 + p);
    ++*launches;
  }
}

void launch_tile_sort(const Work &w, FrameState *fs, int32_t, int32_t, int32_t *launches,
                      cudaStream_t s) {
  set_smem_once();
  const unsigned grid = (unsigned)((w.P_cap + OS_TILE - 1) / OS_TILE);
  const size_t sm = onesweep_smem(false);
  for (int p = 0; p < 2; ++p) {
    k_onesweep<false><<<grid, OS_THREADS, sm, s>>>(w.pairs[p], w.pairs[p ^ 1], nullptr, nullptr,
                                                   &fs->n_pairs, 32 + 8 * p, fs->off_tile[p],
                                                   w.status, fs, TK_TILE0 + p);
    ++*launches;
  }
}

}  // namespace lodge
