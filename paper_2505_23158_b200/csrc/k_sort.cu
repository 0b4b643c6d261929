// K4: onesweep LSD radix sort (Adinets & Merrill 2022) for the two global
// orderings of rasterize (reference src/raster.py:401 and :421-423):
//   1. inputs by fp64 depth, stable over the concatenated input order, which
//      is exactly np.lexsort((source_index, depth)) (the key is the IEEE bit
//      pattern; z > near > 0 so it is monotone as an unsigned integer; culled
//      inputs carry ~0 and sort last);
//   2. duplicated (tile<<32 | splat) pairs by tile id only, stable, which is
//      np.argsort(tile_ids, kind="stable") over pairs emitted in depth order.
// One partition per CTA: keys in registers in warp-contiguous order, stable
// warp-level ranking by per-bit ballots over two independent counter chains
// per warp (ILP), per-digit decoupled look-back across partitions (virtual
// partition ids from an atomic ticket for forward progress), then a
// shared-memory staged, digit-run-coalesced scatter (onesweep.cuh).
#include <algorithm>

#include "internal.cuh"
#include "onesweep.cuh"

namespace lodge {

#ifndef LODGE_OS_ITEMS_D
#define LODGE_OS_ITEMS_D 20  // depth passes (u64 key + u32 value); one wave at config 3
#endif
#ifndef LODGE_OS_ITEMS_T1
#define LODGE_OS_ITEMS_T1 16
#endif
#ifndef LODGE_OS_ITEMS_T2
#define LODGE_OS_ITEMS_T2 32
#endif
// Keys per thread: 16 for the depth passes (key + value), per-build choices
// for the tile passes on u64 and u32 keys.
template <bool VALS, typename KI>
__host__ __device__ constexpr int os_items() {
  return VALS ? LODGE_OS_ITEMS_D : (sizeof(KI) == 8 ? LODGE_OS_ITEMS_T1 : LODGE_OS_ITEMS_T2);
}

// Key maps applied at the scatter (see launch_tile_sort).
enum : int { MAP_ID = 0, MAP_PACK = 1, MAP_LOW = 2 };

template <bool VALS, typename KI, typename KO, int MAP, int NB = 8, bool DROP = false>
#ifndef LODGE_OS_MINB
#define LODGE_OS_MINB 3
#endif
#ifndef LODGE_OS_VMINB
#define LODGE_OS_VMINB 2
#endif
#ifndef LODGE_OS_MINB_T1
#define LODGE_OS_MINB_T1 LODGE_OS_MINB
#endif
__global__ void __launch_bounds__(OS_THREADS, VALS ? LODGE_OS_VMINB
                                                   : (sizeof(KI) == 8 ? LODGE_OS_MINB_T1
                                                                      : LODGE_OS_MINB))
    k_onesweep(
    const KI *__restrict__ kin, KO *__restrict__ kout, const uint32_t *__restrict__ vin,
    uint32_t *__restrict__ vout, const uint32_t *n_ptr, int shift, int sb,
    const uint32_t *__restrict__ digit_off, uint64_t *status, FrameState *fs, int tk) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr int OS_ITEMS = os_items<VALS, KI>();
  constexpr uint32_t OS_TILE = OS_THREADS * OS_ITEMS;
  using Smem = OSmem<OS_ITEMS, VALS, KI, (1 << NB)>;
  Smem &S = *reinterpret_cast<Smem *>(smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) S.misc[0] = atomicAdd(&fs->tickets[tk], 1u);
  __syncthreads();
  const uint32_t part = S.misc[0];
  const uint32_t n = *n_ptr;
  const uint32_t base = part * OS_TILE;
  if (base >= n) return;
  KI k[OS_ITEMS];
  uint32_t vmask = 0;
#pragma unroll
  for (int i = 0; i < OS_ITEMS; ++i) {
    const uint32_t idx = base + warp * (OS_ITEMS * 32) + i * 32 + lane;
    k[i] = idx < n ? kin[idx] : (KI)~(KI)0;
    // drop: culled inputs (key ~0) leave the sort here, the output holds
    // only the survivors (their count, fs->stats.M, is the later passes' n)
    const bool valid = idx < n && !(DROP && k[i] == (KI)~(KI)0);
    vmask |= valid ? (1u << i) : 0u;
  }
  uint32_t cnt = min((uint32_t)OS_TILE, n - base);
  if (DROP) {  // the partition's valid items, not its positional size
    const uint32_t c = __reduce_add_sync(FULL_MASK, (uint32_t)__popc(vmask));
    if (lane == 0) S.misc[2 + warp] = c;
    __syncthreads();
    cnt = 0;
#pragma unroll
    for (int w = 0; w < OS_THREADS / 32; ++w) cnt += S.misc[2 + w];
  }
  const uint32_t lowmask = sb >= 32 ? 0xffffffffu : ((1u << sb) - 1u);
  auto kmap = [&](KI key) -> KO {
    if (MAP == MAP_PACK)  // (tile << 32 | splat) -> (tile >> 8) << sb | splat
      return (KO)((((uint32_t)((uint64_t)key >> 40)) << sb) | (uint32_t)key);
    else if (MAP == MAP_LOW)  // -> splat
      return (KO)((uint32_t)key & lowmask);
    else
      return (KO)key;
  };
  onesweep_partition<OS_ITEMS, NB, VALS>(S, k, vmask, part, cnt, shift, digit_off, status,
                                         fs->epoch + tk, kout, kmap, vout,
                                         [&](uint32_t li) { return vin[base + li]; });
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
    if (k == ~0ull) continue;  // culled: dropped by the first pass
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

// One onesweep pass (dynamic shared memory opted in once per instantiation).
template <bool VALS, typename KI, typename KO, int MAP, int NB, bool DROP = false>
static void os_launch(int64_t cap, cudaStream_t s, const KI *kin, KO *kout, const uint32_t *vin,
                      uint32_t *vout, const uint32_t *n_ptr, int shift, int sb,
                      const uint32_t *digit_off, uint64_t *status, FrameState *fs, int tk) {
  constexpr int64_t TILE = (int64_t)OS_THREADS * os_items<VALS, KI>();
  const unsigned grid = (unsigned)((cap + TILE - 1) / TILE);
  static bool done = false;
  const size_t sm = sizeof(OSmem<os_items<VALS, KI>(), VALS, KI, (1 << NB)>);
  if (!done) {
    cudaFuncSetAttribute(k_onesweep<VALS, KI, KO, MAP, NB, DROP>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    done = true;
  }
  k_onesweep<VALS, KI, KO, MAP, NB, DROP><<<grid, OS_THREADS, sm, s>>>(
      kin, kout, vin, vout, n_ptr, shift, sb, digit_off, status, fs, tk);
}

// Same, with the digit width chosen at run time (nb <= 4 ranks on 4 bits).
template <bool VALS, typename KI, typename KO, int MAP, typename... A>
static void os_launch_nb(int nb, A... args) {
  switch (nb) {
    case 5: os_launch<VALS, KI, KO, MAP, 5>(args...); break;
    case 6: os_launch<VALS, KI, KO, MAP, 6>(args...); break;
    case 7: os_launch<VALS, KI, KO, MAP, 7>(args...); break;
    case 8: os_launch<VALS, KI, KO, MAP, 8>(args...); break;
    default: os_launch<VALS, KI, KO, MAP, 4>(args...); break;
  }
}

void launch_depth_sort(const Work &w, FrameState *fs, int64_t M_cap, int32_t *launches,
                       cudaStream_t s) {
  if (M_cap <= 0) return;
  int hist_blocks = (int)((M_cap + 1023) / 1024);
  if (hist_blocks > 148 * 4) hist_blocks = 148 * 4;
  k_depth_hist<<<hist_blocks, 256, 0, s>>>(w.key_depth[0], fs);
  k_depth_scan<<<1, 256, 0, s>>>(fs);
  *launches += 2;
  for (int p = 0; p < 8; ++p) {
    const int a = p & 1;
    // pass 0 reads all n_sort keys and drops the culled ones; passes 1..7
    // sort the M survivors
    auto launch = p == 0 ? os_launch<true, uint64_t, uint64_t, MAP_ID, 8, true>
                         : os_launch<true, uint64_t, uint64_t, MAP_ID, 8, false>;
    launch(M_cap, s, (const uint64_t *)w.key_depth[a], w.key_depth[a ^ 1],
           (const uint32_t *)w.val_depth[a], w.val_depth[a ^ 1],
           p == 0 ? &fs->n_sort : &fs->stats.M, 8 * p, 32, fs->off_depth[p], w.status, fs,
           TK_DEPTH0 + p);
    ++*launches;
  }
}

static int bit_width(uint64_t v) {
  int b = 0;
  while (v) { ++b; v >>= 1; }
  return b;
}

// The tile-digit passes over the emitted (tile << 32 | splat) pairs, which
// leave the bare u32 splat ids of the per-tile lists in w.list:
//   T <= 256  one pass pairs[0] -> list (u32 in pairs[1])
//   else      pass 1 on tile & 255, pairs[0] -> pairs[1] packed as
//             (tile >> 8) << sb | splat in u32 when it fits (sb = the bits a
//             splat id of this workspace needs), else kept u64;
//             pass 2 on tile >> 8 -> list (u32 in pairs[0]).
// Tile ranges come from tile_start, so the lists need no tile bits.
void launch_tile_sort(Work &w, FrameState *fs, int32_t tiles_x, int32_t tiles_y,
                      int32_t *launches, cudaStream_t s) {
  const int64_t grid = w.P_cap;  // keys: the launchers size their grids
  const uint32_t T = (uint32_t)tiles_x * (uint32_t)tiles_y;
  const int lo_bits = std::min(8, std::max(1, bit_width(T - 1)));
  uint32_t *u32_1 = reinterpret_cast<uint32_t *>(w.pairs[1]);
  uint32_t *u32_0 = reinterpret_cast<uint32_t *>(w.pairs[0]);
  const uint32_t *nin = &fs->n_pairs;
  const uint32_t *no_v = nullptr;
  uint32_t *no_vo = nullptr;
  const uint64_t *p0 = w.pairs[0];
  if (T <= 256) {
    os_launch_nb<false, uint64_t, uint32_t, MAP_LOW>(lo_bits, grid, s, p0, u32_1, no_v, no_vo,
                                                     nin, 32, 32, (const uint32_t *)fs->off_tile[0],
                                                     w.status, fs, (int)TK_TILE0);
    ++*launches;
    w.list = u32_1;
    return;
  }
  const int hi_bits = bit_width((T - 1) >> 8);
  const int sb = std::max(1, bit_width((uint64_t)std::max<int64_t>(w.M_cap, 1) - 1));
  if (hi_bits + sb <= 32) {
    os_launch<false, uint64_t, uint32_t, MAP_PACK, 8>(grid, s, p0, u32_1, no_v, no_vo, nin, 32, sb,
                                                      fs->off_tile[0], w.status, fs, TK_TILE0);
    os_launch_nb<false, uint32_t, uint32_t, MAP_LOW>(
        hi_bits, grid, s, (const uint32_t *)u32_1, u32_0, no_v, no_vo, nin, sb, sb,
        (const uint32_t *)fs->off_tile[1], w.status, fs, (int)TK_TILE0 + 1);
  } else {
    os_launch<false, uint64_t, uint64_t, MAP_ID, 8>(grid, s, p0, w.pairs[1], no_v, no_vo, nin, 32,
                                                    32, fs->off_tile[0], w.status, fs, TK_TILE0);
    os_launch_nb<false, uint64_t, uint32_t, MAP_LOW>(
        hi_bits, grid, s, (const uint64_t *)w.pairs[1], u32_0, no_v, no_vo, nin, 40, 32,
        (const uint32_t *)fs->off_tile[1], w.status, fs, (int)TK_TILE0 + 1);
  }
  *launches += 2;
  w.list = u32_0;
}

}  // namespace lodge
