// K4: onesweep LSD radix sort (Adinets & Merrill 2022) for the two global
// orderings of rasterize (reference src/raster.py:401 and :421-423):
//   1. inputs by fp64 depth, stable over the concatenated input order, which
//      is exactly np.lexsort((source_index, depth)).  Frames sort a 32-bit
//      key -- the fp32 round-toward-zero bit pattern of the depth, monotone
//      in it (z > near > 0) -- in four passes, then k_depth_ties re-orders
//      each run of equal 32-bit keys by the full fp64 depth (and index):
//      the result is the order of the fp64 keys.  Culled inputs carry ~0
//      and leave the sort in its first pass.  The cost tables sort the full
//      64-bit pattern in eight passes.
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
  const uint32_t n = *n_ptr;
  // e.g. a phase that kept block lists: no ticket traffic; and CTAs beyond
  // the partitions of a small sort leave before drawing one
  if ((uint64_t)blockIdx.x * OS_TILE >= n) return;
  // persistent CTAs: partitions in ticket order until the keys run out
  for (;;) {
  if (tid == 0) S.misc[0] = atomicAdd(&fs->tickets[tk], 1u);
  __syncthreads();
  const uint32_t part = S.misc[0];
  const uint32_t base = part * OS_TILE;
  if (base >= n) break;
  KI k[OS_ITEMS];
  uint32_t vmask = 0;
#pragma unroll
  for (int i = 0; i < OS_ITEMS; ++i) {
    const uint32_t idx = base + warp * (OS_ITEMS * 32) + i * 32 + lane;
    k[i] = idx < n ? os_ld(kin + idx) : (KI)~(KI)0;
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
  // the output holds n keys (DROP: the survivors, counted into stats.M)
  onesweep_partition<OS_ITEMS, NB, VALS>(S, k, vmask, part, cnt, shift, digit_off, status,
                                         fs->epoch + tk, kout, kmap, vout,
                                         [&](uint32_t li) { return os_ld(vin + base + li); },
                                         DROP ? fs->stats.M : n, fs);
  __syncthreads();  // the next partition reuses the shared memory
  }
}

// ---- frame depth sort: 32-bit keys + tie repair ----------------------------
// fp32 (round toward zero) bit pattern of a positive fp64 depth key: a
// non-decreasing map, so sorting it leaves only ties of equal 32-bit keys
// to resolve by the full key.  ~0 (culled) stays ~0 (a NaN pattern, never
// produced by a positive depth).
__device__ __forceinline__ uint32_t depth_key32(uint64_t k) {
  return k == ~0ull ? ~0u
                    : __float_as_uint(__double2float_rz(__longlong_as_double((long long)k)));
}

// One pass over 32-bit depth keys; FIRST reads the u64 keys the projection
// wrote (at the concatenated input index), maps them and drops the culled.
#ifndef LODGE_OS_ITEMS_SUB
#define LODGE_OS_ITEMS_SUB 8  // keys per thread of the subset sorts (few partitions: latency)
#endif
template <bool FIRST, int IT = LODGE_OS_ITEMS_D>
__global__ void __launch_bounds__(OS_THREADS, LODGE_OS_VMINB)
    k_depth_pass(const uint64_t *__restrict__ kin64, const uint32_t *__restrict__ kin32,
                 uint32_t *__restrict__ kout, const uint32_t *__restrict__ vin,
                 uint32_t *__restrict__ vout, const uint32_t *n_ptr, int shift,
                 const uint32_t *__restrict__ digit_off, uint64_t *status, FrameState *fs,
                 int tk) {
  extern __shared__ __align__(16) uint8_t smem[];
  constexpr uint32_t TILE = OS_THREADS * IT;
  using Smem = OSmem<IT, true, uint32_t, 256>;
  Smem &S = *reinterpret_cast<Smem *>(smem);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t n = *n_ptr;
  if ((uint64_t)blockIdx.x * TILE >= n) return;  // beyond the partitions (small sorts)
  for (;;) {  // persistent CTAs, partitions in ticket order
  if (tid == 0) S.misc[0] = atomicAdd(&fs->tickets[tk], 1u);
  __syncthreads();
  const uint32_t part = S.misc[0];
  const uint32_t base = part * TILE;
  if (base >= n) break;
  uint32_t k[IT];
  uint32_t vmask = 0;
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    const uint32_t idx = base + warp * (IT * 32) + i * 32 + lane;
    k[i] = idx < n ? (FIRST ? depth_key32(os_ld(kin64 + idx)) : os_ld(kin32 + idx)) : ~0u;
    const bool valid = idx < n && !(FIRST && k[i] == ~0u);
    vmask |= valid ? (1u << i) : 0u;
  }
  uint32_t cnt = min(TILE, n - base);
  if (FIRST) {  // the partition's valid items, not its positional size
    const uint32_t c = __reduce_add_sync(FULL_MASK, (uint32_t)__popc(vmask));
    if (lane == 0) S.misc[2 + warp] = c;
    __syncthreads();
    cnt = 0;
#pragma unroll
    for (int w = 0; w < OS_THREADS / 32; ++w) cnt += S.misc[2 + w];
  }
  onesweep_partition<IT, 8, true>(S, k, vmask, part, cnt, shift, digit_off, status,
                                  fs->epoch + tk, kout, [](uint32_t key) { return key; }, vout,
                                  [&](uint32_t li) { return os_ld(vin + base + li); },
                                  FIRST ? fs->stats.M : n, fs);
  __syncthreads();
  }
}

// Histograms of the four 8-bit digits of the 32-bit depth keys: of the u64
// keys by position (n_sort of them, culled ~0 skipped) or, COMPACT, of the
// projection's M compacted 32-bit survivor keys.
template <bool COMPACT>
__global__ void __launch_bounds__(256) k_depth_hist32(const uint64_t *__restrict__ keys,
                                                     const uint32_t *__restrict__ keys32,
                                                     const uint32_t *n_ptr, FrameState *fs) {
  __shared__ uint32_t h[4][256];
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  const uint32_t n = COMPACT ? *n_ptr : fs->n_sort;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t k32;
    if (COMPACT) {
      k32 = keys32[i];
    } else {
      const uint64_t k = keys[i];
      if (k == ~0ull) continue;  // culled: dropped by the first pass
      k32 = depth_key32(k);
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) atomicAdd(&h[p][(k32 >> (8 * p)) & 255u], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) {
    const uint32_t c = (&h[0][0])[i];
    if (c) atomicAdd(&fs->hist_depth[0][0] + i, c);
  }
}

// Tie repair after the 32-bit passes: every run of equal 32-bit keys is in
// input order (the passes are stable) and must be ordered by (fp64 key,
// index).  One thread per element: an element without an equal neighbour
// is copied; an element of a run finds the run's bounds and its rank in it
// by (full key, index) and is written at run start + rank.  All elements
// are independent (no thread walks a run alone), so the kernel's latency is
// a few dependent loads; a run of n costs O(n^2) loads in all, which only
// adversarial inputs make large (> 32 depths inside one fp32 ulp).
// vin -> vout, both M long.
__global__ void __launch_bounds__(256) k_depth_ties(const uint32_t *__restrict__ k32,
                                                    const uint32_t *__restrict__ vin,
                                                    const uint64_t *__restrict__ full,
                                                    uint32_t *__restrict__ vout,
                                                    const uint32_t *n_ptr) {
  const uint32_t M = *n_ptr;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
    const uint32_t k = k32[i];
    const uint32_t gi = vin[i];
    const bool l = i > 0 && k32[i - 1] == k, r = i + 1 < M && k32[i + 1] == k;
    if (!l && !r) {
      vout[i] = gi;
      continue;
    }
    uint32_t s = i, e = i + 1;
    while (s > 0 && k32[s - 1] == k) --s;
    while (e < M && k32[e] == k) ++e;
    const uint64_t fi = full[gi];
    uint32_t rank = 0;
    for (uint32_t j = s; j < e; ++j) {
      const uint32_t gj = vin[j];
      const uint64_t fj = full[gj];
      rank += (fj < fi || (fj == fi && gj < gi)) ? 1u : 0u;
    }
    vout[s + rank] = gi;
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

// Grid of a persistent kernel: its resident CTAs on this device (at most
// `need`).  Queried once per kernel (static per instantiation at the call).
template <typename K>
static unsigned resident_grid(K kernel, int threads, size_t smem, int64_t need) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem);
  per = std::min(per, LODGE_PERSIST_PER);
  const int64_t r = (int64_t)std::max(per, 1) * std::max(sms, 1);
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(need, r));
}

// One onesweep pass (dynamic shared memory opted in once per instantiation).
template <bool VALS, typename KI, typename KO, int MAP, int NB, bool DROP = false>
static void os_launch(int64_t cap, cudaStream_t s, const KI *kin, KO *kout, const uint32_t *vin,
                      uint32_t *vout, const uint32_t *n_ptr, int shift, int sb,
                      const uint32_t *digit_off, uint64_t *status, FrameState *fs, int tk) {
  constexpr int64_t TILE = (int64_t)OS_THREADS * os_items<VALS, KI>();
  static PerDevice res;
  const size_t sm = sizeof(OSmem<os_items<VALS, KI>(), VALS, KI, (1 << NB)>);
  if (!res()) {
    cudaFuncSetAttribute(k_onesweep<VALS, KI, KO, MAP, NB, DROP>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    res() = resident_grid(k_onesweep<VALS, KI, KO, MAP, NB, DROP>, OS_THREADS, sm, 1 << 30);
  }
  const int64_t resident = res();
#ifndef LODGE_PERSIST
#define LODGE_PERSIST 1
#endif
  const unsigned grid = (unsigned)std::min<int64_t>((cap + TILE - 1) / TILE,
                                                    LODGE_PERSIST ? resident : 0x7fffffff);
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

#ifdef LODGE_VERIFY
// Debug check of one pass: its output is ordered by the pass digit, and the
// value's own key has the output key (bit 8 + pass of stats.fault).
__global__ void k_pass_verify(const uint32_t *kout, const uint32_t *vout, const uint64_t *full,
                              const uint32_t *n_ptr, int shift, int pass, FrameState *fs) {
  const uint32_t n = *n_ptr, U = fs->n_sort;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t g = vout[i];
    bool ok = g < U && depth_key32(full[g]) == kout[i];
    if (i + 1 < n) ok = ok && ((kout[i] >> shift) & 255u) <= ((kout[i + 1] >> shift) & 255u);
    if (!ok) raise_fault(fs, 256u << pass);
  }
}
#endif

#ifdef LODGE_VERIFY
// Debug check of the frame depth order: keys non-decreasing, every value an
// input whose own key is the sorted key.
__global__ void k_depth_verify(const uint32_t *k32, const uint32_t *val, const uint64_t *full,
                               const uint32_t *n_ptr, FrameState *fs) {
  const uint32_t M = *n_ptr, U = fs->n_sort;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
    const uint32_t g = val[i];
    bool ok = g < U && depth_key32(full[g]) == k32[i];
    if (i + 1 < M) ok = ok && k32[i] <= k32[i + 1];
    if (!ok) raise_fault(fs, FAULT_DEPTH);
  }
}
#endif

#ifdef LODGE_VERIFY
// Debug check of the 64-bit frame depth order: (key, index) strictly
// increasing -- np.lexsort((index, depth)) -- and every index an input.
__global__ void k_depth_verify64(const uint64_t *k, const uint32_t *val, FrameState *fs) {
  const uint32_t M = fs->stats.M, U = fs->n_sort;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
    bool ok = val[i] < U && k[i] != ~0ull;
    if (i + 1 < M) ok = ok && (k[i] < k[i + 1] || (k[i] == k[i + 1] && val[i] < val[i + 1]));
    if (!ok) raise_fault(fs, FAULT_DEPTH);
  }
}

// Debug check of the per-tile lists of a tile sort.  List members are input
// indices; vrank holds each survivor's position in the depth order, so a
// tile's members must have strictly increasing ranks (np.lexsort((src,
// depth)) restricted to the tile, src/raster.py:401-423), and the list
// ranges must lie inside the sorted pairs.
__global__ void k_depth_rank(const uint32_t *val, uint32_t *vrank, uint32_t cap,
                             const uint32_t *n_ptr, FrameState *fs) {
  const uint32_t M = *n_ptr;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
    const uint32_t g = val[i];
    if (g < cap) vrank[g] = i;
    else raise_fault(fs, FAULT_LISTORD);
  }
}

__global__ void k_list_verify(const uint32_t *list, const uint32_t *tile_start, uint32_t T,
                              const uint32_t *vrank, uint32_t cap, FrameState *fs, int second) {
  if (fs->stats.overflow) return;  // a discarded attempt: no lists
  if (second ? fs->scan_b : fs->scan_a) return;  // block lists: no per-tile lists
  const uint32_t n = fs->n_pairs;
  for (uint32_t t = blockIdx.x; t < T; t += gridDim.x) {
    const uint32_t s = tile_start[t], e = tile_start[t + 1];
    if (e < s || e > n) {
      if (threadIdx.x == 0) raise_fault(fs, FAULT_LISTORD);
      continue;
    }
    for (uint32_t i = s + threadIdx.x; i + 1 < e; i += blockDim.x) {
      const uint32_t a = list[i], b = list[i + 1];
      if (a >= cap || b >= cap || vrank[a] >= vrank[b]) raise_fault(fs, FAULT_LISTORD);
    }
  }
}

// Debug check of a phase's block lists: per block, the
// length within the capacity, every entry an input with a nonzero mask of
// the block's tiles (alive tiles in phase 2), depth ranks strictly
// increasing, and for every tile of the block the number of entries with
// its bit equal to the tile's list count.
__device__ void k_block_list_verify_body(const uint64_t *blist, const uint32_t *bl_start,
                                         const uint32_t *bl_len, const uint32_t *tile_start,
                                         const uint32_t *alive, int32_t tiles_x,
                                         int32_t tiles_y, const uint32_t *vrank, uint32_t cap,
                                         FrameState *fs) {
  if (fs->stats.overflow) return;
  const uint32_t nbx = (tiles_x + BLK_W - 1) / BLK_W, nb = block_count(tiles_x, tiles_y);
  for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const uint32_t s = bl_start[b], capb = bl_start[b + 1] - s;
    if (capb == 0) continue;  // no pairs of the phase: the block was skipped
    const uint32_t len = bl_len[b];
    if (len > capb) {
      if (threadIdx.x == 0) raise_fault(fs, FAULT_LISTORD);
      continue;
    }
    const uint32_t bx0 = (b % nbx) * BLK_W, by0 = (b / nbx) * BLK_H;
    uint32_t valid = 0;  // the block's tiles inside the frame (and alive in phase 2)
    for (int q = 0; q < BLK_W * BLK_H; ++q) {
      const uint32_t x = bx0 + q % BLK_W, y = by0 + q / BLK_W;
      if (x >= (uint32_t)tiles_x || y >= (uint32_t)tiles_y) continue;
      const uint32_t t = y * tiles_x + x;
      if (!alive || ((alive[t >> 5] >> (t & 31)) & 1u)) valid |= 1u << q;
    }
    for (uint32_t i = threadIdx.x; i < len; i += blockDim.x) {
      const uint64_t e = blist[s + i];
      const uint32_t m = (uint32_t)(e >> 32), id = (uint32_t)e;
      bool ok = m != 0u && (m & ~valid) == 0u && id < cap;
      if (ok && i + 1 < len) {
        const uint32_t id2 = (uint32_t)blist[s + i + 1];
        ok = id2 < cap && vrank[id] < vrank[id2];
      }
      if (!ok) raise_fault(fs, FAULT_LISTORD);
    }
    for (int q = threadIdx.x; q < BLK_W * BLK_H; q += blockDim.x) {
      if (!((valid >> q) & 1u)) continue;
      const uint32_t t = (by0 + q / BLK_W) * tiles_x + bx0 + q % BLK_W;
      uint32_t c = 0;
      for (uint32_t i = 0; i < len; ++i) c += (uint32_t)(blist[s + i] >> (32 + q)) & 1u;
      if (c != tile_start[t + 1] - tile_start[t]) raise_fault(fs, FAULT_LISTORD);
    }
  }
}

// the phase's block-list check, when the phase kept block lists (a device
// flag: the kernel body runs only then)
template <int SECOND>
__global__ void k_block_list_verify_if(const Work w, int32_t tiles_x, int32_t tiles_y,
                                       FrameState *fs) {
  if (!(SECOND ? fs->scan_b : fs->scan_a)) return;
  const uint32_t nb = (uint32_t)block_count(tiles_x, tiles_y);
  k_block_list_verify_body(w.pairs[SECOND], w.bl_start + (SECOND ? nb + 1 : 0),
                           w.bl_len + (SECOND ? nb : 0),
                           SECOND ? w.tile_start_b : w.tile_start, SECOND ? w.alive : nullptr,
                           tiles_x, tiles_y, w.vrank, (uint32_t)w.M_cap, fs);
}

void launch_list_verify(const Work &w, FrameState *fs, uint32_t T, bool second,
                        cudaStream_t s, int32_t tiles_x, int32_t tiles_y) {
  if (!w.vrank) return;
  // depth ranks of the phase's members: the first phase's (or the one
  // pass's) sorted survivors, the second phase's sorted owners
  if (!second)
    k_depth_rank<<<296, 256, 0, s>>>(w.val_depth[0], w.vrank, (uint32_t)w.M_cap,
                                     tiles_x > 0 ? &fs->n_cand : &fs->stats.M, fs);
  else
    k_depth_rank<<<296, 256, 0, s>>>(w.val_depth[1], w.vrank, (uint32_t)w.M_cap,
                                     &fs->n_owners_b, fs);
  k_list_verify<<<std::min<uint32_t>(T, 148 * 8), 128, 0, s>>>(
      w.list, second ? w.tile_start_b : w.tile_start, T, w.vrank, (uint32_t)w.M_cap, fs,
      second ? 1 : 0);
  if (tiles_x > 0) {  // two-phase frames: the phase's block lists, when it kept them
    const uint32_t nb = (uint32_t)block_count(tiles_x, tiles_y);
    if (second)
      k_block_list_verify_if<1><<<std::min<uint32_t>(nb, 148 * 4), 128, 0, s>>>(
          w, tiles_x, tiles_y, fs);
    else
      k_block_list_verify_if<0><<<std::min<uint32_t>(nb, 148 * 4), 128, 0, s>>>(
          w, tiles_x, tiles_y, fs);
  }
}
#endif

// Frames: four passes over 32-bit keys (u32 ping-pong in the two halves of
// key_depth[1]; key_depth[0] keeps the full keys by input index for the tie
// repair), sorted input indices in val_depth[0].
template <int IT>
static void subset_sort(const Work &w, FrameState *fs, int64_t cap, const uint32_t *n_ptr,
                        const uint32_t *kin, const uint32_t *vin, uint32_t *ks0, uint32_t *ks1,
                        uint32_t *vs0, uint32_t *vs1, uint32_t *vout, int tk0,
                        int32_t *launches, cudaStream_t s) {
  cudaMemsetAsync(fs->hist_depth, 0, sizeof(uint32_t) * 4 * 256, s);  // (a frame may sort twice)
  int hist_blocks = (int)((cap + 2047) / 2048);
  if (hist_blocks > 148 * 2) hist_blocks = 148 * 2;
  k_depth_hist32<true><<<hist_blocks, 256, 0, s>>>(nullptr, kin, n_ptr, fs);
  k_depth_scan<<<1, 256, 0, s>>>(fs);
  *launches += 2;
  constexpr int64_t TILE = (int64_t)OS_THREADS * IT;
  const size_t sm = sizeof(OSmem<IT, true, uint32_t, 256>);
  static PerDevice res;
  if (!res()) {
    cudaFuncSetAttribute(k_depth_pass<false, IT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    res() = resident_grid(k_depth_pass<false, IT>, OS_THREADS, sm, 1 << 30);
  }
  const unsigned grid = (unsigned)std::min<int64_t>((cap + TILE - 1) / TILE,
                                                    LODGE_PERSIST ? res() : 0x7fffffff);
  // keys kin -> ks0 -> ks1 -> ks0 -> ks1, values vin -> vs0 -> vs1 -> vs0 -> vs1,
  // then the tie repair vs1 -> vout
  const uint32_t *ki[4] = {kin, ks0, ks1, ks0};
  uint32_t *ko[4] = {ks0, ks1, ks0, ks1};
  const uint32_t *vi[4] = {vin, vs0, vs1, vs0};
  uint32_t *vo[4] = {vs0, vs1, vs0, vs1};
  for (int p = 0; p < 4; ++p) {
    k_depth_pass<false, IT><<<grid, OS_THREADS, sm, s>>>(nullptr, ki[p], ko[p], vi[p], vo[p],
                                                         n_ptr, 8 * p, fs->off_depth[p],
                                                         w.status, fs, tk0 + p);
#ifdef LODGE_VERIFY
    k_pass_verify<<<296, 256, 0, s>>>(ko[p], vo[p], w.key_depth[0], n_ptr, 8 * p, p, fs);
#endif
  }
  const unsigned tgrid = (unsigned)std::min<int64_t>((cap + 255) / 256, 148 * 8);
  k_depth_ties<<<tgrid, 256, 0, s>>>(ks1, vs1, w.key_depth[0], vout, n_ptr);
#ifdef LODGE_VERIFY
  k_depth_verify<<<296, 256, 0, s>>>(ks1, vout, w.key_depth[0], n_ptr, fs);
#endif
  *launches += 5;
}

void launch_subset_sort(const Work &w, FrameState *fs, int64_t cap, const uint32_t *n_ptr,
                        const uint32_t *kin, const uint32_t *vin, uint32_t *ks0, uint32_t *ks1,
                        uint32_t *vs0, uint32_t *vs1, uint32_t *vout, int tk0,
                        int32_t *launches, cudaStream_t s) {
  if (cap <= 0) return;
  // all survivors of a one-pass frame: the large-partition passes; a two-phase
  // frame's candidates and owners (a few partitions): small ones
  if (n_ptr == &fs->stats.M)
    subset_sort<LODGE_OS_ITEMS_D>(w, fs, cap, n_ptr, kin, vin, ks0, ks1, vs0, vs1, vout, tk0,
                                  launches, s);
  else
    subset_sort<LODGE_OS_ITEMS_SUB>(w, fs, cap, n_ptr, kin, vin, ks0, ks1, vs0, vs1, vout, tk0,
                                    launches, s);
}

// Frames: four passes over 32-bit keys (u32 ping-pong in the two halves of
// key_depth[1]; key_depth[0] keeps the full keys by input index for the tie
// repair), sorted input indices in val_depth[0].
void launch_depth_sort(const Work &w, FrameState *fs, int64_t M_cap, int32_t *launches,
                       cudaStream_t s, bool compacted) {
  if (M_cap <= 0) return;
#ifdef LODGE_DEPTH64
  // opt-in: the eight 64-bit passes (0.17 vs 0.12 ms per config-3 frame),
  // which take their input values in val_depth[0]
  cudaMemcpyAsync(w.val_depth[0], w.val_depth[1], 4 * (size_t)M_cap, cudaMemcpyDeviceToDevice, s);
  launch_depth_sort64(w, fs, M_cap, launches, s);
  return;
#endif
  uint32_t *k32[2] = {depth_keys32(w, 0), depth_keys32(w, 1)};
  if (compacted) {  // the projection's compacted survivors (keys in k32[1], values val_depth[1])
    launch_subset_sort(w, fs, M_cap, &fs->stats.M, k32[1], w.val_depth[1], k32[0], k32[1],
                       w.val_depth[0], w.val_depth[1], w.val_depth[0], TK_DEPTH0, launches, s);
    return;
  }
  int hist_blocks = (int)((M_cap + 1023) / 1024);
  if (hist_blocks > 148 * 4) hist_blocks = 148 * 4;
  k_depth_hist32<false><<<hist_blocks, 256, 0, s>>>(w.key_depth[0], nullptr, nullptr, fs);
  k_depth_scan<<<1, 256, 0, s>>>(fs);
  *launches += 2;
  constexpr int64_t TILE = (int64_t)OS_THREADS * LODGE_OS_ITEMS_D;
  const size_t sm = sizeof(OSmem<LODGE_OS_ITEMS_D, true, uint32_t, 256>);
  static PerDevice res;
  if (!res()) {
    cudaFuncSetAttribute(k_depth_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_depth_pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    res() = resident_grid(k_depth_pass<true>, OS_THREADS, sm, 1 << 30);
  }
  const unsigned grid = (unsigned)std::min<int64_t>((M_cap + TILE - 1) / TILE,
                                                    LODGE_PERSIST ? res() : 0x7fffffff);
  // keys 0: u64 -> k32[0], then as launch_subset_sort; values from val_depth[1]
  k_depth_pass<true><<<grid, OS_THREADS, sm, s>>>(w.key_depth[0], nullptr, k32[0],
                                                  w.val_depth[1], w.val_depth[0], &fs->n_sort,
                                                  0, fs->off_depth[0], w.status, fs, TK_DEPTH0);
#ifdef LODGE_VERIFY
  k_pass_verify<<<296, 256, 0, s>>>(k32[0], w.val_depth[0], w.key_depth[0], &fs->stats.M, 0, 0,
                                    fs);
#endif
  for (int p = 1; p < 4; ++p) {
    const int a = p & 1;  // keys: k32[a ^ 1] -> k32[a]; values: [a ^ 1] -> [a]
    k_depth_pass<false><<<grid, OS_THREADS, sm, s>>>(
        nullptr, k32[a ^ 1], k32[a], w.val_depth[a ^ 1], w.val_depth[a], &fs->stats.M, 8 * p,
        fs->off_depth[p], w.status, fs, TK_DEPTH0 + p);
#ifdef LODGE_VERIFY
    k_pass_verify<<<296, 256, 0, s>>>(k32[a], w.val_depth[a], w.key_depth[0], &fs->stats.M,
                                      8 * p, p, fs);
#endif
  }
  const unsigned tgrid = (unsigned)std::min<int64_t>((M_cap + 255) / 256, 148 * 8);
  k_depth_ties<<<tgrid, 256, 0, s>>>(k32[1], w.val_depth[1], w.key_depth[0], w.val_depth[0],
                                     &fs->stats.M);
#ifdef LODGE_VERIFY
  k_depth_verify<<<296, 256, 0, s>>>(k32[1], w.val_depth[0], w.key_depth[0], &fs->stats.M, fs);
#endif
  *launches += 5;
}

// Diagnostic entry (lodge_debug_depth_sort): caller keys -> key_depth[0],
// identity values, n_sort = n, M = the keys that are not ~0.
__global__ void k_debug_sort_in(const uint64_t *keys, uint32_t n, uint64_t *k0, uint32_t *v0,
                                FrameState *fs) {
  __shared__ uint32_t s_m;
  if (threadIdx.x == 0) s_m = 0;
  __syncthreads();
  uint32_t m = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    k0[i] = k;
    v0[i] = i;
    m += k != ~0ull ? 1u : 0u;
  }
  atomicAdd(&s_m, m);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(&fs->stats.M, s_m);
    if (blockIdx.x == 0) fs->n_sort = n;
  }
}

__global__ void k_debug_sort_out(const uint64_t *k0, const uint32_t *v0, FrameState *fs,
                                 uint64_t *ko, uint32_t *vo, uint32_t *m_out) {
  const uint32_t M = fs->stats.M;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < M; i += gridDim.x * blockDim.x) {
    ko[i] = k0[i];
    vo[i] = v0[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    m_out[0] = M;
    m_out[1] = fs->stats.fault;
  }
}

void launch_debug_depth_sort(const Work &w, FrameState *fs, const uint64_t *keys, uint32_t n,
                             uint64_t *ko, uint32_t *vo, uint32_t *m_out, cudaStream_t s) {
  k_debug_sort_in<<<296, 256, 0, s>>>(keys, n, w.key_depth[0], w.val_depth[1], fs);
  int32_t nl = 0;
  launch_depth_sort(w, fs, n, &nl, s);
  k_debug_sort_out<<<296, 256, 0, s>>>(w.key_depth[0], w.val_depth[0], fs, ko, vo, m_out);
}

#ifdef LODGE_VERIFY_PASS
// Debug check after 64-bit pass p: the output is ordered by the digits
// 0..p (the LSD invariant), stable (equal digit prefixes keep the index
// order of pass 0's input), fault bit 1 << (16 + p).
__global__ void k_pass_verify64(const uint64_t *k, const uint32_t *v, int shift, int p,
                                FrameState *fs) {
  const uint32_t M = fs->stats.M;
  const uint64_t mask = shift >= 56 ? ~0ull : ((1ull << (shift + 8)) - 1ull);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i + 1 < M;
       i += gridDim.x * blockDim.x) {
    const uint64_t a = k[i] & mask, b = k[i + 1] & mask;
    if (a > b || (a == b && v[i] >= v[i + 1])) raise_fault(fs, 1u << (16 + p));
  }
}
#endif

// Cost tables: eight passes over the full 64-bit keys (the sorted keys are
// read back in key_depth[0]).
void launch_depth_sort64(const Work &w, FrameState *fs, int64_t M_cap, int32_t *launches,
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
#ifdef LODGE_VERIFY_PASS
    k_pass_verify64<<<296, 256, 0, s>>>(w.key_depth[a ^ 1], w.val_depth[a ^ 1], 8 * p, p, fs);
#endif
  }
#ifdef LODGE_VERIFY
  k_depth_verify64<<<296, 256, 0, s>>>(w.key_depth[0], w.val_depth[0], fs);
#endif
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
                      int32_t *launches, cudaStream_t s, int tk0, const uint32_t *n_keys) {
  const int64_t grid = w.P_cap;  // keys: the launchers size their grids
  const uint32_t T = (uint32_t)tiles_x * (uint32_t)tiles_y;
  const int lo_bits = std::min(8, std::max(1, bit_width(T - 1)));
  uint32_t *u32_1 = reinterpret_cast<uint32_t *>(w.pairs[1]);
  uint32_t *u32_0 = reinterpret_cast<uint32_t *>(w.pairs[0]);
  const uint32_t *nin = n_keys ? n_keys : &fs->n_pairs;
  const uint32_t *no_v = nullptr;
  uint32_t *no_vo = nullptr;
  const uint64_t *p0 = w.pairs[0];
  if (T <= 256) {
    os_launch_nb<false, uint64_t, uint32_t, MAP_LOW>(lo_bits, grid, s, p0, u32_1, no_v, no_vo,
                                                     nin, 32, 32, (const uint32_t *)fs->off_tile[0],
                                                     w.status, fs, tk0);
    ++*launches;
    w.list = u32_1;
    return;
  }
  const int hi_bits = bit_width((T - 1) >> 8);
  const int sb = std::max(1, bit_width((uint64_t)std::max<int64_t>(w.M_cap, 1) - 1));
  if (hi_bits + sb <= 32) {
    os_launch<false, uint64_t, uint32_t, MAP_PACK, 8>(grid, s, p0, u32_1, no_v, no_vo, nin, 32, sb,
                                                      fs->off_tile[0], w.status, fs, tk0);
    os_launch_nb<false, uint32_t, uint32_t, MAP_LOW>(
        hi_bits, grid, s, (const uint32_t *)u32_1, u32_0, no_v, no_vo, nin, sb, sb,
        (const uint32_t *)fs->off_tile[1], w.status, fs, tk0 + 1);
  } else {
    os_launch<false, uint64_t, uint64_t, MAP_ID, 8>(grid, s, p0, w.pairs[1], no_v, no_vo, nin, 32,
                                                    32, fs->off_tile[0], w.status, fs, tk0);
    os_launch_nb<false, uint64_t, uint32_t, MAP_LOW>(
        hi_bits, grid, s, (const uint64_t *)w.pairs[1], u32_0, no_v, no_vo, nin, 40, 32,
        (const uint32_t *)fs->off_tile[1], w.status, fs, tk0 + 1);
  }
  *launches += 2;
  w.list = u32_0;
}

}  // namespace lodge
