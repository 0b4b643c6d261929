// Pair emission (k_dup_emit, k_bin.cu).  Restates the duplication of
// reference src/raster.py:409-418: every depth-sorted splat emits the tiles
// of its rectangle row-major, pairs in global depth order.  A CTA emits a
// fixed range [j0, j1) of the global pair sequence regardless of splat
// sizes: the owners of its pairs are the contiguous depth-order range
// [r0, r1] (from the EMIT_CHUNK splitters k_dup_count writes), staged in
// shared memory; each owner marks its first pair and an inclusive max-scan
// gives every pair its owner.
#pragma once
#include "internal.cuh"

namespace lodge {

constexpr int DUP_THREADS = 256;
constexpr int EMIT_CHUNK = 2048;  // splitter granularity (chunk_first)

template <int NP>  // pairs per CTA
struct EmitSmem {
  uint32_t off[NP + 2];   // pair offset of each owner
  uint64_t rect[NP + 1];  // owner rectangles
  uint32_t m[NP + 1];     // owner splat ids
  uint16_t own[NP];       // owner (local index) of each pair
  uint32_t wmax[DUP_THREADS / 32];
};

// Stages the owners of pairs [j0, j1) (owners [r0, r1]) and fills E.own.
// Block of DUP_THREADS threads; ends with a __syncthreads.
template <int NP>
__device__ __forceinline__ void emit_stage(EmitSmem<NP> &E, const uint32_t *__restrict__ order,
                                           const Work &w, uint32_t j0, uint32_t j1,
                                           uint32_t r0, uint32_t r1, FrameState *fs) {
  constexpr int IT = NP / DUP_THREADS;
  static_assert(NP % DUP_THREADS == 0, "whole pairs per thread");
  uint32_t nr = r1 - r0 + 1;
  if (r1 < r0 || nr > (uint32_t)NP + 1u || r1 >= (uint32_t)w.M_cap) {
    // owners have >= 1 pair: nr <= pairs + 1
    if (threadIdx.x == 0) raise_fault(fs, FAULT_OWNERS);
    nr = 1;
    r0 = 0;
  }
  const uint32_t npair = j1 - j0;
  for (uint32_t k = threadIdx.x; k < NP; k += DUP_THREADS) E.own[k] = 0;
  for (uint32_t q = threadIdx.x; q < nr; q += DUP_THREADS) {
    E.off[q] = w.splat_off[r0 + q];
    E.rect[q] = w.rect_sorted[r0 + q];
    E.m[q] = order[r0 + q];
  }
  __syncthreads();
  // owners with >= 1 pair mark their first pairs, which differ (an owner
  // without pairs -- a second-phase splat that meets no alive tile -- marks
  // nothing)
  for (uint32_t q = threadIdx.x; q < nr; q += DUP_THREADS) {
    const uint32_t next = (q + 1 < nr) ? E.off[q + 1] : w.splat_off[r0 + q + 1];
    const uint32_t st = E.off[q] > j0 ? E.off[q] - j0 : 0u;
    if (st < npair && next > E.off[q]) E.own[st] = (uint16_t)q;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t v[IT], run = 0;
#pragma unroll
  for (int i = 0; i < IT; ++i) {
    v[i] = E.own[threadIdx.x * IT + i];
    run = max(run, v[i]);
    v[i] = run;
  }
  uint32_t inc = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(FULL_MASK, inc, o);
    if (lane >= o) inc = max(inc, t);
  }
  if (lane == 31) E.wmax[warp] = inc;
  __syncthreads();
  uint32_t pre = __shfl_up_sync(FULL_MASK, inc, 1);
  if (lane == 0) pre = 0;
#pragma unroll
  for (int w2 = 0; w2 < DUP_THREADS / 32; ++w2)
    if (w2 < warp) pre = max(pre, E.wmax[w2]);
#pragma unroll
  for (int i = 0; i < IT; ++i) E.own[threadIdx.x * IT + i] = (uint16_t)max(pre, v[i]);
  __syncthreads();
}

// The (tile << 32 | splat) pair at global position j (j0 <= j < j1).
template <int NP>
__device__ __forceinline__ uint64_t emit_pair(const EmitSmem<NP> &E, uint32_t j, uint32_t j0,
                                              int32_t tiles_x) {
  const uint32_t lo = E.own[j - j0];
  const uint64_t rc = E.rect[lo];
  const uint32_t x0 = rc & 0xffff, x1 = (rc >> 16) & 0xffff, y0 = (rc >> 32) & 0xffff;
  const uint32_t wdt = x1 - x0 + 1;
  const uint32_t local = j - E.off[lo];
  // local / wdt by an fp32 reciprocal, corrected to the exact quotient
  // (local < T < 2^16, the tile count check_tile_smem allows, keeps the
  // estimate within one of it)
  uint32_t q = (uint32_t)__fmul_rz((float)local, __frcp_rn((float)wdt));
  int32_t r = (int32_t)(local - q * wdt);
  if (r < 0) { --q; r += (int32_t)wdt; }
  if (r >= (int32_t)wdt) { ++q; r -= (int32_t)wdt; }
  const uint32_t ty = y0 + q, tx = x0 + (uint32_t)r;
  return ((uint64_t)(ty * (uint32_t)tiles_x + tx) << 32) | E.m[lo];
}

// Owner range of the pairs [j0, j1) from the splitters.
__device__ __forceinline__ void emit_owners(const Work &w, uint32_t j0, uint32_t j1, uint32_t P,
                                            uint32_t M, uint32_t &r0, uint32_t &r1) {
  r0 = w.chunk_first[j0 / EMIT_CHUNK];
  r1 = (j1 < P) ? w.chunk_first[j1 / EMIT_CHUNK] : M - 1;
}

}  // namespace lodge
