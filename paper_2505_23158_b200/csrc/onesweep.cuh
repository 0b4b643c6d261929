// One onesweep partition (the radix passes of k_sort.cu).  Input keys KI are
// ranked on the digit (k >> shift) & (D - 1), D = 2^NB <= 256 (a pass whose
// digit has fewer significant bits ranks with fewer ballots and does all of
// its per-digit work -- counters, scans, look-back -- over D digits only);
// the scatter writes kmap(key), which lets a pass narrow the key it hands to
// the next one.
#pragma once
#include <type_traits>

#include "internal.cuh"

namespace lodge {

constexpr int OS_THREADS = 256;

template <typename T>
__device__ __forceinline__ T os_ld(const T *p) {
  return *p;
}

// peers &= lanes whose bit (d & MASK) equals this lane's (bit test, ballot and
// two predicated ANDs; nvcc's own lowering spends six instructions here).
template <uint32_t MASK>
__device__ __forceinline__ void peer_bit(uint32_t &peers, uint32_t d) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 t, bal;\n\t"
      "and.b32 t, %1, %2;\n\t"
      "setp.ne.u32 p, t, 0;\n\t"
      "vote.sync.ballot.b32 bal, p, 0xffffffff;\n\t"
      "@p and.b32 %0, %0, bal;\n\t"
      "not.b32 bal, bal;\n\t"
      "@!p and.b32 %0, %0, bal;\n\t}"
      : "+r"(peers)
      : "r"(d), "n"(MASK));
}

// Lanes holding the same digit d from NB ballots, plus one on bit NB (which
// marks invalid items, d = D) when the partition is ragged: cheaper than
// MATCH.ANY, whose latency dominated the ranking.
template <int NB, bool CHECKV>
__device__ __forceinline__ uint32_t digit_peers(uint32_t d) {
  uint32_t peers = FULL_MASK;
  if (NB > 0) peer_bit<1u>(peers, d);
  if (NB > 1) peer_bit<2u>(peers, d);
  if (NB > 2) peer_bit<4u>(peers, d);
  if (NB > 3) peer_bit<8u>(peers, d);
  if (NB > 4) peer_bit<16u>(peers, d);
  if (NB > 5) peer_bit<32u>(peers, d);
  if (NB > 6) peer_bit<64u>(peers, d);
  if (NB > 7) peer_bit<128u>(peers, d);
  if (CHECKV) peer_bit<(1u << NB)>(peers, d);
  return peers;
}

template <int ITEMS, bool VALS, typename KI, int D>
struct OSmem {
  KI keys[OS_THREADS * ITEMS];
  uint32_t vals[VALS ? OS_THREADS * ITEMS : 1];
  uint32_t whist[2][OS_THREADS / 32][D + 1];  // two ranking chains per warp (+ invalid bucket)
  uint32_t dstart[D];
  uint32_t gbase[D];
  uint32_t misc[32];
  uint16_t rank[OS_THREADS * ITEMS];
};

// Keys are in registers in warp-contiguous order: item i of lane l in warp w
// is partition element w*(ITEMS*32) + i*32 + l (the first half of a warp's
// items forms ranking chain 0, the second half chain 1, so the two chains
// are independent and the element order is (warp, chain, item, lane)).
// vmask marks valid items; cnt_valid = number of valid elements, which are
// the partition's first cnt_valid.  Writes keys (and vget(li) values) to
// their digit-sorted global positions digit_off[d] + prefix + local rank.
// Look-back status words: D per partition.
template <int ITEMS, int NB, bool VALS, typename KI, typename KO, typename KMap, typename VGet>
__device__ __forceinline__ void onesweep_partition(OSmem<ITEMS, VALS, KI, (1 << NB)> &S,
                                                   KI (&k)[ITEMS], uint32_t vmask,
                                                   uint32_t part, uint32_t cnt_valid, int shift,
                                                   const uint32_t *__restrict__ digit_off,
                                                   uint64_t *status, uint32_t epoch,
                                                   KO *__restrict__ kout, KMap kmap,
                                                   uint32_t *__restrict__ vout, VGet vget,
                                                   uint32_t n_out, FrameState *fs) {
  static_assert(ITEMS % 2 == 0, "two ranking chains");
  static_assert(NB >= 1 && NB <= 8, "digit of 1..8 bits");
  constexpr int H = ITEMS / 2;
  constexpr uint32_t D = 1u << NB, DM = D - 1u;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 2 * (OS_THREADS / 32) * (int)(D + 1); i += OS_THREADS)
    (&S.whist[0][0][0])[i] = 0;
  __syncthreads();
  uint32_t *wh0 = S.whist[0][warp], *wh1 = S.whist[1][warp];
  auto rank_items = [&](auto ragged) {
    constexpr bool CV = decltype(ragged)::value;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const uint32_t d0 = (!CV || ((vmask >> i) & 1u)) ? (uint32_t)((k[i] >> shift) & DM) : D;
      const uint32_t d1 =
          (!CV || ((vmask >> (i + H)) & 1u)) ? (uint32_t)((k[i + H] >> shift) & DM) : D;
      const uint32_t p0 = digit_peers<NB, CV>(d0);
      const uint32_t p1 = digit_peers<NB, CV>(d1);
      const uint32_t c0 = wh0[d0], c1 = wh1[d1];
      const uint32_t lt = lanemask_lt();
      __syncwarp();
      if ((p0 & lt) == 0u) wh0[d0] = c0 + __popc(p0);  // lowest peer lane updates
      if ((p1 & lt) == 0u) wh1[d1] = c1 + __popc(p1);
      __syncwarp();
      S.rank[warp * (ITEMS * 32) + i * 32 + lane] = (uint16_t)(c0 + __popc(p0 & lt));
      S.rank[warp * (ITEMS * 32) + (i + H) * 32 + lane] = (uint16_t)(c1 + __popc(p1 & lt));
    }
  };
  if (cnt_valid == (uint32_t)(OS_THREADS * ITEMS)) rank_items(std::false_type{});
  else rank_items(std::true_type{});
  __syncthreads();
  // thread dg < D: digit dg's exclusive offsets over (warp, chain) and its
  // partition total
  const uint32_t dg = tid;
  uint32_t tot = 0;
  if (dg < D) {
#pragma unroll
    for (int w = 0; w < OS_THREADS / 32; ++w) {
      const uint32_t a = S.whist[0][w][dg], b = S.whist[1][w][dg];
      S.whist[0][w][dg] = tot;
      S.whist[1][w][dg] = tot + a;
      tot += a + b;
    }
  }
  // partition-local exclusive scan of the digit totals (zero beyond D)
  constexpr int DW = (int)((D + 31) / 32);  // warps holding digits
  uint32_t inc = tot;
  if (warp < DW) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL_MASK, inc, o);
      if (lane >= o) inc += t;
    }
    if (DW > 1 && lane == 31) S.misc[1 + warp] = inc;
  }
  if (DW > 1) __syncthreads();
  if (dg < D) {
    uint32_t wpre = 0;
#pragma unroll
    for (int w = 0; w < DW; ++w) wpre += (w < warp) ? S.misc[1 + w] : 0u;
    S.dstart[dg] = wpre + inc - tot;
  }
  __syncthreads();
#ifdef LODGE_VERIFY
  if (dg < D) {  // debug builds: digit runs tile [0, cnt_valid)
    const uint32_t nxt = dg + 1 < D ? S.dstart[dg + 1] : cnt_valid;
    if (S.dstart[dg] + tot != nxt) raise_fault(fs, FAULT_STAGE);
  }
#endif
  // look-back across partitions for digit dg (threads < D), overlapped with
  // the staging of this partition's keys by every warp: the staging needs only
  // the partition-local offsets, the global scatter below needs the look-back
  if (dg < D) {
    uint64_t *st = status + (size_t)part * D;
    uint32_t excl = 0;
    if (part == 0) {
      st_store(st + dg, st_pack(epoch, ST_PREFIX, tot));
    } else {
      st_store(st + dg, st_pack(epoch, ST_AGG, tot));
#ifndef LODGE_OS_LB
#define LODGE_OS_LB 8
#endif
      constexpr int LB = LODGE_OS_LB;  // partitions read per round trip
      int64_t q = (int64_t)part - 1;
      bool done = false;
      while (!done) {
        uint64_t sv[LB];
#pragma unroll
        for (int i = 0; i < LB; ++i)
          sv[i] = (q - i >= 0) ? st_load(status + (size_t)(q - i) * D + dg)
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
    S.gbase[dg] = os_ld(digit_off + dg) + excl;
  }
  // Reconverge the warp.  Each lane spun on its own digit's predecessor cell
  // above, so the lanes leave the look-back at different times, and the
  // compiler cannot force reconvergence after a spin loop (forward progress
  // under independent thread scheduling).  A warp still diverged here would
  // reach the staging and then __syncthreads() -- bar.sync, an *aligned*
  // barrier that every lane of a warp must execute together -- part by part:
  // the barrier could release the CTA before the late lanes staged their
  // keys, and the scatter then read stale slots (round 1's intermittent
  // wrong orders under concurrent contexts).  LODGE_OS_NO_RECONVERGE
  // rebuilds that defect, for the stress tests' positive control.
#ifndef LODGE_OS_NO_RECONVERGE
  __syncwarp();
#endif
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if ((vmask >> i) & 1u) {
      const uint32_t li = warp * (ITEMS * 32) + i * 32 + lane;
      const uint32_t di = (uint32_t)((k[i] >> shift) & DM);
      const uint32_t lp = S.dstart[di] + S.whist[i < H ? 0 : 1][warp][di] + S.rank[li];
      S.keys[lp] = k[i];
      if (VALS) S.vals[lp] = vget(li);
    }
  }
  __syncthreads();
  for (uint32_t j = tid; j < cnt_valid; j += OS_THREADS) {
    const KI key = S.keys[j];
    const uint32_t dd = (uint32_t)((key >> shift) & DM);
#ifdef LODGE_VERIFY
    {  // debug builds: the staged key lies in its digit's run
      const uint32_t e = dd + 1 < D ? S.dstart[dd + 1] : cnt_valid;
      if (j < S.dstart[dd] || j >= e) raise_fault(fs, FAULT_STAGE);
    }
#endif
    const uint32_t out = S.gbase[dd] + (j - S.dstart[dd]);
    if (out >= n_out) {  // digit offsets inconsistent with the keys
      raise_fault(fs, FAULT_SCATTER);
      continue;
    }
    kout[out] = kmap(key);
    if (VALS) vout[out] = S.vals[j];
  }
}

}  // namespace lodge
