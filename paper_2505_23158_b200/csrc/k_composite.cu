// K6: per-tile front-to-back alpha compositing (reference
// src/raster.py:327-377 _composite_tile and :440-449 combine).
//
// One CTA per 16x16 tile (heaviest tiles first).  FAST: 64 threads, 4 pixels
// per thread, each warp owning a 16x8 pixel block; EXACT: 128 threads, 2
// pixels per thread, 16x4 blocks.  The tile's member list -- its sorted
// per-tile list, or its members extracted from its block's list (DESIGN.md
// 3.4) -- is consumed in batches (128 members FAST, 256 EXACT) through a
// two-stage pipeline: for batch b+1 the threads issue 16-byte cp.async
// copies of the members' 64 B payloads (plus the 64 B fp64 records in EXACT
// mode) into the idle shared-memory stage, each thread arriving on that
// stage's mbarrier when its copies land, while the warps composite batch b.
// After a stage lands each member's mean is converted once to tile-local
// fp32 in place.  Each warp then compacts (ballots) the members whose
// ellipse can reach one of its pixel centres -- the extremum of the
// quadratic form over the block's centre rectangle against the member's
// cut-off -- and walks only those, in list order.  Warp votes stop a warp
// when all its pixels have T < t_min and the CTA when all pixels have (the
// reference's per-block break is the same per-pixel rule).  Per-member max
// weights reduce in-warp with redux.sync into per-warp shared slots, maxed
// per batch, then one global atomicMax on the float bits per member and
// batch.  An optional 8-bit sRGB image is written with the final pixels.
//
// FAST: fp32 FMA/MUFU.  Both skip tests of src/raster.py:356 are folded into
// one per-splat cut-off on the quadratic form, stored with the conic in
// exponent units (internal.cuh Payload) as a guard band [lo, hi]; pixels
// whose fp32 value lies in the band re-decide in fp64 with the reference's
// operation order (rare, warp-voted branch), so skip decisions match the fp64
// reference.  The list is walked in groups of LODGE_COMP_GROUP members: their
// quadratic forms and alphas first (independent of T), then the blends in
// order.  EXACT: fp64, reproducing the blocked cumprod transmittance of the
// reference (blocks of 1024 members), so per_pixel_visible and max weights
// match it to the ulp of exp.
// Compiled with -fmad=false; the fast path fuses explicitly with fmaf.
#include <algorithm>

#include "internal.cuh"

namespace lodge {

// PH 2 (the second depth phase: few, long tiles) may use fewer pixels per
// thread, i.e. more warps per tile, than the first (LODGE_COMP_PX2).
template <bool EXACT, int PH = 0>
struct CC {
  static constexpr int CB = EXACT ? 256 : 128;  // members per batch (divides 1024)
#ifndef LODGE_COMP_PX
#define LODGE_COMP_PX 4
#endif
#ifndef LODGE_COMP_PX2
#define LODGE_COMP_PX2 2  // phase 2: 16 x 4 blocks, four warps per tile (few, long tiles)
#endif
  static constexpr int PX = EXACT ? 2 : (PH == 2 ? LODGE_COMP_PX2 : LODGE_COMP_PX);  // pixels per thread
  static constexpr int CT = 256 / PX;       // threads per CTA
  static constexpr int NW = CT / 32;        // warps; warp w owns rows [w*ROWS, (w+1)*ROWS)
  static constexpr int ROWS = 2 * PX;
};

__device__ __forceinline__ double q_ref64(double A, double B, double C, double dx, double dy) {
  // cn0*dx*dx + 2.0*cn1*dx*dy + cn2*dy*dy, NumPy left-to-right
  return __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(A, dx), dx),
                             __dmul_rn(__dmul_rn(__dmul_rn(2.0, B), dx), dy)),
                   __dmul_rn(__dmul_rn(C, dy), dy));
}

// fp64 skip decision and alpha of the reference (src/raster.py:353-357).
__device__ __forceinline__ bool ref_decide(double gx, double gy, double mx, double my,
                                           const Precise &pr, const lodge_raster_params &rp,
                                           double &alpha) {
  const double q = q_ref64(pr.A, pr.B, pr.C, __dsub_rn(gx, mx), __dsub_rn(gy, my));
  double a = __dmul_rn(pr.o, exp(__dmul_rn(-0.5, fmax(q, 0.0))));
  a = fmin(a, rp.alpha_clamp);
  alpha = a;
  return (a < rp.alpha_min) || (q > LODGE_SUPPORT_Q);  // skipped
}

// Can the ellipse {q <= cut} reach a pixel centre in [xlo,xhi] x [ylo,yhi]
// (tile-local)?  Exact minimum of the convex quadratic form over the
// rectangle (interior, else the four edges), with a margin for fp32 rounding.
// In the scaled form qs = KQ * q (KQ < 0) the minimum of q is the maximum of
// qs; the extremal points do not depend on the scale.
__device__ __forceinline__ bool ellipse_meets_block(float mx, float my, float A, float B2, float C,
                                                    float lo, float xlo, float xhi, float ylo,
                                                    float yhi) {
  if (!(lo < INFINITY)) return false;
  if (mx >= xlo && mx <= xhi && my >= ylo && my <= yhi) return true;
  const float ex0 = xlo - mx, ex1 = xhi - mx, ey0 = ylo - my, ey1 = yhi - my;
  float qmax = -INFINITY;
  // an approximate extremal coordinate only lowers the evaluated maximum at
  // second order (C * err^2), far inside the margin below
  const float hc = __fdividef(-0.5f * B2, C), ha = __fdividef(-0.5f * B2, A);
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const float dx = s ? ex1 : ex0;  // vertical edge: extremise over dy
    const float dy = fminf(fmaxf(hc * dx, ey0), ey1);
    qmax = fmaxf(qmax, A * dx * dx + B2 * dx * dy + C * dy * dy);
    const float dy2 = s ? ey1 : ey0;  // horizontal edge: extremise over dx
    const float dx2 = fminf(fmaxf(ha * dy2, ex0), ex1);
    qmax = fmaxf(qmax, A * dx2 * dx2 + B2 * dx2 * dy2 + C * dy2 * dy2);
  }
  return !(qmax < lo - 1e-3f * (1.f + fabsf(lo)));  // NaN -> meets
}

// Does every pixel centre of the block [xlo,xhi] x [ylo,yhi] keep the member
// for certain (fp32 qs > hi at every pixel, so no pixel lies in the guard
// band)?  qs = A dx^2 + B2 dx dy + C dy^2 is concave (KQ < 0), so its minimum
// over the block is at a corner; the per-pixel values the blend loop
// computes differ from exact values by a few fp32 roundings of the terms,
// and the corner values here likewise, so the test keeps a relative margin
// of 4e-6 (about 60 ulps) over the terms' magnitude.
__device__ __forceinline__ bool keeps_whole_block(float mx, float my, float A, float B2, float C,
                                                  float hi, float xlo, float xhi, float ylo,
                                                  float yhi) {
  float qmin = INFINITY, mag = 0.f;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const float dx = ((c & 1) ? xhi : xlo) - mx, dy = ((c & 2) ? yhi : ylo) - my;
    const float a = A * dx * dx, b = B2 * dx * dy, cc = C * dy * dy;
    qmin = fminf(qmin, (a + b) + cc);
    mag = fmaxf(mag, (fabsf(a) + fabsf(b)) + fabsf(cc));
  }
  return qmin > hi + 4e-6f * (mag + fabsf(hi)) + 1e-30f;  // NaN -> false
}

// Packed fp32 pairs (sm_100 FADD2 / FMUL2 / FFMA2): two independent IEEE
// round-to-nearest fp32 operations per instruction, lane by lane the same
// result as the scalar add.rn / mul.rn / fma.rn, so the FAST blend keeps its
// exact arithmetic while two pixels share each instruction.
struct __align__(8) F2 {
  float x, y;
};
__device__ __forceinline__ uint64_t f2u(F2 a) { return *reinterpret_cast<uint64_t *>(&a); }
__device__ __forceinline__ F2 u2f(uint64_t v) { return *reinterpret_cast<F2 *>(&v); }
__device__ __forceinline__ F2 f2_fma(F2 a, F2 b, F2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
  return u2f(d);
}
__device__ __forceinline__ F2 f2_add(F2 a, F2 b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(d);
}
__device__ __forceinline__ F2 f2_sub(F2 a, F2 b) {
  uint64_t d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(d);
}
__device__ __forceinline__ F2 f2_mul(F2 a, F2 b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
  return u2f(d);
}
__device__ __forceinline__ F2 f2b(float v) { return F2{v, v}; }

// 1.0f when T >= t_min (and qs > hi), else 0.0f (PTX set: FSET.BF)
__device__ __forceinline__ float keep_f(float T, float tmin) {
  float d;
  asm("set.ge.f32.f32 %0, %1, %2;" : "=f"(d) : "f"(T), "f"(tmin));
  return d;
}
__device__ __forceinline__ float keep_f(float T, float tmin, float qs, float hi) {
  float d;
  asm("{\n\t.reg .pred p;\n\t"
      "setp.ge.f32 p, %1, %2;\n\t"
      "set.gt.and.f32.f32 %0, %3, %4, p;\n\t}"
      : "=f"(d)
      : "f"(T), "f"(tmin), "f"(qs), "f"(hi));
  return d;
}

// Per-thread pixel values, addressable as scalars (s[p]) or pixel pairs
// (v[h] = pixels 2h, 2h + 1).
template <int PX>
union PxF {
  F2 v[(PX + 1) / 2];
  float s[PX];
};

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared, completion counted on `bar` (tx bytes).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

// Member staging.  cp.async (LDGSTS) 16-byte copies, four per 64 B record,
// issued by consecutive lanes, completion tracked per thread on the stage's
// mbarrier (cp.async.mbarrier.arrive.noinc: the barrier counts one arrival
// per thread).  A per-thread cp.async.bulk of each record needs uniform
// operands, and ptxas issues it lane by lane in an elect loop (~8
// instructions per lane and record: 0.5k per warp and batch, ~7% of the
// compositor's instructions at config 3); LODGE_COMP_TMA keeps that form.
__device__ __forceinline__ void cp16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_arrive(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_addr(bar))
               : "memory");
}
// the c-th 16-byte chunk of member m's staged record(s) into stage slot j
template <bool EXACT, typename Sm>
__device__ __forceinline__ void stage_chunk(Sm &S, int k, int j, int c, uint32_t m,
                                            const Payload *payload, const Precise *precise) {
  if (EXACT && c >= 4)
    cp16(reinterpret_cast<char *>(&S.pr[k][j]) + 16 * (c - 4),
         reinterpret_cast<const char *>(precise + m) + 16 * (c - 4));
  else
    cp16(reinterpret_cast<char *>(&S.pl[k][j]) + 16 * c,
         reinterpret_cast<const char *>(payload + m) + 16 * c);
}

template <bool EXACT, int PH = 0>
struct CompSmem {
  static constexpr int CB = CC<EXACT, PH>::CB;
  Payload pl[2][CB];                         // TMA destinations (64 B each)
  Precise pr[EXACT ? 2 : 1][EXACT ? CB : 1];  // EXACT: fp64 records
  uint32_t m[2][CB];                           // member splat ids (guard re-check)
  unsigned long long maxw[EXACT ? CB : 1];
  uint32_t maxw32[CC<EXACT, PH>::NW][CB];  // FAST: per warp (each member once per warp and batch)
  uint8_t wlist[CC<EXACT, PH>::NW * CB];
  uint64_t bar[2];
  uint32_t mt;  // end of the members the tile iterated (max over warps)
  uint32_t bl_mask[32];  // block-list refill: member ballots per (round item, warp), 2 rounds
  uint32_t bl_on, bl_cur, bl_end, bl_bit, bl_par;  // block-list walk (CTA-uniform, not in registers)
};

struct CompParams {
  lodge_raster_params rp;
  float tmin_f, clamp_f;
  int32_t flags, tiles_x, W, H;
  // two-phase frames
  const uint32_t *count_all;  // pairs per tile over all splats
  uint32_t *alive;            // bitmap of tiles the second phase resumes
  float4 *state;              // (T, r, g, b) per pixel of those tiles
  uint32_t n_list, n_payload;  // capacities of the list and payload buffers (bounds checks)
  uint32_t n_maxw;             // entries of the caller's max-weight buffer (bounds check)
  // block lists (phases 1 and 2 when fs->scan_a / scan_b): this phase's
  // lists, their capacity offsets and lengths (k_block_lists)
  const uint64_t *blist;
  const uint32_t *bl_start, *bl_len;
  // FAST: optional 8-bit sRGB output (lodge_frame_out.srgb8_dev) and the
  // level thresholds of lodge_to_srgb8
  uint8_t *srgb8;
  const float *srgb_thr;
};

// The number of level thresholds <= v (lodge_to_srgb8's binary search over
// the 255 thresholds in shared memory).
__device__ __forceinline__ uint32_t srgb_level(const float *thr, float v) {
  uint32_t k = 0;
#pragma unroll
  for (int st = 128; st >= 1; st >>= 1) k += (v >= thr[k + st]) ? st : 0;
  return k;
}

// A finished tile's 8-bit sRGB image as 16-byte row segments (48 B per tile
// row; the caller checks the alignment): whole sectors, so a destination in
// pinned host memory (zero-copy read-back) takes full PCIe writes.  Kept out
// of line: the compositor's walk compiles as without it.  Every thread of
// the CTA calls it (one barrier).
template <int PX, int CT>
__device__ __noinline__ void srgb_tile_rows(PxF<PX> r, PxF<PX> g, PxF<PX> b, const float *thr,
                                            uint8_t *t8, int lx, int ly0, int tx, int ty,
                                            uint8_t *out, int32_t W, int32_t H) {
#pragma unroll
  for (int p = 0; p < PX; ++p) {
    uint8_t *o8 = t8 + 3 * ((ly0 + 2 * p) * 16 + lx);
    o8[0] = (uint8_t)srgb_level(thr, fminf(fmaxf(r.s[p], 0.f), 1.f));
    o8[1] = (uint8_t)srgb_level(thr, fminf(fmaxf(g.s[p], 0.f), 1.f));
    o8[2] = (uint8_t)srgb_level(thr, fminf(fmaxf(b.s[p], 0.f), 1.f));
  }
  __syncthreads();
  for (int q = threadIdx.x; q < 48; q += CT) {
    const int row = q / 3, part = q - 3 * row, py = ty * 16 + row;
    if (py < H)
      *reinterpret_cast<uint4 *>(out + 3 * ((size_t)py * W + tx * 16) + 16 * part) =
          *reinterpret_cast<const uint4 *>(t8 + 48 * row + 16 * part);
  }
}

// MODE < 0: need_image / record_max from cpar.flags at run time (EXACT);
// otherwise bit 0 = image, bit 1 = max weights, fixed at compile time (FAST:
// no per-member branches on either)
// PH (FAST only): 0 one pass over the full lists; 1 the first depth phase of
// a two-phase frame -- a tile that still has live pixels and pairs beyond
// the phase saves (T, colour) per pixel and its visible counts and sets its
// alive bit instead of writing its image; 2 the second phase -- alive tiles
// only (tile_order lists them first, fs->n_alive of them), resumed from the
// saved state.  The per-pixel blend sequence is the one-pass sequence split
// at a member boundary, so the outputs are bitwise those of one pass.
template <bool EXACT, int MODE, int PH = 0>
#ifndef LODGE_COMP_MINB
#define LODGE_COMP_MINB 9  // FAST: resident CTAs per SM (register cap; 9 x 64 threads)
#endif
#ifndef LODGE_COMP_GROUP
#define LODGE_COMP_GROUP 4  // list members per FAST iteration
#endif
#ifndef LODGE_COMP_MINB2
#define LODGE_COMP_MINB2 7  // phase 2 with LODGE_COMP_PX2 = 2 (128 threads): 72 registers
#endif
__global__ void __launch_bounds__(CC<EXACT, PH>::CT,
                                  EXACT ? 1
                                        : (CC<EXACT, PH>::PX < LODGE_COMP_PX ? LODGE_COMP_MINB2
                                                                             : LODGE_COMP_MINB))
    k_composite(
    const uint32_t *__restrict__ list, const uint32_t *__restrict__ tile_start,
    const uint32_t *__restrict__ tile_order, const Payload *__restrict__ payload,
    const Precise *__restrict__ precise, FrameState *fs, const CompParams cpar, void *image,
    int32_t *visible, void *maxw) {
  constexpr int PX = CC<EXACT, PH>::PX, CT = CC<EXACT, PH>::CT, ROWS = CC<EXACT, PH>::ROWS;
  constexpr int CB = CC<EXACT, PH>::CB;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  CompSmem<EXACT, PH> &S = *reinterpret_cast<CompSmem<EXACT, PH> *>(smem_raw);
  const lodge_raster_params &rp = cpar.rp;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (PH == 2 && blockIdx.x >= fs->n_alive) return;
  const uint32_t t = tile_order ? tile_order[blockIdx.x] : blockIdx.x;
  const int tx = t % cpar.tiles_x, ty = t / cpar.tiles_x;
  const int lx = lane & 15, ly0 = warp * ROWS + (lane >> 4);  // pixel p at row ly0 + 2p
  const float wx_lo = 0.5f, wx_hi = 15.5f;
  const float wy_lo = (float)(warp * ROWS) + 0.5f, wy_hi = wy_lo + (float)(ROWS - 1);
  const int px = tx * 16 + lx, py0 = ty * 16 + ly0;
  const bool need_image = MODE < 0 ? (cpar.flags & LODGE_NEED_IMAGE) != 0 : (MODE & 1) != 0;
  const bool record_max =
      MODE < 0 ? (cpar.flags & LODGE_RECORD_MAX) && maxw != nullptr : (MODE & 2) != 0;
  const uint32_t s = tile_start[t];
  uint32_t e = tile_start[t + 1];
  if (fs->stats.overflow) {
    e = s;  // the pair buffers overflowed: this attempt is discarded and re-rendered
            // after they grow, and its tile ranges are stale, so they are not checked
  } else if (e < s || e > cpar.n_list) {
    if (tid == 0) raise_fault(fs, FAULT_LIST);
    e = s;
  }

  const float fpx = (float)lx + 0.5f, fpy0 = (float)ly0 + 0.5f;
  const float clamp_l2 = log2f(cpar.clamp_f) - 1e-3f;  // all-keep members stay below the clamp
  const double gx = (double)px + 0.5, gy0 = (double)py0 + 0.5;
  const double ox = (double)(tx * 16), oy = (double)(ty * 16);
  constexpr uint32_t REC = EXACT ? 128u : 64u;  // bytes staged per member

  uint32_t alive = 0;  // bit p: pixel p composites (T_before >= t_min)
#pragma unroll
  for (int p = 0; p < PX; ++p)
    if (px < cpar.W && py0 + 2 * p < cpar.H) alive |= 1u << p;

  if (tid == 0) {
#ifdef LODGE_COMP_TMA
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
#else
    mbar_init(&S.bar[0], CT);  // one cp.async arrival per thread and stage
    mbar_init(&S.bar[1], CT);
#endif
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    S.mt = s;
  }
  __syncthreads();
  // list position just past the last member this warp blended before all its
  // pixels were done (compositing work, stats.comp_members)
  uint32_t wend = s;

  // Block lists (fs->scan_a / scan_b): the tile's members are the entries of
  // its block's list with the tile's mask bit, in order; the CTA walks the
  // list from bl_cur (CTA-uniform) as it stages batches.
  if (tid == 0) {
    S.bl_on = PH == 1 ? fs->scan_a : (PH == 2 ? fs->scan_b : 0u);
    if (S.bl_on) {
      const uint32_t nbx = (cpar.tiles_x + BLK_W - 1) / BLK_W;
      const uint32_t bi = (ty / BLK_H) * nbx + tx / BLK_W;
      const uint32_t c0 = cpar.bl_start[bi];
      S.bl_cur = c0;
      S.bl_end = c0 + min(cpar.bl_len[bi], cpar.bl_start[bi + 1] - c0);
      S.bl_bit = 32u + (ty % BLK_H) * BLK_W + tx % BLK_W;
      S.bl_par = 0u;
    }
  }
  __syncthreads();
  // stage the tile's next n members from the block list into buffer k:
  // rounds of BR entries per thread; each warp publishes its member ballot
  // per round item (double-buffered by round parity, so one barrier per
  // round), every thread ranks its members from the scanned ballot counts
  // and finds the entry after the batch's last member itself
  auto issue_block = [&](int n, int k) {
    constexpr int BR = 4;
    constexpr int NW = CC<EXACT, PH>::NW;
    constexpr int NQ = BR * NW;  // (item, warp) slots of a round, item-major
    static_assert(NQ <= 16, "two rounds of slots in bl_mask");
    uint32_t bl_cur = S.bl_cur, par = S.bl_par;
    const uint32_t bl_end = S.bl_end, bl_bit = S.bl_bit;
    int got = 0;
    while (got < n) {
      uint64_t v[BR];
#pragma unroll
      for (int i = 0; i < BR; ++i) {
        const uint32_t at = bl_cur + (uint32_t)(i * CT + tid);
        v[i] = at < bl_end ? cpar.blist[at] : 0ull;
      }
      uint32_t mem = 0;
#pragma unroll
      for (int i = 0; i < BR; ++i) {
        const bool h = (v[i] >> bl_bit) & 1ull;
        const uint32_t bal = __ballot_sync(FULL_MASK, h);
        if (lane == 0) S.bl_mask[par * 16 + i * NW + warp] = bal;
        mem |= h ? (1u << i) : 0u;
      }
      __syncthreads();
      const uint32_t mk = lane < NQ ? S.bl_mask[par * 16 + lane] : 0u;
      const uint32_t c = __popc(mk);
      uint32_t inc = c;
#pragma unroll
      for (int o = 1; o < NQ; o <<= 1) {
        const uint32_t t2 = __shfl_up_sync(FULL_MASK, inc, o);
        if (lane >= o) inc += t2;
      }
      const int tot = (int)__shfl_sync(FULL_MASK, inc, NQ - 1);
      const uint32_t ex = inc - c;
#pragma unroll
      for (int i = 0; i < BR; ++i) {
        const bool h = (mem >> i) & 1u;
        const uint32_t bal = __ballot_sync(FULL_MASK, h);
        const uint32_t off = __shfl_sync(FULL_MASK, ex, i * NW + warp);
        if (h) {
          const int rank = got + (int)(off + __popc(bal & lanemask_lt()));
          if (rank < n) {
            uint32_t m = (uint32_t)v[i];
            if (m >= cpar.n_payload) {
              raise_fault(fs, FAULT_MEMBER);
              m = 0;
            }
            S.m[k][rank] = m;
#ifdef LODGE_COMP_TMA
            bulk_g2s(&S.pl[k][rank], payload + m, 64, &S.bar[k]);
#else
#pragma unroll
            for (int c = 0; c < 4; ++c) stage_chunk<EXACT>(S, k, rank, c, m, payload, precise);
#endif
          }
        }
      }
      if (got + tot >= n) {
        // the member of rank n - 1: slot q (item q / NW, warp q % NW), its
        // (need - ex_q)-th set bit
        const uint32_t need = (uint32_t)(n - 1 - got);
        const uint32_t qm = __ballot_sync(FULL_MASK, lane < NQ && ex <= need && need < ex + c);
        const int q = __ffs(qm) - 1;
        const uint32_t mq = __shfl_sync(FULL_MASK, mk, q);
        const uint32_t eq = __shfl_sync(FULL_MASK, ex, q);
        const uint32_t bitpos = __fns(mq, 0, (int)(need - eq) + 1);
        bl_cur += (uint32_t)((q / NW) * CT + (q % NW) * 32) + bitpos + 1u;
        got = n;
      } else {
        got += tot;
        bl_cur += (uint32_t)(BR * CT);
        if (bl_cur >= bl_end) {  // the list ran out before the tile's count: fill the
          if (tid == 0) raise_fault(fs, FAULT_LIST);  // stage with record 0 (no hang)
          for (int r = got + tid; r < n; r += CT) {
            S.m[k][r] = 0;
#ifdef LODGE_COMP_TMA
            bulk_g2s(&S.pl[k][r], payload, 64, &S.bar[k]);
#else
            for (int c = 0; c < 4; ++c) stage_chunk<EXACT>(S, k, r, c, 0u, payload, precise);
#endif
          }
          got = n;
        }
      }
      par ^= 1u;
    }
    // every thread stores the (identical) walk state, so its own next read
    // sees it even when no barrier separates two refills
    S.bl_cur = bl_cur;
    S.bl_par = par;
  };

  auto issue = [&](uint32_t bb, int k) {  // stage members [bb, bb+CB) into buffer k
    const int n = (int)min((uint32_t)CB, e - bb);
#ifdef LODGE_COMP_TMA
    if (tid == 0) mbar_expect_tx(&S.bar[k], (uint32_t)n * REC);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (!EXACT && PH != 0 && S.bl_on) {
      issue_block(n, k);
      return;
    }
#pragma unroll
    for (int h = 0; h < CB / CT; ++h) {
      const int j = tid + h * CT;
      if (j < n) {
        uint32_t m = list[bb + j];
        if (m >= cpar.n_payload) {
          raise_fault(fs, FAULT_MEMBER);
          m = 0;
        }
        S.m[k][j] = m;
        bulk_g2s(&S.pl[k][j], payload + m, 64, &S.bar[k]);
        if (EXACT) bulk_g2s(&S.pr[k][j], precise + m, 64, &S.bar[k]);
      }
    }
#else
    if (!EXACT && PH != 0 && S.bl_on) {
      issue_block(n, k);
    } else {
      // chunk q: member q / CPM, 16-byte piece q % CPM (consecutive lanes
      // copy one record's consecutive pieces)
      constexpr int CPM = (int)(REC / 16);
#pragma unroll
      for (int h = 0; h < CB * CPM / CT; ++h) {
        const int q = tid + h * CT, j = q / CPM, c = q % CPM;
        if (j < n) {
          uint32_t m = list[bb + j];
          if (m >= cpar.n_payload) {
            if (c == 0) raise_fault(fs, FAULT_MEMBER);
            m = 0;
          }
          if (c == 0) S.m[k][j] = m;
          stage_chunk<EXACT>(S, k, j, c, m, payload, precise);
        }
      }
    }
    cp_arrive(&S.bar[k]);  // completes when this thread's copies land
#endif
  };

  PxF<PX> Tu, cru, cgu, cbu;                           // FAST (pixel pairs for FFMA2)
  double tr[EXACT ? PX : 1], cp[EXACT ? PX : 1];      // EXACT transmittance
  double ir[EXACT ? PX : 1], ig[EXACT ? PX : 1], ib[EXACT ? PX : 1];
  double br[EXACT ? PX : 1], bg[EXACT ? PX : 1], bb[EXACT ? PX : 1];
  int32_t vis[PX];   // EXACT visible counts
  PxF<PX> vf;         // FAST visible counts, as floats (FADD2 with the 0/1 keep factors)
#pragma unroll
  for (int p = 0; p < PX; ++p) {
    Tu.s[p] = 1.f;
    cru.s[p] = cgu.s[p] = cbu.s[p] = 0.f;
    vis[p] = 0;
    vf.s[p] = 0.f;
  }
  if (EXACT) {
#pragma unroll
    for (int p = 0; p < (EXACT ? PX : 1); ++p) {
      tr[p] = cp[p] = 1.0;
      ir[p] = ig[p] = ib[p] = br[p] = bg[p] = bb[p] = 0.0;
    }
  }
  // FAST tracks liveness in T itself (T >= t_min); out-of-image pixels hold
  // T = 0: never live, and their blend factors T * a stay 0
  if (!EXACT) {
#pragma unroll
    for (int p = 0; p < PX; ++p) {
      if (!((alive >> p) & 1u)) {
        Tu.s[p] = 0.f;
      } else if (PH == 2) {  // resume the first phase's state
        const size_t pix = (size_t)(py0 + 2 * p) * cpar.W + px;
        const float4 st = cpar.state[pix];
        Tu.s[p] = st.x;
        cru.s[p] = st.y;
        cgu.s[p] = st.z;
        cbu.s[p] = st.w;
        vf.s[p] = (float)visible[pix];  // < 2^24: exact
      }
    }
  }
  auto live_any = [&]() -> bool {
    if (EXACT) return alive != 0u;
    float m = Tu.s[0];
#pragma unroll
    for (int p = 1; p < PX; ++p) m = fmaxf(m, Tu.s[p]);
    return m >= cpar.tmin_f;
  };
  uint32_t guard = 0;
#ifdef LODGE_COUNTERS
  unsigned long long c_list = 0, c_iter = 0, c_hit = 0, c_px = 0, c_batch = 0;
  unsigned long long c_akg = 0, c_nakg = 0;  // groups taken all-keep / with the band tests
#endif
  uint32_t phase0 = 0u, phase1 = 0u;

  int k = 0;
  for (uint32_t b = s; b < e; b += CB, k ^= 1) {
    const int n = (int)min((uint32_t)CB, e - b);
    // the first pass stages batches 0 and 1, later ones the next batch (in
    // flight while this one composites); one call site keeps the code small
#pragma unroll 1
    for (uint32_t bi = (b == s ? s : b + CB); bi <= b + CB && bi < e; bi += CB)
      issue(bi, (int)(((bi - s) / CB) & 1u));
    if (EXACT && b > s && ((b - s) & 1023u) == 0) {
      // block boundary of the reference's 1024-member cumprod
#pragma unroll
      for (int p = 0; p < (EXACT ? PX : 1); ++p) {
        tr[p] = __dmul_rn(cp[p], tr[p]);
        cp[p] = 1.0;
        ir[p] = __dadd_rn(ir[p], br[p]);
        ig[p] = __dadd_rn(ig[p], bg[p]);
        ib[p] = __dadd_rn(ib[p], bb[p]);
        br[p] = bg[p] = bb[p] = 0.0;
      }
    }
    if (k == 0) { mbar_wait(&S.bar[0], phase0); phase0 ^= 1u; }
    else { mbar_wait(&S.bar[1], phase1); phase1 ^= 1u; }
    Payload *PL = S.pl[k];
    // tile-local fp32 mean, written over the fp64 mean in FAST mode (the
    // fp64 mean stays in global memory for the rare re-check)
#pragma unroll
    for (int h = 0; h < CB / CT; ++h) {
      const int j = tid + h * CT;
      if (j < n) {
        Payload &pj = PL[j];
        if (!EXACT) {
          // (mx, my, mid, half): the guard band [lo, hi] as a centre and a
          // half-width that covers it after rounding, so the per-pixel near
          // test is |qs - mid| <= half (half = inf: always near; -1: never)
          const float mxl = (float)(pj.mx - ox), myl = (float)(pj.my - oy);
          const float hi = pj.hi, lo = pj.lo;
          float mid = 0.f, half = -1.f;
          if (lo <= hi && fabsf(lo) < INFINITY && fabsf(hi) < INFINITY) {
            mid = 0.5f * (lo + hi);
            half = fmaxf(__fsub_ru(hi, mid), __fsub_ru(mid, lo));
          } else if (lo < INFINITY) {
            half = INFINITY;
          }
          reinterpret_cast<float4 *>(&pj.mx)[0] = make_float4(mxl, myl, mid, half);
#pragma unroll
          for (int w2 = 0; w2 < CC<EXACT, PH>::NW; ++w2) S.maxw32[w2][j] = 0u;
        } else {
          S.maxw[j] = 0ull;
        }
      }
    }
    __syncthreads();
    // per-warp member list: members whose ellipse can reach a pixel centre
    uint8_t *wl = S.wlist + warp * CB;
    const uint32_t wl_sa = smem_addr(wl);  // read back with 32-bit shared addressing
    int cnt = 0;
    const bool alive0 = __any_sync(FULL_MASK, live_any());
    int done_i = 0;  // list entries this warp went through in this batch
    if (alive0) {
      for (int q0 = 0; q0 < n; q0 += 32) {
        const int j = q0 + lane;
        bool hit = false;
        if (j < n) {
          const Payload &pj = PL[j];
          float mxl, myl;
          if (EXACT) {
            mxl = (float)(pj.mx - ox);
            myl = (float)(pj.my - oy);
          } else {
            const float2 mm = reinterpret_cast<const float2 *>(&pj.mx)[0];
            mxl = mm.x;
            myl = mm.y;
          }
          hit = !(mxl + pj.bx < wx_lo || mxl - pj.bx > wx_hi || myl + pj.by < wy_lo ||
                  myl - pj.by > wy_hi) &&
                ellipse_meets_block(mxl, myl, pj.As, pj.B2s, pj.Cs, pj.lo, wx_lo, wx_hi, wy_lo,
                                    wy_hi);
        }
        // FAST (128-member batches): bit 7 of the entry marks a member every
        // pixel of the block keeps for certain (the blend loop then skips the
        // guard band)
        bool ak = false;
        if (!EXACT && hit) {
          const Payload &pj = PL[j];
          const float2 mm = reinterpret_cast<const float2 *>(&pj.mx)[0];
          // ... and whose alpha never reaches the clamp (log2 o a margin below
          // log2 clamp; qs <= 0 up to rounding), so the clamp is a no-op too
          ak = pj.lo2 < clamp_l2 &&
               keeps_whole_block(mm.x, mm.y, pj.As, pj.B2s, pj.Cs, pj.hi, wx_lo, wx_hi, wy_lo,
                                 wy_hi);
        }
        const uint32_t hm = __ballot_sync(FULL_MASK, hit);
        if (hit) wl[cnt + __popc(hm & lanemask_lt())] = (uint8_t)(j | (ak ? 0x80 : 0));
        cnt += __popc(hm);
      }
    }
    __syncwarp();
#ifdef LODGE_COUNTERS
    c_list += cnt;
    c_batch += 1;
#endif
    if (EXACT) {
      for (int i = 0; i < cnt; ++i, done_i = i) {
        if (!__any_sync(FULL_MASK, live_any())) break;
#ifdef LODGE_COUNTERS
        c_iter += 1;
#endif
        const int j = lds_u8(wl_sa + (uint32_t)i);  // EXACT: 256-member batches, no flag
        const Payload &pj = PL[j];
          const Precise &d = S.pr[k][j];
          double wmax = 0.0;
  #pragma unroll
          for (int p = 0; p < PX; ++p) {
            if (!((alive >> p) & 1u)) continue;
            double a;
            const bool sk = ref_decide(gx, gy0 + 2.0 * p, pj.mx, pj.my, d, rp, a);
            if (sk) a = 0.0;
            const double before = __dmul_rn(cp[p], tr[p]);
            cp[p] = __dmul_rn(cp[p], __dsub_rn(1.0, a));
            const double w = __dmul_rn(before, a);
            if (need_image) {
              br[p] = __dadd_rn(br[p], __dmul_rn(w, d.r));
              bg[p] = __dadd_rn(bg[p], __dmul_rn(w, d.g));
              bb[p] = __dadd_rn(bb[p], __dmul_rn(w, d.b));
            }
            vis[p] += sk ? 0 : 1;
            if (!(__dmul_rn(cp[p], tr[p]) >= rp.t_min)) alive &= ~(1u << p);
            wmax = fmax(wmax, w);
          }
          if (record_max) {
            unsigned long long wb = (unsigned long long)__double_as_longlong(wmax);
  #pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              const unsigned long long ob = __shfl_xor_sync(FULL_MASK, wb, o);
              wb = ob > wb ? ob : wb;
            }
            if (lane == 0 && wb) atomicMax(&S.maxw[j], wb);
          }
      }
    } else {
      // qs = KQ * q in exponent units: keep iff qs > hi (and the pixel is
      // alive: T >= t_min; out-of-image pixels hold T = -inf), re-decide in
      // fp64 iff lo <= qs <= hi, alpha = min(exp2(qs + log2 o), clamp)
      // band: test the guard band (members not flagged all-keep)
      auto quad = [&](const Payload &pj, float (&qs)[PX], float4 &mm, float4 &cn,
                      const bool band) -> bool {
        mm = reinterpret_cast<const float4 *>(&pj.mx)[0];  // mx, my, mid, half
        cn = *reinterpret_cast<const float4 *>(&pj.As);   // KQ*(A, 2B, C), log2 o
        const float dx = fpx - mm.x;
        const float adx2 = cn.x * dx * dx, bdx = cn.y * dx;
        bool near = false;  // dead pixels may vote too; the fp64 path re-checks
#pragma unroll
        for (int p = 0; p < PX; ++p) {
          const float dy = (fpy0 + 2.f * p) - mm.y;
          qs[p] = fmaf(dy, fmaf(cn.z, dy, bdx), adx2);
          if (band) near |= fabsf(qs[p] - mm.z) <= mm.w;
        }
        return near;
      };
      // the same quadratic forms two pixels at a time (FFMA2; lane for lane
      // the scalar fmaf chain above)
      auto quad2 = [&](const Payload &pj, PxF<PX> &qs, float4 &mm, float4 &cn,
                       const bool band) -> bool {
        mm = reinterpret_cast<const float4 *>(&pj.mx)[0];  // mx, my, mid, half
        cn = *reinterpret_cast<const float4 *>(&pj.As);   // KQ*(A, 2B, C), log2 o
        const float dx = fpx - mm.x;
        const float adx2 = cn.x * dx * dx, bdx = cn.y * dx;
        bool near = false;
#pragma unroll
        for (int h = 0; h < PX / 2; ++h) {
          const F2 dy = f2_sub(F2{fpy0 + 4.f * h, fpy0 + 4.f * h + 2.f}, f2b(mm.y));
          qs.v[h] = f2_fma(dy, f2_fma(f2b(cn.z), dy, f2b(bdx)), f2b(adx2));
          if (band) {
            near |= fabsf(qs.v[h].x - mm.z) <= mm.w;
            near |= fabsf(qs.v[h].y - mm.z) <= mm.w;
          }
        }
        return near;
      };
      auto colour = [&](const Payload &pj) {
        return need_image ? *reinterpret_cast<const float4 *>(&pj.r)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
      };
      // lane 0 stores a member's warp-wide weight into the warp's own slot
      // (a member comes once per warp and batch: a plain predicated store;
      // ptxas branches around predicated shared atomics), the warps' slots
      // are maxed when the batch is flushed
      const uint32_t maxw_sa = smem_addr(&S.maxw32[warp][0]);
      auto record = [&](int j, unsigned wb) {
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "setp.eq.u32 p, %2, 0;\n\t"
                     "@p st.shared.u32 [%0], %1;\n\t}"
                     :: "r"(maxw_sa + 4u * (uint32_t)j), "r"(wb), "r"(lane)
                     : "memory");
      };
      auto finish = [&](int j, float wmax) {
#ifdef LODGE_COUNTERS
        c_hit += __any_sync(FULL_MASK, wmax > 0.f) ? 1 : 0;
#endif
        if (record_max) record(j, __reduce_max_sync(FULL_MASK, __float_as_uint(wmax)));
      };
      // one pixel's blend step with every decision certain in fp32; one PTX
      // block keeps the keep test a predicate (nvcc otherwise materialises
      // the count increment as a select and a copy)
      auto step = [&](int p, float qs, float hi, float a, const float4 &c, float &wmax,
                      const bool all_keep) {
        float w;
        if (all_keep) {  // qs > hi at every pixel of the block
          asm("{\n\t.reg .pred k;\n\t"
              "setp.ge.f32 k, %2, %3;\n\t"
              "mul.rn.f32 %0, %2, %4;\n\t"
              "selp.f32 %0, %0, 0f00000000, k;\n\t"
              "@k add.rn.f32 %1, %1, 0f3F800000;\n\t}"
              : "=f"(w), "+f"(vf.s[p])
              : "f"(Tu.s[p]), "f"(cpar.tmin_f), "f"(a));
        } else {
          asm("{\n\t.reg .pred k;\n\t"
              "setp.ge.f32 k, %2, %4;\n\t"
              "setp.gt.and.f32 k, %3, %5, k;\n\t"
              "mul.rn.f32 %0, %2, %6;\n\t"
              "selp.f32 %0, %0, 0f00000000, k;\n\t"
              "@k add.rn.f32 %1, %1, 0f3F800000;\n\t}"
              : "=f"(w), "+f"(vf.s[p])
              : "f"(Tu.s[p]), "f"(qs), "f"(cpar.tmin_f), "f"(hi), "f"(a));
        }
        if (need_image) {
          cru.s[p] = fmaf(w, c.x, cru.s[p]);
          cgu.s[p] = fmaf(w, c.y, cgu.s[p]);
          cbu.s[p] = fmaf(w, c.z, cbu.s[p]);
        }
        Tu.s[p] -= w;
        wmax = fmaxf(wmax, w);
#ifdef LODGE_COUNTERS
        c_px += (w > 0.f) ? 1 : 0;
#endif
      };
      // the blend step for pixels 2h and 2h + 1 (the same operations as
      // step, paired): the keep decisions as 0/1 factors (PTX set.f32:
      // FSET, one ALU op per pixel), w = (T * a) * k -- bitwise the selected
      // T * a or +0, T * a being finite and >= 0 -- and the visible counts
      // += k, all as FMUL2 / FADD2 on the FMA pipe
      auto step2 = [&](int h, F2 qs, float hi, F2 a, const float4 &c, float &wmax,
                       const bool all_keep) {
        const int p0 = 2 * h, p1 = 2 * h + 1;
        F2 kf;
        if (all_keep) {
          kf.x = keep_f(Tu.s[p0], cpar.tmin_f);
          kf.y = keep_f(Tu.s[p1], cpar.tmin_f);
        } else {
          kf.x = keep_f(Tu.s[p0], cpar.tmin_f, qs.x, hi);
          kf.y = keep_f(Tu.s[p1], cpar.tmin_f, qs.y, hi);
        }
        const F2 w = f2_mul(f2_mul(Tu.v[h], a), kf);
        vf.v[h] = f2_add(vf.v[h], kf);
        if (need_image) {
          cru.v[h] = f2_fma(w, f2b(c.x), cru.v[h]);
          cgu.v[h] = f2_fma(w, f2b(c.y), cgu.v[h]);
          cbu.v[h] = f2_fma(w, f2b(c.z), cbu.v[h]);
        }
        Tu.v[h] = f2_sub(Tu.v[h], w);
        wmax = fmaxf(wmax, fmaxf(w.x, w.y));
#ifdef LODGE_COUNTERS
        c_px += (w.x > 0.f ? 1 : 0) + (w.y > 0.f ? 1 : 0);
#endif
      };
      // one member, including the guard band: pixels whose fp32 qs is within
      // the band re-decide in fp64 with the reference's op order (rare)
      auto one = [&](int j) {
#ifdef LODGE_COUNTERS
        c_iter += 1;
#endif
        const Payload &pj = PL[j];
        float qs[PX];
        float4 mm, cn;
        const bool near = quad(pj, qs, mm, cn, true);
        const float hi = pj.hi;
        const float4 c = colour(pj);
        float wmax = 0.f;
        if (__any_sync(FULL_MASK, near)) {
          const float lo = pj.lo;
          bool kp[PX];
          float a[PX];
#pragma unroll
          for (int p = 0; p < PX; ++p) {
            kp[p] = Tu.s[p] >= cpar.tmin_f && qs[p] > hi;
            a[p] = fminf(ex2_approx(qs[p] + cn.w), cpar.clamp_f);
          }
          if (near) {
            const uint32_t m = S.m[k][j];
            const Payload pg = payload[m];
            const Precise pr = precise[m];
#pragma unroll
            for (int p = 0; p < PX; ++p) {
              if (Tu.s[p] >= cpar.tmin_f && qs[p] >= lo && !(qs[p] > hi)) {
                double ad;
                kp[p] = !ref_decide(gx, gy0 + 2.0 * p, pg.mx, pg.my, pr, rp, ad);
                a[p] = (float)ad;
                ++guard;
              }
            }
          }
#pragma unroll
          for (int p = 0; p < PX; ++p) {
            const float w = kp[p] ? Tu.s[p] * a[p] : 0.f;
            if (need_image) {
              cru.s[p] = fmaf(w, c.x, cru.s[p]);
              cgu.s[p] = fmaf(w, c.y, cgu.s[p]);
              cbu.s[p] = fmaf(w, c.z, cbu.s[p]);
            }
            Tu.s[p] -= w;
            if (kp[p]) vf.s[p] += 1.f;
            wmax = fmaxf(wmax, w);
#ifdef LODGE_COUNTERS
            c_px += kp[p] ? 1 : 0;
#endif
          }
        } else {
#pragma unroll
          for (int p = 0; p < PX; ++p)
            step(p, qs[p], hi, fminf(ex2_approx(qs[p] + cn.w), cpar.clamp_f), c, wmax, false);
        }
        finish(j, wmax);
      };
      // G consecutive members: all quadratic forms and alphas first (they do
      // not depend on T), then the blend steps in list order
      // ak: every member of the group is flagged all-keep for this warp's
      // block: no guard band, no keep test beyond T >= t_min
      constexpr int G = LODGE_COMP_GROUP;
      // returns false (nothing blended) when a pixel of the warp falls in a
      // member's guard band: the caller then takes the members one by one
      auto group = [&](const int (&js)[G], const bool AK) -> bool {
        static_assert(PX % 2 == 0, "pixel pairs");
        PxF<PX> q[G];
        float4 mm[G], cn[G];
        bool near = false;
#pragma unroll
        for (int u = 0; u < G; ++u)
          near |= quad2(PL[js[u]], q[u], mm[u], cn[u], !AK);
        if (!AK && __any_sync(FULL_MASK, near)) return false;
#ifdef LODGE_COUNTERS
        c_iter += G;
        if (AK) ++c_akg;
        else ++c_nakg;
#endif
        PxF<PX> a[G];
#pragma unroll
        for (int u = 0; u < G; ++u)
#pragma unroll
          for (int h = 0; h < PX / 2; ++h) {
            const F2 e = f2_add(q[u].v[h], f2b(cn[u].w));
            const float a0 = ex2_approx(e.x), a1 = ex2_approx(e.y);
            a[u].v[h] = AK ? F2{a0, a1}
                           : F2{fminf(a0, cpar.clamp_f), fminf(a1, cpar.clamp_f)};
          }
        float wm[G];
#pragma unroll
        for (int u = 0; u < G; ++u) {
          const Payload &pj = PL[js[u]];
          const float hi = pj.hi;
          const float4 c = colour(pj);
          wm[u] = 0.f;
#pragma unroll
          for (int h = 0; h < PX / 2; ++h) step2(h, q[u].v[h], hi, a[u].v[h], c, wm[u], AK);
        }
        if (record_max) {  // the group's warp reductions back to back
          unsigned wb[G];
#pragma unroll
          for (int u = 0; u < G; ++u) wb[u] = __reduce_max_sync(FULL_MASK, __float_as_uint(wm[u]));
#pragma unroll
          for (int u = 0; u < G; ++u) record(js[u], wb[u]);
        }
#ifdef LODGE_COUNTERS
#pragma unroll
        for (int u = 0; u < G; ++u) c_hit += __any_sync(FULL_MASK, wm[u] > 0.f) ? 1 : 0;
#endif
        return true;
      };
      // groups of G members; a member is taken alone (one, a single call
      // site: the kernel's code stays small) at the list's tail and when its
      // group meets the guard band -- the next group then starts after it
      int i = 0;
      while (i < cnt) {
        if (!__any_sync(FULL_MASK, live_any())) break;
        if (i + G <= cnt) {
          int js[G];
          uint32_t allk = 0x80;
#pragma unroll
          for (int u = 0; u < G; ++u) {
            const uint32_t ent = lds_u8(wl_sa + (uint32_t)(i + u));
            js[u] = (int)(ent & 0x7f);
            allk &= ent;
          }
          if (allk ? group(js, true) : group(js, false)) {
            i += G;
            continue;
          }
        }
        one(lds_u8(wl_sa + (uint32_t)i) & 0x7f);
        ++i;
      }
      done_i = i;
    }
    if (alive0 && done_i > 0 && !__any_sync(FULL_MASK, live_any()))
      wend = b + (lds_u8(wl_sa + (uint32_t)(done_i - 1)) & (EXACT ? 0xffu : 0x7fu)) + 1u;
    __syncthreads();
    if (record_max) {
#pragma unroll
      for (int h = 0; h < CB / CT; ++h) {
        const int j = tid + h * CT;
        if (j < n) {
          const uint32_t src = PL[j].src;
          if (src >= cpar.n_maxw) {  // an input beyond the max-weight buffer
            raise_fault(fs, FAULT_SRC);
            continue;
          }
          if (EXACT) {
            if (S.maxw[j]) atomicMax(reinterpret_cast<unsigned long long *>(maxw) + src, S.maxw[j]);
          } else {
            uint32_t mw = S.maxw32[0][j];
#pragma unroll
            for (int w2 = 1; w2 < CC<EXACT, PH>::NW; ++w2) mw = max(mw, S.maxw32[w2][j]);
            if (mw) atomicMax(reinterpret_cast<unsigned int *>(maxw) + src, mw);
          }
        }
      }
    }
    // also the WAR barrier: buffer k is re-filled by the next-but-one issue
    if (__syncthreads_count(live_any()) == 0) {
      if (b + CB < e) {  // drain the stage already in flight before exiting
        if (k == 0) mbar_wait(&S.bar[1], phase1);
        else mbar_wait(&S.bar[0], phase0);
      }
      break;
    }
  }
  if (!EXACT && guard) atomicAdd(&fs->stats.guard_hits, guard);
#ifdef LODGE_COUNTERS
  if (lane == 0) {  // per warp: list entries, iterations, iterations with a hit, batches
    atomicAdd(&fs->counters[0], c_list);
    atomicAdd(&fs->counters[1], c_iter);
    atomicAdd(&fs->counters[2], c_hit);
    atomicAdd(&fs->counters[4], c_batch);
    atomicAdd(&fs->counters[5], c_akg);
    atomicAdd(&fs->counters[6], c_nakg);
  }
  atomicAdd(&fs->counters[3], c_px);  // pixel evaluations inside the cut-off
  // counters[5] / [6]: all-keep / band-tested groups (per warp)
#endif
  {  // members iterated (SURVEY.md 8d m_t): the whole list while a pixel is
     // still alive, else the furthest member a warp blended before its pixels
     // were done
    if (lane == 0) atomicMax(&S.mt, wend);
    const int live = __syncthreads_or(live_any());
    if (tid == 0) atomicAdd(&fs->stats.comp_members, live ? e - s : S.mt - s);
  }
  bool resume = false;  // PH 1: the second phase continues this tile
  if (PH == 1) {
    resume = __syncthreads_count(live_any()) > 0 && cpar.count_all[t] > e - s;
    if (resume && tid == 0) atomicOr(&cpar.alive[t >> 5], 1u << (t & 31));
  }
  // 8-bit sRGB of the final pixels (FAST): the level thresholds in the
  // staging buffers, free after the batch loop (no copies in flight)
  const bool srgb = !EXACT && need_image && cpar.srgb8 != nullptr && !(PH == 1 && resume);
  float *thr = reinterpret_cast<float *>(&S.pl[0][0]);
  if (!EXACT && need_image && cpar.srgb8 != nullptr) {  // CTA-uniform
    __syncthreads();
    for (int i = tid; i < 256; i += CT) thr[i] = cpar.srgb_thr[i];
    __syncthreads();
  }
  auto level = [&](float v) -> uint32_t {  // the number of thresholds <= v
    uint32_t k = 0;
#pragma unroll
    for (int st = 128; st >= 1; st >>= 1) k += (v >= thr[k + st]) ? st : 0;
    return k;
  };
  // the 8-bit tile goes out as 16-byte row segments when the frame width
  // keeps them aligned (srgb_tile_rows)
#ifndef LODGE_SRGB_ROWS
#define LODGE_SRGB_ROWS 1
#endif
  const bool srgb_rows = LODGE_SRGB_ROWS && srgb && (cpar.W & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(cpar.srgb8) & 15) == 0;
  if (srgb_rows)  // CTA-uniform
    srgb_tile_rows<PX, CT>(cru, cgu, cbu, thr, reinterpret_cast<uint8_t *>(&S.pl[1][0]), lx, ly0,
                           tx, ty, cpar.srgb8, cpar.W, cpar.H);
#pragma unroll
  for (int p = 0; p < PX; ++p) {
    const int py = py0 + 2 * p;
    if (!(px < cpar.W && py < cpar.H)) continue;
    const size_t pix = (size_t)py * cpar.W + px;
    if (visible) visible[pix] = EXACT ? vis[p] : (int32_t)vf.s[p];
    if (srgb && !srgb_rows) {  // byte for byte lodge_to_srgb8 of the clipped float image
      uint8_t *o8 = cpar.srgb8 + 3 * pix;
      o8[0] = (uint8_t)level(fminf(fmaxf(cru.s[p], 0.f), 1.f));
      o8[1] = (uint8_t)level(fminf(fmaxf(cgu.s[p], 0.f), 1.f));
      o8[2] = (uint8_t)level(fminf(fmaxf(cbu.s[p], 0.f), 1.f));
    }
    if (PH == 1 && resume) {
      cpar.state[pix] = make_float4(Tu.s[p], cru.s[p], cgu.s[p], cbu.s[p]);
      continue;
    }
    if (!(need_image && image)) continue;
    if (EXACT) {
      const int pe = EXACT ? p : 0;
      const double r = __dadd_rn(ir[pe], br[pe]), g = __dadd_rn(ig[pe], bg[pe]),
                   b2 = __dadd_rn(ib[pe], bb[pe]);
      double *im = reinterpret_cast<double *>(image) + 3 * pix;
      im[0] = fmin(fmax(r, 0.0), 1.0);
      im[1] = fmin(fmax(g, 0.0), 1.0);
      im[2] = fmin(fmax(b2, 0.0), 1.0);
    } else {
      float *im = reinterpret_cast<float *>(image) + 3 * pix;
      im[0] = fminf(fmaxf(cru.s[p], 0.f), 1.f);
      im[1] = fminf(fmaxf(cgu.s[p], 0.f), 1.f);
      im[2] = fminf(fmaxf(cbu.s[p], 0.f), 1.f);
    }
  }
}

template <bool EXACT, int MODE, int PH = 0>
static void launch_comp(const Work &w, FrameState *fs, int32_t W, int32_t H,
                        const lodge_raster_params &rp, int32_t flags, const lodge_frame_out &out,
                        uint32_t n_maxw, cudaStream_t s) {
  const int32_t tiles_x = (W + 15) / 16, tiles_y = (H + 15) / 16;
  const unsigned T = (unsigned)(tiles_x * tiles_y);
  const size_t sm = sizeof(CompSmem<EXACT, PH>);
  static PerDevice attr;
  if (!attr()) {
    cudaFuncSetAttribute(k_composite<EXACT, MODE, PH>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr() = 1;
  }
  CompParams cp;
  cp.rp = rp;
  cp.tmin_f = (float)rp.t_min;
  cp.clamp_f = (float)rp.alpha_clamp;
  cp.flags = flags;
  cp.tiles_x = tiles_x;
  cp.W = W;
  cp.H = H;
  cp.count_all = w.count_all;
  cp.alive = w.alive;
  cp.state = w.state;
  cp.n_list = (uint32_t)std::min<int64_t>(2 * w.P_cap, 0xffffffffll);
  cp.n_payload = (uint32_t)w.M_cap;
  cp.n_maxw = n_maxw;
  const uint32_t nb = (uint32_t)block_count(tiles_x, tiles_y);
  cp.blist = PH ? w.pairs[PH - 1] : nullptr;
  cp.bl_start = w.bl_start + (PH == 2 ? nb + 1 : 0);
  cp.bl_len = w.bl_len + (PH == 2 ? nb : 0);
  cp.srgb8 = EXACT ? nullptr : reinterpret_cast<uint8_t *>(out.srgb8_dev);
  cp.srgb_thr = w.srgb_thr;
  k_composite<EXACT, MODE, PH><<<T, CC<EXACT, PH>::CT, sm, s>>>(
      w.list, PH == 2 ? w.tile_start_b : w.tile_start, PH == 2 ? w.tile_order_b : w.tile_order,
      w.payload, w.precise, fs, cp, out.image_dev, out.visible_dev, out.maxw_dev);
}

template <int MODE>
static void launch_fast(const Work &w, FrameState *fs, int32_t W, int32_t H,
                        const lodge_raster_params &rp, int32_t flags, const lodge_frame_out &out,
                        uint32_t n_maxw, cudaStream_t s, int phase) {
  switch (phase) {
    case 1: launch_comp<false, MODE, 1>(w, fs, W, H, rp, flags, out, n_maxw, s); break;
    case 2: launch_comp<false, MODE, 2>(w, fs, W, H, rp, flags, out, n_maxw, s); break;
    default: launch_comp<false, MODE, 0>(w, fs, W, H, rp, flags, out, n_maxw, s); break;
  }
}

void launch_composite(const Work &w, FrameState *fs, const lodge_camera *, int32_t W, int32_t H,
                      const lodge_raster_params &rp, int32_t flags, int32_t exact,
                      const lodge_frame_out &out, uint32_t n_maxw, cudaStream_t s, int phase) {
  if (exact) {
    launch_comp<true, -1>(w, fs, W, H, rp, flags, out, n_maxw, s);
    return;
  }
  const int mode = ((flags & LODGE_NEED_IMAGE) ? 1 : 0) |
                   (((flags & LODGE_RECORD_MAX) && out.maxw_dev) ? 2 : 0);
  switch (mode) {
    case 3: launch_fast<3>(w, fs, W, H, rp, flags, out, n_maxw, s, phase); break;
    case 2: launch_fast<2>(w, fs, W, H, rp, flags, out, n_maxw, s, phase); break;
    case 1: launch_fast<1>(w, fs, W, H, rp, flags, out, n_maxw, s, phase); break;
    default: launch_fast<0>(w, fs, W, H, rp, flags, out, n_maxw, s, phase); break;
  }
}

// Compat / inspection: export the sorted per-tile lists as source indices.
__global__ void k_export_lists(const uint32_t *list, const uint32_t *tile_start,
                               const Payload *payload, FrameState *fs, int32_t T,
                               int64_t *tile_offsets, int64_t *tile_src, int64_t cap) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= T) tile_offsets[i] = tile_start[i];
  const uint32_t P = fs->n_pairs;
  if (i < P && i < cap) tile_src[i] = payload[list[i]].src;
}

void launch_export_lists(const Work &w, FrameState *fs, int32_t T, int64_t *tile_offsets,
                         int64_t *tile_src, int64_t cap, cudaStream_t s) {
  const int64_t n = cap > (int64_t)T + 1 ? cap : (int64_t)T + 1;
  k_export_lists<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(w.list, w.tile_start, w.payload,
                                                             fs, T, tile_offsets, tile_src, cap);
}

}  // namespace lodge
