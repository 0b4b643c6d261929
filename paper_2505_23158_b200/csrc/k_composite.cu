// K6: per-tile front-to-back alpha compositing (reference
// src/raster.py:327-377 _composite_tile and :440-449 combine).
//
// One CTA of 128 threads per 16x16 tile (heaviest tiles first); each warp
// owns an 8x8 pixel block, each thread two pixels (rows ly and ly+4).  The
// tile's sorted member list is consumed in batches of 256 members through a
// two-stage TMA pipeline: for batch b+1 each thread issues cp.async.bulk
// copies of two members' 64 B payloads (plus the 64 B fp64 records in EXACT
// mode) into the idle shared-memory stage, completing on that stage's
// mbarrier, while the warps composite batch b.  After a stage lands, each
// member's mean is converted once to tile-local fp32 in place.  Each warp
// then compacts (8 ballots) the members whose pixel box meets its 8x8 block
// -- the others give its pixels weight 0 -- and walks only those, in list
// order.  Warp votes stop a warp when all its pixels have T < t_min and the
// CTA when all pixels have (the reference's per-block break is the same
// per-pixel rule).  Per-member max weights reduce in-warp with redux.sync,
// per CTA with shared-memory atomics, then one global atomicMax on the float
// bits per member and batch.
//
// FAST: fp32 FMA/MUFU, branch-free.  Both skip tests of src/raster.py:356
// are folded into one per-splat cut-off q_eff on the quadratic form; pixels
// whose fp32 q lies within the splat's error bound of q_eff re-decide in fp64
// with the reference's operation order (rare, warp-voted branch), so skip
// decisions match the fp64 reference.  EXACT: fp64, reproducing the blocked
// cumprod transmittance of the reference (blocks of 1024 members), so
// per_pixel_visible and max weights match it to the ulp of exp.
// Compiled with -fmad=false; the fast path fuses explicitly with fmaf.
#include "internal.cuh"

namespace lodge {

constexpr int CB = 256;      // members per batch
constexpr int CT = 128;      // threads per CTA (4 warps x 8x8 pixels, 2 per thread)
constexpr int NW = CT / 32;

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

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
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

template <bool EXACT>
struct CompSmem {
  Payload pl[2][CB];                           // TMA destinations (64 B each)
  Precise pr[EXACT ? 2 : 1][EXACT ? CB : 1];  // EXACT: fp64 records
  uint32_t m[2][CB];                           // member splat ids (guard re-check)
  unsigned long long maxw[EXACT ? CB : 1];
  uint32_t maxw32[CB];
  uint8_t wlist[NW * CB];
  uint64_t bar[2];
};

struct CompParams {
  lodge_raster_params rp;
  float tmin_f, clamp_f;
  int32_t flags, tiles_x, W, H;
};

template <bool EXACT>
__global__ void __launch_bounds__(CT) k_composite(const uint64_t *__restrict__ pairs,
                                                  const uint32_t *__restrict__ tile_start,
                                                  const uint32_t *__restrict__ tile_order,
                                                  const Payload *__restrict__ payload,
                                                  const Precise *__restrict__ precise,
                                                  FrameState *fs, const CompParams cpar,
                                                  void *image, int32_t *visible, void *maxw) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  CompSmem<EXACT> &S = *reinterpret_cast<CompSmem<EXACT> *>(smem_raw);
  const lodge_raster_params &rp = cpar.rp;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t t = tile_order ? tile_order[blockIdx.x] : blockIdx.x;
  const int tx = t % cpar.tiles_x, ty = t / cpar.tiles_x;
  const int lx = (warp & 1) * 8 + (lane & 7), ly0 = (warp >> 1) * 8 + (lane >> 3);
  const float wx_lo = (float)((warp & 1) * 8) + 0.5f, wx_hi = wx_lo + 7.0f;
  const float wy_lo = (float)((warp >> 1) * 8) + 0.5f, wy_hi = wy_lo + 7.0f;
  const int px = tx * 16 + lx, py0 = ty * 16 + ly0, py1 = py0 + 4;
  const bool in0 = px < cpar.W && py0 < cpar.H, in1 = px < cpar.W && py1 < cpar.H;
  const bool need_image = cpar.flags & LODGE_NEED_IMAGE;
  const bool record_max = (cpar.flags & LODGE_RECORD_MAX) && maxw != nullptr;
  const uint32_t s = tile_start[t];
  uint32_t e = tile_start[t + 1];
  if (fs->stats.overflow) e = s;

  const float fpx = (float)lx + 0.5f, fpy0 = (float)ly0 + 0.5f, fpy1 = fpy0 + 4.0f;
  const double gx = (double)px + 0.5, gy0 = (double)py0 + 0.5, gy1 = gy0 + 4.0;
  const double ox = (double)(tx * 16), oy = (double)(ty * 16);
  constexpr uint32_t REC = EXACT ? 128u : 64u;  // bytes staged per member

  if (tid == 0) {
    mbar_init(&S.bar[0], 1);
    mbar_init(&S.bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto issue = [&](uint32_t bb, int k) {  // stage members [bb, bb+256) into buffer k
    const int n = (int)min((uint32_t)CB, e - bb);
    if (tid == 0) mbar_expect_tx(&S.bar[k], (uint32_t)n * REC);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
    for (int h = 0; h < CB / CT; ++h) {
      const int j = tid + h * CT;
      if (j < n) {
        const uint32_t m = (uint32_t)pairs[bb + j];
        S.m[k][j] = m;
        bulk_g2s(&S.pl[k][j], payload + m, 64, &S.bar[k]);
        if (EXACT) bulk_g2s(&S.pr[k][j], precise + m, 64, &S.bar[k]);
      }
    }
  };

  // FAST state (two pixels)
  float T0 = 1.f, T1 = 1.f, r0 = 0.f, g0 = 0.f, b0 = 0.f, r1 = 0.f, g1 = 0.f, b1 = 0.f;
  // EXACT state: per pixel trans, block cumprod, image, block image
  double tr0 = 1.0, cp0 = 1.0, tr1 = 1.0, cp1 = 1.0;
  double ir0 = 0, ig0 = 0, ib0 = 0, br0 = 0, bg0 = 0, bb0 = 0;
  double ir1 = 0, ig1 = 0, ib1 = 0, br1 = 0, bg1 = 0, bb1 = 0;
  int32_t vis0 = 0, vis1 = 0;
  uint32_t guard = 0;
  bool alive0 = in0, alive1 = in1;
  uint32_t phase0 = 0u, phase1 = 0u;

  if (s < e) issue(s, 0);
  int k = 0;
  for (uint32_t b = s; b < e; b += CB, k ^= 1) {
    const int n = (int)min((uint32_t)CB, e - b);
    if (b + CB < e) issue(b + CB, k ^ 1);  // next batch in flight while this one composites
    if (EXACT && b > s && ((b - s) & 1023u) == 0) {
      // block boundary of the reference's 1024-member cumprod
      tr0 = __dmul_rn(cp0, tr0); cp0 = 1.0;
      tr1 = __dmul_rn(cp1, tr1); cp1 = 1.0;
      ir0 = __dadd_rn(ir0, br0); ig0 = __dadd_rn(ig0, bg0); ib0 = __dadd_rn(ib0, bb0);
      ir1 = __dadd_rn(ir1, br1); ig1 = __dadd_rn(ig1, bg1); ib1 = __dadd_rn(ib1, bb1);
      br0 = bg0 = bb0 = br1 = bg1 = bb1 = 0.0;
    }
    if (k == 0) { mbar_wait(&S.bar[0], phase0); phase0 ^= 1u; }
    else { mbar_wait(&S.bar[1], phase1); phase1 ^= 1u; }
    Payload *PL = S.pl[k];
    // tile-local fp32 mean, written over the fp64 mean (kept in S.m -> global
    // payload for the rare fp64 re-check); zero the batch's max slots
#pragma unroll
    for (int h = 0; h < CB / CT; ++h) {
      const int j = tid + h * CT;
      if (j < n) {
        Payload &p = PL[j];
        if (!EXACT) {
          const float mxl = (float)(p.mx - ox), myl = (float)(p.my - oy);
          reinterpret_cast<float2 *>(&p.mx)[0] = make_float2(mxl, myl);
          S.maxw32[j] = 0u;
        } else {
          S.maxw[j] = 0ull;
        }
      }
    }
    __syncthreads();
    // per-warp member list: members whose box meets this warp's 8x8 pixels
    uint8_t *wl = S.wlist + warp * CB;
    int cnt = 0;
    if (__any_sync(FULL_MASK, alive0 || alive1)) {
      for (int q0 = 0; q0 < n; q0 += 32) {
        const int j = q0 + lane;
        bool hit = false;
        if (j < n) {
          const Payload &p = PL[j];
          float mxl, myl;
          if (EXACT) {
            mxl = (float)(p.mx - ox);
            myl = (float)(p.my - oy);
          } else {
            const float2 mm = reinterpret_cast<const float2 *>(&p.mx)[0];
            mxl = mm.x;
            myl = mm.y;
          }
          hit = !(mxl + p.bx < wx_lo || mxl - p.bx > wx_hi || myl + p.by < wy_lo ||
                  myl - p.by > wy_hi);
        }
        const uint32_t hm = __ballot_sync(FULL_MASK, hit);
        if (hit) wl[cnt + __popc(hm & lanemask_lt())] = (uint8_t)j;
        cnt += __popc(hm);
      }
    }
    __syncwarp();
    for (int i = 0; i < cnt; ++i) {
      if (!__any_sync(FULL_MASK, alive0 || alive1)) break;
      const int j = wl[i];
      const Payload &p = PL[j];
      if (EXACT) {
        const Precise &d = S.pr[k][j];
        double w0 = 0.0, w1 = 0.0;
        if (alive0) {
          double a;
          const bool sk = ref_decide(gx, gy0, p.mx, p.my, d, rp, a);
          if (sk) a = 0.0;
          const double before = __dmul_rn(cp0, tr0);
          cp0 = __dmul_rn(cp0, __dsub_rn(1.0, a));
          w0 = __dmul_rn(before, a);
          if (need_image) {
            br0 = __dadd_rn(br0, __dmul_rn(w0, d.r));
            bg0 = __dadd_rn(bg0, __dmul_rn(w0, d.g));
            bb0 = __dadd_rn(bb0, __dmul_rn(w0, d.b));
          }
          vis0 += sk ? 0 : 1;
          alive0 = __dmul_rn(cp0, tr0) >= rp.t_min;
        }
        if (alive1) {
          double a;
          const bool sk = ref_decide(gx, gy1, p.mx, p.my, d, rp, a);
          if (sk) a = 0.0;
          const double before = __dmul_rn(cp1, tr1);
          cp1 = __dmul_rn(cp1, __dsub_rn(1.0, a));
          w1 = __dmul_rn(before, a);
          if (need_image) {
            br1 = __dadd_rn(br1, __dmul_rn(w1, d.r));
            bg1 = __dadd_rn(bg1, __dmul_rn(w1, d.g));
            bb1 = __dadd_rn(bb1, __dmul_rn(w1, d.b));
          }
          vis1 += sk ? 0 : 1;
          alive1 = __dmul_rn(cp1, tr1) >= rp.t_min;
        }
        if (record_max) {
          unsigned long long wb = (unsigned long long)__double_as_longlong(fmax(w0, w1));
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ob = __shfl_xor_sync(FULL_MASK, wb, o);
            wb = ob > wb ? ob : wb;
          }
          if (lane == 0 && wb) atomicMax(&S.maxw[j], wb);
        }
      } else {
        const float2 mm = reinterpret_cast<const float2 *>(&p.mx)[0];
        const float4 cn = *reinterpret_cast<const float4 *>(&p.A);    // A, 2B, C, o
        const float2 qt = *reinterpret_cast<const float2 *>(&p.q_eff);  // q_eff, tol
        const float dx = fpx - mm.x, dy0 = fpy0 - mm.y, dy1 = fpy1 - mm.y;
        const float adx = cn.x * dx, bdx = cn.y * dx;
        const float q0 = fmaf(adx, dx, fmaf(bdx, dy0, cn.z * dy0 * dy0));
        const float q1 = fmaf(adx, dx, fmaf(bdx, dy1, cn.z * dy1 * dy1));
        const float d0 = q0 - qt.x, d1 = q1 - qt.x;
        bool keep0 = alive0 && d0 < -qt.y, keep1 = alive1 && d1 < -qt.y;
        float a0 = fminf(cn.w * ex2_approx(fmaxf(q0, 0.f) * -0.72134752044448170f), cpar.clamp_f);
        float a1 = fminf(cn.w * ex2_approx(fmaxf(q1, 0.f) * -0.72134752044448170f), cpar.clamp_f);
        const bool inb0 = alive0 && fabsf(d0) <= qt.y, inb1 = alive1 && fabsf(d1) <= qt.y;
        if (__any_sync(FULL_MASK, inb0 || inb1)) {
          // guard band: re-decide in fp64 with the reference's op order (rare)
          if (inb0 || inb1) {
            const uint32_t m = S.m[k][j];
            const Payload pg = payload[m];
            const Precise pr = precise[m];
            double a;
            if (inb0) { keep0 = !ref_decide(gx, gy0, pg.mx, pg.my, pr, rp, a); a0 = (float)a; ++guard; }
            if (inb1) { keep1 = !ref_decide(gx, gy1, pg.mx, pg.my, pr, rp, a); a1 = (float)a; ++guard; }
          }
        }
        const float w0 = keep0 ? T0 * a0 : 0.f, w1 = keep1 ? T1 * a1 : 0.f;
        if (need_image) {
          const float4 c = *reinterpret_cast<const float4 *>(&p.r);
          r0 = fmaf(w0, c.x, r0); g0 = fmaf(w0, c.y, g0); b0 = fmaf(w0, c.z, b0);
          r1 = fmaf(w1, c.x, r1); g1 = fmaf(w1, c.y, g1); b1 = fmaf(w1, c.z, b1);
        }
        T0 = keep0 ? T0 * (1.f - a0) : T0;
        T1 = keep1 ? T1 * (1.f - a1) : T1;
        vis0 += keep0;
        vis1 += keep1;
        alive0 = alive0 && T0 >= cpar.tmin_f;
        alive1 = alive1 && T1 >= cpar.tmin_f;
        if (record_max) {
          const unsigned wb = __reduce_max_sync(FULL_MASK, __float_as_uint(fmaxf(w0, w1)));
          if (lane == 0 && wb) atomicMax(&S.maxw32[j], wb);
        }
      }
    }
    __syncthreads();
    if (record_max) {
#pragma unroll
      for (int h = 0; h < CB / CT; ++h) {
        const int j = tid + h * CT;
        if (j < n) {
          const uint32_t src = PL[j].src;
          if (EXACT) {
            if (S.maxw[j]) atomicMax(reinterpret_cast<unsigned long long *>(maxw) + src, S.maxw[j]);
          } else if (S.maxw32[j]) {
            atomicMax(reinterpret_cast<unsigned int *>(maxw) + src, S.maxw32[j]);
          }
        }
      }
    }
    // also the WAR barrier: buffer k is re-filled by the next-but-one issue
    if (__syncthreads_count(alive0 || alive1) == 0) {
      if (b + CB < e) {  // drain the stage already in flight before exiting
        if (k == 0) mbar_wait(&S.bar[1], phase1);
        else mbar_wait(&S.bar[0], phase0);
      }
      break;
    }
  }
  if (!EXACT && guard) atomicAdd(&fs->stats.guard_hits, guard);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const bool in = h ? in1 : in0;
    if (!in) continue;
    const size_t pix = (size_t)(h ? py1 : py0) * cpar.W + px;
    if (visible) visible[pix] = h ? vis1 : vis0;
    if (!(need_image && image)) continue;
    if (EXACT) {
      double ir = h ? ir1 : ir0, ig = h ? ig1 : ig0, ib = h ? ib1 : ib0;
      ir = __dadd_rn(ir, h ? br1 : br0);
      ig = __dadd_rn(ig, h ? bg1 : bg0);
      ib = __dadd_rn(ib, h ? bb1 : bb0);
      double *im = reinterpret_cast<double *>(image) + 3 * pix;
      im[0] = fmin(fmax(ir, 0.0), 1.0);
      im[1] = fmin(fmax(ig, 0.0), 1.0);
      im[2] = fmin(fmax(ib, 0.0), 1.0);
    } else {
      float *im = reinterpret_cast<float *>(image) + 3 * pix;
      im[0] = fminf(fmaxf(h ? r1 : r0, 0.f), 1.f);
      im[1] = fminf(fmaxf(h ? g1 : g0, 0.f), 1.f);
      im[2] = fminf(fmaxf(h ? b1 : b0, 0.f), 1.f);
    }
  }
}

template <bool EXACT>
static void launch_comp(const Work &w, FrameState *fs, int32_t W, int32_t H,
                        const lodge_raster_params &rp, int32_t flags, const lodge_frame_out &out,
                        cudaStream_t s) {
  const int32_t tiles_x = (W + 15) / 16, tiles_y = (H + 15) / 16;
  const unsigned T = (unsigned)(tiles_x * tiles_y);
  const size_t sm = sizeof(CompSmem<EXACT>);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_composite<EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  CompParams cp;
  cp.rp = rp;
  cp.tmin_f = (float)rp.t_min;
  cp.clamp_f = (float)rp.alpha_clamp;
  cp.flags = flags;
  cp.tiles_x = tiles_x;
  cp.W = W;
  cp.H = H;
  k_composite<EXACT><<<T, CT, sm, s>>>(w.pairs[0], w.tile_start, w.tile_order, w.payload,
                                       w.precise, fs, cp, out.image_dev, out.visible_dev,
                                       out.maxw_dev);
}

void launch_composite(const Work &w, FrameState *fs, const lodge_camera *, int32_t W, int32_t H,
                      const lodge_raster_params &rp, int32_t flags, int32_t exact,
                      const lodge_frame_out &out, uint32_t, cudaStream_t s) {
  if (exact) launch_comp<true>(w, fs, W, H, rp, flags, out, s);
  else launch_comp<false>(w, fs, W, H, rp, flags, out, s);
}

// Compat / inspection: export the sorted per-tile lists as source indices.
__global__ void k_export_lists(const uint64_t *pairs, const uint32_t *tile_start,
                               const Payload *payload, FrameState *fs, int32_t T,
                               int64_t *tile_offsets, int64_t *tile_src, int64_t cap) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= T) tile_offsets[i] = tile_start[i];
  const uint32_t P = fs->n_pairs;
  if (i < P && i < cap) tile_src[i] = payload[(uint32_t)pairs[i]].src;
}

void launch_export_lists(const Work &w, FrameState *fs, int32_t T, int64_t *tile_offsets,
                         int64_t *tile_src, int64_t cap, cudaStream_t s) {
  const int64_t n = cap > (int64_t)T + 1 ? cap : (int64_t)T + 1;
  k_export_lists<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(w.pairs[0], w.tile_start, w.payload,
                                                             fs, T, tile_offsets, tile_src, cap);
}

}  // namespace lodge
