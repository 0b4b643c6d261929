// K6: per-tile front-to-back alpha compositing (reference
// src/raster.py:327-377 _composite_tile and :440-449 combine).
//
// One CTA per 16x16 tile, one pixel per thread.  The tile's sorted member
// list is consumed in batches of 256: each thread stages one member's 64 B
// payload into shared memory (converted to tile-local fp32 coordinates),
// then every pixel thread walks the batch.  Warp votes skip batches for
// warps whose pixels all have T < t_min and end the tile when the whole CTA
// is done (the reference's block-level break is the same rule per pixel).
// Per-member max weights reduce in-warp with redux.sync, per-CTA in shared
// memory, then one global atomicMax on the float bits per member.
//
// FAST: fp32 FMA/MUFU.  Both skip tests of src/raster.py:356 are folded into
// one per-splat cut-off q_eff on the quadratic form; pixels whose fp32 q
// lies within the splat's error bound of q_eff re-decide in fp64 with the
// reference's operation order, so skip decisions match the fp64 reference.
// EXACT: fp64, reproducing the blocked cumprod transmittance of the
// reference (blocks of 1024 members) so per_pixel_visible and max weights
// match it to the ulp of exp.
// Compiled with -fmad=false; the fast path fuses explicitly with fmaf.
#include "internal.cuh"

namespace lodge {

constexpr int CB = 256;  // members per batch == threads per CTA

__device__ __forceinline__ double q_ref64(double A, double B, double C, double dx, double dy) {
  // cn0*dx*dx + 2.0*cn1*dx*dy + cn2*dy*dy, NumPy left-to-right
  return __dadd_rn(__dadd_rn(__dmul_rn(__dmul_rn(A, dx), dx),
                             __dmul_rn(__dmul_rn(__dmul_rn(2.0, B), dx), dy)),
                   __dmul_rn(__dmul_rn(C, dy), dy));
}

template <bool EXACT>
__global__ void __launch_bounds__(CB) k_composite(const uint64_t *__restrict__ pairs,
                                                  const uint32_t *__restrict__ tile_start,
                                                  const Payload *__restrict__ payload,
                                                  const Precise *__restrict__ precise,
                                                  FrameState *fs, lodge_raster_params rp,
                                                  int32_t flags, int32_t tiles_x, int32_t W,
                                                  int32_t H, void *image, int32_t *visible,
                                                  void *maxw) {
  __shared__ float4 s_pos[CB];   // FAST: mx_l, my_l, q_eff, tol
  __shared__ float4 s_con[CB];   // FAST: A, 2B, C, o
  __shared__ float4 s_col[CB];   // r, g, b, src bits
  __shared__ double s_d[EXACT ? CB * 9 : 1];  // EXACT: mx, my, A, B, C, o, r, g, b
  __shared__ unsigned long long s_maxw[CB];
  __shared__ uint32_t s_m[CB];

  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t t = blockIdx.x;
  const int tx = t % tiles_x, ty = t / tiles_x;
  const int px = tx * 16 + (tid & 15), py = ty * 16 + (tid >> 4);
  const bool inside = px < W && py < H;
  const bool need_image = flags & LODGE_NEED_IMAGE;
  const bool record_max = (flags & LODGE_RECORD_MAX) && maxw != nullptr;
  uint32_t s = tile_start[t], e = tile_start[t + 1];
  if (fs->stats.overflow) e = s;

  const float fpx = (float)(tid & 15) + 0.5f, fpy = (float)(tid >> 4) + 0.5f;
  const double gx = (double)px + 0.5, gy = (double)py + 0.5;
  const double ox = (double)(tx * 16), oy = (double)(ty * 16);
  const float tmin_f = (float)rp.t_min, clamp_f = (float)rp.alpha_clamp;

  // FAST state
  float T = 1.0f, cr = 0.f, cg = 0.f, cb = 0.f;
  // EXACT state
  double trans = 1.0, cp = 1.0, ir = 0, ig = 0, ib = 0, br = 0, bg = 0, bb = 0;
  int32_t vis = 0;
  uint32_t guard = 0;
  bool alive = inside;

  for (uint32_t b = s; b < e; b += CB) {
    const int n = (int)min((uint32_t)CB, e - b);
    if (tid < n) {
      const uint32_t m = (uint32_t)pairs[b + tid];
      const Payload pl = payload[m];
      s_m[tid] = m;
      s_maxw[tid] = 0ull;
      s_col[tid] = make_float4(pl.r, pl.g, pl.b, __uint_as_float(pl.src));
      if (EXACT) {
        const Precise pr = precise[m];
        double *d = s_d + tid * 9;
        d[0] = pl.mx;
        d[1] = pl.my;
        d[2] = pr.A;
        d[3] = pr.B;
        d[4] = pr.C;
        d[5] = pr.o;
        d[6] = pr.r;
        d[7] = pr.g;
        d[8] = pr.b;
      } else {
        s_pos[tid] = make_float4((float)(pl.mx - ox), (float)(pl.my - oy), pl.q_eff, pl.tol);
        s_con[tid] = make_float4(pl.A, pl.B2, pl.C, pl.o);
      }
    }
    if (EXACT && b > s && ((b - s) & 1023u) == 0) {
      // block boundary of the reference's 1024-member cumprod
      trans = __dmul_rn(cp, trans);
      cp = 1.0;
      ir = __dadd_rn(ir, br); ig = __dadd_rn(ig, bg); ib = __dadd_rn(ib, bb);
      br = bg = bb = 0.0;
    }
    __syncthreads();
    for (int j = 0; j < n; ++j) {
      if (!__any_sync(FULL_MASK, alive)) break;
      if (EXACT) {
        double w = 0.0;
        if (alive) {
          const double *d = s_d + j * 9;
          const double dx = __dsub_rn(gx, d[0]), dy = __dsub_rn(gy, d[1]);
          const double q = q_ref64(d[2], d[3], d[4], dx, dy);
          double alpha = __dmul_rn(d[5], exp(__dmul_rn(-0.5, fmax(q, 0.0))));
          alpha = fmin(alpha, rp.alpha_clamp);
          const bool skipped = (alpha < rp.alpha_min) || (q > LODGE_SUPPORT_Q);
          const double a = skipped ? 0.0 : alpha;
          const double before = __dmul_rn(cp, trans);
          cp = __dmul_rn(cp, __dsub_rn(1.0, a));
          // before >= t_min holds (alive)
          w = __dmul_rn(before, a);
          if (need_image) {
            br = __dadd_rn(br, __dmul_rn(w, d[6]));
            bg = __dadd_rn(bg, __dmul_rn(w, d[7]));
            bb = __dadd_rn(bb, __dmul_rn(w, d[8]));
          }
          vis += skipped ? 0 : 1;
          alive = __dmul_rn(cp, trans) >= rp.t_min;
        }
        if (record_max) {
          unsigned long long wb = (unsigned long long)__double_as_longlong(w);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            unsigned long long ob = __shfl_xor_sync(FULL_MASK, wb, o);
            wb = ob > wb ? ob : wb;
          }
          if (lane == 0 && wb) atomicMax(&s_maxw[j], wb);
        }
      } else {
        float w = 0.f;
        if (alive) {
          const float4 P0 = s_pos[j];
          const float4 P1 = s_con[j];
          const float dx = fpx - P0.x, dy = fpy - P0.y;
          const float q = fmaf(P1.x * dx, dx, fmaf(P1.y * dx, dy, P1.z * dy * dy));
          const float dq = q - P0.z;
          bool skip;
          float alpha = 0.f;
          if (dq > P0.w) {
            skip = true;
          } else if (dq >= -P0.w) {
            // guard band: re-decide in fp64 with the reference's op order
            ++guard;
            const uint32_t m = s_m[j];
            const Payload pl = payload[m];
            const Precise pr = precise[m];
            const double ddx = __dsub_rn(gx, pl.mx), ddy = __dsub_rn(gy, pl.my);
            const double q64 = q_ref64(pr.A, pr.B, pr.C, ddx, ddy);
            double a64 = __dmul_rn(pr.o, exp(__dmul_rn(-0.5, fmax(q64, 0.0))));
            a64 = fmin(a64, rp.alpha_clamp);
            skip = (a64 < rp.alpha_min) || (q64 > LODGE_SUPPORT_Q);
            alpha = (float)a64;
          } else {
            skip = false;
            alpha = fminf(P1.w * ex2_approx(fmaxf(q, 0.f) * -0.72134752044448170f), clamp_f);
          }
          if (!skip) {
            w = T * alpha;
            if (need_image) {
              const float4 c = s_col[j];
              cr = fmaf(w, c.x, cr);
              cg = fmaf(w, c.y, cg);
              cb = fmaf(w, c.z, cb);
            }
            T = T * (1.f - alpha);
            ++vis;
            alive = T >= tmin_f;
          }
        }
        if (record_max) {
          const unsigned wb = __reduce_max_sync(FULL_MASK, __float_as_uint(w));
          if (lane == 0 && wb) atomicMax(&s_maxw[j], (unsigned long long)wb);
        }
      }
    }
    __syncthreads();
    if (record_max && tid < n && s_maxw[tid]) {
      const uint32_t src = __float_as_uint(s_col[tid].w);
      if (EXACT) atomicMax(reinterpret_cast<unsigned long long *>(maxw) + src, s_maxw[tid]);
      else atomicMax(reinterpret_cast<unsigned int *>(maxw) + src, (unsigned int)s_maxw[tid]);
    }
    if (__syncthreads_count(alive) == 0) break;
  }
  if (!EXACT && guard) atomicAdd(&fs->stats.guard_hits, guard);
  if (!inside) return;
  const size_t pix = (size_t)py * W + px;
  if (visible) visible[pix] = vis;
  if (need_image && image) {
    if (EXACT) {
      ir = __dadd_rn(ir, br); ig = __dadd_rn(ig, bg); ib = __dadd_rn(ib, bb);
      double *im = reinterpret_cast<double *>(image) + 3 * pix;
      im[0] = fmin(fmax(ir, 0.0), 1.0);
      im[1] = fmin(fmax(ig, 0.0), 1.0);
      im[2] = fmin(fmax(ib, 0.0), 1.0);
    } else {
      float *im = reinterpret_cast<float *>(image) + 3 * pix;
      im[0] = fminf(fmaxf(cr, 0.f), 1.f);
      im[1] = fminf(fmaxf(cg, 0.f), 1.f);
      im[2] = fminf(fmaxf(cb, 0.f), 1.f);
    }
  }
}

void launch_composite(const Work &w, FrameState *fs, const lodge_camera *, int32_t W, int32_t H,
                      const lodge_raster_params &rp, int32_t flags, int32_t exact,
                      const lodge_frame_out &out, uint32_t, cudaStream_t s) {
  const int32_t tiles_x = (W + 15) / 16, tiles_y = (H + 15) / 16;
  const unsigned T = (unsigned)(tiles_x * tiles_y);
  if (exact)
    k_composite<true><<<T, CB, 0, s>>>(w.pairs[0], w.tile_start, w.payload, w.precise, fs, rp,
                                       flags, tiles_x, W, H, out.image_dev, out.visible_dev,
                                       out.maxw_dev);
  else
    k_composite<false><<<T, CB, 0, s>>>(w.pairs[0], w.tile_start, w.payload, w.precise, fs, rp,
                                        flags, tiles_x, W, H, out.image_dev, out.visible_dev,
                                        out.maxw_dev);
}

// Compat: export the sorted per-tile lists as source indices.
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
