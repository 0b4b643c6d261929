// K0 chunk selection and K1 two-chunk union with blend tags.
//
// K0 restates nearest_two_chunks + blend_factor (reference
// src/blending.py:77-99) in fp64 with NumPy's operation order: norms as
// sqrt((x*x + y*y) + z*z) (add.reduce over a length-3 axis), 1-D np.dot as
// OpenBLAS's fma chain.  Compiled with -fmad=false so nothing else fuses.
//
// K1 restates compose_active (src/blending.py:119-128): per level, the
// sorted union of the two chunks' sets with tag 3 (both, mod 1), 1 (primary
// only, mod t), 2 (other only, mod 1-t).  Each set element finds its union
// slot by a binary search in the other set: slot(a_i) = i + |{b < a_i}|,
// slot(b_j) = j + |{a < b_j}| (b_j not in A).  Union sizes follow from the
// intersection count, accumulated with one atomic per warp.
#include "internal.cuh"

namespace lodge {

__device__ __forceinline__ double dot3_blas(double a0, double a1, double a2, double b0,
                                            double b1, double b2) {
  return fma(a2, b2, fma(a1, b1, a0 * b0));
}

// One thread per query position.
__device__ void select_one(const double *centers, int32_t K, double px, double py, double pz,
                           int32_t *f, int32_t *o, double *tb, double *t) {
  int32_t b0 = -1, b1 = -1;
  double d0 = 0.0, d1 = 0.0;
  for (int32_t j = 0; j < K; ++j) {
    double x = centers[3 * j] - px, y = centers[3 * j + 1] - py, z = centers[3 * j + 2] - pz;
    double d = sqrt((x * x + y * y) + z * z);
    if (b0 < 0 || d < d0) {
      b1 = b0; d1 = d0; b0 = j; d0 = d;
    } else if (b1 < 0 || d < d1) {
      b1 = j; d1 = d;
    }
  }
  *f = b0;
  if (K > 1) {
    *o = b1;
    const double *mf = centers + 3 * b0, *mo = centers + 3 * b1;
    double fo0 = mf[0] - mo[0], fo1 = mf[1] - mo[1], fo2 = mf[2] - mo[2];
    double co0 = px - mo[0], co1 = py - mo[1], co2 = pz - mo[2];
    double d2 = dot3_blas(fo0, fo1, fo2, fo0, fo1, fo2);
    double tbar = dot3_blas(co0, co1, co2, fo0, fo1, fo2) / d2;
    *tb = tbar;
    *t = fmin(1.0, fmax(0.0, tbar));
  } else {
    *o = -1;
    *tb = 1.0;
    *t = 1.0;
  }
}

__global__ void k_select(const double *centers, int32_t K, const double *pos, int32_t n,
                         int32_t *f, int32_t *o, double *tb, double *t) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  select_one(centers, K, pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], f + i, o + i, tb + i, t + i);
}

void launch_select(const double *centers, int32_t K, const double *pos, int32_t n, int32_t *f,
                   int32_t *o, double *tb, double *t, cudaStream_t s) {
  if (n <= 0) return;
  k_select<<<(n + 127) / 128, 128, 0, s>>>(centers, K, pos, n, f, o, tb, t);
}

__global__ void k_blend_factor(const double *in, int32_t n, double *out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double *r = in + 9 * i;
  const double fo0 = r[3] - r[6], fo1 = r[4] - r[7], fo2 = r[5] - r[8];
  const double co0 = r[0] - r[6], co1 = r[1] - r[7], co2 = r[2] - r[8];
  const double d2 = dot3_blas(fo0, fo1, fo2, fo0, fo1, fo2);
  out[3 * i] = d2;
  if (d2 <= 0) {
    out[3 * i + 1] = out[3 * i + 2] = 0.0;
    return;
  }
  const double tb = dot3_blas(co0, co1, co2, fo0, fo1, fo2) / d2;
  out[3 * i + 1] = tb;
  out[3 * i + 2] = fmin(1.0, fmax(0.0, tb));
}

void launch_blend_factor(const double *in, int32_t n, double *out, cudaStream_t s) {
  if (n <= 0) return;
  k_blend_factor<<<(n + 127) / 128, 128, 0, s>>>(in, n, out);
}

// Per-frame selection into the frame state; also zeroes intersection counts.
__global__ void k_select_frame(const double *centers, int32_t K, const lodge_camera *cam,
                               int32_t have_pair, int32_t pf, int32_t po, double t_val,
                               FrameState *fs) {
  if (threadIdx.x == 0) {
    lodge_frame_stats &st = fs->stats;
    if (have_pair) {
      st.f = pf;
      st.o = po;
      st.t = (po < 0) ? 1.0 : t_val;
      st.t_bar = st.t;
    } else {
      select_one(centers, K, cam->pos[0], cam->pos[1], cam->pos[2], &st.f, &st.o, &st.t_bar,
                 &st.t);
    }
  }
  if (threadIdx.x < LODGE_MAX_LEVELS) fs->stats.U_level[threadIdx.x] = 0;
}

void launch_select_frame(const double *centers, int32_t K, const lodge_camera *cam,
                         const int32_t *, const double *, int32_t have_pair, int32_t pair_f,
                         int32_t pair_o, double t_val, FrameState *fs, cudaStream_t s) {
  k_select_frame<<<1, 32, 0, s>>>(centers, K, cam, have_pair, pair_f, pair_o, t_val, fs);
}

struct UnionArgs {
  const int64_t *offsets;
  const uint32_t *data;
  int32_t L;
  uint32_t status_stride;  // look-back words per level
  uint32_t slot_base[LODGE_MAX_LEVELS + 1];
};

// grid.y = level.  Element t of the stable merge S = merge(A, B) (A first on
// ties) is located by a merge-path search on diagonal t; the B copy of a
// value present in both sets is dropped, and survivors are compacted in S
// order (ordered look-back), which yields np.union1d(A, B) with its tags.
__global__ void __launch_bounds__(256) k_union(UnionArgs a, FrameState *fs, uint64_t *status,
                                               uint32_t *union_idx, uint8_t *union_tag) {
  __shared__ uint32_t s_warp[32];
  __shared__ uint32_t s_base;
  const int l = blockIdx.y;
  const int32_t f = fs->stats.f, o = fs->stats.o;
  const int64_t fa = a.offsets[(int64_t)f * a.L + l];
  const uint32_t na = (uint32_t)(a.offsets[(int64_t)f * a.L + l + 1] - fa);
  const uint32_t *A = a.data + fa;
  uint32_t nb = 0;
  const uint32_t *B = A;
  if (o >= 0) {
    const int64_t fb = a.offsets[(int64_t)o * a.L + l];
    nb = (uint32_t)(a.offsets[(int64_t)o * a.L + l + 1] - fb);
    B = a.data + fb;
  }
  const uint32_t part = take_ticket(&fs->tickets[TK_UNION0 + l], &s_base);
  const uint32_t n = na + nb;
  if (part * 256u >= n) return;  // block-uniform
  const uint32_t t = part * 256u + threadIdx.x;
  bool keep = false;
  uint32_t v = 0;
  uint8_t tag = 0;
  if (t < n) {
    uint32_t lo = t > nb ? t - nb : 0u, hi = t < na ? t : na;
    while (lo < hi) {  // i = #A among the first t merged elements
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(A + mid) <= __ldg(B + (t - 1 - mid))) lo = mid + 1;
      else hi = mid;
    }
    const uint32_t i = lo, j = t - lo;
    if (i < na && (j >= nb || __ldg(A + i) <= __ldg(B + j))) {
      v = __ldg(A + i);
      tag = (j < nb && __ldg(B + j) == v) ? 3 : 1;
      keep = true;
    } else {
      v = __ldg(B + j);
      keep = !(i > 0 && __ldg(A + i - 1) == v);
      tag = 2;
    }
  }
  const int64_t m = compact_slot(keep, status + (size_t)l * a.status_stride,
                                 fs->epoch + TK_UNION0 + l, part, s_warp, &s_base);
  if (m < 0) return;
  union_idx[a.slot_base[l] + m] = v;
  union_tag[a.slot_base[l] + m] = tag;
  atomicMax(&fs->stats.U_level[l], (uint32_t)(m + 1));
}

__global__ void k_union_sizes(int32_t L, FrameState *fs) {
  if (threadIdx.x != 0) return;
  uint32_t U = 0;
  for (int l = 0; l < L; ++l) U += fs->stats.U_level[l];
  fs->stats.U = U;
  fs->n_sort = U;  // fused path: every input is a depth-sort key (culled -> ~0)
}

void launch_union(const lodge_chunks &ch, const LevelSlots &ls, FrameState *fs, uint64_t *status,
                  uint32_t *union_idx, uint8_t *union_tag, cudaStream_t s) {
  UnionArgs a;
  a.offsets = ch.offsets_dev;
  a.data = ch.data_dev;
  a.L = ch.L;
  uint32_t max_slots = 0;
  for (int l = 0; l <= LODGE_MAX_LEVELS; ++l) a.slot_base[l] = (l <= ch.L) ? ls.slot_base[l] : 0;
  for (int l = 0; l < ch.L; ++l) max_slots = max(max_slots, ls.slot_base[l + 1] - ls.slot_base[l]);
  a.status_stride = union_status_stride(max_slots);
  if (max_slots > 0) {
    dim3 grid((max_slots + 255) / 256, ch.L);
    k_union<<<grid, 256, 0, s>>>(a, fs, status, union_idx, union_tag);
  }
  k_union_sizes<<<1, 32, 0, s>>>(ch.L, fs);
}

__global__ void k_begin_frame(FrameState *fs) {
  int i = threadIdx.x;
  if (i == 0) {
    fs->epoch += 32;
    fs->stats.M = 0;
    fs->stats.P = 0;
    fs->stats.overflow = 0;
    fs->stats.guard_hits = 0;
  }
  if (i < 32) fs->tickets[i] = 0;
  if (i < 8) fs->counters[i] = 0;
  for (int k = i; k < 8 * 256; k += blockDim.x) (&fs->hist_depth[0][0])[k] = 0;
}

void launch_begin_frame(FrameState *fs, cudaStream_t s) { k_begin_frame<<<1, 256, 0, s>>>(fs); }

}  // namespace lodge
