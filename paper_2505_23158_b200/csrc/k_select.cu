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
  uint32_t part_base[LODGE_MAX_LEVELS + 1];  // CTA-count table offsets per level
};

// One CTA = 256 consecutive diagonals of level l's stable merge S =
// merge(A, B) (A first on ties).  The CTA's window of A and B is found by two
// merge-path searches and staged in shared memory; each thread then locates
// its element by a short search there.  The B copy of a value present in
// both sets is dropped (keep = false).  Compacting the kept elements in S
// order yields np.union1d(A, B) with its tags (count -> scan -> write, so no
// look-back chain serialises the CTAs).  Returns false if the CTA is idle.
struct UnionLevel {
  const uint32_t *A, *B;
  uint32_t na, nb;
};

__device__ __forceinline__ UnionLevel union_level(const UnionArgs &a, const FrameState *fs, int l) {
  const int32_t f = fs->stats.f, o = fs->stats.o;
  UnionLevel u;
  const int64_t fa = a.offsets[(int64_t)f * a.L + l];
  u.na = (uint32_t)(a.offsets[(int64_t)f * a.L + l + 1] - fa);
  u.A = a.data + fa;
  u.nb = 0;
  u.B = u.A;
  if (o >= 0) {
    const int64_t fb = a.offsets[(int64_t)o * a.L + l];
    u.nb = (uint32_t)(a.offsets[(int64_t)o * a.L + l + 1] - fb);
    u.B = a.data + fb;
  }
  return u;
}

// Flattened CTA index -> (level, part) over a.part_base.
__device__ __forceinline__ int union_level_of(const UnionArgs &a, uint32_t g, uint32_t &part) {
  int l = 0;
  while (l + 1 < a.L && g >= a.part_base[l + 1]) ++l;
  part = g - a.part_base[l];
  return l;
}

// Merge-path splits for every CTA boundary of every level, all in parallel:
// splits[part_base[l] + l + p] = #A among the first min(256 p, n_l) merged
// elements, p = 0 .. ceil(n_l / 256).
__global__ void k_union_split(UnionArgs a, FrameState *fs, uint32_t *splits) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.part_base[a.L] + a.L) return;
  int l = 0;
  while (l + 1 < a.L && g >= a.part_base[l + 1] + l + 1) ++l;
  const uint32_t p = g - a.part_base[l] - l;
  const UnionLevel u = union_level(a, fs, l);
  const uint32_t n = u.na + u.nb;
  if (p > (n + 255u) / 256u) return;
  const uint32_t d = min(p * 256u, n);
  uint32_t lo = d > u.nb ? d - u.nb : 0u, hi = d < u.na ? d : u.na;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(u.A + mid) <= __ldg(u.B + (d - 1 - mid))) lo = mid + 1;
    else hi = mid;
  }
  splits[g] = lo;
}

__device__ __forceinline__ bool union_block(const UnionArgs &a, const FrameState *fs, int l,
                                            uint32_t part, const uint32_t *splits, bool &keep,
                                            uint32_t &v, uint8_t &tag) {
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
  __shared__ uint32_t s_a[258], s_b[258];  // A[i0-1 .. i1], B[j0 .. j1]
  const uint32_t n = na + nb;
  if (part * 256u >= n) return false;  // block-uniform
  const uint32_t d0 = part * 256u, d1 = min(d0 + 256u, n);
  const uint32_t *sp = splits + a.part_base[l] + l + part;
  const uint32_t i0 = sp[0], i1 = sp[1], j0 = d0 - i0, j1 = d1 - i1;
  // stage A[i0-1 .. i1] (one element back for the duplicate test, one ahead
  // for the tie test) and B[j0 .. j1]
  for (uint32_t q = threadIdx.x; q < i1 - i0 + 2; q += 256) {
    const int64_t ia = (int64_t)i0 - 1 + q;
    s_a[q] = (ia >= 0 && ia < na) ? __ldg(A + ia) : 0xffffffffu;
  }
  for (uint32_t q = threadIdx.x; q < j1 - j0 + 1; q += 256)
    s_b[q] = (j0 + q < nb) ? __ldg(B + j0 + q) : 0xffffffffu;
  __syncthreads();
  const uint32_t t = d0 + threadIdx.x;
  keep = false;
  v = 0;
  tag = 0;
  if (t < n) {
    // merge-path search inside the staged window (local diagonal t - d0)
    const uint32_t dl = t - d0;
    uint32_t lo = dl > (j1 - j0) ? dl - (j1 - j0) : 0u, hi = min(dl, i1 - i0);
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (s_a[mid + 1] <= s_b[dl - 1 - mid]) lo = mid + 1;
      else hi = mid;
    }
    const uint32_t i = i0 + lo, j = j0 + (dl - lo);  // global positions
    const uint32_t av = s_a[lo + 1], bv = s_b[dl - lo];
    if (i < na && (j >= nb || av <= bv)) {
      v = av;
      tag = (j < nb && bv == v) ? 3 : 1;
      keep = true;
    } else {
      v = bv;
      keep = !(i > 0 && s_a[lo] == v);
      tag = 2;
    }
  }
  return true;
}

// flattened grid over all levels' CTAs: kept elements per CTA.
__global__ void __launch_bounds__(256) k_union_count(UnionArgs a, FrameState *fs,
                                                     const uint32_t *splits, uint32_t *cnt) {
  uint32_t part;
  const int l = union_level_of(a, blockIdx.x, part);
  bool keep;
  uint32_t v;
  uint8_t tag;
  if (!union_block(a, fs, l, part, splits, keep, v, tag)) return;
  const uint32_t c = __syncthreads_count(keep);
  if (threadIdx.x == 0) cnt[a.part_base[l] + part] = c;
}

// grid L x 1024 threads: exclusive scan of the CTA counts of level l, U_l.
__global__ void __launch_bounds__(1024) k_union_scan(UnionArgs a, FrameState *fs, uint32_t *cnt) {
  __shared__ uint32_t s_sum[1024];
  const int l = blockIdx.x;
  const int32_t f = fs->stats.f, o = fs->stats.o;
  uint32_t n = (uint32_t)(a.offsets[(int64_t)f * a.L + l + 1] - a.offsets[(int64_t)f * a.L + l]);
  if (o >= 0) n += (uint32_t)(a.offsets[(int64_t)o * a.L + l + 1] - a.offsets[(int64_t)o * a.L + l]);
  const uint32_t np = (n + 255u) / 256u;
  uint32_t *c = cnt + a.part_base[l];
  const uint32_t per = (np + 1023u) / 1024u, b = threadIdx.x * per, e = min(np, b + per);
  uint32_t loc = 0;
  for (uint32_t q = b; q < e; ++q) loc += c[q];
  s_sum[threadIdx.x] = loc;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    const uint32_t t = threadIdx.x >= off ? s_sum[threadIdx.x - off] : 0u;
    __syncthreads();
    s_sum[threadIdx.x] += t;
    __syncthreads();
  }
  uint32_t run = s_sum[threadIdx.x] - loc;
  for (uint32_t q = b; q < e; ++q) {
    const uint32_t x = c[q];
    c[q] = run;
    run += x;
  }
  if (threadIdx.x == 1023) fs->stats.U_level[l] = s_sum[1023];
}

// flattened grid: recompute the CTA's merge and write the kept elements in order.
__global__ void __launch_bounds__(256) k_union_write(UnionArgs a, FrameState *fs,
                                                     const uint32_t *splits, const uint32_t *cnt,
                                                     uint32_t *union_idx, uint8_t *union_tag) {
  __shared__ uint32_t s_w[8];
  uint32_t part;
  const int l = union_level_of(a, blockIdx.x, part);
  bool keep;
  uint32_t v;
  uint8_t tag;
  if (!union_block(a, fs, l, part, splits, keep, v, tag)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t bal = __ballot_sync(FULL_MASK, keep);
  if (lane == 0) s_w[warp] = __popc(bal);
  __syncthreads();
  uint32_t pre = cnt[a.part_base[l] + part];
  for (int w = 0; w < warp; ++w) pre += s_w[w];
  if (!keep) return;
  const uint32_t m = pre + __popc(bal & lanemask_lt());
  union_idx[a.slot_base[l] + m] = v;
  union_tag[a.slot_base[l] + m] = tag;
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
  a.part_base[0] = 0;
  for (int l = 0; l < ch.L; ++l)
    a.part_base[l + 1] = a.part_base[l] + (ls.slot_base[l + 1] - ls.slot_base[l] + 255) / 256;
  // scratch in the look-back buffer: CTA counts, then the merge-path splits
  // (count words have zero flag bits, so no look-back ever reads them as ready)
  uint32_t *cnt = reinterpret_cast<uint32_t *>(status);
  uint32_t *splits = cnt + a.part_base[ch.L];
  const uint32_t nparts = a.part_base[ch.L];
  if (max_slots > 0 && nparts > 0) {
    k_union_split<<<(nparts + ch.L + 255) / 256, 256, 0, s>>>(a, fs, splits);
    k_union_count<<<nparts, 256, 0, s>>>(a, fs, splits, cnt);
    k_union_scan<<<ch.L, 1024, 0, s>>>(a, fs, cnt);
    k_union_write<<<nparts, 256, 0, s>>>(a, fs, splits, cnt, union_idx, union_tag);
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
