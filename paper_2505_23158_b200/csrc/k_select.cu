// K0 chunk selection and K1 two-chunk union with blend tags.
//
// K0 restates nearest_two_chunks + blend_factor (reference
// src/blending.py:77-99) in fp64 with NumPy's operation order: norms as
// sqrt((x*x + y*y) + z*z) (add.reduce over a length-3 axis), 1-D np.dot as
// OpenBLAS's fma chain.  Compiled with -fmad=false so nothing else fuses.
//
// K1 restates compose_active (src/blending.py:119-128): per level, the
// sorted union of the two chunks' sets with tag 3 (both, mod 1), 1 (primary
// only, mod t), 2 (other only, mod 1-t), as a stable merge-path merge of the
// two sets that drops the second copy of common values (k_union_merge).
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

// (d, j) ordered lexicographically, i.e. lexsort((arange, dist)) order.
__device__ __forceinline__ bool dist_before(double da, int32_t ja, double db, int32_t jb) {
  if (jb < 0) return ja >= 0;
  if (ja < 0) return false;
  return da < db || (!(db < da) && ja < jb);
}

// Warp arg-min of (d, j) over the lanes' candidates (j < 0: none).
__device__ __forceinline__ void warp_argmin(double &d, int32_t &j) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double od = __shfl_xor_sync(FULL_MASK, d, o);
    const int32_t oj = __shfl_xor_sync(FULL_MASK, j, o);
    if (dist_before(od, oj, d, j)) {
      d = od;
      j = oj;
    }
  }
}

// Per-frame selection into the frame state (one warp): the same fp64
// distances as select_one, lanes over chunks, then the two smallest (d, j).
__global__ void k_select_frame(const double *centers, int32_t K, const lodge_camera *cam,
                               int32_t have_pair, int32_t pf, int32_t po, double t_val,
                               FrameState *fs) {
  lodge_frame_stats &st = fs->stats;
  const int lane = threadIdx.x & 31;
  if (have_pair) {
    if (lane == 0) {
      st.f = pf;
      st.o = po;
      st.t = (po < 0) ? 1.0 : t_val;
      st.t_bar = st.t;
    }
  } else if (threadIdx.x < 32) {
    const double px = cam->pos[0], py = cam->pos[1], pz = cam->pos[2];
    // each lane keeps its best two (d, j) over chunks lane, lane + 32, ...
    double d0 = 0.0, d1 = 0.0;
    int32_t b0 = -1, b1 = -1;
    for (int32_t j = lane; j < K; j += 32) {
      const double x = centers[3 * j] - px, y = centers[3 * j + 1] - py,
                   z = centers[3 * j + 2] - pz;
      const double d = sqrt((x * x + y * y) + z * z);
      if (dist_before(d, j, d0, b0)) {
        d1 = d0; b1 = b0; d0 = d; b0 = j;
      } else if (dist_before(d, j, d1, b1)) {
        d1 = d; b1 = j;
      }
    }
    double bd = d0;
    int32_t bj = b0;
    warp_argmin(bd, bj);  // the nearest chunk
    // runner-up: each lane's best candidate other than the winner
    double cd = (b0 == bj) ? d1 : d0;
    int32_t cj = (b0 == bj) ? b1 : b0;
    warp_argmin(cd, cj);
    if (lane == 0) {
      st.f = bj;
      if (K > 1) {
        st.o = cj;
        const double *mf = centers + 3 * bj, *mo = centers + 3 * cj;
        const double fo0 = mf[0] - mo[0], fo1 = mf[1] - mo[1], fo2 = mf[2] - mo[2];
        const double co0 = px - mo[0], co1 = py - mo[1], co2 = pz - mo[2];
        const double d2 = dot3_blas(fo0, fo1, fo2, fo0, fo1, fo2);
        const double tbar = dot3_blas(co0, co1, co2, fo0, fo1, fo2) / d2;
        st.t_bar = tbar;
        st.t = fmin(1.0, fmax(0.0, tbar));
      } else {
        st.o = -1;
        st.t_bar = 1.0;
        st.t = 1.0;
      }
    }
  }
  if (threadIdx.x < LODGE_MAX_LEVELS) fs->stats.U_level[threadIdx.x] = 0;
}

void launch_select_frame(const double *centers, int32_t K, const lodge_camera *cam,
                         const int32_t *, const double *, int32_t have_pair, int32_t pair_f,
                         int32_t pair_o, double t_val, FrameState *fs, cudaStream_t s) {
  k_select_frame<<<1, 32, 0, s>>>(centers, K, cam, have_pair, pair_f, pair_o, t_val, fs);
}

constexpr int UN_THREADS = 256, UN_ITEMS = 8;
constexpr uint32_t UN_TILE = UN_THREADS * UN_ITEMS;  // merged elements per CTA

struct UnionArgs {
  const int64_t *offsets;
  const uint32_t *data;
  int32_t L;
  uint32_t status_stride;  // look-back words per level
  uint32_t slot_base[LODGE_MAX_LEVELS + 1];
  uint32_t part_base[LODGE_MAX_LEVELS + 1];  // CTA-count table offsets per level
  int32_t slab;                              // write set positions (chunk slabs)
  uint64_t uid;                              // lodge_chunks.uid (0: no reuse)
};

// Reuse of the previous frame's union (same plan contents and chunk pair):
// decided once per frame by k_union_check, read by the union kernels.
__global__ void k_union_check(uint64_t uid, FrameState *fs) {
  if (threadIdx.x != 0) return;
  fs->uc_hit = (uid != 0 && fs->uc_uid == uid && fs->uc_f == fs->stats.f &&
                fs->uc_o == fs->stats.o) ? 1u : 0u;
}

// The two sorted sets of level l for the frame's chunk pair.
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
// splits[part_base[l] + l + p] = #A among the first min(UN_TILE p, n_l)
// merged elements, p = 0 .. ceil(n_l / UN_TILE).
__global__ void k_union_split(UnionArgs a, FrameState *fs, uint32_t *splits) {
  if (fs->uc_hit) return;
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.part_base[a.L] + a.L) return;
  int l = 0;
  while (l + 1 < a.L && g >= a.part_base[l + 1] + l + 1) ++l;
  const uint32_t p = g - a.part_base[l] - l;
  const UnionLevel u = union_level(a, fs, l);
  const uint32_t n = u.na + u.nb;
  if (p > (n + UN_TILE - 1) / UN_TILE) return;
  const uint32_t d = min(p * UN_TILE, n);
  uint32_t lo = d > u.nb ? d - u.nb : 0u, hi = d < u.na ? d : u.na;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(u.A + mid) <= __ldg(u.B + (d - 1 - mid))) lo = mid + 1;
    else hi = mid;
  }
  splits[g] = lo;
}

// One CTA = UN_TILE consecutive diagonals of level l's stable merge
// S = merge(A, B) (A first on ties), CTAs in ticket order.  The CTA's windows
// of A and B (from the precomputed merge-path splits) are staged in shared
// memory; each thread finds the start of its UN_ITEMS diagonals by one
// merge-path search there and merges them sequentially.  The B copy of a
// value present in both sets is dropped; the kept elements are compacted in
// S order by a block scan and a per-level decoupled look-back, which yields
// np.union1d(A, B) with its tags in one pass.
__global__ void __launch_bounds__(UN_THREADS) k_union_merge(UnionArgs a, FrameState *fs,
                                                           const uint32_t *splits,
                                                           uint64_t *lb_status,
                                                           uint32_t *union_idx,
                                                           uint8_t *union_tag) {
  __shared__ uint32_t s_a[UN_TILE + 2], s_b[UN_TILE + 1];  // A[i0-1 .. i1], B[j0 .. j1]
  __shared__ uint32_t s_w[UN_THREADS / 32 + 1];
  __shared__ uint32_t s_tk;
  if (fs->uc_hit) return;  // block-uniform: the previous frame's union is this one
  const uint32_t g = take_ticket(&fs->tickets[TK_UNION0], &s_tk);
  uint32_t part;
  const int l = union_level_of(a, g, part);
  const UnionLevel u = union_level(a, fs, l);
  const uint32_t n = u.na + u.nb;
  if (part * UN_TILE >= n) return;  // block-uniform: idle slot of this level
  const uint32_t d0 = part * UN_TILE, d1 = min(d0 + UN_TILE, n);
  const uint32_t *sp = splits + a.part_base[l] + l + part;
  const uint32_t i0 = sp[0], i1 = sp[1], j0 = d0 - i0, j1 = d1 - i1;
  for (uint32_t q = threadIdx.x; q < i1 - i0 + 2; q += UN_THREADS) {
    const int64_t ia = (int64_t)i0 - 1 + q;
    s_a[q] = (ia >= 0 && ia < u.na) ? __ldg(u.A + ia) : 0xffffffffu;
  }
  for (uint32_t q = threadIdx.x; q < j1 - j0 + 1; q += UN_THREADS)
    s_b[q] = (j0 + q < u.nb) ? __ldg(u.B + j0 + q) : 0xffffffffu;
  __syncthreads();
  // this thread's diagonals [dl, dl + UN_ITEMS) of the window
  const uint32_t wa = i1 - i0, wb = j1 - j0, dn = d1 - d0;
  const uint32_t dl = min((uint32_t)threadIdx.x * UN_ITEMS, dn);
  uint32_t lo = dl > wb ? dl - wb : 0u, hi = min(dl, wa);
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (s_a[mid + 1] <= s_b[dl - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  uint32_t ia = lo, jb = dl - lo;  // window positions
  uint32_t vals[UN_ITEMS];
  uint8_t tags[UN_ITEMS];
  uint32_t kmask = 0, kc = 0;
#pragma unroll
  for (int it = 0; it < UN_ITEMS; ++it) {
    if (dl + it < dn) {
      const uint32_t av = s_a[ia + 1], bv = s_b[jb];
      const bool a_ok = i0 + ia < u.na, b_ok = j0 + jb < u.nb;
      // slab mode: the position in the owning chunk's set (tag 3/1: the
      // primary, 2: the other) instead of the Gaussian's index
      if (a_ok && (!b_ok || av <= bv)) {
        vals[it] = a.slab ? i0 + ia : av;
        tags[it] = (b_ok && bv == av) ? 3 : 1;
        kmask |= 1u << it;
        ++ia;
      } else {
        vals[it] = a.slab ? j0 + jb : bv;
        tags[it] = 2;
        if (!(i0 + ia > 0 && s_a[ia] == bv)) kmask |= 1u << it;
        ++jb;
      }
    }
  }
  kc = __popc(kmask);
  // block exclusive scan of the kept counts
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = kc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(FULL_MASK, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) s_w[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t wv = lane < UN_THREADS / 32 ? s_w[lane] : 0u;
    uint32_t wi = wv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL_MASK, wi, o);
      if (lane >= o) wi += t;
    }
    const uint32_t total = __shfl_sync(FULL_MASK, wi, UN_THREADS / 32 - 1);
    const uint32_t pre = lookback_warp(lb_status + a.part_base[l], part, total,
                                       fs->epoch + TK_UNION0);
    if (lane < UN_THREADS / 32) s_w[lane] = pre + wi - wv;
    if (lane == 0 && (part + 1) * UN_TILE >= n) fs->stats.U_level[l] = pre + total;
  }
  __syncthreads();
  uint32_t m = a.slot_base[l] + s_w[warp] + inc - kc;
#pragma unroll
  for (int it = 0; it < UN_ITEMS; ++it) {
    if ((kmask >> it) & 1u) {
      union_idx[m] = vals[it];
      union_tag[m] = tags[it];
      ++m;
    }
  }
}

// mode 1: chunk union (record or reuse the cache); 0: band selection (the
// union buffers now hold something else: drop the cache)
__global__ void k_union_sizes(int32_t L, FrameState *fs, int32_t mode, uint64_t uid) {
  if (threadIdx.x != 0) return;
  if (mode == 0) {
    fs->uc_uid = 0;
  } else if (fs->uc_hit) {
    for (int l = 0; l < L; ++l) fs->stats.U_level[l] = fs->uc_U[l];
  } else {
    for (int l = 0; l < L; ++l) fs->uc_U[l] = fs->stats.U_level[l];
    fs->uc_uid = uid;
    fs->uc_f = fs->stats.f;
    fs->uc_o = fs->stats.o;
  }
  uint32_t U = 0;
  for (int l = 0; l < L; ++l) U += fs->stats.U_level[l];
  fs->stats.U = U;
  fs->n_sort = U;  // fused path: every input is a depth-sort key (culled -> ~0)
}

// LOD-mode selection (select_active, reference src/lod.py:192-211): level l
// keeps the Gaussians whose camera distance ||mean - position|| (NumPy's
// sqrt((dx*dx + dy*dy) + dz*dz)) lies in [lo_l, hi_l); full mode is level 0
// with [0, inf) and empty bands elsewhere.  Kept indices are compacted in
// index order into the level's slots (tag 3: modulation 1), UN_TILE inputs
// per CTA in ticket order, block scan + per-level decoupled look-back.
struct BandArgs {
  const void *geom[LODGE_MAX_LEVELS];
  int64_t n[LODGE_MAX_LEVELS];
  double lo[LODGE_MAX_LEVELS], hi[LODGE_MAX_LEVELS];
  uint32_t slot_base[LODGE_MAX_LEVELS + 1];
  uint32_t part_base[LODGE_MAX_LEVELS + 1];
  int32_t L, geom32;
};

__global__ void __launch_bounds__(UN_THREADS) k_band_select(BandArgs a, FrameState *fs,
                                                           const double *__restrict__ pos,
                                                           uint64_t *lb_status,
                                                           uint32_t *union_idx,
                                                           uint8_t *union_tag) {
  // item-major: item it of lane l in warp w is input part*UN_TILE +
  // it*UN_THREADS + w*32 + l, so each load instruction of a warp reads 32
  // consecutive records (coalesced); kept inputs are ranked over (item,
  // warp, lane) -- index order -- by ballots and a scan of the per-(item,
  // warp) counts
  constexpr int NW = UN_THREADS / 32;
  static_assert(UN_ITEMS * NW <= 64, "two (item, warp) counts per lane");
  __shared__ uint32_t s_c[UN_ITEMS * NW];
  __shared__ uint32_t s_tk;
  const uint32_t g = take_ticket(&fs->tickets[TK_UNION0], &s_tk);
  int l = 0;
  while (l + 1 < a.L && g >= a.part_base[l + 1]) ++l;
  const uint32_t part = g - a.part_base[l];
  const int64_t n = a.n[l];
  const int64_t i0 = (int64_t)part * UN_TILE;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double px = pos[0], py = pos[1], pz = pos[2];
  uint32_t bal[UN_ITEMS];
#pragma unroll
  for (int it = 0; it < UN_ITEMS; ++it) {
    const int64_t i = i0 + it * UN_THREADS + tid;
    bool keep = false;
    if (i < n) {
      double mx, my, mz;
      if (a.geom32) {
        const float4 r = *reinterpret_cast<const float4 *>(
            reinterpret_cast<const float *>(a.geom[l]) + i * 12);  // 48 B records: 16-B aligned
        mx = r.x; my = r.y; mz = r.z;
      } else {
        const double *r = reinterpret_cast<const double *>(a.geom[l]) + i * 12;
        const double2 r01 = *reinterpret_cast<const double2 *>(r);
        mx = r01.x; my = r01.y; mz = r[2];
      }
      const double dx = mx - px, dy = my - py, dz = mz - pz;
      const double d = sqrt((dx * dx + dy * dy) + dz * dz);
      keep = d >= a.lo[l] && d < a.hi[l];
    }
    bal[it] = __ballot_sync(FULL_MASK, keep);
    if (lane == 0) s_c[it * NW + warp] = __popc(bal[it]);
  }
  __syncthreads();
  if (warp == 0) {  // exclusive offsets over (item, warp), then the level's look-back
    const uint32_t c0 = 2 * lane < UN_ITEMS * NW ? s_c[2 * lane] : 0u;
    const uint32_t c1 = 2 * lane + 1 < UN_ITEMS * NW ? s_c[2 * lane + 1] : 0u;
    const uint32_t v = c0 + c1;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL_MASK, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t total = __shfl_sync(FULL_MASK, inc, 31);
    const uint32_t pre = lookback_warp(lb_status + a.part_base[l], part, total,
                                       fs->epoch + TK_UNION0);
    if (2 * lane < UN_ITEMS * NW) s_c[2 * lane] = pre + inc - v;
    if (2 * lane + 1 < UN_ITEMS * NW) s_c[2 * lane + 1] = pre + inc - v + c0;
    if (lane == 0 && (int64_t)(part + 1) * UN_TILE >= n) fs->stats.U_level[l] = pre + total;
  }
  __syncthreads();
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int it = 0; it < UN_ITEMS; ++it) {
    if ((bal[it] >> lane) & 1u) {
      const uint32_t m = a.slot_base[l] + s_c[it * NW + warp] + __popc(bal[it] & lt);
      union_idx[m] = (uint32_t)(i0 + it * UN_THREADS + tid);
      union_tag[m] = 3;
    }
  }
}

void launch_band_select(const lodge_level *levels, int32_t L, const double *bounds, int32_t full,
                        const LevelSlots &ls, FrameState *fs, const double *pos,
                        uint64_t *status, uint32_t *union_idx, uint8_t *union_tag,
                        cudaStream_t s) {
  BandArgs a;
  a.L = L;
  a.geom32 = (levels[0].flags & LODGE_GEOM_FP32) ? 1 : 0;
  a.part_base[0] = 0;
  for (int l = 0; l < LODGE_MAX_LEVELS; ++l) {
    const bool on = l < L && (!full || l == 0);
    a.geom[l] = l < L ? levels[l].geom_dev : nullptr;
    a.n[l] = on ? levels[l].n : 0;
    a.lo[l] = full ? 0.0 : (l < L ? bounds[l] : 0.0);
    a.hi[l] = full ? INFINITY : (l < L ? bounds[l + 1] : 0.0);
  }
  for (int l = 0; l <= LODGE_MAX_LEVELS; ++l) a.slot_base[l] = l <= L ? ls.slot_base[l] : 0;
  for (int l = 0; l < L; ++l)
    a.part_base[l + 1] = a.part_base[l] + (uint32_t)((a.n[l] + UN_TILE - 1) / UN_TILE);
  for (int l = L + 1; l <= LODGE_MAX_LEVELS; ++l) a.part_base[l] = a.part_base[L];
  const uint32_t nparts = a.part_base[L];
  if (nparts > 0)
    k_band_select<<<nparts, UN_THREADS, 0, s>>>(a, fs, pos, status, union_idx, union_tag);
  k_union_sizes<<<1, 32, 0, s>>>(L, fs, 0, 0ull);
}

int launch_union(const lodge_chunks &ch, const LevelSlots &ls, FrameState *fs, uint64_t *status,
                  uint32_t *union_idx, uint8_t *union_tag, cudaStream_t s) {
  UnionArgs a;
  a.offsets = ch.offsets_dev;
  a.data = ch.data_dev;
  a.L = ch.L;
  uint32_t max_slots = 0;
  for (int l = 0; l <= LODGE_MAX_LEVELS; ++l) a.slot_base[l] = (l <= ch.L) ? ls.slot_base[l] : 0;
  for (int l = 0; l < ch.L; ++l) max_slots = max(max_slots, ls.slot_base[l + 1] - ls.slot_base[l]);
  a.status_stride = union_status_stride(max_slots);
  a.slab = ch.slab_geom_dev != nullptr ? 1 : 0;
  a.uid = ch.uid;
  a.part_base[0] = 0;
  for (int l = 0; l < ch.L; ++l)
    a.part_base[l + 1] =
        a.part_base[l] + (ls.slot_base[l + 1] - ls.slot_base[l] + UN_TILE - 1) / UN_TILE;
  // scratch in the look-back buffer: the merge-path splits as u32 (values
  // < 2^30 leave the flag bits clear, so no look-back reads them as ready),
  // then the per-level look-back words
  const uint32_t nparts = a.part_base[ch.L];
  uint32_t *splits = reinterpret_cast<uint32_t *>(status);
  uint64_t *lb = status + (nparts + ch.L + 2) / 2 + 1;
  int launches = 2;
  k_union_check<<<1, 32, 0, s>>>(a.uid, fs);
  if (max_slots > 0 && nparts > 0) {
    k_union_split<<<(nparts + ch.L + 255) / 256, 256, 0, s>>>(a, fs, splits);
    k_union_merge<<<nparts, UN_THREADS, 0, s>>>(a, fs, splits, lb, union_idx, union_tag);
    launches += 2;
  }
  k_union_sizes<<<1, 32, 0, s>>>(ch.L, fs, 1, a.uid);
  return launches;  // kernels enqueued
}

__global__ void k_begin_frame(FrameState *fs) {
  int i = threadIdx.x;
  if (i == 0) {
    fs->epoch += 32;
    fs->stats.M = 0;
    fs->stats.P = 0;
    fs->stats.overflow = 0;
    fs->stats.guard_hits = 0;
    fs->stats.P_first = 0;
    fs->stats.P_second = 0;
    fs->stats.fault = 0;
    fs->stats.M_first = 0;
    fs->stats.M_second = 0;
    fs->stats.comp_members = 0;
    fs->stats.block_lists = 0;
    fs->stats.sorted_first = 0;
    fs->split_S = 0;
    fs->P_A = 0;
    fs->n_alive = 0;
    fs->n_owners_b = 0;
    fs->n_cand = fs->n_ocand = 0;
    fs->sel_B = 0;
    fs->scan_a = fs->scan_b = 0;
    fs->n_sort_a = fs->n_sort_b = 0;
    fs->stats.f = -1;  // set by k_select_frame on the chunk paths
    fs->stats.o = -1;
    fs->stats.t = 1.0;
    fs->stats.t_bar = 1.0;
  }
  if (i < LODGE_MAX_LEVELS) fs->stats.U_level[i] = 0;
  if (i < 32) fs->tickets[i] = 0;
  if (i < 8) fs->counters[i] = 0;
  for (int k = i; k < 8 * 256; k += blockDim.x) (&fs->hist_depth[0][0])[k] = 0;
}

void launch_begin_frame(FrameState *fs, cudaStream_t s) { k_begin_frame<<<1, 256, 0, s>>>(fs); }

}  // namespace lodge
