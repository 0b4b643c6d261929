// K7: per-frame report metrics of the reference bench (src/cli.py:283-320)
// on the device: the visibility histogram (src/raster.py:464-479), the mean
// per-tile count, the visible-Gaussian count (nonzero max weights) and the
// squared error against another image (psnr_vs_full).  One pass over each
// output buffer, block-local shared histograms, one atomic per bin per CTA.
#include <algorithm>

#include "internal.cuh"

namespace lodge {

constexpr int REPORT_MAX_BINS = 256;

// out[0 .. n_bins): histogram; out[n_bins]: sum of tile counts;
// out[n_bins + 1]: inputs with a nonzero max weight.
__global__ void __launch_bounds__(256) k_frame_report(const int32_t *__restrict__ visible,
                                                      int64_t n_px, const double *__restrict__ edges,
                                                      int32_t n_edges,
                                                      const int32_t *__restrict__ tile_count,
                                                      int64_t n_tiles, const void *maxw,
                                                      int32_t maxw_fp64, int64_t n_inputs,
                                                      unsigned long long *out) {
  __shared__ unsigned long long h[REPORT_MAX_BINS];
  __shared__ double e[REPORT_MAX_BINS + 1];
  __shared__ unsigned long long s_tiles, s_vis;
  const int n_bins = n_edges - 1;
  for (int i = threadIdx.x; i < n_bins; i += blockDim.x) h[i] = 0ull;
  for (int i = threadIdx.x; i < n_edges; i += blockDim.x) e[i] = edges[i];
  if (threadIdx.x == 0) s_tiles = s_vis = 0ull;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t first = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = first; i < n_px; i += stride) {
    // np.searchsorted(edges, v, side="right") - 1, clipped to [0, n_bins)
    const double v = (double)visible[i];
    int lo = 0, hi = n_edges;  // first edge > v
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (e[mid] <= v) lo = mid + 1;
      else hi = mid;
    }
    const int b = min(max(lo - 1, 0), n_bins - 1);
    atomicAdd(&h[b], 1ull);
  }
  unsigned long long t = 0, nz = 0;
  for (int64_t i = first; i < n_tiles; i += stride) t += (unsigned long long)tile_count[i];
  if (maxw) {
    for (int64_t i = first; i < n_inputs; i += stride) {
      const bool pos = maxw_fp64 ? reinterpret_cast<const double *>(maxw)[i] != 0.0
                                 : reinterpret_cast<const float *>(maxw)[i] != 0.f;
      nz += pos ? 1ull : 0ull;
    }
  }
  t = __reduce_add_sync(FULL_MASK, (unsigned)t) + 0ull;  // per-warp partials fit 32 bits
  nz = __reduce_add_sync(FULL_MASK, (unsigned)nz) + 0ull;
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&s_tiles, t);
    atomicAdd(&s_vis, nz);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n_bins; i += blockDim.x)
    if (h[i]) atomicAdd(&out[i], h[i]);
  if (threadIdx.x == 0) {
    if (s_tiles) atomicAdd(&out[n_bins], s_tiles);
    if (s_vis) atomicAdd(&out[n_bins + 1], s_vis);
  }
}

// Sum of squared differences of two fp32 images (n values), fp64.
__global__ void __launch_bounds__(256) k_sq_err(const float *__restrict__ a,
                                                const float *__restrict__ b, int64_t n,
                                                double *out) {
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double d = (double)a[i] - (double)b[i];
    acc = fma(d, d, acc);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL_MASK, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

static unsigned report_grid(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 8));
}

void launch_frame_report(const int32_t *visible, int64_t n_px, const double *edges_dev,
                         int32_t n_edges, const int32_t *tile_count, int64_t n_tiles,
                         const void *maxw, int32_t maxw_fp64, int64_t n_inputs,
                         unsigned long long *out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(unsigned long long) * (size_t)(n_edges + 1), s);
  k_frame_report<<<report_grid(std::max(n_px, std::max(n_tiles, n_inputs))), 256, 0, s>>>(
      visible, n_px, edges_dev, n_edges, tile_count, n_tiles, maxw, maxw_fp64, n_inputs, out);
}

void launch_sq_err(const float *a, const float *b, int64_t n, double *out, cudaStream_t s) {
  cudaMemsetAsync(out, 0, sizeof(double), s);
  k_sq_err<<<report_grid(n), 256, 0, s>>>(a, b, n, out);
}

}  // namespace lodge
