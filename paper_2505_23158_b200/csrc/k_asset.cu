// Asset upload: the decode and value checks of
// read_asset's _parse_level_blob (reference src/assets.py:257-282) and its
// index-set checks (:448-453), on the device.
//
// A level blob is n little-endian fp32 records of W = 12 + 3*(deg+1)^2
// floats [mean3, scale3, rot4, opacity, fv, sh...] (src/assets.py:240-254).
// k_asset_split walks the blob as a flat float array (coalesced reads), writes
// each float to the geometry store (n x 12) or the SH store (n x 3T) and
// records which of the reference's checks fail.  The checks run on the fp32
// values: the reference converts to fp64 first, which is exact, so every
// comparison decides identically.  The rotation check needs the fp64 norm in
// NumPy's order, np.linalg.norm(axis=1) = sqrt(((w*w + x*x) + y*y) + z*z)
// (add.reduce over a length-4 row), which k_asset_rot computes per record.
#include "internal.cuh"

namespace lodge {

__global__ void __launch_bounds__(256) k_asset_split(const float *__restrict__ blob, int64_t n,
                                                     int32_t width, float *__restrict__ geom,
                                                     float *__restrict__ sh,
                                                     int32_t *__restrict__ flags) {
  const int64_t total = n * width;
  const int32_t terms3 = width - 12;
  int32_t bad = 0;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < total;
       f += (int64_t)gridDim.x * blockDim.x) {
    const float x = blob[f];
    const int64_t i = f / width;
    const int32_t c = (int32_t)(f - i * width);
    if (!isfinite(x)) bad |= LODGE_ASSET_NONFINITE;
    if (c >= 3 && c < 6 && !(x > 0.f)) bad |= LODGE_ASSET_SCALE;
    if (c == 10 && (x < 0.f || x > 1.f)) bad |= LODGE_ASSET_OPACITY;
    if (c == 11 && x < 0.f) bad |= LODGE_ASSET_FV;
    if (c < 12) geom[i * 12 + c] = x;
    else sh[i * terms3 + (c - 12)] = x;
  }
  // NaN compares false everywhere above, like NumPy's comparisons
  bad = __reduce_or_sync(FULL_MASK, bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicOr(flags, bad);
}

__global__ void __launch_bounds__(256) k_asset_rot(const float *__restrict__ geom, int64_t n,
                                                   int32_t *__restrict__ flags) {
  int32_t bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    // rot starts 24 bytes into the 48-byte record: two 8-byte loads
    const float2 q0 = *reinterpret_cast<const float2 *>(geom + i * 12 + 6);
    const float2 q1 = *reinterpret_cast<const float2 *>(geom + i * 12 + 8);
    const double w = q0.x, x = q0.y, y = q1.x, z = q1.y;
    const double nn = sqrt(((w * w + x * x) + y * y) + z * z);
    if (fabs(nn - 1.0) > 1e-3) bad = LODGE_ASSET_ROTATION;
  }
  bad = __reduce_or_sync(FULL_MASK, bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicOr(flags, bad);
}

// One CTA per index set (j, l): bit 0 not strictly increasing, bit 1 an
// index >= level_size[l].
__global__ void __launch_bounds__(256) k_asset_sets(const int64_t *__restrict__ offsets,
                                                    const uint32_t *__restrict__ data, int32_t L,
                                                    const int64_t *__restrict__ level_size,
                                                    int32_t *__restrict__ set_flags) {
  const int32_t s = blockIdx.x;
  const int64_t b = offsets[s], e = offsets[s + 1];
  const int64_t lim = level_size[s % L];
  int32_t bad = 0;
  for (int64_t k = b + threadIdx.x; k < e; k += blockDim.x) {
    const uint32_t v = data[k];
    if (k + 1 < e && !(data[k + 1] > v)) bad |= 1;
    if ((int64_t)v >= lim) bad |= 2;
  }
  bad = __reduce_or_sync(FULL_MASK, bad);
  if ((threadIdx.x & 31) == 0 && bad) atomicOr(set_flags + s, bad);
}

void launch_asset_split(const float *blob, int64_t n, int32_t width, float *geom, float *sh,
                        int32_t *flags_dev, cudaStream_t s) {
  if (n <= 0) return;
  const int64_t total = n * width;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_asset_split<<<(unsigned)blocks, 256, 0, s>>>(blob, n, width, geom, sh, flags_dev);
  int64_t rb = (n + 255) / 256;
  if (rb > 148 * 16) rb = 148 * 16;
  k_asset_rot<<<(unsigned)rb, 256, 0, s>>>(geom, n, flags_dev);
}

void launch_asset_sets(const lodge_chunks &ch, const int64_t *level_size_dev, int32_t *flags_dev,
                       cudaStream_t s) {
  const int32_t nsets = ch.K * ch.L;
  if (nsets <= 0) return;
  k_asset_sets<<<nsets, 256, 0, s>>>(ch.offsets_dev, ch.data_dev, ch.L, level_size_dev,
                                     flags_dev);
}

}  // namespace lodge
