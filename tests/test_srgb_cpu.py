"""lodge_to_srgb8's level thresholds (csrc/lodge_api.cu): the reference's
to_uint8 (src/images.py:10-17) is a non-decreasing step function of the
fp32 input, so `levels(x) = #{k: t_k <= x}` with t_k the smallest fp32 x
where to_uint8(x) >= k.  Restates the bisection in NumPy and checks it
against to_uint8 itself on every fp32 value within 64 ulps of each
threshold, on 2M random values in [-0.1, 1.1] and on the special values."""

import numpy as np


def to_uint8(x):
    """The reference's formula (src/images.py:10-17)."""
    x = np.clip(np.asarray(x, dtype=np.float64), 0.0, 1.0)
    e = np.where(x <= 0.0031308, 12.92 * x, 1.055 * np.power(x, 1 / 2.4) - 0.055)
    return np.round(e * 255.0).astype(np.uint8)


def thresholds():
    t = np.empty(256, np.float32)
    t[0] = -np.inf
    for k in range(1, 256):
        lo, hi = 0, 0x3F800000
        while lo < hi:
            mid = (lo + hi) // 2
            if int(to_uint8(np.array([mid], np.uint32).view(np.float32))[0]) >= k:
                hi = mid
            else:
                lo = mid + 1
        t[k] = np.array([lo], np.uint32).view(np.float32)[0]
    return t


def levels(x, t):
    return np.searchsorted(t, np.asarray(x, np.float32), side="right") - 1


def test_thresholds_reproduce_to_uint8():
    t = thresholds()
    assert np.all(np.diff(t[1:]) > 0)
    bits = t[1:].view(np.uint32).astype(np.int64)
    near = (bits[:, None] + np.arange(-64, 65)[None, :]).ravel()
    near = near[(near >= 0) & (near <= 0x3F800000)].astype(np.uint32).view(np.float32)
    rng = np.random.default_rng(7)
    rand = rng.uniform(-0.1, 1.1, 2_000_000).astype(np.float32)
    special = np.array([0.0, -0.0, 1.0, -1.0, 2.0, np.inf, -np.inf, 1e-45, 0.0031308,
                        np.nextafter(np.float32(1.0), np.float32(0.0))], np.float32)
    for x in (near, rand, special):
        got = levels(x, t)
        ref = to_uint8(x)
        assert np.array_equal(got.astype(np.uint8), ref)
