"""GPU: the frame depth sort (32-bit keys + tie repair, csrc/k_sort.cu) gives
exactly np.lexsort((source_index, depth)) (reference src/raster.py:401) on
adversarial depths -- long runs of depths inside one fp32 ulp (> 32 members,
the CTA path of k_depth_ties), short runs, exactly equal depths (index order)
-- checked through the per-tile lists against the CPU oracle and, on a
one-tile image where every splat covers the tile, against NumPy's lexsort."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_23158_b200 as L  # noqa: E402
from paper_2505_23158_b200 import device as D  # noqa: E402
from paper_2505_23158_b200.raster import DeviceBatch, rasterize_device  # noqa: E402
from oracle import oracle as O  # noqa: E402


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    yield
    D.set_default_precision("exact")


def adversarial_depths(rng):
    d = []
    d += list(5.0 + rng.permutation(300) * 1e-10)           # one long run (one fp32 ulp)
    d += list(7.25 + rng.permutation(40) * 3e-9)            # a run just over 32
    for k in range(60):                                      # short runs of 2..5
        base = 2.0 + 0.37 * k
        d += list(base + rng.permutation(rng.integers(2, 6)) * 1e-12)
    d += [3.5] * 25 + [11.0] * 3                             # equal fp64 depths
    d += list(rng.uniform(0.06, 40.0, 400))                  # untied
    d = np.array(d)
    return d[rng.permutation(len(d))]


def make_batch(rng, depth, w, h, spread):
    M = depth.shape[0]
    mean2d = np.stack([rng.uniform(0.5 * w - spread, 0.5 * w + spread, M),
                       rng.uniform(0.5 * h - spread, 0.5 * h + spread, M)], axis=1)
    s = rng.uniform(2.0, 9.0, M)
    cov = np.zeros((M, 2, 2))
    cov[:, 0, 0] = cov[:, 1, 1] = s * s
    conic = np.stack([1.0 / (s * s), np.zeros(M), 1.0 / (s * s)], axis=1)
    extent = np.stack([3.0 * s, 3.0 * s], axis=1)
    opac = rng.uniform(0.05, 0.3, M)
    color = rng.uniform(0.0, 1.0, (M, 3))
    src = np.arange(M, dtype=np.int64)
    return L.Splat2DBatch(M, src, mean2d, cov, conic, extent, depth, opac, color)


def oracle_batch(b):
    return {"src": b.source_index, "mean2d": b.mean2d, "conic": b.conic, "extent": b.extent,
            "depth": b.depth, "opacity": b.opacity_eff, "color": b.color,
            "n_inputs": b.n_inputs}


def camera(w, h):
    return L.Camera(np.zeros(3), np.array([1.0, 0.0, 0.0, 0.0]), np.array([100.0, 100.0]),
                    np.array([w / 2, h / 2]), (w, h), 0.05)


@pytest.mark.parametrize("prec", ["exact", "fast"])
def test_tied_depths_lists_match_oracle(prec):
    rng = np.random.default_rng(11)
    w, h = 96, 80
    b = make_batch(rng, adversarial_depths(rng), w, h, 30.0)
    cam = camera(w, h)
    db = DeviceBatch.from_host(b, D.context().device)
    res = rasterize_device(db, cam, L.RasterConfig(), True, True, precision=prec, lists=True)
    ref = O.rasterize(oracle_batch(b), w, h, O.cfg_struct(L.RasterConfig()), lists=True)
    assert np.array_equal(res["tile_offsets"].cpu().numpy(), ref["tile_offsets"])
    assert np.array_equal(res["tile_src"].cpu().numpy(), ref["tile_src"])


def test_tied_depths_single_tile_is_lexsort():
    rng = np.random.default_rng(5)
    w, h = 16, 16
    depth = adversarial_depths(rng)
    b = make_batch(rng, depth, w, h, 2.0)  # every splat covers the one tile
    db = DeviceBatch.from_host(b, D.context().device)
    res = rasterize_device(db, camera(w, h), L.RasterConfig(), False, False, precision="fast",
                           lists=True)
    got = res["tile_src"].cpu().numpy()
    assert np.array_equal(got, np.lexsort((b.source_index, depth)))
