"""Threshold-search cost tables on the device against
the reference's ThresholdSearcher (tests/golden/thresholds.npz)."""

import numpy as np
import pytest

from .golden_util import load
from .test_importance_cpu import golden_cameras

pytestmark = pytest.mark.gpu

TH = load("thresholds.npz")
C1 = load("config1.npz")


def make_level(L, p, d, k):
    sc = L.Scene(d[p + "means"], d[p + "scales"], d[p + "rotations"], d[p + "opacities"],
                 d[p + "sh"], d[p + "fv"], int(d[p + "deg"]))
    prov = d[p + "provenance"] if (p + "provenance") in d else np.arange(len(sc))
    return L.LodLevel(k, float(TH["depths"][k]), sc, prov)


@pytest.fixture(scope="module")
def lodge():
    import paper_2505_23158_b200 as L
    from paper_2505_23158_b200 import thresholds
    levels = [make_level(L, "L0/", C1, 0), make_level(L, "P1/", TH, 1),
              make_level(L, "P2/", TH, 2)]
    return L, thresholds, levels


@pytest.mark.parametrize("k", [0, 1, 2])
def test_cover_tables_bit_exact(lodge, k):
    L, T, levels = lodge
    for vi, cam in enumerate(golden_cameras([0, 1, 2, 3])):
        dist, prefix = T.cover_table(levels[k], cam, L.RasterConfig())
        assert np.array_equal(dist, TH[f"T{k}/{vi}/dist"]), (k, vi)
        assert np.array_equal(prefix, TH[f"T{k}/{vi}/prefix"]), (k, vi)


def test_searcher_evaluate_matches_reference(lodge):
    L, T, levels = lodge
    by_depth = {float(TH["depths"][k]): levels[k] for k in (1, 2)}

    def builder(base, depth, cfg, single_round, subsample_views):
        assert single_round
        return by_depth[float(depth)], {}

    from types import SimpleNamespace
    cfg = SimpleNamespace(raster=L.RasterConfig())
    s = T.ThresholdSearcher(levels[0], golden_cameras([0, 1, 2, 3]), cfg, level_builder=builder)
    for name in ("e1", "e2"):
        ev = s.evaluate(list(TH[name + "/thresholds"]))
        assert ev.mean_gaussians_per_tile == float(TH[name + "/mean"])
        assert ev.per_view_cost == tuple(TH[name + "/per_view"])
        assert ev.build_cost_proxy == int(TH[name + "/build"])
    with pytest.raises(ValueError, match="strictly increasing"):
        s.evaluate([3.0, 1.0])


def test_cover_table_subset_and_empty(lodge):
    L, T, levels = lodge
    cam = golden_cameras([0])[0]
    idx = np.arange(0, 10000, 3)
    dist, prefix = T.cover_table(levels[0], cam, L.RasterConfig(), indices=idx)
    full_d, full_p = T.cover_table(levels[0], cam, L.RasterConfig())
    assert prefix[0] == 0 and np.all(np.diff(dist) >= 0)
    assert dist.shape[0] <= full_d.shape[0] and prefix[-1] <= full_p[-1]
    d0, p0 = T.cover_table(levels[0], cam, L.RasterConfig(), indices=np.zeros(0, np.int64))
    assert d0.shape == (0,) and list(p0) == [0]
