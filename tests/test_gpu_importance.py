"""Importance scoring on the device against the
reference's own outputs (tests/golden/importance.npz) and the oracle.
EXACT reproduces the reference's fp64 weights; FAST has fp32 weights with
the reference's skip decisions."""

from types import SimpleNamespace

import numpy as np
import pytest

from .golden_util import config1_levels, config1_sets, load
from .test_importance_cpu import golden_cameras

pytestmark = pytest.mark.gpu

IMP = load("importance.npz")
C1 = load("config1.npz")


@pytest.fixture(scope="module")
def lodge():
    import paper_2505_23158_b200 as L
    return L


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_compute_importance(lodge, precision):
    levels = config1_levels(C1)
    cfg = SimpleNamespace(raster=lodge.RasterConfig(), gamma=float(IMP["a/gamma"]))
    imp = lodge.compute_importance(levels[0], golden_cameras([0, 1, 2, 3]), cfg,
                                   lodge.PerturbSpec(2, 5), precision=precision)
    assert isinstance(imp, lodge.ImportanceScores)
    assert imp.threshold_base == cfg.gamma
    ref = IMP["a/scores"]
    assert imp.scores.shape == ref.shape and imp.scores.dtype == np.float64
    if precision == "exact":
        np.testing.assert_allclose(imp.scores, ref, rtol=1e-12, atol=0)
        assert np.array_equal(imp.scores > 0, ref > 0)
    else:
        np.testing.assert_allclose(imp.scores, ref, rtol=1e-4, atol=1e-7)
        assert np.mean((imp.scores > 0) != (ref > 0)) <= 1e-3


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_score_active_selection_two_levels(lodge, precision):
    levels = config1_levels(C1)
    sets = config1_sets(C1)[2]
    got = lodge.score_active_selection(levels, sets, golden_cameras([4, 5]),
                                       lodge.RasterConfig(), lodge.PerturbSpec(1, 9),
                                       precision=precision)
    for l in range(len(levels)):
        ref = IMP[f"b/scores{l}"]
        if precision == "exact":
            np.testing.assert_allclose(got[l], ref, rtol=1e-12, atol=0)
        else:
            np.testing.assert_allclose(got[l], ref, rtol=1e-4, atol=1e-7)


def test_visibility_filter_chunk_exact(lodge):
    levels = config1_levels(C1)
    sets = config1_sets(C1)
    plan = lodge.ChunkPlan(C1["centers"], C1["radii"], tuple(tuple(s) for s in sets),
                           np.zeros(0, np.int64))
    cfg = SimpleNamespace(perturb_count=2, perturb_seed=3, perturb_law="uniform",
                          vis_threshold=float(IMP["c/vis_threshold"]))
    kept = lodge.visibility_filter_chunk(plan, 0, levels, golden_cameras([0, 1]), cfg,
                                         precision="exact")
    for l in range(len(levels)):
        assert np.array_equal(np.asarray(kept[l]), IMP[f"c/kept{l}"])


def test_accumulate_is_max_over_views(lodge):
    """One call over views {a, b} equals the element-wise max of two calls."""
    levels = config1_levels(C1)
    sets = config1_sets(C1)[1]
    rc = lodge.RasterConfig()
    both = lodge.score_active_selection(levels, sets, golden_cameras([2, 6]), rc,
                                        precision="exact")
    a = lodge.score_active_selection(levels, sets, golden_cameras([2]), rc, precision="exact")
    b = lodge.score_active_selection(levels, sets, golden_cameras([6]), rc, precision="exact")
    for l in range(len(levels)):
        assert np.array_equal(both[l], np.maximum(a[l], b[l]))


def test_errors(lodge):
    levels = config1_levels(C1)
    sets = config1_sets(C1)[0]
    rc = lodge.RasterConfig()
    with pytest.raises(ValueError, match="at least one view"):
        lodge.score_active_selection(levels, sets, [], rc)
    with pytest.raises(ValueError, match="sorted and unique"):
        lodge.score_active_selection(levels, [sets[0][::-1], sets[1]], golden_cameras([0]), rc)
