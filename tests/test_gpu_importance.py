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


# ---- the reference's TestImportance / TestVisibilityFilter cases
# (tests/test_lod.py:73-112, tests/test_chunks.py:183-229 of the reference
# package) on the device path

C0 = 0.28209479177387814


def _cam(L):
    return L.Camera(np.zeros(3), np.array([1.0, 0, 0, 0]), np.array([50.0, 50.0]),
                    np.array([32.0, 32.0]), (64, 64), near_plane=0.05)


def _wall(L, z, half=4.0, opacity=0.99, color=0.6):
    sh = np.zeros((3, 1))
    sh[:, 0] = (color - 0.5) / C0
    return L.Gaussian(np.array([0, 0, z], float), np.array([half, half, 0.05]),
                      np.array([1.0, 0, 0, 0]), opacity, sh)


def _cfg(L):
    return SimpleNamespace(raster=L.RasterConfig(), gamma=0.02)


def _random_level(L, seed, n):
    from .test_gpu_raster_props import random_scene
    return L.LodLevel.base(random_scene(seed, n))


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_lone_fullframe_gaussian_scores_its_opacity(lodge, precision):
    L = lodge
    level = L.LodLevel.base(L.Scene.from_gaussians([_wall(L, 6.0, half=6.0, opacity=0.9)], 0))
    s = L.compute_importance(level, [_cam(L)], _cfg(L), precision=precision).scores
    assert s[0] == pytest.approx(0.9, abs=1e-3)


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_occluded_gaussian_scores_below_transmittance_bound(lodge, precision):
    L = lodge
    g = [_wall(L, 4.0, half=6.0, opacity=0.99), _wall(L, 8.0, half=2.0, opacity=0.9)]
    level = L.LodLevel.base(L.Scene.from_gaussians(g, 0))
    s = L.compute_importance(level, [_cam(L)], _cfg(L), precision=precision).scores
    assert s[1] < 0.02


def test_outside_frustum_scores_zero(lodge):
    L = lodge
    level = L.LodLevel.base(L.Scene.from_gaussians([_wall(L, -5.0)], 0))
    assert L.compute_importance(level, [_cam(L)], _cfg(L)).scores[0] == 0.0


def test_requires_views(lodge):
    L = lodge
    with pytest.raises(ValueError, match="view"):
        L.compute_importance(_random_level(L, 0, 5), [], _cfg(L))


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_perturbed_views_are_deterministic_and_monotone(lodge, precision):
    L = lodge
    level = _random_level(L, 3, 60)
    p = L.PerturbSpec(count=3, seed=11)
    a = L.compute_importance(level, [_cam(L)], _cfg(L), perturb=p, precision=precision).scores
    b = L.compute_importance(level, [_cam(L)], _cfg(L), perturb=p, precision=precision).scores
    np.testing.assert_array_equal(a, b)
    base = L.compute_importance(level, [_cam(L)], _cfg(L), precision=precision).scores
    assert np.all(a >= base - 1e-15)  # more views only raise a max over views


def test_behind_camera_gaussian_retained_via_perturbations(lodge):
    L = lodge
    front = L.Gaussian(np.array([0, 0, 6.0]), np.array([3, 3, 0.1]), np.array([1.0, 0, 0, 0]),
                       0.9, np.zeros((3, 1)))
    behind = L.Gaussian(np.array([0, 0, -6.0]), np.array([3, 3, 0.1]),
                        np.array([1.0, 0, 0, 0]), 0.9, np.zeros((3, 1)))
    levels = [L.LodLevel.base(L.Scene.from_gaussians([front, behind], 0))]
    plan = L.build_chunk_active_sets(levels, np.zeros((1, 3)), np.array([1.0]),
                                     np.zeros(1, np.int64))
    ccfg = SimpleNamespace(perturb_count=8, perturb_seed=2, perturb_law="uniform",
                           vis_threshold=0.02)
    cam = _cam(L)
    got = L.visibility_filter_chunk(plan, 0, levels, [cam], ccfg)
    assert 1 in got[0]
    sc = L.score_active_selection(levels, plan.active_sets[0], [cam], L.RasterConfig(),
                                  L.PerturbSpec(count=8, seed=2))[0]
    assert sc[1] >= 0.02
    plain = L.score_active_selection(levels, plan.active_sets[0], [cam], L.RasterConfig())[0]
    assert plain[1] == 0.0


def test_zero_threshold_drops_nothing_and_monotone(lodge):
    L = lodge
    levels = config1_levels(C1)
    plan = L.ChunkPlan(C1["centers"], C1["radii"], tuple(tuple(s) for s in config1_sets(C1)),
                       np.zeros(0, np.int64))
    cams = golden_cameras([0, 1])
    kept = {}
    for thr in (0.0, 0.005, 0.05):
        ccfg = SimpleNamespace(perturb_count=2, perturb_seed=0, perturb_law="uniform",
                               vis_threshold=thr)
        kept[thr] = L.visibility_filter_chunk(plan, 0, levels, cams, ccfg)
    for l in range(len(levels)):
        np.testing.assert_array_equal(kept[0.0][l], plan.active_sets[0][l])
        assert np.isin(kept[0.05][l], kept[0.005][l]).all()


def test_chunk_without_cameras_warns_and_skips(lodge):
    L = lodge
    levels = config1_levels(C1)
    plan = L.ChunkPlan(C1["centers"], C1["radii"], tuple(tuple(s) for s in config1_sets(C1)),
                       np.zeros(0, np.int64))
    ccfg = SimpleNamespace(perturb_count=2, perturb_seed=0, perturb_law="uniform",
                           vis_threshold=0.02)
    with pytest.warns(UserWarning, match="no assigned cameras"):
        got = L.visibility_filter_chunk(plan, 1, levels, [], ccfg)
    for l in range(len(levels)):
        np.testing.assert_array_equal(got[l], plan.active_sets[1][l])
