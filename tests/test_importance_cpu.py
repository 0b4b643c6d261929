"""Importance scoring, CPU side: the oracle's
score_active_selection and the package's host logic for perturbed views
(random_rotations, scoring_views) against the reference's own outputs
(tests/golden/importance.npz, oracle/make_golden.py make_importance)."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2505_23158_b200.importance import random_rotations, scoring_views
from paper_2505_23158_b200.types import Camera, PerturbSpec, RasterConfig

from .golden_util import config1_levels, config1_sets, load

IMP = load("importance.npz")
C1 = load("config1.npz")


def golden_cameras(ids):
    out = []
    for v in ids:
        p = f"v{v}/"
        out.append(Camera(C1[p + "pos"], C1[p + "quat"], C1[p + "focal"], C1[p + "pp"],
                          tuple(int(x) for x in C1[p + "res"]), float(C1[p + "near"]), f"v{v}"))
    return out


def oracle_scores(levels, sets, views):
    cams = [O.camera_from(v) for v in views]
    return O.importance(levels, sets, cams, O.cfg_struct(RasterConfig()))


def test_random_rotations_unit_and_deterministic():
    q1 = random_rotations(np.random.default_rng(5), 64)
    q2 = random_rotations(np.random.default_rng(5), 64)
    assert q1.shape == (64, 4) and np.array_equal(q1, q2)
    assert np.allclose(np.linalg.norm(q1, axis=1), 1.0, atol=1e-12)


def test_scoring_views_layout():
    base = golden_cameras([0, 1])
    views = scoring_views(base, PerturbSpec(3, 7))
    assert len(views) == 2 + 2 * 3
    q = random_rotations(np.random.default_rng(7), 6)
    for vi in range(2):
        for k in range(3):
            v = views[2 + vi * 3 + k]
            assert np.array_equal(v.position, base[vi].position)
            assert np.allclose(v.orientation, q[vi * 3 + k] / np.linalg.norm(q[vi * 3 + k]))
    assert scoring_views(base, None) == base
    assert scoring_views(base, PerturbSpec(0, 1)) == base


def test_perturb_spec_validation():
    with pytest.raises(ValueError):
        PerturbSpec(-1)
    with pytest.raises(ValueError):
        PerturbSpec(1, 0, "gaussian")


def test_oracle_compute_importance_matches_reference():
    levels = config1_levels(C1)
    views = scoring_views(golden_cameras([0, 1, 2, 3]), PerturbSpec(2, 5))
    got = oracle_scores([levels[0]], [np.arange(len(levels[0].means))], views)[0]
    ref = IMP["a/scores"]
    assert got.shape == ref.shape
    # the C oracle's exp is glibc's, NumPy's is AVX-512 (<= 1 ulp apart)
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=0)
    assert np.array_equal(got > 0, ref > 0)


def test_oracle_score_active_selection_matches_reference():
    levels = config1_levels(C1)
    sets = config1_sets(C1)[2]
    views = scoring_views(golden_cameras([4, 5]), PerturbSpec(1, 9))
    got = oracle_scores(levels, sets, views)
    for l in range(len(levels)):
        np.testing.assert_allclose(got[l], IMP[f"b/scores{l}"], rtol=1e-13, atol=0)


def test_oracle_visibility_filter_matches_reference():
    levels = config1_levels(C1)
    sets = config1_sets(C1)[0]
    views = scoring_views(golden_cameras([0, 1]), PerturbSpec(2, 3 + 0))
    sc = oracle_scores(levels, sets, views)
    thr = float(IMP["c/vis_threshold"])
    for l in range(len(levels)):
        kept = np.asarray(sets[l])[sc[l] >= thr]
        assert np.array_equal(kept, IMP[f"c/kept{l}"])
