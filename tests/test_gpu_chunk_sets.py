"""Band selection on the device without a frame (lodge_select_active):
select_active (src/lod.py:192-211) against the reference's sets in
modes.npz, build_chunk_active_sets (src/chunks.py:122-135) against the
reference's street plan in street.npz (built by exactly that function), and
the reference's TestChunkActiveSets properties (tests/test_chunks.py:127-145
of the reference package).  Bit-exact: the sets are index lists."""

import numpy as np
import pytest

from .golden_util import config1_levels, config1_sets, load
from .test_importance_cpu import golden_cameras
from .test_modes_cpu import c1_levels

pytestmark = pytest.mark.gpu

MD = load("modes.npz")
S = load("street.npz")


@pytest.fixture(scope="module")
def L():
    import paper_2505_23158_b200 as lodge
    return lodge


def street_levels(L):
    return [L.LodLevel(l, float(S[f"L{l}/depth_threshold"]),
                       L.Scene(s.means, s.scales, s.rotations, s.opacities, s.sh_coeffs,
                               s.filter_variance, s.sh_degree),
                       np.arange(len(s.means)))
            for l, s in enumerate(config1_levels(S))]


@pytest.mark.parametrize("v", [1, 5])
@pytest.mark.parametrize("tag,offs", [("lod", None), ("lodoff", [0.0, 1.5])])
def test_select_active_matches_reference(L, v, tag, offs):
    lv = c1_levels()
    cam = golden_cameras([v])[0]
    got = L.select_active(lv, cam.position, offs)
    for l in range(len(lv)):
        ref = MD[f"v{v}/{tag}/set{l}"]
        assert got[l].dtype == np.int64 and np.array_equal(got[l], ref)


def test_build_chunk_active_sets_matches_reference(L):
    lv = street_levels(L)
    plan = L.build_chunk_active_sets(lv, S["centers"], S["radii"])
    ref = config1_sets(S)
    assert plan.n_chunks == len(ref)
    for j in range(plan.n_chunks):
        for l in range(len(lv)):
            assert np.array_equal(plan.active_sets[j][l], ref[j][l]), (j, l)
    np.testing.assert_array_equal(plan.radii, S["radii"])


def test_zero_radius_matches_plain_selection(L):
    lv = street_levels(L)
    plan = L.build_chunk_active_sets(lv, np.zeros((1, 3)), np.array([0.0]))
    for got, want in zip(plan.active_sets[0], L.select_active(lv, np.zeros(3))):
        np.testing.assert_array_equal(got, want)


def test_offset_keeps_midband_gaussian_in_fine_level(L):
    d1, r = 10.0, 4.0
    g = L.Gaussian(np.array([0, 0, d1 + r / 2]), np.full(3, 0.1), np.array([1.0, 0, 0, 0]),
                   0.5, np.zeros((3, 1)))
    scene = L.Scene.from_gaussians([g], 0)
    levels = [L.LodLevel.base(scene), L.LodLevel(1, d1, scene, np.zeros(1, np.int64))]
    plan = L.build_chunk_active_sets(levels, np.zeros((1, 3)), np.array([r]))
    np.testing.assert_array_equal(plan.active_sets[0][0], [0])
    assert plan.active_sets[0][1].size == 0


@pytest.mark.parametrize("seed", range(4))
def test_band_membership_brute_force(L, seed):
    """Random query points and offsets against a direct evaluation of the
    band predicate (NumPy's norm op order: ((dx^2 + dy^2) + dz^2))."""
    rng = np.random.default_rng(seed)
    lv = street_levels(L)
    q = rng.uniform([-3, -1, 0], [3, 3, 70])
    offs = [0.0, float(rng.uniform(0, 6))]
    got = L.select_active(lv, q, offs)
    bounds = L.lod_bounds(lv, offs)
    for l, level in enumerate(lv):
        d = np.linalg.norm(level.scene.means - q, axis=1)
        want = np.flatnonzero((d >= bounds[l]) & (d < bounds[l + 1]))
        np.testing.assert_array_equal(got[l], want)


def test_unsorted_levels_rejected(L):
    lv = street_levels(L)
    with pytest.raises(ValueError, match="strictly increasing depth thresholds"):
        L.select_active(lv[::-1], np.zeros(3))
    with pytest.raises(ValueError, match="one depth offset per level"):
        L.select_active(lv, np.zeros(3), [0.0])
