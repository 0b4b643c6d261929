"""LOD-mode and full-mode renders, CPU side: the band
bounds' host logic and the oracle's select_active + render against the
reference (tests/golden/modes.npz, oracle/make_golden.py make_modes)."""

from types import SimpleNamespace

import numpy as np
import pytest

from oracle import oracle as O
from paper_2505_23158_b200.lod import lod_bounds
from paper_2505_23158_b200.types import RasterConfig

from .golden_util import config1_levels, load
from .test_importance_cpu import golden_cameras

MD = load("modes.npz")
C1 = load("config1.npz")


def c1_levels():
    scenes = config1_levels(C1)
    return [SimpleNamespace(scene=s, depth_threshold=float(C1[f"L{l}/depth_threshold"]))
            for l, s in enumerate(scenes)]


def test_bounds_and_validation():
    lv = c1_levels()
    d1 = lv[1].depth_threshold
    assert lod_bounds(lv) == [0.0, d1, np.inf]
    assert lod_bounds(lv, [0.0, 1.5]) == [0.0, d1 + 1.5, np.inf]
    with pytest.raises(ValueError, match="one depth offset per level"):
        lod_bounds(lv, [0.0])
    bad = [lv[1], lv[0]]
    with pytest.raises(ValueError, match="strictly increasing depth thresholds"):
        lod_bounds(bad)


@pytest.mark.parametrize("v", [1, 5])
@pytest.mark.parametrize("tag,offs", [("lod", None), ("lodoff", [0.0, 1.5]), ("full", None)])
def test_oracle_modes_match_reference(v, tag, offs):
    lv = c1_levels()
    cam = golden_cameras([v])[0]
    if tag == "full":
        sets = [np.arange(len(lv[0].scene.means))] + [np.zeros(0, np.int64)]
    else:
        sets = O.select_active(lv, cam.position, lod_bounds(lv, offs))
        for l in range(2):
            assert np.array_equal(sets[l], MD[f"v{v}/{tag}/set{l}"])
    out = O.render_selection(lv, sets, None, O.camera_from(cam), O.cfg_struct(RasterConfig()))
    p = f"v{v}/{tag}/"
    assert np.array_equal(out["per_tile_count"], MD[p + "tile_count"])
    assert np.array_equal(out["per_pixel_visible"], MD[p + "visible"])
    np.testing.assert_allclose(out["image"], MD[p + "image"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(out["per_gaussian_max_weight"], MD[p + "maxw"], rtol=1e-13)
