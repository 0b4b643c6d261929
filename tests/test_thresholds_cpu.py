"""Threshold-search cost tables, CPU side: the oracle's
_table restatement and the package's host-side band sums against the
reference (tests/golden/thresholds.npz, oracle/make_golden.py
make_thresholds)."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2505_23158_b200.thresholds import CostEvaluation
from paper_2505_23158_b200.types import RasterConfig

from .golden_util import load, scene
from .test_importance_cpu import golden_cameras

TH = load("thresholds.npz")
C1 = load("config1.npz")


def level_scene(k):
    return scene(C1, "L0/") if k == 0 else scene(TH, f"P{k}/")


@pytest.mark.parametrize("k", [0, 1, 2])
def test_oracle_cover_tables_match_reference(k):
    sc = level_scene(k)
    for vi, cam in enumerate(golden_cameras([0, 1, 2, 3])):
        dist, prefix = O.cover_table(sc, O.camera_from(cam), O.cfg_struct(RasterConfig()),
                                     cam.position)
        assert np.array_equal(dist, TH[f"T{k}/{vi}/dist"])
        assert np.array_equal(prefix, TH[f"T{k}/{vi}/prefix"])


def test_cost_evaluation_validation():
    with pytest.raises(ValueError, match="strictly increasing"):
        CostEvaluation((2.0, 1.0), 0.0, (), (), 0)
