"""The reference bench's report fields on the host side (src/raster.py:464-479,
src/cli.py:283-320): the drop-in visibility_histogram and its edge checks
against vectors the reference produced (tests/golden/report.npz,
oracle/make_golden.py make_report)."""

from types import SimpleNamespace

import numpy as np
import pytest

from paper_2505_23158_b200.raster import check_bin_edges, visibility_histogram

from .golden_util import load

G = load("report.npz")
C1 = load("config1.npz")
EDGES = sorted(k.split("/", 1)[1] for k in G.files if k.startswith("edges/"))


@pytest.mark.parametrize("name", EDGES)
@pytest.mark.parametrize("v", range(8))
def test_host_histogram_matches_reference(v, name):
    out = SimpleNamespace(per_pixel_visible=C1[f"v{v}/o_visible"])
    got = visibility_histogram(out, G["edges/" + name])
    assert np.array_equal(got, G[f"v{v}/hist/{name}"])
    assert got.sum() == C1[f"v{v}/o_visible"].size


@pytest.mark.parametrize("i,bad", enumerate(([1.0], [3.0, 2.0], [0.0, 1.0, 1.0])))
def test_edge_messages_match_reference(i, bad):
    with pytest.raises(ValueError) as e:
        check_bin_edges(np.asarray(bad))
    assert str(e.value) == str(G["bad_edges_messages"][i])
