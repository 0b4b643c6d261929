"""Host-side error behaviour of the drop-in API: the same exceptions and
messages as the reference (messages cited from src/blending.py, src/raster.py
and src/scene.py).  These checks run before any device work."""

import numpy as np
import pytest

import paper_2505_23158_b200 as L
from paper_2505_23158_b200.types import BlendState, StreamEvent


def plan2():
    sets = ((np.array([0, 2]), np.array([1])), (np.array([1, 3]), np.array([0])))
    return L.ChunkPlan(np.array([[0.0, 0, 0], [1.0, 0, 0]]), np.array([1.0, 1.0]), sets,
                       np.zeros(0, np.int64))


def test_compose_active_errors():  # src/blending.py:110-118
    p = plan2()
    with pytest.raises(ValueError, match="^chunk 5 is not in the plan$"):
        L.compose_active(p, [None, None], 5, None, 1.0)
    with pytest.raises(ValueError, match="^chunk -1 is not in the plan$"):
        L.compose_active(p, [None, None], -1, None, 1.0)
    with pytest.raises(ValueError, match="^chunk 7 is not in the plan$"):
        L.compose_active(p, [None, None], 0, 7, 0.5)
    with pytest.raises(ValueError, match="^blending needs two distinct chunks$"):
        L.compose_active(p, [None, None], 1, 1, 0.5)


def test_compose_active_single_chunk_is_host_only():  # src/blending.py:112-114
    sel = L.compose_active(plan2(), [None, None], 1, None, 0.3)
    assert [list(s) for s in sel.sets] == [[1, 3], [0]]
    assert all(np.all(m == 1.0) for m in sel.modulations)


def test_visibility_histogram_errors():  # src/raster.py:473-475
    out = L.TileRenderOutput(None, np.zeros((1, 1)), np.zeros((2, 2), np.int64), None, {})
    with pytest.raises(ValueError, match="need at least two bin edges"):
        L.visibility_histogram(out, [1.0])
    with pytest.raises(ValueError, match="bin edges must be strictly increasing"):
        L.visibility_histogram(out, [0.0, 2.0, 1.0])
    assert list(L.visibility_histogram(out, [0, 1, 5])) == [4, 0]


def test_chunk_plan_and_level_validation():  # src/scene.py:215-256
    with pytest.raises(ValueError, match="a chunk plan needs at least one chunk"):
        L.ChunkPlan(np.zeros((0, 3)), np.zeros(0), (), np.zeros(0, np.int64))
    with pytest.raises(ValueError, match="centers, radii and active_sets must have equal length"):
        L.ChunkPlan(np.zeros((2, 3)), np.zeros(1), ((np.zeros(0),),), np.zeros(0, np.int64))
    with pytest.raises(ValueError, match="chunk radii must be non-negative"):
        L.ChunkPlan(np.zeros((1, 3)), np.array([-1.0]), ((np.zeros(0),),), np.zeros(0, np.int64))


def test_stream_types_validation():  # src/blending.py:28-63
    with pytest.raises(ValueError, match="unknown stream event kind"):
        StreamEvent("teleport", 0, (0.0, 0.0, 0.0))
    with pytest.raises(ValueError, match="exactly one or two chunks may be resident"):
        BlendState((), 0, 1.0, 1.0)
    with pytest.raises(ValueError, match="resident chunk ids must be distinct"):
        BlendState((1, 1), 1, 1.0, 1.0)
    with pytest.raises(ValueError, match="primary chunk must be resident"):
        BlendState((0, 1), 2, 1.0, 1.0)


def test_camera_validation():  # src/scene.py:100-109
    q = np.array([1.0, 0, 0, 0])
    with pytest.raises(ValueError, match="focal must be positive"):
        L.Camera(np.zeros(3), q, np.array([0.0, 1.0]), np.zeros(2), (4, 4))
    with pytest.raises(ValueError, match="resolution must be positive"):
        L.Camera(np.zeros(3), q, np.ones(2), np.zeros(2), (0, 4))
    with pytest.raises(ValueError, match="orientation quaternion norm"):
        L.Camera(np.zeros(3), 2 * q, np.ones(2), np.zeros(2), (4, 4))
