"""Residency streaming (stream_step, src/blending.py:140-194) and the blend
factor along a path, against the reference's own walk on its street_runtime
fixture (tests/test_blending.py:21-33, 136-235 of the reference package),
recorded by oracle/make_golden.py make_street.  The state machine is host
control plane, but its nearest-two query is the device selection kernel
(no host fallback), so these run on the GPU."""

import numpy as np
import pytest

import paper_2505_23158_b200 as L
from paper_2505_23158_b200.types import BlendState

from .golden_util import config1_sets, load

pytestmark = pytest.mark.gpu

S = load("street.npz")
KINDS = ("load", "unload", "swap_primary")


def street_plan():
    return L.ChunkPlan(S["centers"], S["radii"], tuple(tuple(ch) for ch in config1_sets(S)),
                       np.zeros(0, np.int64))


def walk(plan, zs):
    """(events, states) in the golden layout: events (step, kind, chunk, x, y, z),
    states (loaded0, loaded1 or -1, primary, t_bar, t)."""
    state, ev, st = None, [], []
    for i, z in enumerate(zs):
        state, events = L.stream_step(state, plan, np.array([0.0, 0.5, z]))
        ev += [(i, KINDS.index(e.kind), e.chunk_id) + tuple(e.camera_position) for e in events]
        lc = state.loaded_chunks + (-1,) * (2 - len(state.loaded_chunks))
        st.append(lc + (state.primary_id, state.t_bar, state.t))
        assert 1 <= len(state.loaded_chunks) <= 2
    return np.array(ev, np.float64).reshape(-1, 6), np.array(st, np.float64)


@pytest.mark.parametrize("tag", ["walk", "teleport"])
def test_walk_matches_reference_bit_exact(tag):
    ev, st = walk(street_plan(), S[tag + "/zs"])
    assert np.array_equal(ev, S[tag + "/events"])
    assert np.array_equal(st, S[tag + "/states"])  # t_bar, t bit-exact


def test_initial_load_and_stationary():
    plan = street_plan()
    pos = np.array([0.0, 0.5, 10.0])
    state, events = L.stream_step(None, plan, pos)
    assert [e.kind for e in events] == ["load", "load"]
    assert set(state.loaded_chunks) == {0, 1}
    state2, events2 = L.stream_step(state, plan, pos)
    assert events2 == [] and state2.loaded_chunks == state.loaded_chunks


def test_collinear_walk_event_sequence():
    ev, _ = walk(street_plan(), np.linspace(8.0, 44.0, 400))
    kinds = [(KINDS[int(k)], int(c)) for k, c in ev[:, 1:3]]
    assert kinds == [("load", 0), ("load", 1), ("swap_primary", 1),
                     ("unload", 0), ("load", 2), ("swap_primary", 2)]


def test_secondary_swap_waits_for_full_fade():
    plan = street_plan()
    state, prev, saw = None, None, False
    for z in np.linspace(8.0, 44.0, 400):
        prev = state
        state, events = L.stream_step(state, plan, np.array([0.0, 0.5, z]))
        for e in events:
            if e.kind == "unload":
                saw = True
                _, t_out = L.blend_factor(np.array(e.camera_position),
                                          plan.centers[prev.primary_id], plan.centers[e.chunk_id])
                assert t_out == 1.0
    assert saw and state.loaded_chunks == (2, 1)


def test_single_chunk_plan_never_swaps():
    plan = L.ChunkPlan(np.zeros((1, 3)), np.array([1.0]), ((np.arange(10),),),
                       np.zeros(0, np.int64))
    state, events = L.stream_step(None, plan, np.zeros(3))
    assert [e.kind for e in events] == ["load"]
    for x in np.linspace(-20, 20, 50):
        state, events = L.stream_step(state, plan, np.array([x, 0, 0]))
        assert events == [] and state.t == 1.0


def test_teleport_reloads():
    plan = street_plan()
    state, _ = L.stream_step(None, plan, np.array([0.0, 0.5, 10.0]))
    state, events = L.stream_step(state, plan, np.array([0.0, 0.5, 60.0]))
    kinds = [e.kind for e in events]
    assert kinds.count("unload") == 2 and kinds.count("load") == 2
    assert set(state.loaded_chunks) == {2, 1}


def test_modulation_piecewise_linear_along_path():
    plan = street_plan()
    a, b = plan.centers[0], plan.centers[1]
    ts = []
    for lam in np.linspace(0, 1, 11):
        c = (1 - lam) * a + lam * b
        f, o = L.nearest_two_chunks(plan, c)[:2]
        pair = (f, o if o is not None else f)
        ts.append(L.blend_factor(c, plan.centers[pair[0]], plan.centers[pair[1]])[1])
    assert ts[0] == pytest.approx(1.0) and ts[5] == pytest.approx(0.5)
    assert ts[-1] == pytest.approx(1.0)
    diffs = np.diff(ts)
    assert np.allclose(np.abs(diffs), np.abs(diffs[0]), atol=1e-9)


def test_blend_state_secondary():
    s = BlendState((0, 1), 0, 1.5, 1.0)
    assert s.secondary_id == 1
    assert BlendState((3,), 3, 1.0, 1.0).secondary_id is None
