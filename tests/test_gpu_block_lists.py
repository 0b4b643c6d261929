"""GPU: block lists (csrc/k_bin.cu k_block_lists, the
compositor's block walk in csrc/k_composite.cu) give bitwise the outputs of
sorted per-tile lists -- image, per_pixel_visible, per_tile_count, max
weights, P and M.  lodge_set_block_lists FORCE takes them for every phase
that fits (<= 128k splats) whatever the splat sizes, OFF never: the street
sweep at 1080p for budgets from one pair per tile to more than P, an odd
resolution (partial blocks on the right and bottom edges), a frame smaller
than one block, LOD and full modes, and frames in flight.  The one-pass
frame they are compared with is pinned to the oracle (tests/test_gpu_scale.py);
the config-2/3/4 frames of tests/test_gpu_bench_parity.py take block lists
in AUTO mode."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_23158_b200 as L  # noqa: E402
from paper_2505_23158_b200.device import DeviceLevel, DevicePlan  # noqa: E402
from fixtures import scenes  # noqa: E402

from .test_gpu_two_phase import assert_same, outputs  # noqa: E402


@pytest.fixture(scope="module")
def street():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cfg = scenes.build("street1080")
    dev = torch.device("cuda", 0)
    levels = [DeviceLevel.from_tensors(torch.from_numpy(g).to(dev), torch.from_numpy(s).to(dev),
                                       cfg.degree) for g, s, _ in cfg.levels]
    plan = DevicePlan.from_arrays(cfg.centers, cfg.offsets, cfg.data, cfg.L, dev)
    one = L.Renderer(levels, plan, storage="fp32", precision="fast", full_lists=True)
    return cfg, levels, plan, one


def renderer(street, mode, budget, **kw):
    _, levels, plan, _ = street
    return L.Renderer(levels, plan, storage="fp32", precision="fast", phase_budget=budget,
                      block_lists=mode, **kw)


@pytest.mark.parametrize("budget", [1, 40, 300, 1536, 2048, 1 << 20])
@pytest.mark.parametrize("z", [6.0, 47.0, 118.0])
def test_forced_block_lists_equal_sorted_lists(street, budget, z):
    cfg, levels, plan, one = street
    cam = scenes.camera(z)
    ref = outputs(*one.render_camera(cam))
    frf, stf = renderer(street, "force", budget).render_camera(cam)
    fro, sto = renderer(street, "off", budget).render_camera(cam)
    assert_same(outputs(frf, stf), ref)
    assert_same(outputs(fro, sto), ref)
    assert stf.fault == 0 and sto.fault == 0
    assert sto.block_lists == 0
    if stf.M_first <= 131072 and stf.P_first > 0:
        assert stf.block_lists & 1  # the first phase took block lists
    if stf.M_second and stf.M_second <= 131072:
        assert stf.block_lists & 2


@pytest.mark.parametrize("w,h", [(1277, 719), (100, 50), (16, 16)])
def test_forced_block_lists_partial_blocks(street, w, h):
    cfg, levels, plan, one = street
    cam = scenes.camera(31.0, width=w, height=h, focal=scenes.FOCAL * w / 1920)
    ref = outputs(*one.render_camera(cam))
    for budget in (8, 64):
        fr, st = renderer(street, "force", budget).render_camera(cam)
        assert_same(outputs(fr, st), ref)
        assert st.fault == 0


@pytest.mark.parametrize("full", [False, True])
def test_forced_block_lists_lod_and_full_modes(street, full):
    cfg, levels, plan, one = street
    bounds = [0.0] + [float(cfg.levels[l][2]) for l in range(1, cfg.L)] + [float("inf")]
    cam = scenes.camera(52.0)
    ref = outputs(*one.render_lod_camera(cam, bounds, full))
    fr, st = renderer(street, "force", 200).render_lod_camera(cam, bounds, full)
    assert_same(outputs(fr, st), ref)
    assert st.fault == 0


def test_forced_block_lists_frames_in_flight(street):
    cfg, levels, plan, one = street
    r = renderer(street, "force", 300, n_streams=3)
    cams_h = [scenes.camera(z) for z in (9.0, 23.0, 61.0, 90.0, 14.0, 77.0)]
    refs = [outputs(*one.render_camera(c)) for c in cams_h]
    r.reserve(max(x["P"] for x in refs) + 4096)
    cams = r.upload_cameras(cams_h)
    frames = [r.alloc_frame(1920, 1080) for _ in cams_h]
    for j in range(len(cams_h)):
        r.render(cams[j], frames[j], slot=j % 3)
    torch.cuda.synchronize()
    for j, fr in enumerate(frames):
        st = fr.read_stats()
        assert_same(outputs(fr, st), refs[j])
        assert st.block_lists & 1
    assert r.fault_flags() == 0


def test_block_list_mode_is_validated(street):
    with pytest.raises(ValueError):
        renderer(street, "sometimes", 300)


@pytest.mark.parametrize("share", [1, 2, 7])
@pytest.mark.parametrize("z", [6.0, 47.0])
def test_grid_share_same_outputs(street, share, z):
    """lodge_set_grid_share caps the projection's and the record gather's
    persistent grids (frames in flight); the outputs do not depend on it."""
    cfg, levels, plan, one = street
    cam = scenes.camera(z)
    ref = outputs(*one.render_camera(cam))
    base = renderer(street, "auto", 1536)
    assert base.grid_share == 0
    fr0, st0 = base.render_camera(cam)
    fr, st = renderer(street, "auto", 1536, grid_share=share).render_camera(cam)
    assert_same(outputs(fr, st), outputs(fr0, st0))
    assert_same(outputs(fr, st), ref)
    assert st.fault == 0


def test_grid_share_rejects_negative(street):
    with pytest.raises(ValueError):
        renderer(street, "auto", 1536, grid_share=-1)
