"""GPU: two-phase FAST frames (csrc/k_bin.cu k_dup_count / k_setup_b /
k_emit_b, k_composite phases 1 and 2) give bitwise the outputs of
one pass over the full per-tile lists -- image, per_pixel_visible,
per_tile_count, max weights, P and M -- for first-phase budgets from one pair
per tile (almost everything in the second phase) to more than P (no second
phase), along the street sweep at 1080p, an odd resolution, in LOD and full
modes, and with frames in flight on two streams.  One pass is itself pinned
to the oracle (tests/test_gpu_scale.py)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_23158_b200 as L  # noqa: E402
from paper_2505_23158_b200.device import DeviceLevel, DevicePlan  # noqa: E402
from fixtures import scenes  # noqa: E402


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


def outputs(fr, st):
    torch.cuda.synchronize()
    return {"image": fr.image.cpu().numpy().copy(), "visible": fr.visible.cpu().numpy().copy(),
            "tile_count": fr.tile_count.cpu().numpy().copy(),
            "maxw": fr.maxw[:st.U].cpu().numpy().copy(), "P": st.P, "M": st.M, "U": st.U}


def assert_same(a, b):
    for k in ("P", "M", "U"):
        assert a[k] == b[k], k
    for k in ("tile_count", "visible", "image", "maxw"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("budget", [1, 40, 300, 1280, 1536, 2048, 1 << 20])
@pytest.mark.parametrize("z", [6.0, 47.0, 118.0])
def test_two_phase_equals_one_pass(street, budget, z):
    cfg, levels, plan, one = street
    two = L.Renderer(levels, plan, storage="fp32", precision="fast", phase_budget=budget)
    cam = scenes.camera(z)
    fr1, st1 = one.render_camera(cam)
    ref = outputs(fr1, st1)
    fr2, st2 = two.render_camera(cam)
    got = outputs(fr2, st2)
    assert_same(got, ref)
    assert st2.fault == 0 and st1.fault == 0
    assert st2.P_first <= st2.P and st2.P_first + st2.P_second <= st2.P
    if budget >= (1 << 20):
        assert st2.P_first == st2.P and st2.P_second == 0
    assert st1.P_first == st1.P and st1.P_second == 0


def test_two_phase_odd_resolution(street):
    cfg, levels, plan, one = street
    two = L.Renderer(levels, plan, storage="fp32", precision="fast", phase_budget=64)
    cam = scenes.camera(31.0, width=1277, height=719, focal=scenes.FOCAL * 1277 / 1920)
    assert_same(outputs(*two.render_camera(cam)), outputs(*one.render_camera(cam)))


@pytest.mark.parametrize("full", [False, True])
def test_two_phase_lod_and_full_modes(street, full):
    cfg, levels, plan, one = street
    two = L.Renderer(levels, plan, storage="fp32", precision="fast", phase_budget=200)
    bounds = [0.0] + [float(cfg.levels[l][2]) for l in range(1, cfg.L)] + [float("inf")]
    cam = scenes.camera(52.0)
    fr1, st1 = one.render_lod_camera(cam, bounds, full)
    fr2, st2 = two.render_lod_camera(cam, bounds, full)
    assert_same(outputs(fr2, st2), outputs(fr1, st1))


def test_two_phase_frames_in_flight(street):
    """Two slots (own contexts and streams) interleaving two-phase frames."""
    cfg, levels, plan, one = street
    two = L.Renderer(levels, plan, storage="fp32", precision="fast", n_streams=2,
                     phase_budget=500)
    cams_h = [scenes.camera(z) for z in (9.0, 23.0, 61.0, 90.0)]
    refs = [outputs(*one.render_camera(c)) for c in cams_h]
    two.reserve(max(r["P"] for r in refs) + 4096)
    cams = two.upload_cameras(cams_h)
    frames = [two.alloc_frame(1920, 1080) for _ in cams_h]
    for j in range(len(cams_h)):
        two.render(cams[j], frames[j], slot=j % 2)
    torch.cuda.synchronize()
    for j, fr in enumerate(frames):
        assert_same(outputs(fr, fr.read_stats()), refs[j])
    assert two.fault_flags() == 0 and one.fault_flags() == 0
