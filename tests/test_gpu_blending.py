"""Blend renders on the reference's street_runtime fixture (tests/
test_blending.py:94-235 of the reference package): render_blend_state along
the recorded walk against the reference's own frames, the same frames
through the fused device path (lodge_render_frame with the state's pair and
t), and the TestComposeActive / TestSwapConsistency properties.  Bars as in
test_gpu_parity: EXACT image <= 1e-12 with exact visibility, FAST max-abs
<= 1e-3 and PSNR >= 60 dB."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_23158_b200 as L  # noqa: E402
from paper_2505_23158_b200 import device as D  # noqa: E402

from .golden_util import camera, config1_levels, load  # noqa: E402
from .test_gpu_stream_step import street_plan  # noqa: E402

S = load("street.npz")
WALK_RENDERS = sorted(int(k.split("/")[1][1:]) for k in S.files
                      if k.startswith("walk/r") and k.endswith("/image"))


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    yield
    D.set_default_precision("exact")


@pytest.fixture(scope="module")
def street():
    levels = [L.LodLevel(l, float(S[f"L{l}/depth_threshold"]),
                         L.Scene(s.means, s.scales, s.rotations, s.opacities, s.sh_coeffs,
                                 s.filter_variance, s.sh_degree),
                         np.arange(len(s.means)))
              for l, s in enumerate(config1_levels(S))]
    return levels, street_plan(), [camera(S, f"v{v}/") for v in range(8)]


def psnr(a, b):
    mse = float(np.mean((a - b) ** 2))
    return float("inf") if mse == 0 else -10.0 * np.log10(mse)


def view_at(cam, pos):
    return L.Camera(np.asarray(pos, float), cam.orientation, cam.focal, cam.principal_point,
                    cam.resolution, cam.near_plane)


def states_along_walk(plan):
    state, out = None, {}
    for i, z in enumerate(S["walk/zs"]):
        state, _ = L.stream_step(state, plan, np.array([0.0, 0.5, z]))
        if i in WALK_RENDERS:
            out[i] = (state, np.array([0.0, 0.5, z]))
    return out


def check(img, vis, mw, p, prec):
    ref = S[p + "image"]
    if prec == "exact":
        np.testing.assert_allclose(img, ref, atol=1e-12, rtol=0)
        assert np.array_equal(vis, S[p + "visible"])
        if mw is not None:
            np.testing.assert_allclose(mw, S[p + "maxw"], rtol=1e-12, atol=1e-300)
    else:
        assert np.abs(img - ref).max() <= 1e-3
        assert psnr(img, ref) >= 60.0


@pytest.mark.parametrize("prec", ["exact", "fast"])
def test_render_blend_state_along_walk(street, prec):
    D.set_default_precision(prec)
    levels, plan, cams = street
    for i, (state, pos) in states_along_walk(plan).items():
        out = L.render_blend_state(state, plan, levels, view_at(cams[0], pos))
        p = f"walk/r{i}/"
        assert np.array_equal(out.per_tile_count, S[p + "tile_count"])
        check(out.image, out.per_pixel_visible, out.per_gaussian_max_weight, p, prec)


@pytest.mark.parametrize("prec", ["exact", "fast"])
def test_fused_frame_with_state_pair(street, prec):
    """The state's pair and t passed to lodge_render_frame (select, union,
    projection, sort, composite fused on the device) give the same frames."""
    levels, plan, cams = street
    r = L.Renderer(levels, plan, storage="fp64", precision=prec)
    for i, (state, pos) in states_along_walk(plan).items():
        view = view_at(cams[0], pos)
        row = r.upload_cameras([view])[0]
        fr = r.alloc_frame(*view.resolution)
        r.render(row, fr, pair=(state.primary_id, state.secondary_id), t=state.t)
        p = f"walk/r{i}/"
        assert np.array_equal(fr.tile_count.cpu().numpy(), S[p + "tile_count"])
        img = fr.image.double().cpu().numpy()
        check(img, fr.visible.cpu().numpy(), None, p, prec)


def test_identical_sets_full_opacity_and_t_independent(street):
    levels, plan, cams = street
    same = L.ChunkPlan(plan.centers[:2], plan.radii[:2],
                       (plan.active_sets[0], plan.active_sets[0]), np.zeros(0, np.int64))
    imgs = []
    for t in (0.2, 0.9):
        sel = L.compose_active(same, levels, 0, 1, t)
        for mod in sel.modulations:
            assert np.all(mod == 1.0)
        imgs.append(L.render_selection(levels, sel, cams[2]).image)
    np.testing.assert_array_equal(imgs[0], imgs[1])


def test_t_one_matches_primary_alone_and_reference(street):
    levels, plan, cams = street
    blended = L.render_selection(levels, L.compose_active(plan, levels, 0, 1, 1.0),
                                 cams[2]).image
    single = L.render_selection(levels, L.compose_active(plan, levels, 0, None, 1.0),
                                cams[2]).image
    np.testing.assert_allclose(blended, single, atol=1e-12)
    np.testing.assert_allclose(blended, S["t_one/image"], atol=1e-12)


def test_half_t_disjoint_singletons():
    rng = np.random.default_rng(0)
    sc = L.Scene(rng.uniform(-1, 1, (2, 3)) + [0, 0, 5], np.full((2, 3), 0.3),
                 np.tile([1.0, 0, 0, 0], (2, 1)), np.full(2, 0.5), np.zeros((2, 3, 1)),
                 np.zeros(2), 0)
    levels = [L.LodLevel.base(sc)]
    plan = L.ChunkPlan(np.array([[0, 0, 0], [1, 0, 0]], float), np.array([1.0, 1.0]),
                       ((np.array([0]),), (np.array([1]),)), np.zeros(0, np.int64))
    sel = L.compose_active(plan, levels, 0, 1, 0.5)
    np.testing.assert_array_equal(sel.sets[0], [0, 1])
    np.testing.assert_allclose(sel.modulations[0], [0.5, 0.5])


def test_swap_instant_renders_match(street):
    levels, plan, cams = street
    swap_pos = plan.centers[1]
    view = view_at(cams[0], swap_pos)
    imgs = {}
    for tag, o in (("swap_old", 0), ("swap_new", 2)):
        t = L.blend_factor(swap_pos, plan.centers[1], plan.centers[o])[1]
        assert t == float(S[tag + "/t"])
        imgs[tag] = L.render_selection(levels, L.compose_active(plan, levels, 1, o, t),
                                       view).image
        np.testing.assert_allclose(imgs[tag], S[tag + "/image"], atol=1e-12)
    np.testing.assert_allclose(imgs["swap_old"], imgs["swap_new"], atol=1e-6)
