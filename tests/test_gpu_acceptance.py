"""The reference's release criteria that sit on the render path
(tests/test_acceptance.py:207-345 of the reference package), on config 1
(the reference-built 10k-Gaussian street: 2 levels, 4 chunks, 8 views) and
through the device path: active-set soundness, blending continuity (the
fused frame along a trajectory through the middle chunk pair), swap
consistency, and the residency bound of the streaming state machine."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2505_23158_b200 as L  # noqa: E402

from .golden_util import camera, config1_levels, config1_sets, load  # noqa: E402

C1 = load("config1.npz")


@pytest.fixture(scope="module")
def pipe():
    levels = [L.LodLevel(l, float(C1[f"L{l}/depth_threshold"]),
                         L.Scene(s.means, s.scales, s.rotations, s.opacities, s.sh_coeffs,
                                 s.filter_variance, s.sh_degree),
                         np.arange(len(s.means)))
              for l, s in enumerate(config1_levels(C1))]
    plan = L.ChunkPlan(C1["centers"], C1["radii"],
                       tuple(tuple(ch) for ch in config1_sets(C1)), np.zeros(0, np.int64))
    return levels, plan, [camera(C1, f"v{v}/") for v in range(8)]


def cam_at(template, pos):
    return L.Camera(np.asarray(pos, float), template.orientation, template.focal,
                    template.principal_point, template.resolution, template.near_plane)


def test_active_set_soundness(pipe):
    levels, plan, _ = pipe
    pre = L.build_chunk_active_sets(levels, plan.centers, plan.radii)
    bounds_of = [L.lod_bounds(levels, [0.0] + [float(r)] * (len(levels) - 1))
                 for r in plan.radii]
    for j in range(plan.n_chunks):
        for l, lv in enumerate(levels):
            d = np.linalg.norm(lv.scene.means - plan.centers[j], axis=1)
            b = bounds_of[j]
            want = np.flatnonzero((d >= b[l]) & (d < b[l + 1]))
            assert np.array_equal(pre.active_sets[j][l], want)       # exact predicate
            assert np.isin(plan.active_sets[j][l], want).all()       # shipped ⊆ band


def _window(plan, half_width=1.0, steps=201):
    order = np.argsort(plan.centers[:, 2])
    a, b = int(order[len(order) // 2]), int(order[len(order) // 2 + 1])
    ca, cb = plan.centers[a], plan.centers[b]
    mid = 0.5 * (ca + cb)
    axis = (cb - ca) / np.linalg.norm(cb - ca)
    lo, hi = mid - half_width * axis, mid + half_width * axis
    return ca, cb, [lo + s * (hi - lo) for s in np.linspace(0, 1, steps)]


@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_blending_continuity(pipe, precision):
    levels, plan, cams = pipe
    ca, cb, positions = _window(plan)
    r = L.Renderer(levels, plan, storage="fp64", precision=precision)
    imgs, nearest = [], []
    for pos in positions:
        fr, st = r.render_camera(cam_at(cams[0], pos))
        imgs.append(fr.image.double().cpu().numpy())
        nearest.append(int(st.f))
    blend_max = max(float(np.abs(imgs[i + 1] - imgs[i]).max()) for i in range(len(imgs) - 1))
    swap = next(i for i in range(len(nearest) - 1) if nearest[i + 1] != nearest[i])
    hard = []
    for i in (swap, swap + 1):
        sel = L.compose_active(plan, levels, nearest[i], None, 1.0)
        hard.append(L.render_selection(levels, sel, cam_at(cams[0], positions[i])).image)
    hard_delta = float(np.abs(hard[1] - hard[0]).max())
    assert blend_max <= 0.1 * hard_delta, (blend_max, hard_delta)
    assert abs(L.blend_factor(ca, ca, cb)[0] - 1.0) <= 1e-12
    assert abs(L.blend_factor(0.5 * (ca + cb), ca, cb)[0] - 0.5) <= 1e-12


def test_swap_consistency(pipe):
    levels, plan, cams = pipe
    order = np.argsort(plan.centers[:, 2])
    a, b, c = (int(order[len(order) // 2 - 1]), int(order[len(order) // 2]),
               int(order[len(order) // 2 + 1]))
    swap_pos = plan.centers[b].copy()
    cam = cam_at(cams[0], swap_pos)
    t_old = L.blend_factor(swap_pos, plan.centers[b], plan.centers[a])[1]
    t_new = L.blend_factor(swap_pos, plan.centers[b], plan.centers[c])[1]
    img_old = L.render_selection(levels, L.compose_active(plan, levels, b, a, t_old), cam).image
    img_new = L.render_selection(levels, L.compose_active(plan, levels, b, c, t_new), cam).image
    assert float(np.abs(img_old - img_new).max()) <= 1e-6


def test_residency_bound(pipe):
    levels, plan, _ = pipe
    order = np.argsort(plan.centers[:, 2])
    bound = max(plan.resident_count([int(x), int(y)]) for x, y in zip(order, order[1:]))
    full = len(levels[0].scene.means)
    state, worst = None, 0
    z0, z1 = plan.centers[:, 2].min(), plan.centers[:, 2].max()
    for z in np.linspace(z0, z1, 240):
        state, _ = L.stream_step(state, plan, np.array([0.0, 0.5, z]))
        worst = max(worst, plan.resident_count(list(state.loaded_chunks)))
    assert worst <= bound and worst < full
