"""LOD-mode and full-mode frames on the device:
render_lod / render_full (band predicate and selection inside the fused
frame) against the reference's render_lod and full-mode renders
(tests/golden/modes.npz)."""

import numpy as np
import pytest

from .golden_util import load
from .test_importance_cpu import golden_cameras
from .test_modes_cpu import c1_levels

pytestmark = pytest.mark.gpu

MD = load("modes.npz")


@pytest.fixture(scope="module")
def lodge():
    import paper_2505_23158_b200 as L
    from paper_2505_23158_b200 import lod
    return L, lod


def check(res, p, exact):
    assert np.array_equal(res.per_tile_count, MD[p + "tile_count"])
    if exact:
        assert np.array_equal(res.per_pixel_visible, MD[p + "visible"])
        np.testing.assert_allclose(res.image, MD[p + "image"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(res.per_gaussian_max_weight, MD[p + "maxw"], rtol=1e-12)
    else:
        vis = res.per_pixel_visible != MD[p + "visible"]
        assert vis.mean() <= 1e-3
        assert np.abs(res.image - MD[p + "image"]).max() <= 1e-3
        np.testing.assert_allclose(res.per_gaussian_max_weight, MD[p + "maxw"], rtol=1e-4,
                                   atol=1e-7)


@pytest.mark.parametrize("precision", ["exact", "fast"])
@pytest.mark.parametrize("v", [1, 5])
@pytest.mark.parametrize("tag,offs", [("lod", None), ("lodoff", [0.0, 1.5])])
def test_render_lod(lodge, precision, v, tag, offs):
    L, lod = lodge
    L.set_default_precision(precision)
    try:
        res = lod.render_lod(c1_levels(), golden_cameras([v])[0], L.RasterConfig(),
                             depth_offsets=offs)
    finally:
        L.set_default_precision("exact")
    check(res, f"v{v}/{tag}/", precision == "exact")


@pytest.mark.parametrize("precision", ["exact", "fast"])
@pytest.mark.parametrize("v", [1, 5])
def test_render_full(lodge, precision, v):
    L, lod = lodge
    L.set_default_precision(precision)
    try:
        res = lod.render_full(c1_levels(), golden_cameras([v])[0], L.RasterConfig())
    finally:
        L.set_default_precision("exact")
    check(res, f"v{v}/full/", precision == "exact")


def test_lod_sets_on_device(lodge):
    """The device band selection yields select_active's sets (per-level
    counts via the frame stats, members via lodge_frame_union)."""
    L, lod = lodge
    from paper_2505_23158_b200 import _native as N
    lv = c1_levels()
    r = lod._lod_renderer(lv, L.RasterConfig())
    cam = golden_cameras([1])[0]
    fr, st = r.render_lod_camera(cam, lod.lod_bounds(lv), False, False, False)
    import ctypes as C
    import torch
    for l in range(2):
        ref = MD[f"v1/lod/set{l}"]
        assert st.U_level[l] == ref.shape[0]
        idx = torch.empty(max(ref.shape[0], 1), dtype=torch.int32, device=r.device)
        tag = torch.empty(max(ref.shape[0], 1), dtype=torch.uint8, device=r.device)
        N.check(N.lib().lodge_frame_union(r.ctx.ptr, l, C.c_void_p(idx.data_ptr()),
                                          C.c_void_p(tag.data_ptr()), ref.shape[0]),
                "lodge_frame_union")
        got = idx[:ref.shape[0]].cpu().numpy().view(np.uint32)
        assert np.array_equal(got, ref)
        assert np.all(tag[:ref.shape[0]].cpu().numpy() == 3)
