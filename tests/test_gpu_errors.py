"""Error behaviour that needs the device: the drop-in messages the
reference raises after computing (src/blending.py:97, src/raster.py:206) and
the C ABI's argument checks surfacing as ValueError with the library's
message (BAD_ARG) through the Python binding."""

import numpy as np
import pytest

from .golden_util import config1_levels, config1_sets, load
from .test_importance_cpu import golden_cameras

pytestmark = pytest.mark.gpu

C1 = load("config1.npz")


@pytest.fixture(scope="module")
def L():
    import paper_2505_23158_b200 as lodge
    return lodge


def test_blend_factor_same_centres(L):
    c = np.array([1.0, 2.0, 3.0])
    with pytest.raises(ValueError, match="blend_factor needs distinct chunk centers"):
        L.blend_factor(np.zeros(3), c, c)


def test_project_scene_modulation_length(L):
    sc = config1_levels(C1)[1]
    cam = golden_cameras([0])[0]
    with pytest.raises(ValueError, match="modulation length must match the input list"):
        L.project_scene(sc, cam, L.RasterConfig(), indices=np.arange(5),
                        modulation=np.ones(4))


def test_render_frame_pair_errors(L):
    from paper_2505_23158_b200.device import DevicePlan
    levels = config1_levels(C1)
    plan = L.ChunkPlan(C1["centers"], C1["radii"], tuple(tuple(s) for s in config1_sets(C1)),
                       np.zeros(0, np.int64))
    r = L.Renderer(levels, plan)
    cam = golden_cameras([0])[0]
    fr = r.alloc_frame(128, 128)
    row = r.upload_cameras([cam])[0]
    with pytest.raises(ValueError, match="chunk 9 is not in the plan"):
        r.render(row, fr, pair=(9, None))
    with pytest.raises(ValueError, match="chunk 9 is not in the plan"):
        r.render(row, fr, pair=(0, 9))
    with pytest.raises(ValueError, match="blending needs two distinct chunks"):
        r.render(row, fr, pair=(2, 2))
    with pytest.raises(ValueError, match="one distance bound per level"):
        r.render_lod(row, fr, bounds=[0.0, 1.0])
    # the context stays usable after rejected calls
    fr, st = r.render_camera(cam)
    assert st.U > 0 and not st.overflow


def test_c_abi_argument_checks(L):
    import ctypes as C
    from paper_2505_23158_b200 import _native as N
    from paper_2505_23158_b200.device import context
    ctx = context()
    lib = N.lib()
    lvl = N.Level()
    cam = N.Camera()  # zero resolution and focal
    rp = N.RasterParams()
    m = C.c_int64()
    with pytest.raises(ValueError, match="resolution must be positive"):
        N.check(lib.lodge_cover_table(ctx.bind(), C.byref(lvl), None, 0, C.byref(cam),
                                      C.byref(rp), None, None, C.byref(m)), "lodge_cover_table")
    bad = C.c_int32()
    with pytest.raises(ValueError, match="sh degree must be in 0..3"):
        N.check(lib.lodge_asset_split(ctx.bind(), None, 0, 7, None, None, C.byref(bad)),
                "lodge_asset_split")
    assert "sh degree" in lib.lodge_last_error().decode()
    with pytest.raises(ValueError, match="CTAs per SM must be >= 0"):
        N.check(lib.lodge_set_grid_share(ctx.bind(), -1), "lodge_set_grid_share")
    N.check(lib.lodge_set_grid_share(ctx.bind(), 0), "lodge_set_grid_share")
