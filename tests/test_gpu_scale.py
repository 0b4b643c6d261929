"""GPU parity at 1080p on the bench fixtures (fixtures/scenes.py) against the
pinned CPU oracle, through the fused device path (lodge_render_frame).

Bit-exact: chunk pair and t, union sets, per_tile_count, sorted per-tile
lists; FAST image max-abs <= 1e-3 and PSNR >= 60 dB; deterministic reruns.
Size-independent properties at full size: sum(per_tile_count) == P, lists
sorted by (depth, source) within every tile, max weights in [0, 1].
"""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from fixtures import scenes  # noqa: E402
from oracle import oracle as O  # noqa: E402

import paper_2505_23158_b200 as L  # noqa: E402
from paper_2505_23158_b200 import _native as N  # noqa: E402
from paper_2505_23158_b200.device import DeviceLevel, DevicePlan  # noqa: E402


@pytest.fixture(scope="module")
def street():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cfg = scenes.build("street1080")
    dev = torch.device("cuda", 0)
    levels = [DeviceLevel.from_tensors(torch.from_numpy(g).to(dev), torch.from_numpy(s).to(dev),
                                       cfg.degree) for g, s, _ in cfg.levels]
    plan = DevicePlan.from_arrays(cfg.centers, cfg.offsets, cfg.data, cfg.L, dev)
    r = L.Renderer(levels, plan, storage="fp32", precision="fast", full_lists=True)
    return cfg, r


def oracle_frame(cfg, cam):
    f, o, tb, t = O.select(cfg.centers, cam.position)
    sel, mods = [], []
    for l in range(cfg.L):
        b = cfg.set(o, l).astype(np.int64) if o is not None else np.zeros(0, np.int64)
        idx, mod, _ = O.union(cfg.set(f, l).astype(np.int64), b, t)
        sel.append(idx)
        mods.append(mod)
    levels = [scenes.scene_objects(cfg, l) for l in range(cfg.L)]
    out = O.render_selection(levels, sel, mods, O.camera_from(cam),
                             O.cfg_struct(L.RasterConfig()), lists=True)
    return (f, o, t), sel, out


def frame_lists(r, fr, st):
    T = fr.tile_count.numel()
    offs = torch.zeros(T + 1, dtype=torch.int64, device=r.device)
    src = torch.zeros(max(int(st.P), 1), dtype=torch.int64, device=r.device)
    N.check(N.lib().lodge_frame_lists(r.ctx.ptr, T, offs.data_ptr(), src.data_ptr(), int(st.P)))
    torch.cuda.synchronize()
    return offs.cpu().numpy(), src[:int(st.P)].cpu().numpy()


@pytest.mark.parametrize("z", [6.0, 40.0, 71.0, 118.0])
def test_street_1080p_vs_oracle(street, z):
    cfg, r = street
    cam = scenes.camera(z)
    fr, st = r.render_camera(cam)
    (f, o, t), sel, ref = oracle_frame(cfg, cam)
    assert (st.f, st.o if st.o >= 0 else None) == (f, o) and st.t == t
    assert [st.U_level[l] for l in range(cfg.L)] == [len(s) for s in sel]
    assert st.M == len(ref["batch"]["src"]) and st.P == ref["P"]
    assert np.array_equal(fr.tile_count.cpu().numpy(), ref["per_tile_count"])
    offs, src = frame_lists(r, fr, st)
    assert np.array_equal(offs, ref["tile_offsets"])
    assert np.array_equal(src, ref["tile_src"])
    img = fr.image.double().cpu().numpy()
    err = np.abs(img - ref["image"]).max()
    mse = np.mean((img - ref["image"]) ** 2)
    assert err <= 1e-3, err
    assert mse == 0 or -10 * np.log10(mse) >= 60
    dv = np.abs(fr.visible.cpu().numpy() - ref["per_pixel_visible"])
    assert dv.max() <= 1 and np.count_nonzero(dv) <= dv.size // 1000
    mw = fr.maxw[:st.U].double().cpu().numpy()
    assert np.abs(mw - ref["per_gaussian_max_weight"]).max() <= 2e-3


def test_street_properties_and_determinism(street):
    cfg, r = street
    cam = scenes.camera(30.0)
    fr, st = r.render_camera(cam)
    tc = fr.tile_count.cpu().numpy()
    assert tc.sum() == st.P and st.overflow == 0
    offs, src = frame_lists(r, fr, st)
    assert np.array_equal(np.diff(offs), tc.reshape(-1))
    img0, vis0 = fr.image.clone(), fr.visible.clone()
    mw0 = fr.maxw.clone()
    for _ in range(2):
        fr2, st2 = r.render_camera(cam)
        assert torch.equal(fr2.image, img0) and torch.equal(fr2.visible, vis0)
        assert torch.equal(fr2.maxw, mw0)
    mw = mw0[:st.U]
    assert float(mw.min()) >= 0 and float(mw.max()) <= 1


def test_overflow_recovers(street):
    """A pair buffer smaller than P reports overflow; render_camera grows it."""
    cfg, r = street
    cam = scenes.camera(12.0)
    fr, st = r.render_camera(cam)
    assert st.overflow == 0 and st.P > 0


@pytest.mark.parametrize("res", [(3840, 2160), (1277, 719), (17, 1)])
@pytest.mark.parametrize("precision", ["fast", "exact"])
def test_street_other_resolutions_vs_oracle(street, res, precision):
    """4K (8160 -> 32640 tiles: the tile sort's high digit grows to 8 bits),
    an odd size with partial edge tiles, and a one-row strip (single tile
    pass), through the fused path in both precisions."""
    cfg, _ = street
    w, h = res
    r = L.Renderer(street[1].levels, street[1].plan, precision=precision, full_lists=True)
    cam = scenes.camera(47.0, width=w, height=h, focal=scenes.FOCAL * max(w, 64) / 1920)
    fr, st = r.render_camera(cam)
    (f, o, t), sel, ref = oracle_frame(cfg, cam)
    assert st.M == len(ref["batch"]["src"]) and st.P == ref["P"]
    assert np.array_equal(fr.tile_count.cpu().numpy(), ref["per_tile_count"])
    offs, src = frame_lists(r, fr, st)
    assert np.array_equal(offs, ref["tile_offsets"]) and np.array_equal(src, ref["tile_src"])
    img = fr.image.double().cpu().numpy()
    if precision == "exact":
        assert np.abs(img - ref["image"]).max() <= 1e-12
        assert np.array_equal(fr.visible.cpu().numpy(), ref["per_pixel_visible"])
        mw = fr.maxw[:st.U].double().cpu().numpy()
        np.testing.assert_allclose(mw, ref["per_gaussian_max_weight"], rtol=1e-12)
    else:
        assert np.abs(img - ref["image"]).max() <= 1e-3
