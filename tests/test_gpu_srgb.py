"""GPU: lodge_to_srgb8 (csrc/lodge_api.cu, binary search over the level
thresholds) equals the reference's to_uint8 (src/images.py:10-17) on every
fp32 value within 64 ulps of each level threshold, on random values in
[-0.1, 1.1], on special values, and on odd lengths and unaligned buffers
(the kernel's vector path and its tail)."""

import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2505_23158_b200 import _native as N  # noqa: E402
from paper_2505_23158_b200.device import context  # noqa: E402

from .test_srgb_cpu import thresholds, to_uint8  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    return context(torch.device("cuda", 0))


def srgb8(ctx, x, offset=0):
    dev = torch.device("cuda", 0)
    n3 = x.size
    buf = torch.zeros(n3 + offset + 4, dtype=torch.float32, device=dev)
    buf[offset:offset + n3] = torch.from_numpy(x)
    out = torch.zeros(n3 + offset + 4, dtype=torch.uint8, device=dev)
    src = buf[offset:]
    dst = out[offset:]
    N.check(N.lib().lodge_to_srgb8(ctx.bind("fast"), C.c_void_p(src.data_ptr()), n3 // 3,
                                   C.c_void_p(dst.data_ptr())), "lodge_to_srgb8")
    torch.cuda.synchronize()
    return out[offset:offset + n3].cpu().numpy()


def test_srgb8_matches_reference(ctx):
    t = thresholds()
    bits = t[1:].view(np.uint32).astype(np.int64)
    near = (bits[:, None] + np.arange(-64, 65)[None, :]).ravel()
    near = near[(near >= 0) & (near <= 0x3F800000)].astype(np.uint32).view(np.float32)
    rng = np.random.default_rng(11)
    rand = rng.uniform(-0.1, 1.1, 3 * 700_001).astype(np.float32)
    special = np.array([0.0, -0.0, 1.0, -1.0, 2.0, np.inf, -np.inf, 1e-45, 0.0031308,
                        0.5, 0.25, 0.75], np.float32)
    for x in (near, rand, special):
        x = x[: 3 * (x.size // 3)]
        assert np.array_equal(srgb8(ctx, x), to_uint8(x))


@pytest.mark.parametrize("offset", [0, 1, 2, 3])
@pytest.mark.parametrize("n", [1, 2, 5, 1277 * 719])
def test_srgb8_tails_and_alignment(ctx, n, offset):
    rng = np.random.default_rng(n + offset)
    x = rng.uniform(-0.05, 1.05, 3 * n).astype(np.float32)
    assert np.array_equal(srgb8(ctx, x, offset), to_uint8(x))


@pytest.mark.parametrize("budget", [0, 300, 2048])
@pytest.mark.parametrize("res", [(1920, 1080), (1277, 719)])
def test_render_srgb8_out_equals_to_srgb8(budget, res):
    """Renderer.render(srgb8_out=...) -- the compositor's own 8-bit output,
    one pass and two phases -- equals to_srgb8 of the float image."""
    from fixtures import scenes
    import paper_2505_23158_b200 as L
    from paper_2505_23158_b200.device import DeviceLevel, DevicePlan
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    cfg = scenes.build("street1080")
    dev = torch.device("cuda", 0)
    levels = [DeviceLevel.from_tensors(torch.from_numpy(g).to(dev), torch.from_numpy(s).to(dev),
                                       cfg.degree) for g, s, _ in cfg.levels]
    plan = DevicePlan.from_arrays(cfg.centers, cfg.offsets, cfg.data, cfg.L, dev)
    r = L.Renderer(levels, plan, storage="fp32", precision="fast", phase_budget=budget)
    w, h = res
    for z in (8.0, 60.0):
        cam = scenes.camera(z, width=w, height=h, focal=scenes.FOCAL * w / 1920)
        cams = r.upload_cameras([cam])
        fr = r.alloc_frame(w, h)
        r.reserve(64 << 20)
        r.render(cams[0], fr)
        ref = torch.empty((h, w, 3), dtype=torch.uint8, device=dev)
        r.to_srgb8(fr, ref)
        got = torch.zeros((h, w, 3), dtype=torch.uint8, device=dev)
        fr2 = r.alloc_frame(w, h)
        r.render(cams[0], fr2, srgb8_out=got, float_image=False)
        torch.cuda.synchronize()
        assert torch.equal(got, ref)
        assert fr2.read_stats().fault == 0
        # zero-copy into pinned host memory (16-byte row segments at width
        # 1920, bytes at 1277), and a device buffer off 16-byte alignment
        host = torch.zeros((h, w, 3), dtype=torch.uint8).pin_memory()
        r.render(cams[0], fr2, srgb8_out=host, float_image=False)
        torch.cuda.synchronize()
        assert torch.equal(host, ref.cpu())
        raw = torch.zeros(h * w * 3 + 1, dtype=torch.uint8, device=dev)
        odd = raw[1:].view(h, w, 3)
        r.render(cams[0], fr2, srgb8_out=odd, float_image=False)
        torch.cuda.synchronize()
        assert torch.equal(odd, ref)
        with pytest.raises(ValueError, match="pinned host memory"):
            r.render(cams[0], fr2, srgb8_out=torch.zeros((h, w, 3), dtype=torch.uint8))
