"""GPU: the device frame report (csrc/k_report.cu, lodge_frame_report /
lodge_sq_err) -- visibility histogram, per-tile sum, visible-Gaussian count,
PSNR -- bit-exact against the reference's own values on the reference's
config-1 frames (tests/golden/report.npz), and Renderer.report on a fused
frame against the host computation of the same fields."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from .golden_util import load  # noqa: E402

G = load("report.npz")
C1 = load("config1.npz")
EDGES = sorted(k.split("/", 1)[1] for k in G.files if k.startswith("edges/"))


@pytest.fixture(autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.mark.parametrize("name", EDGES)
@pytest.mark.parametrize("v", range(8))
@pytest.mark.parametrize("fp64", [False, True])
def test_device_report_matches_reference(v, name, fp64):
    from paper_2505_23158_b200.raster import frame_report_device
    p = f"v{v}/"
    dev = torch.device("cuda", 0)
    vis = torch.from_numpy(C1[p + "o_visible"].astype(np.int32)).to(dev)
    tc = torch.from_numpy(C1[p + "o_tile_count"].astype(np.int32)).to(dev)
    mw = torch.from_numpy(C1[p + "o_maxw"]).to(dev)
    mw = mw if fp64 else mw.float()
    hist, tsum, nvis = frame_report_device(vis, tc, mw, mw.numel(), G["edges/" + name])
    assert np.array_equal(hist, G[p + "hist/" + name])
    assert tsum / tc.numel() == float(G[p + "mean_per_tile"])
    if fp64:  # fp32 max weights may round a tiny weight to zero
        assert nvis == int(G[p + "visible_gaussians"])


def test_device_report_edge_errors():
    from paper_2505_23158_b200.raster import frame_report_device
    dev = torch.device("cuda", 0)
    z = torch.zeros(16, dtype=torch.int32, device=dev)
    for i, bad in enumerate(([1.0], [3.0, 2.0], [0.0, 1.0, 1.0])):
        with pytest.raises(ValueError) as e:
            frame_report_device(z, z, None, 0, np.asarray(bad))
        assert str(e.value) == str(G["bad_edges_messages"][i])
    with pytest.raises(ValueError):
        frame_report_device(z, z, None, 0, np.arange(300.0))


def test_renderer_report_and_psnr():
    """Renderer.report on a fused config-1 frame: every field equals the host
    computation over the frame's own outputs; psnr_vs_full against a
    full-mode frame of the same view equals the host PSNR."""
    import paper_2505_23158_b200 as L
    from paper_2505_23158_b200.raster import visibility_histogram
    from types import SimpleNamespace
    from .golden_util import camera, config1_levels, config1_sets
    lv = config1_levels(C1)
    levels = [L.LodLevel(l, 0.0 if l == 0 else float(C1[f"L{l}/depth_threshold"]),
                         L.Scene(s.means, s.scales, s.rotations, s.opacities, s.sh_coeffs,
                                 s.filter_variance, s.sh_degree), np.arange(len(s.means)))
              for l, s in enumerate(lv)]
    sets = config1_sets(C1)
    plan = L.ChunkPlan(C1["centers"], C1["radii"], tuple(tuple(ch) for ch in sets))
    r = L.Renderer(levels, plan, storage="fp32", precision="fast")
    cam = camera(C1, "v2/")
    fr, st = r.render_camera(cam)
    full, _ = r.render_lod_camera(cam, full=True)
    rep = r.report(fr, st, full_frame=full)
    vis = fr.visible.cpu().numpy()
    host = visibility_histogram(SimpleNamespace(per_pixel_visible=vis),
                                np.asarray([0, 1, 2, 4, 8, 16, 32, 64, 128, 256]))
    assert rep["visibility_histogram"] == host.tolist()
    assert rep["mean_per_tile"] == float(fr.tile_count.double().mean())
    assert rep["visible_gaussians"] == int((fr.maxw[:st.U] != 0).sum())
    assert rep["resident_gaussians"] == plan.resident_count([st.f, st.o])
    assert rep["chunk_pair"] == [st.f, st.o]
    a = fr.image.double().cpu().numpy()
    b = full.image.double().cpu().numpy()
    mse = float(np.mean((a - b) ** 2))
    assert rep["psnr_vs_full"] == pytest.approx(-10 * np.log10(mse), rel=1e-9)
