"""Residency-bounded store: frames rendered from chunk
slabs loaded asynchronously into a few device slots are bit-identical to
frames rendered from the fully resident store (same fp32 records, same
kernels), including across evictions and with frames in flight on several
streams; and slab-mode frames built from the reference's own asset equal the
reference's renders of it (golden vectors)."""

import numpy as np
import pytest

from .golden_util import config1_levels, config1_sets, load
from .test_importance_cpu import golden_cameras

pytestmark = pytest.mark.gpu

C1 = load("config1.npz")


def host_store():
    levels = []
    for sc in config1_levels(C1):
        g = np.concatenate([sc.means, sc.scales, sc.rotations, sc.opacities[:, None],
                            sc.filter_variance[:, None]], axis=1).astype(np.float32)
        levels.append((g, np.asarray(sc.sh_coeffs, np.float32)))
    sets = config1_sets(C1)
    K, L = len(sets), len(levels)
    offsets = np.zeros(K * L + 1, np.int64)
    offsets[1:] = np.cumsum([len(sets[j][l]) for j in range(K) for l in range(L)])
    data = np.concatenate([np.asarray(sets[j][l], np.uint32) for j in range(K)
                           for l in range(L)])
    return levels, C1["centers"], offsets, data


@pytest.fixture(scope="module")
def setup():
    import torch
    import paper_2505_23158_b200 as Lg
    from paper_2505_23158_b200.device import DeviceLevel, DevicePlan
    from paper_2505_23158_b200.streaming import StreamingStore, host_pair
    dev = torch.device("cuda", 0)
    levels, centers, offsets, data = host_store()
    full = [DeviceLevel.from_tensors(torch.from_numpy(g).to(dev), torch.from_numpy(s).to(dev), 1)
            for g, s in levels]
    plan = DevicePlan.from_arrays(centers, offsets, data, len(levels), dev)
    return Lg, torch, dev, levels, centers, offsets, data, full, plan, StreamingStore, host_pair


@pytest.mark.parametrize("n_streams,n_slots", [(1, 2), (2, 3)])
def test_slab_frames_equal_resident_frames(setup, n_streams, n_slots):
    (Lg, torch, dev, levels, centers, offsets, data, full, plan, StreamingStore,
     host_pair) = setup
    from paper_2505_23158_b200.device import DevicePlan
    ref_r = Lg.Renderer(full, plan, dev, storage="fp32", precision="fast")
    store = StreamingStore(levels, centers, offsets, data, dev, n_slots=n_slots)
    splan = store.attach(DevicePlan.from_arrays(centers, offsets, data, len(levels), dev))
    r = Lg.Renderer(store.device_levels(), splan, dev, storage="fp32", precision="fast",
                    n_streams=n_streams)
    cams = golden_cameras(list(range(8)))
    order = [0, 7, 1, 6, 2, 5, 3, 4, 0, 7]  # walks back and forth: evictions
    r.reserve(1 << 20)
    ref_r.reserve(1 << 20)
    rows = r.upload_cameras([cams[v] for v in order])
    frames = [r.alloc_frame(128, 128) for _ in order]
    for i, v in enumerate(order):
        f, o, t = host_pair(centers, cams[v].position)
        slot = i % n_streams
        s = r.stream_of(slot)
        store.require([f, o], s)
        r.render(rows[i], frames[i], pair=(f, o), t=t, slot=slot)
        store.release([f, o], s)
    torch.cuda.synchronize()
    assert store.loads >= 4
    for i, v in enumerate(order):
        ref, st_ref = ref_r.render_camera(cams[v])  # device-side pair selection
        st = frames[i].read_stats()
        assert (st.f, st.o) == (st_ref.f, st_ref.o) and st.t == st_ref.t
        assert torch.equal(frames[i].image, ref.image)
        assert torch.equal(frames[i].tile_count, ref.tile_count)
        assert torch.equal(frames[i].visible, ref.visible)
        assert torch.equal(frames[i].maxw[:st.U], ref.maxw[:st.U])
    assert store.resident_bytes() < sum(g.nbytes + s.nbytes for g, s in levels) * 2


def test_host_pair_matches_device_selection(setup):
    (Lg, torch, dev, levels, centers, offsets, data, full, plan, StreamingStore,
     host_pair) = setup
    for v in range(8):
        cam = golden_cameras([v])[0]
        f, o, t = host_pair(centers, cam.position)
        ff, oo = Lg.nearest_two_chunks(Lg.ChunkPlan(centers, C1["radii"],
                                                    tuple(tuple(s) for s in config1_sets(C1)),
                                                    np.zeros(0, np.int64)), cam.position)
        assert (f, o) == (ff, oo)
        assert t == float(C1[f"v{v}/t"][1])


def test_slab_frames_match_reference_asset():
    """Slab mode against the reference itself: the chunk slabs are built from
    the asset the reference wrote (tests/golden/asset_c1, fp32 records with
    raw rotations, LODGE_GEOM_QNORM), rendered in EXACT precision with the
    chunk pair decided on the host, and compared with the reference rendering
    its own read_asset result (tests/golden/asset.npz; reference
    src/blending.py:132-137, src/raster.py:380-449)."""
    import torch
    import paper_2505_23158_b200 as Lg
    from paper_2505_23158_b200 import _native as N
    from paper_2505_23158_b200 import asset as A
    from paper_2505_23158_b200.device import DevicePlan
    from paper_2505_23158_b200.streaming import StreamingStore, host_pair
    from .golden_util import GOLDEN
    import os
    gold = load("asset.npz")
    ast = A.load_asset(os.path.join(GOLDEN, "asset_c1"))
    dev = torch.device("cuda", 0)
    levels = [(lv.geom.cpu().numpy(), lv.sh.cpu().numpy()) for lv in ast.levels]
    centers = ast.plan.centers.cpu().numpy()
    offsets = ast.plan.offsets.cpu().numpy()
    data = ast.plan.data.cpu().numpy().view(np.uint32)
    store = StreamingStore(levels, centers, offsets, data, dev, n_slots=2,
                           level_flags=N.GEOM_QNORM)
    plan = store.attach(DevicePlan.from_arrays(centers, offsets, data, len(levels), dev))
    r = Lg.Renderer(store.device_levels(), plan, dev, precision="exact")
    r.reserve(1 << 20)
    for v in (1, 6):
        cam = golden_cameras([v])[0]
        f, o, t = host_pair(centers, cam.position)
        p = f"v{v}/"
        assert (f, o) == tuple(int(x) for x in gold[p + "pair"])
        assert t == float(gold[p + "t"][1])
        row = r.upload_cameras([cam])
        fr = r.alloc_frame(128, 128)
        s = r.stream_of(0)
        store.require([f, o], s)
        r.render(row[0], fr, pair=(f, o), t=t)
        store.release([f, o], s)
        torch.cuda.synchronize()
        st = fr.read_stats()
        assert st.fault == 0 and st.overflow == 0
        assert np.array_equal(fr.tile_count.cpu().numpy(), gold[p + "tile_count"])
        assert np.array_equal(fr.visible.cpu().numpy(), gold[p + "visible"])
        np.testing.assert_allclose(fr.image.cpu().numpy(), gold[p + "image"], rtol=0,
                                   atol=1e-12)
        U = int(st.U)
        assert U == gold[p + "maxw"].shape[0]
        np.testing.assert_allclose(fr.maxw[:U].cpu().numpy(), gold[p + "maxw"], rtol=1e-12,
                                   atol=0)
