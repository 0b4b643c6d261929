"""Asset loader -> device store on the GPU: the split
store against the blob's fp32 values, every device-side check against the
reference's read_asset messages, and whole frames rendered from the loaded
store against the reference's render of its own read_asset result
(tests/golden/asset.npz, oracle/make_golden.py make_asset)."""

import json
import os

import numpy as np
import pytest

from .asset_util import clean, corrupt
from .golden_util import GOLDEN, load
from .test_importance_cpu import golden_cameras

pytestmark = pytest.mark.gpu

GOLD = load("asset.npz")
MSGS = json.loads(str(GOLD["messages"]))
SRC = os.path.join(GOLDEN, "asset_c1")

DEVICE_CASES = [
    ("nan_mean", "f32", ("L0", 5, 0, "nan")),
    ("neg_scale", "f32", ("L0", 7, 4, -0.5)),
    ("opacity_gt1", "f32", ("L1", 3, 10, 1.5)),
    ("neg_fv", "f32", ("L1", 0, 11, -1.0)),
    ("bad_rot", "f32", ("L0", 11, 6, 3.0)),
    ("nan_sh", "f32", ("L1", 9, 13, "inf")),
    ("unsorted_set", "u32swap", (1, 0, 2)),
    ("set_oob", "u32set", (2, 1, -1, 4076)),
    ("count_mismatch", "level_field", (1, "gaussian_count", 4075)),
    ("prov_mismatch", "level_field", (0, "provenance_length", 4)),
    ("set_count", "set_field", (3, 1, "count", 1)),
    ("missing_sets", "drop_set", (2,)),
]


@pytest.fixture(scope="module")
def lodge():
    import paper_2505_23158_b200 as L
    from paper_2505_23158_b200 import asset
    return L, asset


@pytest.mark.parametrize("name,kind,args", DEVICE_CASES, ids=[c[0] for c in DEVICE_CASES])
def test_device_checks_match_reference(lodge, tmp_path, name, kind, args):
    _, A = lodge
    dst = str(tmp_path / "a")
    path = corrupt(SRC, dst, kind, args)
    with pytest.raises(A.AssetError) as ei:
        A.load_asset(path)
    assert str(ei.value).replace(str(path), "<path>") == MSGS[name]
    clean(dst)


def test_store_matches_blob(lodge):
    _, A = lodge
    asset = A.load_asset(SRC)
    m = json.load(open(os.path.join(SRC, "manifest.json")))
    data = open(os.path.join(SRC, "data.bin"), "rb").read()
    deg = m["sh_degree"]
    T = (deg + 1) ** 2
    assert asset.n_levels == len(m["levels"])
    for l, row in enumerate(m["levels"]):
        n = row["gaussian_count"]
        rec = np.frombuffer(data[row["offset"]:row["offset"] + row["length"]], "<f4")
        rec = rec.reshape(n, 12 + 3 * T)
        lv = asset.levels[l]
        assert lv.flags & 4  # LODGE_GEOM_QNORM
        assert np.array_equal(lv.geom.cpu().numpy(), rec[:, :12])
        assert np.array_equal(lv.sh.cpu().numpy().reshape(n, -1), rec[:, 12:])
        assert np.array_equal(asset.provenance[l], GOLD[f"L{l}/provenance"])
    assert asset.plan.K == len(m["chunks"]) and asset.plan.L == len(m["levels"])
    for j, ch in enumerate(m["chunks"]):
        for l, s in enumerate(ch["index_sets"]):
            ref = np.frombuffer(data[s["offset"]:s["offset"] + s["length"]], "<u4")
            b, e = (int(x) for x in asset.plan.offsets.cpu().numpy()[j * asset.plan.L + l:
                                                                   j * asset.plan.L + l + 2])
            got = asset.plan.data.cpu().numpy().view(np.uint32)[b:e]
            assert np.array_equal(got, ref)


def test_container_loads_same_store(lodge, tmp_path):
    _, A = lodge
    dst = str(tmp_path / "c")
    path = corrupt(SRC, dst, "container", ())
    a = A.load_asset(path)
    b = A.load_asset(SRC)
    for la, lb in zip(a.levels, b.levels):
        assert np.array_equal(la.geom.cpu().numpy(), lb.geom.cpu().numpy())
    clean(dst)


@pytest.mark.parametrize("v", [1, 6])
def test_frames_from_loaded_store_match_reference(lodge, v):
    """Device selection + union + projection (rotations normalised in fp64 at
    read time) + rasterisation from the loaded store, EXACT precision, vs the
    reference rendering its read_asset result."""
    L, A = lodge
    asset = A.load_asset(SRC)
    r = L.Renderer(asset.levels, asset.plan, precision="exact")
    cam = golden_cameras([v])[0]
    fr, st = r.render_camera(cam)
    p = f"v{v}/"
    assert (st.f, st.o) == tuple(int(x) for x in GOLD[p + "pair"])
    assert st.t == float(GOLD[p + "t"][1])
    assert np.array_equal(fr.tile_count.cpu().numpy(), GOLD[p + "tile_count"])
    assert np.array_equal(fr.visible.cpu().numpy(), GOLD[p + "visible"])
    np.testing.assert_allclose(fr.image.cpu().numpy(), GOLD[p + "image"], rtol=0, atol=1e-12)
    U = int(st.U)
    ref_w = GOLD[p + "maxw"]
    assert U == ref_w.shape[0]
    np.testing.assert_allclose(fr.maxw[:U].cpu().numpy(), ref_w, rtol=1e-12, atol=0)
