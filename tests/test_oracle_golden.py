"""Pin the CPU oracle (oracle/lodge_oracle.c) against vectors produced by the
reference itself (oracle/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import oracle as O

from .golden_util import batch, camera, cfg, config1_levels, config1_sets, load, scene

BATCH_FIELDS = [("src", "src"), ("mean2d", "mean2d"), ("cov2d", "cov2d"), ("conic", "conic"),
                ("extent", "extent"), ("depth", "depth"), ("opacity", "opacity"),
                ("color", "color")]

CASES = load("cases.npz")
CASE_NAMES = [str(n) for n in CASES["names"]]


def check_batch_exact(got, d, p):
    assert got["src"].shape[0] == d[p + "src"].shape[0]
    for gk, rk in BATCH_FIELDS:
        ref = d[p + rk]
        g = got[gk].reshape(ref.shape)
        # bit-exact: the oracle restates NumPy's fp64 operation order
        assert np.array_equal(g, ref), f"{gk}: {np.sum(g != ref)} mismatches"


def check_raster(out, d, p, image_atol=1e-12):
    assert np.array_equal(out["per_tile_count"], d[p + "tile_count"])
    assert np.array_equal(out["per_pixel_visible"], d[p + "visible"])
    assert np.array_equal(out["tile_offsets"], d[p + "tile_offsets"])
    assert np.array_equal(out["tile_src"], d[p + "tile_src"])
    if p + "image" in d:
        np.testing.assert_allclose(out["image"], d[p + "image"], atol=image_atol, rtol=0)
    if p + "maxw" in d:
        # NumPy's SIMD exp and glibc's exp differ by <= 1 ulp on ~5% of inputs;
        # the ulps propagate through the transmittance product
        np.testing.assert_allclose(out["per_gaussian_max_weight"], d[p + "maxw"],
                                   rtol=1e-13, atol=1e-300)


@pytest.mark.parametrize("name", CASE_NAMES)
def test_case_projection_and_raster(name):
    d, p = CASES, name + "/"
    sc, cam, rc = scene(d, p), camera(d, p), cfg(d, p)
    c, r = O.camera_from(cam), O.cfg_struct(rc)
    idx = d[p + "idx"] if p + "idx" in d else None
    mod = d[p + "mod"] if p + "mod" in d else None
    got = O.project(sc, idx, c, r, mod)
    check_batch_exact(got, d, p + "b_")
    out = O.rasterize(batch(d, p + "b_"), cam.resolution[0], cam.resolution[1], r, lists=True)
    check_raster(out, d, p + "o_")


@pytest.fixture(scope="module")
def c1():
    return load("config1.npz")


def test_config1_sizes(c1):
    sets = config1_sets(c1)
    assert [[len(s) for s in ch] for ch in sets] == [[3928, 427], [1046, 868], [744, 194],
                                                      [2208, 384]]
    assert [len(l.means) for l in config1_levels(c1)] == [10000, 4076]


@pytest.mark.parametrize("v", range(8))
def test_config1_view(c1, v):
    d, p = c1, f"v{v}/"
    levels, sets = config1_levels(d), config1_sets(d)
    cam = camera(d, p)
    f, o, tb, t = O.select(d["centers"], cam.position)
    assert (f, o) == tuple(int(x) for x in d[p + "pair"])
    assert tb == d[p + "t"][0] and t == d[p + "t"][1]          # bit-exact fp64
    L = len(levels)
    sel, mods = [], []
    for l in range(L):
        idx, mod, _ = O.union(sets[f][l], sets[o][l], t)
        assert np.array_equal(idx, d[p + f"sel{l}"])
        assert np.array_equal(mod, d[p + f"mod{l}"])
        sel.append(idx)
        mods.append(mod)
    out = O.render_selection(levels, sel, mods, O.camera_from(cam), O.cfg_struct(cfg(d, "")),
                             lists=True)
    check_batch_exact(out["batch"], d, p + "b_")
    check_raster(out, d, p + "o_")
