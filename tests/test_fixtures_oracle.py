"""CPU: the bench fixtures are deterministic and the oracle's fp32-storage
projection equals its fp64 restatement on widened values."""

import numpy as np

from fixtures import scenes
from oracle import oracle as O


def test_fixture_deterministic_and_sized():
    a = scenes.build("street1080")
    b = scenes.build("street1080")
    assert np.array_equal(a.levels[0][0], b.levels[0][0])
    assert np.array_equal(a.data, b.data) and np.array_equal(a.offsets, b.offsets)
    assert len(a.levels[0][0]) == 47620
    for j in range(a.K):
        for l in range(a.L):
            s = a.set(j, l)
            assert np.all(np.diff(s.astype(np.int64)) > 0)


def test_config2_level_sizes():
    c = scenes.build("config2")
    assert c.n_gaussians() == [1_000_000, 310_000, 130_000]
    assert c.K == 16 and c.L == 3


def test_project_f32_equals_fp64_restatement():
    c = scenes.build("street1080")
    cam = scenes.camera(40.0)
    oc, rc = O.camera_from(cam), O.cfg_struct(__import__("paper_2505_23158_b200").RasterConfig())
    f, o, tb, t = O.select(c.centers, cam.position)
    for l in range(c.L):
        idx, mod, _ = O.union(c.set(f, l).astype(np.int64), c.set(o, l).astype(np.int64), t)
        a = O.project(scenes.scene_objects(c, l), idx, oc, rc, mod)
        g, s, _ = c.levels[l]
        b = O.project_f32(g, s, c.degree, idx, oc, rc, mod)
        for k in ("src", "mean2d", "conic", "depth", "opacity", "color", "rect"):
            assert np.array_equal(a[k], b[k]), k


def test_config4_room_fixture():
    """Config 4: 6M Gaussians, 4 LODs at d = 0.2 (10, 28, 47),
    32 chunks from k-means over a 2-D camera grid at eye height (a Voronoi
    tiling of the floor plan), and a 1024-view Lissajous path that changes
    chunk pair often and passes near junctions of three or more chunks."""
    c = scenes.build("config4")
    assert c.n_gaussians() == [6_000_000, 1_860_000, 780_000, 456_000]
    assert c.K == 32 and c.L == 4 and c.degree == 3
    assert [lv[2] for lv in c.levels[1:]] == [2.0, 5.6, 9.4]
    assert np.allclose(c.centers[:, 1], scenes.ROOM_EYE)  # 2-D tiling at eye height
    path = c.sweep(1024)
    assert len(path) == 1024
    pairs = [O.select(c.centers, cam.position)[:2] for cam in path]
    changes = sum(1 for i in range(1, len(pairs)) if pairs[i] != pairs[i - 1])
    assert changes >= 50 and len(set(pairs)) >= 40
    near3 = 0
    for cam in path:
        d = np.sort(np.linalg.norm(c.centers - cam.position, axis=1))
        near3 += int(d[2] < 1.3 * d[0])
    assert near3 >= 20
    for cam in path[:8]:  # the camera looks along the path tangent: R is a rotation
        R = cam.rotation_matrix
        assert np.allclose(R @ R.T, np.eye(3)) and np.isclose(np.linalg.det(R), 1.0)
