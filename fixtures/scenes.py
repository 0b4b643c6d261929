"""Bench/test fixture configs (SURVEY.md 8d recipes) built with fixtures/synth.c.

    cfg = build("config3")     # 20M Gaussians, 5 LODs, 64 chunks, SH3
    cfg = build("config4")     # indoor room, 6M Gaussians, 4 LODs, 32 chunks (2-D Voronoi)
    cfg.levels  -> [(geom fp32 (n,12), sh fp32 (n,3,16), depth_threshold)]
    cfg.plan    -> centers (K,3), radii (K,), offsets (K*L+1), data uint32
    cfg.sweep(n)-> n trajectory cameras along the corridor (config 5)

Levels use the pruning proxy of the recipe (keep the top fraction by
opacity * max(scale)^2, ties by index) with the Eq. 3 filter variance
d / f_ref; chunks are 1-D Lloyd k-means over the rig positions (quantile
initialisation), radii to the nearest other centre, radius-offset distance
bands (src/chunks.py:101-135).  Visibility filtering is off (documented in
DESIGN.md).  Inputs for both bench arms; not part of the render path.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import time
from dataclasses import dataclass, field
from types import SimpleNamespace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libsynth.so")
_lib = None

CONFIGS = {
    # name: n_fine, length, sh_degree, thresholds, keep fractions, K, rig views
    "street1080": dict(n_fine=42000, length=200.0, degree=1, d=(10.0,), keep=(0.31,), K=4,
                       views=64),
    "config2": dict(n_fine=994_380, length=200.0, degree=3, d=(10.0, 28.0), keep=(0.31, 0.13),
                    K=16, views=64),
    "config3": dict(n_fine=19_994_380, length=2000.0, degree=3, d=(10.0, 28.0, 47.0, 63.0),
                    keep=(0.31, 0.13, 0.076, 0.049), K=64, views=256),
    # Zip-NeRF-style room (synth_room), d = 0.2 * (10, 28, 47),
    # a 16 x 12 camera grid at height 1.6, k-means k = 32 over it, a
    # 1024-view Lissajous path crossing the chunk junctions
    "config4": dict(n_fine=5_986_062, length=0.0, degree=3, d=(2.0, 5.6, 9.4),
                    keep=(0.31, 0.13, 0.076), K=32, views=(16, 12), scene="room"),
}
ROOM_X, ROOM_Z, ROOM_EYE = 20.0, 15.0, 1.6
WIDTH, HEIGHT, FOCAL = 1920, 1080, 1560.0


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        L = C.CDLL(_LIB)
        P = C.c_void_p
        L.synth_count.argtypes = [C.c_int64]
        L.synth_count.restype = C.c_int64
        L.synth_room_count.argtypes = [C.c_int64]
        L.synth_room_count.restype = C.c_int64
        L.synth_room.argtypes = [C.c_uint64, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p]
        L.synth_street.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.c_int32, P, P]
        L.synth_prune_key.argtypes = [P, C.c_int64, P]
        L.synth_gather_level.argtypes = [P, P, C.c_int32, P, C.c_int64, C.c_float, P, P]
        L.synth_bands.argtypes = [P, C.c_int64, P, C.c_int32, P, P, P, P, P]
        L.synth_threads.restype = C.c_int32
        L.synth_set_threads.argtypes = [C.c_int32]
        _lib = L
    return _lib


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def camera(z: float, width=WIDTH, height=HEIGHT, focal=FOCAL, x=0.0, y=0.5, yaw=0.0):
    """Trajectory camera at (x, y, z) looking along (sin yaw, 0, cos yaw);
    yaw 0 is the identity orientation of pkg/scripts/make_deep_street.py:34-36.
    rotation_matrix maps world offsets to camera coordinates (src/scene.py:
    116-117); orientation is its wxyz quaternion (a rotation about y by -yaw)."""
    c, s = float(np.cos(yaw)), float(np.sin(yaw))
    R = np.eye(3) if yaw == 0.0 else np.array([[c, 0.0, -s], [0.0, 1.0, 0.0], [s, 0.0, c]])
    quat = np.array([np.cos(-yaw / 2), 0.0, np.sin(-yaw / 2), 0.0])
    return SimpleNamespace(position=np.array([x, y, z], np.float64), orientation=quat,
                           rotation_matrix=R, focal=np.array([focal, focal]),
                           principal_point=np.array([width / 2, height / 2]),
                           resolution=(width, height), near_plane=0.05)


def lissajous(n: int):
    """Config 4 path: n views on x = 0.85 X sin(3s + pi/2), z = 0.8 Z sin(2s),
    s in [0, 2 pi), at eye height, each looking along the path tangent -- a
    dense diagonal sweep through the room that crosses the chunk junctions."""
    s = np.linspace(0.0, 2 * np.pi, n, endpoint=False)
    x = 0.85 * ROOM_X * np.sin(3 * s + np.pi / 2)
    z = 0.8 * ROOM_Z * np.sin(2 * s)
    dx = 0.85 * ROOM_X * 3 * np.cos(3 * s + np.pi / 2)
    dz = 0.8 * ROOM_Z * 2 * np.cos(2 * s)
    yaw = np.arctan2(dx, dz)
    return [camera(float(z[i]), x=float(x[i]), y=ROOM_EYE, yaw=float(yaw[i])) for i in range(n)]


def kmeans_1d(positions: np.ndarray, k: int, iters: int = 50):
    """Lloyd iterations from quantile seeds (deterministic): seeds are the
    positions at evenly spaced list indices (a path for the corridor, the
    row-major grid for the room); any dimension."""
    pts = np.asarray(positions, np.float64)
    seeds = np.round(np.linspace(0, len(pts) - 1, k)).astype(np.int64)
    centers = pts[seeds].copy()
    assign = None
    for _ in range(iters):
        d = np.linalg.norm(pts[:, None, :] - centers[None, :, :], axis=2)
        new = np.argmin(d, axis=1)
        if assign is not None and np.array_equal(new, assign):
            break
        assign = new
        for j in range(k):
            m = pts[assign == j]
            if len(m):
                centers[j] = m.mean(axis=0)
    return centers, assign


def chunk_radii(centers):
    d = np.linalg.norm(centers[:, None, :] - centers[None, :, :], axis=2)
    np.fill_diagonal(d, np.inf)
    return d.min(axis=1)


@dataclass
class Config:
    name: str
    levels: list           # [(geom, sh, depth_threshold)]
    degree: int
    centers: np.ndarray
    radii: np.ndarray
    offsets: np.ndarray    # (K*L+1,) int64
    data: np.ndarray       # uint32
    rig_z: np.ndarray
    length: float
    timings: dict = field(default_factory=dict)
    rig: np.ndarray = None  # (V, 3) rig positions (config 4: the 2-D grid)

    @property
    def K(self):
        return self.centers.shape[0]

    @property
    def L(self):
        return len(self.levels)

    def set(self, j, l):
        return self.data[self.offsets[j * self.L + l]:self.offsets[j * self.L + l + 1]]

    def sweep(self, n: int):
        """Config 5 path: z from 4 to 0.65*length, identity orientation; the
        room (config 4): the Lissajous path."""
        if self.name == "config4":
            return lissajous(n)
        return [camera(float(z)) for z in np.linspace(4.0, 0.65 * self.length, n)]

    def rig_camera(self, i: int):
        if self.rig is not None:
            p = self.rig[i]
            return camera(float(p[2]), x=float(p[0]), y=float(p[1]))
        return camera(float(self.rig_z[i]))

    def n_gaussians(self):
        return [len(g) for g, _, _ in self.levels]

    def store_bytes(self):
        return sum(g.nbytes + s.nbytes for g, s, _ in self.levels)


def build(name: str, seed: int = 7, verbose: bool = False, threads: int = 0) -> Config:
    """threads > 0: OpenMP threads of the generator (else the runtime's default)."""
    spec = CONFIGS[name]
    L = lib()
    if threads > 0:
        L.synth_set_threads(int(threads))
    t0 = time.time()
    deg = spec["degree"]
    terms = (deg + 1) ** 2
    room = spec.get("scene") == "room"
    n = int((L.synth_room_count if room else L.synth_count)(spec["n_fine"]))
    geom = np.empty((n, 12), np.float32)
    sh = np.empty((n, 3, terms), np.float32)
    if room:
        L.synth_room(seed, spec["n_fine"], deg, _p(geom), _p(sh))
    else:
        L.synth_street(seed, spec["n_fine"], spec["length"], deg, _p(geom), _p(sh))
    t1 = time.time()
    levels = [(geom, sh, 0.0)]
    if spec["d"]:
        key = np.empty(n, np.float32)
        L.synth_prune_key(_p(geom), n, _p(key))
        order = np.argsort(-key, kind="stable")
        for d, keep in zip(spec["d"], spec["keep"]):
            idx = np.sort(order[:int(round(keep * n))]).astype(np.int64)
            g = np.empty((len(idx), 12), np.float32)
            s = np.empty((len(idx), 3, terms), np.float32)
            L.synth_gather_level(_p(geom), _p(sh), terms, _p(idx), len(idx), float(d / FOCAL),
                                 _p(g), _p(s))
            levels.append((g, s, float(d)))
    t2 = time.time()
    if room:  # a 2-D camera grid at eye height; k-means over it tiles the floor plan
        nx, nz = spec["views"]
        gx, gz = np.meshgrid(np.linspace(-0.9 * ROOM_X, 0.9 * ROOM_X, nx),
                             np.linspace(-0.9 * ROOM_Z, 0.9 * ROOM_Z, nz), indexing="ij")
        positions = np.stack([gx.reshape(-1), np.full(nx * nz, ROOM_EYE), gz.reshape(-1)], axis=1)
        rig_z = positions[:, 2].copy()
    else:
        rig_z = np.linspace(2.0, 0.7 * spec["length"], spec["views"])
        positions = np.stack([np.zeros_like(rig_z), np.full_like(rig_z, 0.5), rig_z], axis=1)
    centers, _ = kmeans_1d(positions, spec["K"])
    radii = chunk_radii(centers) if spec["K"] > 1 else np.array([1.0])
    K, nl = spec["K"], len(levels)
    ds = [0.0] + list(spec["d"])
    counts = np.zeros((nl, K), np.int64)
    per_level = []
    for l, (g, _, _) in enumerate(levels):
        lo = np.array([0.0 if l == 0 else ds[l] + radii[j] for j in range(K)])
        hi = np.array([np.inf if l + 1 == nl else ds[l + 1] + radii[j] for j in range(K)])
        c = np.zeros(K, np.int64)
        L.synth_bands(_p(g), len(g), _p(centers), K, _p(lo), _p(hi), _p(c), None, None)
        offs = np.zeros(K + 1, np.int64)
        offs[1:] = np.cumsum(c)
        out = np.empty(int(offs[-1]), np.uint32)
        L.synth_bands(_p(g), len(g), _p(centers), K, _p(lo), _p(hi), None, _p(offs), _p(out))
        counts[l] = c
        per_level.append((offs, out))
    sizes = counts.T.reshape(-1)  # (j, l) order
    offsets = np.zeros(K * nl + 1, np.int64)
    offsets[1:] = np.cumsum(sizes)
    data = np.empty(int(offsets[-1]), np.uint32)
    for j in range(K):
        for l in range(nl):
            o, arr = per_level[l]
            data[offsets[j * nl + l]:offsets[j * nl + l + 1]] = arr[o[j]:o[j + 1]]
    t3 = time.time()
    cfg = Config(name, levels, deg, centers, radii, offsets, data, rig_z, spec["length"],
                 {"scene_s": t1 - t0, "levels_s": t2 - t1, "chunks_s": t3 - t2,
                  "threads": int(L.synth_threads())}, positions if room else None)
    if verbose:
        print(f"[fixtures] {name}: levels {cfg.n_gaussians()} sets {len(data)} "
              f"({cfg.timings})", flush=True)
    return cfg


def _scratch_dir(nbytes: int, key: str) -> str:
    """/dev/shm when it has room for the arrays (page cache shared by the
    ranks), else /tmp."""
    import shutil
    for root in ("/dev/shm", "/tmp"):
        try:
            if shutil.disk_usage(root).free > 1.2 * nbytes:
                return os.path.join(root, key)
        except OSError:
            continue
    return os.path.join("/tmp", key)


def build_shared(name: str, local_rank: int, local_world: int, barrier, seed: int = 7,
                 key: str = "") -> Config:
    """One generation per node for multi-rank runs: local rank 0 builds the
    config with every host core and writes its arrays (.npy) to a scratch
    directory; the other local ranks memory-map them (no per-rank copy of the
    ~8 GB host arrays).  barrier() must synchronise the node's ranks."""
    import json
    import shutil
    if local_world <= 1:
        return build(name, seed, threads=os.cpu_count() or 1)
    spec = CONFIGS[name]
    cnt = lib().synth_room_count if spec.get("scene") == "room" else lib().synth_count
    n0 = int(cnt(spec["n_fine"]))
    est = n0 * (48 + 12 * (spec["degree"] + 1) ** 2) * 2
    d = _scratch_dir(est, f"lodge_fixture_{name}_{seed}_{key or os.getppid()}")
    if local_rank == 0:
        cfg = build(name, seed, threads=os.cpu_count() or 1)
        os.makedirs(d, exist_ok=True)
        meta = {"name": cfg.name, "degree": cfg.degree, "length": cfg.length,
                "L": cfg.L, "d": [float(x[2]) for x in cfg.levels], "timings": cfg.timings}
        for l, (g, s, _) in enumerate(cfg.levels):
            np.save(os.path.join(d, f"g{l}.npy"), g)
            np.save(os.path.join(d, f"s{l}.npy"), s)
        for k in ("centers", "radii", "offsets", "data", "rig_z"):
            np.save(os.path.join(d, f"{k}.npy"), getattr(cfg, k))
        if cfg.rig is not None:
            np.save(os.path.join(d, "rig.npy"), cfg.rig)
        with open(os.path.join(d, "meta.json"), "w") as f:
            json.dump(meta, f)
    barrier()
    if local_rank != 0:
        meta = json.load(open(os.path.join(d, "meta.json")))
        ld = lambda k: np.load(os.path.join(d, f"{k}.npy"), mmap_mode="r")  # noqa: E731
        levels = [(ld(f"g{l}"), ld(f"s{l}"), meta["d"][l]) for l in range(meta["L"])]
        cfg = Config(meta["name"], levels, meta["degree"], np.array(ld("centers")),
                     np.array(ld("radii")), np.array(ld("offsets")), ld("data"),
                     np.array(ld("rig_z")), meta["length"],
                     dict(meta["timings"], shared_from=d),
                     np.array(ld("rig")) if os.path.exists(os.path.join(d, "rig.npy")) else None)
    barrier()  # every rank has mapped the files: rank 0 may unlink them
    if local_rank == 0:
        shutil.rmtree(d, ignore_errors=True)
    return cfg


def scene_objects(cfg: Config, l: int):
    """fp64 Scene-like view of level l (for the oracle / drop-in API)."""
    g, s, _ = cfg.levels[l]
    g64 = g.astype(np.float64)
    return SimpleNamespace(means=g64[:, 0:3], scales=g64[:, 3:6], rotations=g64[:, 6:10],
                           opacities=g64[:, 10], filter_variance=g64[:, 11],
                           sh_coeffs=s.astype(np.float64), sh_degree=cfg.degree)
