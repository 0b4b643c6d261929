"""ctypes front-end of the CPU oracle (oracle/lodge_oracle.c).

TEST INFRASTRUCTURE ONLY -- the checker, never the product.  Only tests/,
``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs import this
module.  The product package (paper_2505_23158_b200) never imports it and
fails loudly when its own CUDA library is missing.

Each function restates one reference function (file:line under
/root/reference/pkg/src/splatlod/) in fp64 with NumPy's operation order;
tests/test_oracle_golden.py pins it against vectors generated from the
reference itself (oracle/make_golden.py).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblodge_oracle.so")
_lib = None

_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
_I32 = C.POINTER(C.c_int32)
_I8 = C.POINTER(C.c_int8)


class Camera(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("pos", C.c_double * 3), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("w", C.c_int32), ("h", C.c_int32), ("near_plane", C.c_double)]


class RasterCfg(C.Structure):
    _fields_ = [("alpha_clamp", C.c_double), ("alpha_min", C.c_double),
                ("t_min", C.c_double), ("dilation2d", C.c_double)]


def build() -> str:
    """Compile the oracle library in place (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_select.argtypes = [_D, C.c_int32, _D, _I32, _I32, _D, _D]
        L.orc_union.argtypes = [_I64, C.c_int64, _I64, C.c_int64, C.c_double, _I64, _D, _I8]
        L.orc_union.restype = C.c_int64
        L.orc_project.argtypes = [_D, _D, _D, _D, _D, _D, C.c_int32, _I64, C.c_int64, _D,
                                  C.POINTER(Camera), C.POINTER(RasterCfg), C.c_int32,
                                  _I64, _D, _D, _D, _D, _D, _D, _D, _I32]
        L.orc_project.restype = C.c_int64
        L.orc_rasterize.argtypes = [C.c_int64, C.c_int64, _I64, _D, _D, _D, _D, _D, _D,
                                    C.c_int32, C.c_int32, C.POINTER(RasterCfg), C.c_int32,
                                    C.c_int32, _D, _I64, _I64, _D, _I64, _I64, C.c_int64]
        L.orc_rasterize.restype = C.c_int64
        L.orc_num_threads.restype = C.c_int32
        L.orc_set_threads.argtypes = [C.c_int32]
        L.orc_project_f32.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, _I64, C.c_int64, _D,
                                      C.POINTER(Camera), C.POINTER(RasterCfg), C.c_int32,
                                      _I64, _D, _D, _D, _D, _D, _D, _D, _I32]
        L.orc_project_f32.restype = C.c_int64
        _lib = L
    return _lib


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_threads(n: int) -> None:
    """OpenMP threads of the oracle's parallel loops."""
    lib().orc_set_threads(int(n))


def camera_struct(R, pos, focal, pp, resolution, near) -> Camera:
    c = Camera()
    for i, v in enumerate(np.asarray(R, np.float64).reshape(9)):
        c.R[i] = float(v)
    for i, v in enumerate(np.asarray(pos, np.float64).reshape(3)):
        c.pos[i] = float(v)
    c.fx, c.fy = float(focal[0]), float(focal[1])
    c.cx, c.cy = float(pp[0]), float(pp[1])
    c.w, c.h = int(resolution[0]), int(resolution[1])
    c.near_plane = float(near)
    return c


def camera_from(cam) -> Camera:
    """From any object with the reference Camera's attributes (src/scene.py:80-121)."""
    return camera_struct(cam.rotation_matrix, cam.position, cam.focal, cam.principal_point,
                         cam.resolution, cam.near_plane)


def cfg_struct(cfg) -> RasterCfg:
    r = RasterCfg()
    r.alpha_clamp, r.alpha_min = float(cfg.alpha_clamp), float(cfg.alpha_min)
    r.t_min, r.dilation2d = float(cfg.t_min), float(cfg.dilation2d)
    return r


def select(centers, position):
    """nearest_two_chunks + blend_factor (src/blending.py:77-99)."""
    centers = np.ascontiguousarray(centers, np.float64)
    pos = np.ascontiguousarray(position, np.float64)
    f, o = C.c_int32(), C.c_int32()
    tb, t = C.c_double(), C.c_double()
    lib().orc_select(_p(centers, _D), centers.shape[0], _p(pos, _D), C.byref(f), C.byref(o),
                     C.byref(tb), C.byref(t))
    return f.value, (None if o.value < 0 else o.value), tb.value, t.value


def union(a, b, t):
    """One level of compose_active (src/blending.py:119-128)."""
    a = np.ascontiguousarray(a, np.int64)
    b = np.ascontiguousarray(b, np.int64)
    n = a.shape[0] + b.shape[0]
    idx = np.empty(n, np.int64)
    mod = np.empty(n, np.float64)
    tag = np.empty(n, np.int8)
    k = lib().orc_union(_p(a, _I64), a.shape[0], _p(b, _I64), b.shape[0], float(t),
                        _p(idx, _I64), _p(mod, _D), _p(tag, _I8))
    return idx[:k].copy(), mod[:k].copy(), tag[:k].copy()


def project(scene, indices, camera: Camera, cfg: RasterCfg, modulation=None, shade=True):
    """project_scene (src/raster.py:188-291) for a Scene-like object."""
    means = np.ascontiguousarray(scene.means, np.float64)
    scales = np.ascontiguousarray(scene.scales, np.float64)
    rots = np.ascontiguousarray(scene.rotations, np.float64)
    opac = np.ascontiguousarray(scene.opacities, np.float64)
    fv = np.ascontiguousarray(scene.filter_variance, np.float64)
    sh = np.ascontiguousarray(scene.sh_coeffs, np.float64)
    idx = (np.arange(means.shape[0], dtype=np.int64) if indices is None
           else np.ascontiguousarray(indices, np.int64))
    n = idx.shape[0]
    mod = None if modulation is None else np.ascontiguousarray(modulation, np.float64)
    if mod is not None and mod.shape[0] != n:
        raise ValueError("modulation length must match the input list")
    out = {"src": np.empty(n, np.int64), "mean2d": np.empty((n, 2)), "cov2d": np.empty((n, 2, 2)),
           "conic": np.empty((n, 3)), "extent": np.empty((n, 2)), "depth": np.empty(n),
           "opacity": np.empty(n), "color": np.empty((n, 3)), "rect": np.empty((n, 4), np.int32)}
    m = lib().orc_project(_p(means, _D), _p(scales, _D), _p(rots, _D), _p(opac, _D), _p(fv, _D),
                          _p(sh, _D), int(scene.sh_degree), _p(idx, _I64), n, _p(mod, _D),
                          C.byref(camera), C.byref(cfg), int(bool(shade)),
                          _p(out["src"], _I64), _p(out["mean2d"], _D), _p(out["cov2d"], _D),
                          _p(out["conic"], _D), _p(out["extent"], _D), _p(out["depth"], _D),
                          _p(out["opacity"], _D), _p(out["color"], _D), _p(out["rect"], _I32))
    res = {k: v[:m].copy() for k, v in out.items()}
    res["n_inputs"] = n
    return res


def project_f32(geom, sh, degree, indices, camera: Camera, cfg: RasterCfg, modulation=None,
                shade=True):
    """project_scene over fp32 AoS records (N,12) + SH (N,3,terms), widened to
    fp64 (the device's fp32 store); OpenMP over input chunks, order kept."""
    geom = np.ascontiguousarray(geom, np.float32)
    sh = np.ascontiguousarray(sh, np.float32)
    idx = np.ascontiguousarray(indices, np.int64)
    n = idx.shape[0]
    mod = None if modulation is None else np.ascontiguousarray(modulation, np.float64)
    out = {"src": np.empty(n, np.int64), "mean2d": np.empty((n, 2)), "cov2d": np.empty((n, 2, 2)),
           "conic": np.empty((n, 3)), "extent": np.empty((n, 2)), "depth": np.empty(n),
           "opacity": np.empty(n), "color": np.empty((n, 3)), "rect": np.empty((n, 4), np.int32)}
    m = lib().orc_project_f32(C.c_void_p(geom.ctypes.data), C.c_void_p(sh.ctypes.data),
                              int(degree), _p(idx, _I64), n, _p(mod, _D), C.byref(camera),
                              C.byref(cfg), int(bool(shade)), _p(out["src"], _I64),
                              _p(out["mean2d"], _D), _p(out["cov2d"], _D), _p(out["conic"], _D),
                              _p(out["extent"], _D), _p(out["depth"], _D),
                              _p(out["opacity"], _D), _p(out["color"], _D),
                              _p(out["rect"], _I32))
    if m < 0:
        raise MemoryError("oracle project_f32: allocation failed")
    res = {k: v[:m] for k, v in out.items()}
    res["n_inputs"] = n
    return res


def concat(parts):
    """Splat2DBatch.concat (src/raster.py:98-116): level-major, shifted sources."""
    off = 0
    out = {k: [] for k in ("src", "mean2d", "cov2d", "conic", "extent", "depth", "opacity",
                           "color", "rect")}
    for p in parts:
        for k in out:
            out[k].append(p[k] + off if k == "src" else p[k])
        off += p["n_inputs"]
    res = {k: np.concatenate(v) if v else np.zeros(0) for k, v in out.items()}
    res["n_inputs"] = off
    return res


def rasterize(batch, w, h, cfg: RasterCfg, need_image=True, record_max=True, lists=False):
    """rasterize (src/raster.py:380-449).  With ``lists`` also returns the
    per-tile member lists (source indices, tile-major) and their offsets."""
    tiles_x, tiles_y = -(-w // 16), -(-h // 16)
    T = tiles_x * tiles_y
    M = int(batch["src"].shape[0])
    n_in = int(batch["n_inputs"])
    src = np.ascontiguousarray(batch["src"], np.int64)
    mean2d = np.ascontiguousarray(batch["mean2d"], np.float64).reshape(-1, 2)
    conic = np.ascontiguousarray(batch["conic"], np.float64).reshape(-1, 3)
    extent = np.ascontiguousarray(batch["extent"], np.float64).reshape(-1, 2)
    depth = np.ascontiguousarray(batch["depth"], np.float64)
    opac = np.ascontiguousarray(batch["opacity"], np.float64)
    color = np.ascontiguousarray(batch["color"], np.float64).reshape(-1, 3)
    image = np.zeros((h, w, 3)) if need_image else None
    tile_count = np.zeros((tiles_y, tiles_x), np.int64)
    visible = np.zeros((h, w), np.int64)
    maxw = np.zeros(n_in) if record_max else None
    offs = np.zeros(T + 1, np.int64) if lists else None
    cap = 0
    tile_src = None
    if lists:
        # count first, then fetch
        P = lib().orc_rasterize(n_in, M, _p(src, _I64), _p(mean2d, _D), _p(conic, _D),
                                _p(extent, _D), _p(depth, _D), _p(opac, _D), _p(color, _D),
                                w, h, C.byref(cfg), 0, 0, None, _p(tile_count, _I64),
                                _p(visible, _I64), None, _p(offs, _I64), None, 0)
        cap = max(int(P), 1)
        tile_src = np.zeros(cap, np.int64)
    P = lib().orc_rasterize(n_in, M, _p(src, _I64), _p(mean2d, _D), _p(conic, _D),
                            _p(extent, _D), _p(depth, _D), _p(opac, _D), _p(color, _D),
                            w, h, C.byref(cfg), int(bool(need_image)), int(bool(record_max)),
                            _p(image, _D), _p(tile_count, _I64), _p(visible, _I64),
                            _p(maxw, _D), _p(offs, _I64), _p(tile_src, _I64), cap)
    if P < 0:
        raise MemoryError("oracle rasterize: allocation failed")
    out = {"image": image, "per_tile_count": tile_count, "per_pixel_visible": visible,
           "per_gaussian_max_weight": maxw, "P": int(P)}
    if lists:
        out["tile_offsets"] = offs
        out["tile_src"] = tile_src[:P]
    return out


def select_active(levels, position, bounds):
    """select_active (src/lod.py:192-211) for precomputed band bounds: level l
    keeps flatnonzero(bounds[l] <= ||means - position|| < bounds[l+1])."""
    q = np.asarray(position, float)
    sets = []
    for l, lv in enumerate(levels):
        means = np.asarray(getattr(lv, "scene", lv).means)
        dist = np.linalg.norm(means - q, axis=1)
        sets.append(np.flatnonzero((dist >= bounds[l]) & (dist < bounds[l + 1])))
    return sets


def cover_table(scene, camera: Camera, cfg: RasterCfg, position):
    """ThresholdSearcher._table (src/thresholds.py:80-90): project with
    shade=False, tile_cover_counts (src/raster.py:303-324) of the survivors,
    their distances np.linalg.norm(means[src] - position, axis=1), stable
    argsort by distance, prefix = [0, cumsum(cover[order])]."""
    b = project(scene, None, camera, cfg, None, shade=False)
    tiles_x, tiles_y = -(-camera.w // 16), -(-camera.h // 16)
    mean2d = np.asarray(b["mean2d"]).reshape(-1, 2)
    ext = np.asarray(b["extent"]).reshape(-1, 2)
    x0 = np.clip(np.floor((mean2d[:, 0] - ext[:, 0]) / 16), 0, tiles_x - 1).astype(np.int64)
    x1 = np.clip(np.floor((mean2d[:, 0] + ext[:, 0]) / 16), 0, tiles_x - 1).astype(np.int64)
    y0 = np.clip(np.floor((mean2d[:, 1] - ext[:, 1]) / 16), 0, tiles_y - 1).astype(np.int64)
    y1 = np.clip(np.floor((mean2d[:, 1] + ext[:, 1]) / 16), 0, tiles_y - 1).astype(np.int64)
    cover = (x1 - x0 + 1) * (y1 - y0 + 1)
    src = np.asarray(b["src"], np.int64)
    dist = np.linalg.norm(np.asarray(scene.means)[src] - np.asarray(position), axis=1)
    order = np.argsort(dist, kind="stable")
    return dist[order], np.concatenate([[0], np.cumsum(cover[order])])


def importance(levels, sets, cameras, cfg: RasterCfg):
    """score_active_selection (src/lod.py:95-122) over the given, already
    perturbed views: per view project every level's set with shade=False,
    concat, rasterize with need_image=False / record_max_weight=True, and
    keep the running np.maximum of per_gaussian_max_weight.  Returns one
    score array per level."""
    offsets = np.cumsum([0] + [len(s) for s in sets])
    scores = np.zeros(offsets[-1])
    for cam in cameras:
        out = render_selection(levels, sets, None, cam, cfg, need_image=False, record_max=True)
        np.maximum(scores, out["per_gaussian_max_weight"], out=scores)
    return [scores[offsets[l]:offsets[l + 1]] for l in range(len(sets))]


def render_selection(levels, sets, mods, camera: Camera, cfg: RasterCfg, need_image=True,
                     record_max=True, lists=False):
    """project_selection + rasterize (src/blending.py:132-137, src/lod.py:216-227)."""
    parts = []
    for l, lv in enumerate(levels):
        scene = getattr(lv, "scene", lv)
        parts.append(project(scene, sets[l], camera, cfg,
                             None if mods is None else mods[l], shade=need_image))
    batch = concat(parts)
    out = rasterize(batch, camera.w, camera.h, cfg, need_image, record_max, lists)
    out["batch"] = batch
    return out
