"""Drop-in projection + rasterization API (reference src/raster.py).

project_scene / rasterize / render_scene / project_gaussian keep the
reference's names, signatures and outputs; the work runs in liblodge.so
(K2 projection, K4 onesweep sorts, K3 binning, K6 compositing).  Inputs are
uploaded once per host object and outputs are copied back as the
reference's fp64 / int64 NumPy arrays.
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch

from . import _native as N
from .device import (camera_struct, context, default_precision, level_for, params_struct,
                     ptr)
from .types import (TILE_SIZE, RasterConfig, Scene, Splat2DBatch, TileRenderOutput,
                    empty_batch)

_F64 = torch.float64


def _tiles(camera):
    w, h = camera.resolution
    return -(-int(w) // TILE_SIZE), -(-int(h) // TILE_SIZE)


class DeviceBatch:
    """A Splat2DBatch resident on the device (fp64 fields, int64 sources)."""

    FIELDS = ("src", "mean2d", "cov2d", "conic", "extent", "depth", "opacity", "color")

    def __init__(self, n_inputs, t: dict):
        self.n_inputs = int(n_inputs)
        self.t = t

    def __len__(self):
        return int(self.t["src"].shape[0])

    @staticmethod
    def alloc(n, device):
        shapes = {"src": (n,), "mean2d": (n, 2), "cov2d": (n, 2, 2), "conic": (n, 3),
                  "extent": (n, 2), "depth": (n,), "opacity": (n,), "color": (n, 3)}
        return {k: torch.empty(s, dtype=torch.int64 if k == "src" else _F64, device=device)
                for k, s in shapes.items()}

    def struct(self) -> N.Batch:
        b = N.Batch()
        for k, f in zip(self.FIELDS, ("src_dev", "mean2d_dev", "cov2d_dev", "conic_dev",
                                      "extent_dev", "depth_dev", "opacity_dev", "color_dev")):
            setattr(b, f, self.t[k].data_ptr() if self.t[k].numel() else None)
        return b

    def to_host(self) -> Splat2DBatch:
        if len(self) == 0:
            return empty_batch(self.n_inputs)
        h = {k: v.cpu().numpy() for k, v in self.t.items()}
        return Splat2DBatch(self.n_inputs, h["src"], h["mean2d"], h["cov2d"], h["conic"],
                            h["extent"], h["depth"], h["opacity"], h["color"])

    @staticmethod
    def from_host(batch, device) -> "DeviceBatch":
        src = np.asarray(batch.source_index, np.int64)
        f = {"src": src, "mean2d": batch.mean2d, "cov2d": batch.cov2d, "conic": batch.conic,
             "extent": batch.extent, "depth": batch.depth, "opacity": batch.opacity_eff,
             "color": batch.color}
        if src.shape[0] > 1 and np.any(np.diff(src) <= 0):
            # np.lexsort((source_index, depth)) breaks depth ties by source
            # index; the device sort is stable over rows, so feed rows in
            # source order (a permutation of the input, no arithmetic).
            order = np.argsort(src, kind="stable")
            f = {k: np.asarray(v)[order] for k, v in f.items()}
        t = {k: torch.from_numpy(np.ascontiguousarray(v, np.int64 if k == "src" else np.float64))
             .to(device) for k, v in f.items()}
        return DeviceBatch(batch.n_inputs, t)

    @staticmethod
    def concat(parts, device) -> "DeviceBatch":
        if not parts:
            return DeviceBatch(0, DeviceBatch.alloc(0, device))
        off, srcs = 0, []
        for p in parts:
            srcs.append(p.t["src"] + off)
            off += p.n_inputs
        t = {"src": torch.cat(srcs)}
        for k in DeviceBatch.FIELDS[1:]:
            t[k] = torch.cat([p.t[k] for p in parts])
        return DeviceBatch(off, t)


def project_scene_device(scene, camera, cfg=RasterConfig(), indices=None, modulation=None,
                         shade=True, device=None, storage="fp64") -> DeviceBatch:
    """project_scene into a device-resident batch (src/raster.py:188-291)."""
    ctx = context(device)
    dev = ctx.device
    n_total = len(scene.means)
    if indices is None:
        n = n_total
        idx_t = None
    else:
        idx = np.asarray(indices, dtype=np.int64)
        n = idx.shape[0]
        if n and (idx.min() < -n_total or idx.max() >= n_total):
            raise IndexError("index out of bounds for the scene")
        idx = np.where(idx < 0, idx + n_total, idx)
        idx_t = torch.from_numpy(idx).to(dev) if n else None
    if n == 0:
        return DeviceBatch(0, DeviceBatch.alloc(0, dev))
    mod_t = None
    if modulation is not None:
        mod = np.asarray(modulation, dtype=np.float64)
        if mod.shape[0] != n:
            raise ValueError("modulation length must match the input list")
        mod_t = torch.from_numpy(np.ascontiguousarray(mod)).to(dev)
    lvl = level_for(scene, dev, storage)
    out = DeviceBatch.alloc(n, dev)
    b = DeviceBatch(n, out)
    m = C.c_int64()
    N.check(N.lib().lodge_project(ctx.bind(), C.byref(lvl.struct), ptr(idx_t), n, ptr(mod_t),
                                  C.byref(camera_struct(camera)), C.byref(params_struct(cfg)),
                                  int(bool(shade)), C.byref(b.struct()), C.byref(m)),
            "lodge_project")
    M = int(m.value)
    return DeviceBatch(n, {k: v[:M] for k, v in out.items()})


def project_scene(scene, camera, cfg: RasterConfig = RasterConfig(),
                  indices: Optional[np.ndarray] = None, modulation: Optional[np.ndarray] = None,
                  shade: bool = True) -> Splat2DBatch:
    """Drop-in for reference project_scene (src/raster.py:188)."""
    return project_scene_device(scene, camera, cfg, indices, modulation, shade).to_host()


def project_gaussian(g, camera, cfg: RasterConfig = RasterConfig()):
    """Project a single Gaussian; returns None when culled (src/raster.py:294-300)."""
    degree = int(np.sqrt(np.asarray(g.sh_coeffs).shape[-1])) - 1
    scene = Scene.from_gaussians([g], degree)
    batch = project_scene(scene, camera, cfg)
    return batch.splat(0) if len(batch) else None


def rasterize_device(db: DeviceBatch, camera, cfg=RasterConfig(), need_image=True,
                     record_max_weight=True, precision=None, lists=False, device=None,
                     ctx=None):
    """Bin, sort and composite a device batch; returns device tensors.
    ctx: a device.Context to run on (default: the device's shared one)."""
    ctx = ctx or context(device)
    dev = ctx.device
    w, h = (int(v) for v in camera.resolution)
    tx, ty = _tiles(camera)
    prec = precision or default_precision()
    exact = prec == "exact"
    fdt = torch.float64 if exact else torch.float32
    M = len(db)
    res = {"image": torch.zeros((h, w, 3), dtype=fdt, device=dev) if need_image else None,
           "tile_count": torch.zeros((ty, tx), dtype=torch.int32, device=dev),
           "visible": torch.zeros((h, w), dtype=torch.int32, device=dev),
           "maxw": torch.zeros(db.n_inputs, dtype=fdt, device=dev) if record_max_weight else None,
           "stats": N.FrameStats()}
    if lists:
        res["tile_offsets"] = torch.zeros(tx * ty + 1, dtype=torch.int64, device=dev)
    if M == 0:
        if lists:
            res["tile_src"] = torch.zeros(0, dtype=torch.int64, device=dev)
        return res
    out = N.FrameOut()
    out.image_dev = res["image"].data_ptr() if need_image else None
    out.tile_count_dev = res["tile_count"].data_ptr()
    out.visible_dev = res["visible"].data_ptr()
    out.maxw_dev = (res["maxw"].data_ptr() if record_max_weight and db.n_inputs else None)
    flags = (N.NEED_IMAGE if need_image else 0) | (N.RECORD_MAX if record_max_weight else 0)
    cam = camera_struct(camera)
    rp = params_struct(cfg)
    bs = db.struct()
    lib = N.lib()
    if lists:
        # first pass learns P, second exports the lists (same deterministic result)
        cap = 0
        N.check(lib.lodge_rasterize(ctx.bind(prec), C.byref(bs), M, db.n_inputs, C.byref(cam),
                                    C.byref(rp), flags, C.byref(out), None, None, 0,
                                    C.byref(res["stats"])), "lodge_rasterize")
        cap = int(res["stats"].P)
        res["tile_src"] = torch.zeros(max(cap, 1), dtype=torch.int64, device=dev)
        if need_image:
            res["image"].zero_()
        N.check(lib.lodge_rasterize(ctx.bind(prec), C.byref(bs), M, db.n_inputs, C.byref(cam),
                                    C.byref(rp), flags, C.byref(out),
                                    ptr(res["tile_offsets"]), ptr(res["tile_src"]), cap,
                                    C.byref(res["stats"])), "lodge_rasterize")
        res["tile_src"] = res["tile_src"][:cap]
    else:
        N.check(lib.lodge_rasterize(ctx.bind(prec), C.byref(bs), M, db.n_inputs, C.byref(cam),
                                    C.byref(rp), flags, C.byref(out), None, None, 0,
                                    C.byref(res["stats"])), "lodge_rasterize")
    if res["stats"].fault:
        raise N.LodgeError("lodge_rasterize: device bounds check fired "
                           f"(fault bits {res['stats'].fault:#x})")
    return res


def output_to_host(res, cfg) -> TileRenderOutput:
    img = res["image"]
    mw = res["maxw"]
    return TileRenderOutput(
        None if img is None else img.to(torch.float64).cpu().numpy(),
        res["tile_count"].to(torch.int64).cpu().numpy(),
        res["visible"].to(torch.int64).cpu().numpy(),
        None if mw is None else mw.to(torch.float64).cpu().numpy(),
        cfg.metadata() if hasattr(cfg, "metadata") else {})


def rasterize(batch, camera, cfg: RasterConfig = RasterConfig(), *, need_image: bool = True,
              record_max_weight: bool = True) -> TileRenderOutput:
    """Drop-in for reference rasterize (src/raster.py:380)."""
    ctx = context()
    db = DeviceBatch.from_host(batch, ctx.device)
    return output_to_host(rasterize_device(db, camera, cfg, need_image, record_max_weight), cfg)


def render_scene(scene, camera, cfg: RasterConfig = RasterConfig(),
                 indices: Optional[np.ndarray] = None, modulation: Optional[np.ndarray] = None,
                 need_image: bool = True, record_max_weight: bool = True) -> TileRenderOutput:
    """Drop-in for reference render_scene (src/raster.py:452); the batch stays on the device."""
    db = project_scene_device(scene, camera, cfg, indices, modulation, shade=need_image)
    return output_to_host(rasterize_device(db, camera, cfg, need_image, record_max_weight), cfg)


def tile_cover_counts(batch, camera) -> np.ndarray:
    """Tiles per surviving splat (src/raster.py:316-324); host integer helper."""
    tiles_x, tiles_y = _tiles(camera)
    if len(batch) == 0:
        return np.zeros(0, dtype=np.int64)
    x0 = np.clip(np.floor((batch.mean2d[:, 0] - batch.extent[:, 0]) / TILE_SIZE).astype(np.int64), 0, tiles_x - 1)
    x1 = np.clip(np.floor((batch.mean2d[:, 0] + batch.extent[:, 0]) / TILE_SIZE).astype(np.int64), 0, tiles_x - 1)
    y0 = np.clip(np.floor((batch.mean2d[:, 1] - batch.extent[:, 1]) / TILE_SIZE).astype(np.int64), 0, tiles_y - 1)
    y1 = np.clip(np.floor((batch.mean2d[:, 1] + batch.extent[:, 1]) / TILE_SIZE).astype(np.int64), 0, tiles_y - 1)
    return (x1 - x0 + 1) * (y1 - y0 + 1)


def check_bin_edges(bin_edges) -> np.ndarray:
    """visibility_histogram's edge validation with the reference's messages
    (src/raster.py:471-475)."""
    edges = np.asarray(bin_edges, dtype=np.float64)
    if edges.ndim != 1 or edges.shape[0] < 2:
        raise ValueError("need at least two bin edges")
    if not np.all(np.diff(edges) > 0):
        raise ValueError(f"bin edges must be strictly increasing, got {edges}")
    return edges


def frame_report_device(visible, tile_count, maxw, n_inputs: int, bin_edges, device=None,
                        ctx=None):
    """Device report of one frame (K7, csrc/k_report.cu): the visibility
    histogram of per_pixel_visible (src/raster.py:464-479), the per-tile
    count sum and the number of inputs with a nonzero max weight (the
    reference bench's mean_per_tile / visible_gaussians, src/cli.py:283-320).
    Returns (hist int64 ndarray, tile_count_sum, visible_gaussians)."""
    edges = check_bin_edges(bin_edges)
    if edges.shape[0] > 257:
        raise ValueError("at most 256 histogram bins")
    ctx = ctx or context(device)
    out = torch.zeros(edges.shape[0] + 1, dtype=torch.int64, device=ctx.device)
    e = np.ascontiguousarray(edges)
    vis = visible.contiguous()
    tc = tile_count.contiguous()
    fp64 = 1 if (maxw is not None and maxw.dtype == torch.float64) else 0
    N.check(N.lib().lodge_frame_report(
        ctx.bind(), ptr(vis), vis.numel(), e.ctypes.data_as(C.POINTER(C.c_double)), e.shape[0],
        ptr(tc), tc.numel(), ptr(maxw), fp64, int(n_inputs) if maxw is not None else 0,
        ptr(out)), "lodge_frame_report")
    o = out.cpu().numpy()
    n_bins = edges.shape[0] - 1
    return o[:n_bins].copy(), int(o[n_bins]), int(o[n_bins + 1])


def squared_error_device(a, b, device=None, ctx=None) -> float:
    """Sum of squared differences of two fp32 device images (psnr_vs_full)."""
    if a.dtype != torch.float32 or b.dtype != torch.float32 or a.numel() != b.numel():
        raise ValueError("squared_error_device needs two fp32 images of one size")
    ctx = ctx or context(device)
    out = torch.zeros(1, dtype=torch.float64, device=ctx.device)
    N.check(N.lib().lodge_sq_err(ctx.bind(), ptr(a.contiguous()), ptr(b.contiguous()),
                                 a.numel(), ptr(out)), "lodge_sq_err")
    return float(out.item())


def visibility_histogram(out, bin_edges) -> np.ndarray:
    """Histogram of per-pixel visible counts (src/raster.py:464-479) over a
    host TileRenderOutput, as the reference computes it (the drop-in accepts
    the reference's own output objects); device frames use
    frame_report_device / Renderer.report, the same binning in one kernel."""
    edges = check_bin_edges(bin_edges)
    vals = np.asarray(out.per_pixel_visible).reshape(-1)
    which = np.searchsorted(edges, vals, side="right") - 1
    np.clip(which, 0, edges.shape[0] - 2, out=which)
    return np.bincount(which, minlength=edges.shape[0] - 1)
