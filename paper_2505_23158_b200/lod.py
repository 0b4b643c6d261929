"""Drop-in project_selection (reference src/lod.py:216-227) and the LOD-mode /
full-mode renders (src/lod.py:230-237, src/cli.py:221-243) on the fused path."""

from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .device import _device, context, default_precision, level_for, ptr
from .raster import DeviceBatch, project_scene_device
from .types import ChunkPlan, RasterConfig, TileRenderOutput


def project_selection_device(levels: Sequence, sets: Sequence, camera, raster_cfg,
                             modulations: Optional[Sequence] = None, shade: bool = True,
                             device=None) -> DeviceBatch:
    """Per-level projection concatenated level-major, kept on the device."""
    ctx = context(device)
    parts = []
    for l in range(len(levels)):
        mod = None if modulations is None else np.asarray(modulations[l], float)
        scene = getattr(levels[l], "scene", levels[l])
        parts.append(project_scene_device(scene, camera, raster_cfg,
                                          indices=np.asarray(sets[l], dtype=np.int64),
                                          modulation=mod, shade=shade, device=ctx.device))
    return DeviceBatch.concat(parts, ctx.device)


def project_selection(levels: Sequence, sets: Sequence, camera, raster_cfg: RasterConfig,
                      modulations: Optional[Sequence] = None, shade: bool = True):
    """Project per-level index sets into one splat batch (level-major order)."""
    return project_selection_device(levels, sets, camera, raster_cfg, modulations,
                                    shade).to_host()


def lod_bounds(levels: Sequence, depth_offsets: Optional[Sequence[float]] = None) -> list:
    """The distance bands of select_active (src/lod.py:186-205): level l
    covers [d_l + off_l, d_{l+1} + off_{l+1}), level 0 from 0, the last band
    to infinity.  Validates as the reference does."""
    ds = [lv.depth_threshold for lv in levels]
    if any(b <= a for a, b in zip(ds, ds[1:])):
        raise ValueError(f"levels must have strictly increasing depth thresholds, got {ds}")
    n = len(levels)
    offs = np.zeros(n) if depth_offsets is None else np.asarray(depth_offsets, float)
    if offs.shape[0] != n:
        raise ValueError("need one depth offset per level")
    return [0.0] + [levels[l].depth_threshold + offs[l] for l in range(1, n)] + [np.inf]


def _band_sets(levels, queries, device=None) -> list:
    """[(position, bounds)] -> per-query per-level ascending int64 index sets
    from the device band kernel (lodge_select_active)."""
    ctx = context(device)
    dev = ctx.device
    dl = [level_for(getattr(lv, "scene", lv), dev, "fp64") for lv in levels]
    arr = (N.Level * len(dl))(*[d.struct for d in dl])
    sizes_n = [int(d.struct.n) for d in dl]
    base = np.concatenate([[0], np.cumsum(sizes_n)]).astype(np.int64)
    pos = torch.tensor(np.asarray([q for q, _ in queries], np.float64).reshape(-1, 3),
                       dtype=torch.float64, device=dev)
    idx = torch.empty(max(int(base[-1]), 1), dtype=torch.int32, device=dev)
    sizes = torch.empty((len(queries), len(dl)), dtype=torch.int32, device=dev)
    lib = N.lib()
    out = []
    for k, (_, bounds) in enumerate(queries):
        b = (C.c_double * (len(dl) + 1))(*[float(v) for v in bounds])
        N.check(lib.lodge_select_active(ctx.bind(), arr, len(dl), b, ptr(pos[k]), ptr(idx),
                                        ptr(sizes[k])), "lodge_select_active")
        sz = sizes[k].cpu().numpy()  # syncs the context stream; idx is reused
        flat = idx.cpu().numpy().view(np.uint32)
        out.append([flat[base[l]:base[l] + sz[l]].astype(np.int64) for l in range(len(dl))])
    return out


def select_active(levels: Sequence, query_point, depth_offsets: Optional[Sequence[float]] = None,
                  device=None) -> list:
    """Drop-in select_active (src/lod.py:192-211): per level, the ascending
    indices whose distance to query_point lies in the level's band, chosen
    by the device band kernel (the one lodge_render_lod runs per frame)."""
    bounds = lod_bounds(levels, depth_offsets)
    return _band_sets(levels, [(np.asarray(query_point, np.float64), bounds)], device)[0]


def build_chunk_active_sets(levels: Sequence, centers, radii, camera_assignment=None,
                            device=None) -> ChunkPlan:
    """Drop-in build_chunk_active_sets (src/chunks.py:122-135): each chunk's
    active sets are the band selection at its centre with every boundary
    above level 0 moved out by its radius."""
    centers = np.asarray(centers, dtype=np.float64)
    radii = np.asarray(radii, dtype=np.float64)
    queries = [(centers[j], lod_bounds(levels, [0.0] + [float(radii[j])] * (len(levels) - 1)))
               for j in range(centers.shape[0])]
    sets = tuple(tuple(s) for s in _band_sets(levels, queries, device))
    assignment = (np.zeros(0, dtype=np.int64) if camera_assignment is None
                  else np.asarray(camera_assignment, dtype=np.int64))
    return ChunkPlan(centers, radii, sets, assignment)


def _frame_to_host(fr, st, raster_cfg) -> TileRenderOutput:
    U = int(st.U)
    return TileRenderOutput(
        None if fr.image is None else fr.image.to(torch.float64).cpu().numpy(),
        fr.tile_count.to(torch.int64).cpu().numpy(),
        fr.visible.to(torch.int64).cpu().numpy(),
        None if fr.maxw is None else fr.maxw[:U].to(torch.float64).cpu().numpy(),
        raster_cfg.metadata() if hasattr(raster_cfg, "metadata") else {})


def _lod_renderer(levels, raster_cfg, device=None):
    from .renderer import Renderer
    dev = _device(device)
    dl = [level_for(getattr(lv, "scene", lv), dev, "fp64") for lv in levels]
    return Renderer(dl, None, dev, raster_cfg=raster_cfg, precision=default_precision())


def render_lod(levels: Sequence, camera, raster_cfg: RasterConfig = RasterConfig(),
               depth_offsets: Optional[Sequence[float]] = None, need_image: bool = True):
    """Select active Gaussians at the camera position and rasterize them
    (src/lod.py:230-237): the Eq. 2 band predicate runs on the device inside
    the fused frame (lodge_render_lod)."""
    bounds = lod_bounds(levels, depth_offsets)
    r = _lod_renderer(levels, raster_cfg)
    fr, st = r.render_lod_camera(camera, bounds, False, need_image, True)
    return _frame_to_host(fr, st, raster_cfg)


def render_full(levels: Sequence, camera, raster_cfg: RasterConfig = RasterConfig(),
                need_image: bool = True):
    """The CLI's "full" mode (src/cli.py:221-226, rendered by _render_mode
    :236-243): every Gaussian of level 0, the other levels empty."""
    r = _lod_renderer(levels, raster_cfg)
    fr, st = r.render_lod_camera(camera, None, True, need_image, True)
    return _frame_to_host(fr, st, raster_cfg)
