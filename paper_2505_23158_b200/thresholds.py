"""Threshold-search cost evaluation on the device.

The searcher's cost of a threshold set is a band sum over per-(level, view)
distance-sorted prefix tables of per-splat tile cover counts (reference
src/thresholds.py:56-111).  Building those tables is the expensive part:
project_scene(shade=False), tile_cover_counts, the camera distances, a
stable argsort and a cumulative sum.  lodge_cover_table does all of it on
the GPU in one call (a fused projection + cover + distance kernel compacted
in batch order, the onesweep sort stable over that order, a scan); the band
sums stay two binary searches per band on the host, as in the reference.

ThresholdSearcher mirrors the reference class with device tables.
Restated host code: apart from `_table` (the device tables) and
`evaluate_cost`, the class follows reference src/thresholds.py:51-120 near
verbatim -- the band sums, caching and CostEvaluation fields must come out
identical for the reference's greedy_search to accept it.  The
provisional levels come from a level builder (the reference's own
`splatlod.lod.build_level`; the LOD build is outside this package's scope),
and the reference's greedy_search accepts the searcher as is:

    searcher = ThresholdSearcher(base, views, cfg, level_builder=build_level)
    greedy_search(base, views, cfg, grid, max_levels, searcher=searcher)
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .device import _device, camera_struct, context, level_for, params_struct
from .types import TILE_SIZE, RasterConfig


@dataclass(frozen=True)
class CostEvaluation:
    """Reference src/thresholds.py:27-38."""

    thresholds: tuple
    mean_gaussians_per_tile: float
    per_view_cost: tuple
    views_used: tuple
    build_cost_proxy: int  # total Gaussians across levels (reported, not optimized)

    def __post_init__(self):
        ds = self.thresholds
        if any(b <= a for a, b in zip(ds, ds[1:])):
            raise ValueError(f"thresholds must be strictly increasing, got {ds}")


def cover_table(level, view, raster_cfg: RasterConfig = RasterConfig(), device=None,
                indices=None):
    """(distances sorted ascending, prefix) of ThresholdSearcher._table
    (src/thresholds.py:80-90) for one level (a LodLevel / Scene, or a
    DeviceLevel) and one camera: prefix = [0, cumsum(cover[order])]."""
    from .device import DeviceLevel
    dev = _device(device)
    if isinstance(level, DeviceLevel):
        dl = level
    else:
        dl = level_for(getattr(level, "scene", level), dev, "fp64")
    idx = None
    n = dl.n
    if indices is not None:
        idx = torch.as_tensor(np.ascontiguousarray(indices, np.int64), device=dev)
        n = int(idx.numel())
    dist = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    prefix = torch.empty(n + 1, dtype=torch.int64, device=dev)
    m = C.c_int64()
    ctx = context(dev)
    cam = camera_struct(view)
    rp = params_struct(raster_cfg)
    N.check(N.lib().lodge_cover_table(ctx.bind(), C.byref(dl.struct),
                                      C.c_void_p(idx.data_ptr()) if idx is not None else None,
                                      n, C.byref(cam), C.byref(rp), C.c_void_p(dist.data_ptr()),
                                      C.c_void_p(prefix.data_ptr()), C.byref(m)),
            "lodge_cover_table")
    M = m.value
    return dist[:M].cpu().numpy(), prefix[:M + 1].cpu().numpy()


class ThresholdSearcher:
    """Memoizing cost evaluator over one base level, view set and config
    (src/thresholds.py:52-111) whose (level, view) tables are built on the
    GPU.  level_builder(base, depth, cfg, single_round=True,
    subsample_views=...) -> (LodLevel, report) supplies the provisional
    levels (e.g. splatlod.lod.build_level)."""

    def __init__(self, base, views: Sequence, cfg, subsample_views: bool = True,
                 level_builder: Optional[Callable] = None, device=None):
        if not views:
            raise ValueError("cost evaluation needs at least one view")
        self.base = base
        self.views = list(views)
        self.cfg = cfg
        self.subsample_views = subsample_views
        self.level_builder = level_builder
        self.device = device
        self._levels = {0.0: base}
        self._tables = {}
        self._tiles_per_view = [(-(-int(v.resolution[0]) // TILE_SIZE)) *
                                (-(-int(v.resolution[1]) // TILE_SIZE)) for v in self.views]

    def provisional_level(self, depth: float):
        """Filter + single prune round at gamma (the reference's proxy)."""
        d = float(depth)
        if d not in self._levels:
            if self.level_builder is None:
                raise ValueError("provisional levels need a level_builder "
                                 "(e.g. splatlod.lod.build_level)")
            level, _ = self.level_builder(self.base, d, self.cfg, single_round=True,
                                          subsample_views=self.subsample_views)
            self._levels[d] = level
        return self._levels[d]

    def _table(self, depth: float, view_idx: int):
        key = (float(depth), view_idx)
        if key not in self._tables:
            level = self.provisional_level(depth)
            self._tables[key] = cover_table(level, self.views[view_idx], self.cfg.raster,
                                            self.device)
        return self._tables[key]

    def _band_count(self, depth: float, view_idx: int, lo: float, hi: float) -> int:
        dist, prefix = self._table(depth, view_idx)
        i0 = np.searchsorted(dist, lo, side="left")
        i1 = dist.shape[0] if hi == np.inf else np.searchsorted(dist, hi, side="left")
        return int(prefix[i1] - prefix[i0])

    def evaluate(self, thresholds: Sequence[float]) -> CostEvaluation:
        ds = [float(d) for d in thresholds]
        if any(d <= 0 for d in ds) or any(b <= a for a, b in zip(ds, ds[1:])):
            raise ValueError(f"thresholds must be strictly increasing and > 0, got {ds}")
        bounds = [0.0] + ds + [np.inf]
        depths = [0.0] + ds
        per_view = []
        for vi in range(len(self.views)):
            binned = sum(self._band_count(depths[l], vi, bounds[l], bounds[l + 1])
                         for l in range(len(depths)))
            per_view.append(binned / self._tiles_per_view[vi])
        build_proxy = sum(len(self.provisional_level(d)) for d in depths)
        return CostEvaluation(tuple(ds), float(np.mean(per_view)), tuple(per_view),
                              tuple(getattr(v, "cam_id", "") or str(i)
                                    for i, v in enumerate(self.views)), build_proxy)


def evaluate_cost(base, thresholds: Sequence[float], views: Sequence, cfg,
                  searcher: Optional[ThresholdSearcher] = None,
                  level_builder: Optional[Callable] = None) -> CostEvaluation:
    """Mean per-tile binned count under the given depth thresholds
    (src/thresholds.py:114-120)."""
    if searcher is None:
        searcher = ThresholdSearcher(base, views, cfg, level_builder=level_builder)
    return searcher.evaluate(thresholds)
