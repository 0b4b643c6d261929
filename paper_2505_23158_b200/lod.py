"""Drop-in project_selection (reference src/lod.py:216-227)."""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from .device import context
from .raster import DeviceBatch, project_scene_device
from .types import RasterConfig


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
