"""Importance scoring on the device: the LOD build's and
the chunk visibility filter's inner loop.

score_active_selection (reference src/lod.py:95-122) renders every view --
the given ones plus `perturb.count` orientation-resampled copies of each --
with shade=False, need_image=False, record_max_weight=True over the
concatenation of the per-level sets, and keeps the per-input max blend weight
over all views.  Here the sets become a one-chunk plan, every view is one
lodge_render_frame of the fused path (chunk pair = (0, none): the union of a
single chunk is its own sets with modulation 1, i.e. the reference's
concatenation in level-major order), and LODGE_ACCUMULATE_MAX makes the
compositor's global atomicMax reduce over views in HBM: no per-view host
round trip, one read-back at the end.

compute_importance (src/lod.py:125-131) and visibility_filter_chunk
(src/chunks.py:141-160) are the reference's two callers.
"""

from __future__ import annotations

import warnings
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .device import DevicePlan, _device, default_precision, level_for
from .renderer import STATS_BYTES, Renderer
from .types import ImportanceScores, PerturbSpec, RasterConfig


def random_rotations(rng: np.random.Generator, n: int) -> np.ndarray:
    """Uniform random unit quaternions (w, x, y, z), Shoemake's method; draws
    from `rng` exactly as the reference (src/synthetic.py:17-22)."""
    u1, u2, u3 = rng.random(n), rng.random(n), rng.random(n)
    a, b = np.sqrt(1.0 - u1), np.sqrt(u1)
    return np.stack([a * np.sin(2 * np.pi * u2), a * np.cos(2 * np.pi * u2),
                     b * np.sin(2 * np.pi * u3), b * np.cos(2 * np.pi * u3)], axis=1)


def scoring_views(views: Sequence, perturb: Optional[PerturbSpec]) -> list:
    """The given views, then per view `perturb.count` copies with orientations
    from random_rotations(default_rng(perturb.seed)) (src/lod.py:103-110)."""
    all_views = list(views)
    if perturb is not None and perturb.count > 0:
        rng = np.random.default_rng(perturb.seed)
        quats = random_rotations(rng, perturb.count * len(views))
        for vi, view in enumerate(views):
            for k in range(perturb.count):
                all_views.append(view.replaced_orientation(quats[vi * perturb.count + k]))
    return all_views


def _check_sets(sets) -> list:
    out = []
    for s in sets:
        a = np.asarray(s, dtype=np.int64).reshape(-1)
        if a.size and (a.min() < 0 or a.max() >= 2 ** 32):
            raise ValueError("active-set indices must be in [0, 2^32)")
        if a.size > 1 and not np.all(a[1:] > a[:-1]):
            # the device union consumes sorted unique sets, which is what the
            # reference's producers (np.arange, select_active) hand over
            raise ValueError("active sets must be sorted and unique")
        out.append(a)
    return out


def score_active_selection(levels: Sequence, sets: Sequence, views: Sequence,
                           raster_cfg: RasterConfig = RasterConfig(),
                           perturb: Optional[PerturbSpec] = None, precision: str | None = None,
                           device=None, n_streams: int = 2) -> list:
    """Max blending weight per selected Gaussian over all views, rendered
    jointly across levels (src/lod.py:95-122).  Returns one fp64 score array
    per level, aligned with `sets`.  precision "exact" reproduces the
    reference's weights (fp64 compositing); "fast" is fp32 with the
    reference's skip decisions."""
    if not views:
        raise ValueError("importance scoring needs at least one view")
    if len(sets) != len(levels):
        raise ValueError("one active set per level is required")
    all_views = scoring_views(views, perturb)
    sets = _check_sets(sets)
    dev = _device(device)
    prec = precision or default_precision()
    sizes = np.array([a.size for a in sets], np.int64)
    offsets = np.zeros(len(sets) + 1, np.int64)
    offsets[1:] = np.cumsum(sizes)
    U = int(offsets[-1])
    if U == 0:
        return [np.zeros(0) for _ in sets]
    data = np.concatenate(sets).astype(np.uint32) if U else np.zeros(0, np.uint32)
    plan = DevicePlan.from_arrays(np.zeros((1, 3)), offsets, data, len(sets), dev)
    storage = "fp64"
    dlevels = [level_for(getattr(lv, "scene", lv), dev, storage) for lv in levels]
    r = Renderer(dlevels, plan, dev, storage=storage, precision=prec, raster_cfg=raster_cfg,
                 n_streams=n_streams)
    fdt = torch.float64 if prec == "exact" else torch.float32
    maxw = torch.zeros(max(r.U_cap, 1), dtype=fdt, device=dev)
    cams = r.upload_cameras(all_views)
    frames = {}
    stats = torch.zeros((len(all_views), STATS_BYTES), dtype=torch.uint8, device=dev)

    def frame_for(view, slot):
        w, h = (int(v) for v in view.resolution)
        key = (w, h, slot)
        if key not in frames:
            fr = r.alloc_frame(w, h, need_image=False, record_max=False)
            fr.maxw = maxw  # every view maxes into the same buffer
            frames[key] = fr
        return frames[key]

    def render(idx_list):
        cur = torch.cuda.current_stream(dev)
        ev = torch.cuda.Event()
        ev.record(cur)
        for q in range(r.n_streams):
            r.stream_of(q).wait_event(ev)
        for k, i in enumerate(idx_list):
            slot = k % r.n_streams
            fr = frame_for(all_views[i], slot)
            r.render(cams[i], fr, pair=(0, None), need_image=False, record_max=True, slot=slot,
                     accumulate_max=True)
            with torch.cuda.stream(r.stream_of(slot)):
                stats[i].copy_(fr.stats)
        for q in range(r.n_streams):
            cur.wait_stream(r.stream_of(q))
        torch.cuda.synchronize(dev)

    def read(idx):
        raw = stats.cpu().numpy()
        return {i: N.FrameStats.from_buffer_copy(raw[i].tobytes()) for i in idx}

    # an overflowing frame composites nothing and max is idempotent, so a
    # view whose pairs did not fit is simply rendered again with room
    todo = list(range(len(all_views)))
    for batch in (todo[:1], todo[1:]):  # the first view sizes the pair buffers
        while batch:
            render(batch)
            st = read(batch)
            bad = [i for i in batch if st[i].fault]
            if bad:  # a skipped write would leave the scores too low
                raise RuntimeError("liblodge: device bounds check fired while scoring "
                                   f"(views {bad[:8]}, fault bits {st[bad[0]].fault:#x})")
            redo = [i for i in batch if st[i].overflow]
            if redo:
                r.reserve(int(max(st[i].P for i in redo) * 1.25) + 4096)
            batch = redo
    scores = maxw[:U].double().cpu().numpy()
    return [scores[offsets[l]:offsets[l + 1]].copy() for l in range(len(sets))]


def compute_importance(level, views: Sequence, cfg, perturb: Optional[PerturbSpec] = None,
                       precision: str | None = None, device=None) -> ImportanceScores:
    """Per-Gaussian importance: max alpha-blend contribution over all views
    (src/lod.py:125-131)."""
    n = len(level) if hasattr(level, "__len__") else len(getattr(level, "scene", level).means)
    sets = [np.arange(n, dtype=np.int64)]
    scores = score_active_selection([level], sets, views, cfg.raster, perturb, precision,
                                    device)[0]
    return ImportanceScores(scores, cfg.gamma)


def visibility_filter_chunk(plan, chunk_id: int, levels: Sequence, cameras_in_chunk: Sequence,
                            cfg, raster_cfg: RasterConfig = RasterConfig(),
                            precision: str | None = None, device=None) -> tuple:
    """Importance-prune one chunk's active sets under its own cameras plus
    orientation-perturbed copies; returns the reduced per-level sets
    (src/chunks.py:141-160)."""
    sets = plan.active_sets[chunk_id]
    if not cameras_in_chunk:
        warnings.warn(f"chunk {chunk_id} has no assigned cameras; skipping "
                      "visibility filtering", stacklevel=2)
        return sets
    perturb = PerturbSpec(count=cfg.perturb_count, seed=cfg.perturb_seed + chunk_id,
                          law=cfg.perturb_law)
    scores = score_active_selection(levels, sets, list(cameras_in_chunk), raster_cfg, perturb,
                                    precision, device)
    return tuple(np.asarray(s)[sc >= cfg.vis_threshold] for s, sc in zip(sets, scores))
