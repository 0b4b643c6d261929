"""Device-resident per-frame renderer: the fused hot path.

A Renderer owns the level store and chunk plan on one GPU and renders camera
views end to end with lodge_render_frame: chunk selection -> union +
modulation -> projection -> depth sort -> binning -> tile sort ->
compositing, with no host synchronisation inside a frame.  Outputs stay in
HBM (image, per_tile_count, per_pixel_visible, per_gaussian_max_weight) until
the caller reads them.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _native as N
from .device import (CAMERA_BYTES, Context, DeviceLevel, DevicePlan, camera_bytes, context,
                     params_struct, ptr)
from .types import TILE_SIZE, RasterConfig

STATS_BYTES = C.sizeof(N.FrameStats)
# the reference CLI's default --histogram-bins (src/cli.py)
DEFAULT_HISTOGRAM_EDGES = (0, 1, 2, 4, 8, 16, 32, 64, 128, 256)


@dataclass
class Frame:
    """Device outputs of one view (reference TileRenderOutput fields)."""

    width: int
    height: int
    image: Optional[torch.Tensor]        # (H, W, 3) fp32 (fast) / fp64 (exact)
    tile_count: torch.Tensor             # (tiles_y, tiles_x) int32
    visible: torch.Tensor                # (H, W) int32
    maxw: Optional[torch.Tensor]         # (U_cap,) fp32 / fp64; first stats.U valid
    stats: torch.Tensor                  # lodge_frame_stats bytes

    def read_stats(self) -> N.FrameStats:
        raw = self.stats.cpu().numpy().tobytes()
        return N.FrameStats.from_buffer_copy(raw)


BLOCK_LIST_MODES = {"auto": 0, "off": 1, "force": 2}  # lodge.h LODGE_BLOCK_LISTS_*


class Renderer:
    """n_streams > 1 keeps that many frames in flight: each slot owns a
    liblodge context (workspace + frame state) and a CUDA stream, so the
    latency-bound stages of one frame overlap the bandwidth-bound stages of
    another.  render(..., slot=k) enqueues on slot k's stream.

    FAST frames composite in two depth phases (lodge_set_phase_budget:
    phase_budget first-phase pairs per tile, 0 = one pass); full_lists=True
    keeps one pass so the sorted per-tile lists stay inspectable
    (lodge_frame_lists).  block_lists ("auto", "off", "force";
    lodge_set_block_lists) chooses how a phase of few large splats builds
    its lists.  grid_share (lodge_set_grid_share; default 1 CTA per SM with
    several slots, 0 = the single-frame grids otherwise) caps the
    projection's persistent grids so frames in flight share the SMs.  The
    outputs are the same either way."""

    def __init__(self, levels: Sequence, plan, device=None, storage: str = "fp32",
                 precision: str = "fast", raster_cfg: RasterConfig = RasterConfig(),
                 n_streams: int = 1, full_lists: bool = False, phase_budget: int = 1536,
                 block_lists: str = "auto", grid_share: int = None):
        self.ctx = context(device)
        self.device = self.ctx.device
        if n_streams < 1:
            raise ValueError("n_streams must be >= 1")
        self._slots = [(self.ctx, None)]
        for _ in range(n_streams - 1):
            self._slots.append((Context(self.device), torch.cuda.Stream(self.device)))
        if n_streams > 1:  # slot 0 gets its own stream too
            self._slots[0] = (self.ctx, torch.cuda.Stream(self.device))
        self.levels = []
        for lv in levels:
            if isinstance(lv, DeviceLevel):
                self.levels.append(lv)
            else:
                self.levels.append(DeviceLevel(getattr(lv, "scene", lv), self.device, storage))
        # plan=None: LOD / full modes only (render_lod)
        self.plan = (plan if (plan is None or isinstance(plan, DevicePlan))
                     else DevicePlan(plan, self.device))
        if self.plan is not None and self.plan.L != len(self.levels):
            raise ValueError("chunk plan and level list disagree on the level count")
        self._level_arr = (N.Level * len(self.levels))(*[l.struct for l in self.levels])
        self.precision = precision
        self.full_lists = bool(full_lists)
        if phase_budget < 0:
            raise ValueError("phase_budget must be >= 0")
        self.phase_budget = int(phase_budget)
        if block_lists not in BLOCK_LIST_MODES:
            raise ValueError("block_lists must be 'auto', 'off' or 'force'")
        self.block_lists = BLOCK_LIST_MODES[block_lists]
        # frames in flight: the projection's persistent grids leave room on
        # every SM for the other slots' kernels (lodge_set_grid_share)
        if grid_share is None:
            grid_share = 1 if n_streams > 1 else 0
        if grid_share < 0:
            raise ValueError("grid_share must be >= 0")
        self.grid_share = int(grid_share)
        self.cfg = raster_cfg
        self._rp = params_struct(raster_cfg)
        lod_cap = sum(l.n for l in self.levels)
        self.U_cap = max(self.plan.union_capacity, lod_cap) if self.plan is not None else lod_cap

    # ------------------------------------------------------------------
    @property
    def n_streams(self) -> int:
        return len(self._slots)

    def stream_of(self, slot: int = 0):
        """torch stream of a slot (the current stream for a single-slot renderer)."""
        s = self._slots[slot][1]
        return s if s is not None else torch.cuda.current_stream(self.device)

    def _bind(self, slot: int):
        ctx, s = self._slots[slot]
        if s is None:
            p = ctx.bind(self.precision)
        else:
            with torch.cuda.stream(s):
                p = ctx.bind(self.precision)
        N.check(N.lib().lodge_set_phase_budget(p, self.phase_budget), "lodge_set_phase_budget")
        N.check(N.lib().lodge_set_block_lists(p, self.block_lists), "lodge_set_block_lists")
        N.check(N.lib().lodge_set_grid_share(p, self.grid_share), "lodge_set_grid_share")
        return p

    def reserve(self, max_pairs: int):
        for k in range(self.n_streams):
            N.check(N.lib().lodge_reserve(self._bind(k), self.U_cap, int(max_pairs)),
                    "lodge_reserve")

    def profile(self, enable: bool, max_frames: int = 0):
        for ctx, _ in self._slots:
            N.check(N.lib().lodge_profile(ctx.ptr, int(enable), int(max_frames)), "lodge_profile")

    def profile_read(self):
        """Summed per-stage milliseconds and frame count over all slots."""
        tot = np.zeros(N.N_STAGES)
        frames = 0
        for ctx, _ in self._slots:
            ms = (C.c_double * N.N_STAGES)()
            n = C.c_int32()
            N.check(N.lib().lodge_profile_read(ctx.ptr, ms, C.byref(n)), "lodge_profile_read")
            tot += np.array(ms[:])
            frames += n.value
        return tot, frames

    def alloc_frame(self, width: int, height: int, need_image=True, record_max=True) -> Frame:
        tx, ty = -(-width // TILE_SIZE), -(-height // TILE_SIZE)
        fdt = torch.float64 if self.precision == "exact" else torch.float32
        d = self.device
        fr = Frame(width, height,
                   torch.empty((height, width, 3), dtype=fdt, device=d) if need_image else None,
                   torch.empty((ty, tx), dtype=torch.int32, device=d),
                   torch.empty((height, width), dtype=torch.int32, device=d),
                   # zeroed: a frame clears only the entries its own slot
                   # layout can write, which may be fewer than U_cap
                   torch.zeros(max(self.U_cap, 1), dtype=fdt, device=d) if record_max else None,
                   torch.zeros(STATS_BYTES, dtype=torch.uint8, device=d))
        self._publish()  # the fills land before any slot stream renders into it
        return fr

    def _publish(self):
        """Make every slot stream wait for the work enqueued so far on the
        current stream (a camera upload, a frame's allocation fill)."""
        if self.n_streams == 1 and self._slots[0][1] is None:
            return
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        for _, st in self._slots:
            if st is not None:
                st.wait_event(ev)

    def upload_cameras(self, cameras) -> torch.Tensor:
        """(V, sizeof(lodge_camera)) uint8 device tensor of camera structs,
        visible to every slot stream."""
        host = np.stack([camera_bytes(c) for c in cameras])
        out = torch.from_numpy(host).to(self.device)
        self._publish()
        return out

    def render(self, cam_row: torch.Tensor, frame: Frame, pair=None, t: float = None,
               need_image: bool = True, record_max: bool = True, slot: int = 0,
               accumulate_max: bool = False, srgb8_out: torch.Tensor = None,
               float_image: bool = True) -> Frame:
        """Enqueue one frame on slot `slot`'s stream (the current stream for a
        single-slot renderer).  cam_row: one row of upload_cameras().
        pair=None: nearest two chunks chosen on device.  accumulate_max: max
        this frame's per-input weights into frame.maxw instead of resetting it
        (a device-side max over views, src/lod.py:95-131).  srgb8_out: a
        (h, w, 3) uint8 tensor the compositor fills with the 8-bit sRGB image
        as it finishes each tile (FAST; byte for byte to_srgb8 of the float
        image, which float_image=False then skips writing) -- on the device,
        or in pinned host memory (zero-copy: the image reaches the host as
        the compositor writes it, in 16-byte row segments when the width is
        a multiple of 16)."""
        out = N.FrameOut()
        out.image_dev = (frame.image.data_ptr()
                         if (need_image and float_image and frame.image is not None) else None)
        if srgb8_out is not None:
            if (srgb8_out.dtype != torch.uint8 or not srgb8_out.is_contiguous()
                    or srgb8_out.numel() != 3 * frame.width * frame.height):
                raise ValueError("srgb8_out must be a contiguous uint8 (h, w, 3) tensor")
            if not (srgb8_out.is_cuda or srgb8_out.is_pinned()):
                raise ValueError("srgb8_out must be a device tensor or pinned host memory")
            out.srgb8_dev = srgb8_out.data_ptr()
        out.tile_count_dev = frame.tile_count.data_ptr()
        out.visible_dev = frame.visible.data_ptr()
        out.maxw_dev = frame.maxw.data_ptr() if (record_max and frame.maxw is not None) else None
        flags = ((N.NEED_IMAGE if need_image else 0) | (N.RECORD_MAX if record_max else 0) |
                 (N.FULL_LISTS if self.full_lists else 0))
        if accumulate_max:
            flags |= N.ACCUMULATE_MAX
        pr = None
        tv = None
        if pair is not None:
            f, o = pair
            pr = (C.c_int32 * 2)(int(f), -1 if o is None else int(o))
            tv = C.c_double(1.0 if t is None else float(t))
        N.check(N.lib().lodge_render_frame(
            self._bind(slot), self._level_arr, len(self.levels), C.byref(self.plan.struct),
            ptr(cam_row), frame.width, frame.height, C.byref(self._rp), pr,
            None if tv is None else C.byref(tv), flags, C.byref(out), ptr(frame.stats)),
            "lodge_render_frame")
        return frame

    def render_lod(self, cam_row: torch.Tensor, frame: Frame, bounds=None, full: bool = False,
                   need_image: bool = True, record_max: bool = True, slot: int = 0,
                   accumulate_max: bool = False) -> Frame:
        """Enqueue one LOD-mode frame (level l keeps the Gaussians with
        bounds[l] <= camera distance < bounds[l+1], src/lod.py:192-237) or,
        with full=True, a full-mode frame (all of level 0, src/cli.py:221-226)
        on slot `slot`'s stream."""
        if not full:
            if bounds is None or len(bounds) != len(self.levels) + 1:
                raise ValueError("need one distance bound per level plus one")
            b = (C.c_double * len(bounds))(*[float(x) for x in bounds])
        else:
            b = None
        need = self.levels[0].n if full else sum(l.n for l in self.levels)
        if record_max and frame.maxw is not None and frame.maxw.numel() < need:
            raise ValueError("frame.maxw holds fewer entries than the inputs this mode selects")
        out = N.FrameOut()
        out.image_dev = frame.image.data_ptr() if (need_image and frame.image is not None) else None
        out.tile_count_dev = frame.tile_count.data_ptr()
        out.visible_dev = frame.visible.data_ptr()
        out.maxw_dev = frame.maxw.data_ptr() if (record_max and frame.maxw is not None) else None
        flags = ((N.NEED_IMAGE if need_image else 0) | (N.RECORD_MAX if record_max else 0) |
                 (N.ACCUMULATE_MAX if accumulate_max else 0) |
                 (N.FULL_LISTS if self.full_lists else 0))
        N.check(N.lib().lodge_render_lod(
            self._bind(slot), self._level_arr, len(self.levels), b, int(bool(full)),
            ptr(cam_row), frame.width, frame.height, C.byref(self._rp), flags, C.byref(out),
            ptr(frame.stats)), "lodge_render_lod")
        return frame

    def render_lod_camera(self, camera, bounds=None, full=False, need_image=True,
                          record_max=True):
        """Convenience: one host camera -> device frame + stats (grows the
        pair buffers and renders again on overflow)."""
        w, h = (int(v) for v in camera.resolution)
        fr = self.alloc_frame(w, h, need_image, record_max)
        cams = self.upload_cameras([camera])
        self.render_lod(cams[0], fr, bounds, full, need_image, record_max)
        st = fr.read_stats()
        if st.overflow:
            self.reserve(int(st.P))
            self.render_lod(cams[0], fr, bounds, full, need_image, record_max)
            st = fr.read_stats()
        if st.fault:
            raise RuntimeError(f"liblodge: device bounds check fired (fault bits {st.fault:#x})")
        return fr, st

    def to_srgb8(self, frame: Frame, out: torch.Tensor, slot: int = 0) -> torch.Tensor:
        """8-bit sRGB of the frame's image on the device (src/images.py:10-17)."""
        if frame.image is None or frame.image.dtype != torch.float32:
            raise ValueError("to_srgb8 needs a FAST-precision frame with an image")
        N.check(N.lib().lodge_to_srgb8(self._bind(slot), ptr(frame.image),
                                       frame.width * frame.height, ptr(out)), "lodge_to_srgb8")
        return out

    def report(self, frame: Frame, stats=None, bin_edges=None, full_frame: Frame = None):
        """The reference bench's per-frame report fields (src/cli.py:283-320),
        computed on the device (csrc/k_report.cu): visibility_histogram,
        mean_per_tile, visible_gaussians (nonzero max weights),
        resident_gaussians (the chunk pair's union size: ChunkPlan.
        resident_count, src/scene.py:266-272, is sum over levels of
        |union1d(A_l, B_l)| = U), chunk_pair, and psnr_vs_full when the
        full-mode frame of the same view is given."""
        from .raster import frame_report_device, squared_error_device
        torch.cuda.synchronize(self.device)  # the frame may come from any slot stream
        st = stats if stats is not None else frame.read_stats()
        edges = DEFAULT_HISTOGRAM_EDGES if bin_edges is None else bin_edges
        hist, tsum, vis = frame_report_device(frame.visible, frame.tile_count, frame.maxw,
                                              st.U, edges, ctx=self.ctx)
        rep = {"mean_per_tile": tsum / frame.tile_count.numel(), "visible_gaussians": vis,
               "resident_gaussians": int(st.U), "visibility_histogram": hist.tolist(),
               "chunk_pair": ([int(st.f), None if st.o < 0 else int(st.o)]
                              if st.f >= 0 else None)}
        if full_frame is not None:
            if frame.image is None or full_frame.image is None:
                raise ValueError("psnr_vs_full needs both images")
            sq = squared_error_device(frame.image, full_frame.image, ctx=self.ctx)
            mse = sq / frame.image.numel()
            rep["psnr_vs_full"] = float("inf") if mse == 0 else -10.0 * float(np.log10(mse))
        return rep

    def fault_flags(self) -> int:
        """OR over every frame of every slot of the device bounds-check bits
        (0 = no check ever fired); synchronises the slots."""
        f = 0
        for ctx, _ in self._slots:
            v = C.c_uint32()
            N.check(N.lib().lodge_fault_flags(ctx.ptr, C.byref(v)), "lodge_fault_flags")
            f |= v.value
        return f

    def last_launch_count(self) -> int:
        return int(N.lib().lodge_last_launch_count(self.ctx.ptr))

    def render_camera(self, camera, need_image=True, record_max=True, pair=None, t=None):
        """Convenience: one host camera -> host outputs (image fp64, counts int64)."""
        w, h = (int(v) for v in camera.resolution)
        fr = self.alloc_frame(w, h, need_image, record_max)
        cams = self.upload_cameras([camera])
        self.render(cams[0], fr, pair=pair, t=t, need_image=need_image, record_max=record_max)
        st = fr.read_stats()
        if st.overflow:
            self.reserve(int(st.P))
            self.render(cams[0], fr, pair=pair, t=t, need_image=need_image, record_max=record_max)
            st = fr.read_stats()
        if st.fault:
            raise RuntimeError(f"liblodge: device bounds check fired (fault bits {st.fault:#x})")
        return fr, st
