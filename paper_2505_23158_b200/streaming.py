"""Residency-bounded device store with asynchronous chunk loads (SURVEY.md
8f rank 4; the paper's background reload, reference src/blending.py:140-194).

The full LOD store stays in host memory; the GPU holds only a few chunk
slabs.  A slab is one chunk's Gaussians -- for each level, the records of
its index set in set order (geometry n x 12, then SH n x 3T, fp32), laid out
contiguously and pinned on the host once.  `require(chunks)` makes chunks
resident: a missing chunk is copied host->device on a dedicated copy stream
into a free slot (least recently used, and only after every frame that read
that slot has completed), followed by an update of the per-(chunk, level)
pointer tables that lodge_render_frame reads in slab mode
(lodge_chunks.slab_geom_dev / slab_sh_dev).  The render stream waits on the
slot's copy event, so a frame never reads a slab before it has landed, and
the copies of the next chunk overlap the frames of the current ones.

In slab mode the union emits each element's position in its owning chunk's
set (tags 3/1: the primary chunk, 2: the other), and the projection reads
the record from that chunk's slab: the same values as the full store, so
frames are bit-identical to fully resident ones.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .device import DeviceLevel, DevicePlan


def host_pair(centers, position):
    """(f, o, t) of nearest_two_chunks + blend_factor (src/blending.py:77-99)
    on the host, which must decide residency before the frame is enqueued:
    lexsort by (distance, id); t = clip(dot(c - o, f - o) / dot(f - o, f - o))."""
    centers = np.asarray(centers, np.float64)
    c = np.asarray(position, np.float64)
    dist = np.linalg.norm(centers - c, axis=1)
    order = np.lexsort((np.arange(dist.shape[0]), dist))
    f = int(order[0])
    if centers.shape[0] == 1:
        return f, None, 1.0
    o = int(order[1])
    fo = centers[f] - centers[o]
    d2 = float(np.dot(fo, fo))
    if d2 <= 0:
        raise ValueError("blend_factor needs distinct chunk centers")
    t_bar = float(np.dot(c - centers[o], fo)) / d2
    return f, o, min(1.0, max(0.0, t_bar))


class StreamingStore:
    def __init__(self, levels, centers, offsets, data, device, n_slots: int = 3,
                 level_flags: int = 0):
        """levels: [(geom (n,12) fp32, sh (n,3,T) fp32)] host arrays; the plan
        as centers (K,3), offsets (K*L+1), data (uint32 sets).  level_flags:
        extra lodge_level flags of every level (LODGE_GEOM_QNORM for an
        asset's raw rotations, normalised at projection as read_asset does)."""
        self.level_flags = int(level_flags)
        if n_slots < 2:
            raise ValueError("a blended frame needs two resident chunks")
        self.device = torch.device(device)
        self.L = len(levels)
        self.K = np.asarray(centers).shape[0]
        offsets = np.asarray(offsets, np.int64)
        data = np.asarray(data, np.uint32)
        self.terms3 = [int(np.prod(sh.shape[1:])) for _, sh in levels]
        self.degree = int(round((levels[0][1].shape[2]) ** 0.5)) - 1
        self.level_n = [g.shape[0] for g, _ in levels]
        # host slabs (pinned) and the byte offsets of each level's parts
        self.slabs, self.parts = [], []
        for j in range(self.K):
            chunks, parts, off = [], [], 0
            for l, (g, sh) in enumerate(levels):
                s = data[offsets[j * self.L + l]:offsets[j * self.L + l + 1]].astype(np.int64)
                gb = np.ascontiguousarray(g[s], np.float32).view(np.uint8).reshape(-1)
                sb = np.ascontiguousarray(sh[s].reshape(len(s), -1), np.float32).view(np.uint8)
                sb = sb.reshape(-1)
                parts.append((off, off + gb.size))
                off += gb.size + sb.size
                off = (off + 255) // 256 * 256  # 256-byte aligned parts
                chunks += [gb, sb]
            slab = torch.empty(max(off, 1), dtype=torch.uint8).pin_memory()
            sv = slab.numpy()
            for (go, so), (gb, sb) in zip(parts, zip(chunks[0::2], chunks[1::2])):
                sv[go:go + gb.size] = gb
                sv[so:so + sb.size] = sb
            self.slabs.append(slab)
            self.parts.append(parts)
        self.slot_bytes = max(s.numel() for s in self.slabs)
        self.slots = [torch.empty(self.slot_bytes, dtype=torch.uint8, device=self.device)
                      for _ in range(n_slots)]
        self.slot_chunk = [-1] * n_slots
        self.slot_ready = [None] * n_slots      # copy-stream event: slab landed
        self.slot_free = [dict() for _ in range(n_slots)]  # render stream -> last reader done
        self.slot_tick = [0] * n_slots
        self.tick = 0
        self.where = {}                          # chunk -> slot
        self.copy_stream = torch.cuda.Stream(self.device)
        self.geom_tab = torch.zeros(self.K * self.L, dtype=torch.int64, device=self.device)
        self.sh_tab = torch.zeros(self.K * self.L, dtype=torch.int64, device=self.device)
        # the table rows of (chunk, slot), pinned once, so table updates are
        # plain async copies whose sources never change
        self._rows = {}
        for j in range(self.K):
            for k in range(n_slots):
                base = self.slots[k].data_ptr()
                g = torch.tensor([base + go for go, _ in self.parts[j]], dtype=torch.int64)
                sh = torch.tensor([base + so for _, so in self.parts[j]], dtype=torch.int64)
                self._rows[(j, k)] = (g.pin_memory(), sh.pin_memory())
        self.loads = 0
        self.bytes_loaded = 0

    # ------------------------------------------------------------------
    def device_levels(self):
        """Level descriptors for the Renderer: sizes, degree and fp32 flags,
        no resident store (geom_dev / sh_dev NULL)."""
        out = []
        for n in self.level_n:
            lv = DeviceLevel.__new__(DeviceLevel)
            lv.geom = lv.sh = None
            lv.n, lv.degree = n, self.degree
            lv.flags = N.GEOM_FP32 | N.SH_FP32 | self.level_flags
            s = N.Level()
            s.n, s.sh_degree, s.flags = n, self.degree, lv.flags
            s.geom_dev = None
            s.sh_dev = None
            lv.struct = s
            out.append(lv)
        return out

    def attach(self, plan: DevicePlan) -> DevicePlan:
        """Point a DevicePlan at the slab tables (slab mode)."""
        from .device import _next_uid
        plan.struct.uid = _next_uid()  # slab unions hold set positions, not indices
        plan.struct.slab_geom_dev = self.geom_tab.data_ptr()
        plan.struct.slab_sh_dev = self.sh_tab.data_ptr()
        return plan

    def resident_bytes(self) -> int:
        return len(self.slots) * self.slot_bytes

    def require(self, chunks, stream=None):
        """Make `chunks` resident and make `stream` (the render stream) wait
        until their slabs have landed."""
        stream = stream or torch.cuda.current_stream(self.device)
        need = [int(j) for j in chunks if j is not None and j >= 0]
        for j in need:
            self.tick += 1
            if j in self.where:
                self.slot_tick[self.where[j]] = self.tick
                continue
            cand = [k for k in range(len(self.slots)) if self.slot_chunk[k] not in need]
            k = min(cand, key=lambda s: self.slot_tick[s])
            old = self.slot_chunk[k]
            if old >= 0:
                del self.where[old]
            cs = self.copy_stream
            for ev_free in self.slot_free[k].values():
                cs.wait_event(ev_free)  # frames still reading the old slab
            self.slot_free[k] = {}
            with torch.cuda.stream(cs):
                src = self.slabs[j]
                self.slots[k][:src.numel()].copy_(src, non_blocking=True)
                g, sh = self._rows[(j, k)]
                self.geom_tab[j * self.L:(j + 1) * self.L].copy_(g, non_blocking=True)
                self.sh_tab[j * self.L:(j + 1) * self.L].copy_(sh, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
            self.slot_ready[k] = ev
            self.slot_chunk[k] = j
            self.slot_tick[k] = self.tick
            self.where[j] = k
            self.loads += 1
            self.bytes_loaded += src.numel()
        for j in need:
            stream.wait_event(self.slot_ready[self.where[j]])

    def release(self, chunks, stream=None):
        """Record that the frames enqueued so far on `stream` read `chunks`."""
        stream = stream or torch.cuda.current_stream(self.device)
        for j in chunks:
            if j is None or j < 0 or j not in self.where:
                continue
            ev = torch.cuda.Event()
            ev.record(stream)
            self.slot_free[self.where[j]][stream.cuda_stream] = ev
