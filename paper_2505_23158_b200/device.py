"""Device plumbing: per-GPU liblodge contexts, resident level/plan stores.

PyTorch provides device memory and streams only; every computation of the
render path is a liblodge.so kernel.  Uploads are cached per host object
(by identity, weakly) so repeated compat calls do not re-upload a scene.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import weakref

import numpy as np
import torch

from . import _native as N

_ctx_lock = threading.Lock()
_contexts: dict = {}

PRECISIONS = {"fast": N.PREC_FAST, "exact": N.PREC_EXACT}
_default_precision = os.environ.get("LODGE_PRECISION", "exact")


def set_default_precision(p: str) -> None:
    """Compositing precision of the drop-in API: "exact" (default; fp64,
    the reference's own test tolerances hold) or "fast" (fp32 + fp64 guard
    band; image max-abs <= 1e-3)."""
    global _default_precision
    if p not in PRECISIONS:
        raise ValueError(f"precision must be one of {sorted(PRECISIONS)}")
    _default_precision = p


def default_precision() -> str:
    return _default_precision


def _device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise N.LodgeError("no CUDA device: the LODGE renderer has no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise ValueError("LODGE renders on CUDA devices only")
    return torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())


class Context:
    """One liblodge context per CUDA device (not thread-safe, like the C ABI)."""

    def __init__(self, device: torch.device):
        self.device = device
        self.lib = N.lib()
        ptr = C.c_void_p()
        with torch.cuda.device(device):
            N.check(self.lib.lodge_create(device.index, C.byref(ptr)), "lodge_create")
        self.ptr = ptr
        self._precision = None

    def bind(self, precision: str | None = None):
        """Attach the current torch stream and the precision; returns the raw pointer."""
        s = torch.cuda.current_stream(self.device).cuda_stream
        N.check(self.lib.lodge_set_stream(self.ptr, C.c_void_p(s)), "lodge_set_stream")
        p = precision or _default_precision
        if p != self._precision:
            N.check(self.lib.lodge_set_precision(self.ptr, PRECISIONS[p]), "lodge_set_precision")
            self._precision = p
        return self.ptr


def context(device=None) -> Context:
    d = _device(device)
    with _ctx_lock:
        c = _contexts.get(d.index)
        if c is None:
            c = Context(d)
            _contexts[d.index] = c
    return c


def ptr(t) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())


def camera_struct(cam) -> N.Camera:
    """lodge_camera from any object with the reference Camera's attributes."""
    c = N.Camera()
    R = np.asarray(cam.rotation_matrix, np.float64).reshape(9)
    for i in range(9):
        c.R[i] = float(R[i])
    pos = np.asarray(cam.position, np.float64).reshape(3)
    for i in range(3):
        c.pos[i] = float(pos[i])
    c.fx, c.fy = float(cam.focal[0]), float(cam.focal[1])
    c.cx, c.cy = float(cam.principal_point[0]), float(cam.principal_point[1])
    c.w, c.h = int(cam.resolution[0]), int(cam.resolution[1])
    c.near_plane = float(cam.near_plane)
    return c


CAMERA_BYTES = C.sizeof(N.Camera)


def camera_bytes(cam) -> np.ndarray:
    s = camera_struct(cam)
    return np.frombuffer(C.string_at(C.addressof(s), CAMERA_BYTES), dtype=np.uint8).copy()


def params_struct(cfg) -> N.RasterParams:
    p = N.RasterParams()
    p.alpha_clamp, p.alpha_min = float(cfg.alpha_clamp), float(cfg.alpha_min)
    p.t_min, p.dilation2d = float(cfg.t_min), float(cfg.dilation2d)
    return p


# ---------------------------------------------------------------------------
# resident stores
# ---------------------------------------------------------------------------
class DeviceLevel:
    """One level on the device: AoS geometry (N, 12) + SH (N, 3, terms)."""

    def __init__(self, scene, device: torch.device, storage: str = "fp64"):
        if storage not in ("fp64", "fp32"):
            raise ValueError("storage must be 'fp64' or 'fp32'")
        dt = torch.float64 if storage == "fp64" else torch.float32
        n = len(scene.means)
        deg = int(scene.sh_degree)
        if not 0 <= deg <= 3:
            raise ValueError(f"sh degree must be in 0..3, got {deg}")
        geom = np.empty((n, 12), np.float64)
        geom[:, 0:3] = scene.means
        geom[:, 3:6] = scene.scales
        geom[:, 6:10] = scene.rotations
        geom[:, 10] = scene.opacities
        geom[:, 11] = scene.filter_variance
        self.geom = torch.from_numpy(geom).to(device=device, dtype=dt)
        sh = np.ascontiguousarray(scene.sh_coeffs, np.float64).reshape(n, 3, (deg + 1) ** 2)
        self.sh = torch.from_numpy(sh).to(device=device, dtype=dt)
        self.n = n
        self.degree = deg
        self.flags = 0 if storage == "fp64" else (N.GEOM_FP32 | N.SH_FP32)
        self.struct = self._make_struct()

    @classmethod
    def from_tensors(cls, geom: torch.Tensor, sh: torch.Tensor, degree: int):
        self = cls.__new__(cls)
        self.geom, self.sh = geom.contiguous(), sh.contiguous()
        self.n = int(geom.shape[0])
        self.degree = int(degree)
        self.flags = (N.GEOM_FP32 if geom.dtype == torch.float32 else 0) | (
            N.SH_FP32 if sh.dtype == torch.float32 else 0)
        self.struct = self._make_struct()
        return self

    def _make_struct(self) -> N.Level:
        s = N.Level()
        s.n, s.sh_degree, s.flags = self.n, self.degree, self.flags
        s.geom_dev = self.geom.data_ptr() if self.n else None
        s.sh_dev = self.sh.data_ptr() if self.n else None
        return s

    def nbytes(self) -> int:
        return self.geom.numel() * self.geom.element_size() + self.sh.numel() * self.sh.element_size()


_uid_lock = threading.Lock()
_uid = [0]


def _next_uid() -> int:
    """Process-unique plan identity (lodge_chunks.uid): never reused, so a
    context's union reuse can never mistake a new plan at a recycled address
    for the one it cached."""
    with _uid_lock:
        _uid[0] += 1
        return (os.getpid() << 32) | _uid[0]


class DevicePlan:
    """Chunk centres and all K*L sorted uint32 index sets, resident."""

    def __init__(self, plan, device: torch.device):
        K = plan.centers.shape[0]
        L = len(plan.active_sets[0])
        if L > N.MAX_LEVELS:
            raise ValueError(f"at most {N.MAX_LEVELS} levels are supported")
        sizes = np.array([[len(plan.active_sets[j][l]) for l in range(L)] for j in range(K)],
                         np.int64)
        offsets = np.zeros(K * L + 1, np.int64)
        offsets[1:] = np.cumsum(sizes.reshape(-1))
        data = np.empty(int(offsets[-1]), np.uint32)
        for j in range(K):
            for l in range(L):
                s = np.asarray(plan.active_sets[j][l])
                if s.size and (s.min() < 0 or s.max() >= 2 ** 32):
                    raise ValueError("active-set indices must fit in uint32")
                data[offsets[j * L + l]:offsets[j * L + l + 1]] = s
        self.K, self.L = K, L
        self.centers = torch.from_numpy(np.ascontiguousarray(plan.centers, np.float64)).to(device)
        self.offsets = torch.from_numpy(offsets).to(device)
        self.data = torch.from_numpy(data.view(np.int32)).to(device)
        self.max_set = sizes.max(axis=0)
        self.struct = N.Chunks()
        self.struct.uid = _next_uid()
        self.struct.K, self.struct.L = K, L
        self.struct.centers_dev = self.centers.data_ptr()
        self.struct.offsets_dev = self.offsets.data_ptr()
        self.struct.data_dev = self.data.data_ptr() if data.size else self.offsets.data_ptr()
        for l in range(L):
            self.struct.max_set[l] = int(self.max_set[l])

    @classmethod
    def from_arrays(cls, centers, offsets, data, L: int, device: torch.device):
        """From flat arrays: centers (K,3) fp64, offsets (K*L+1) int64, data uint32
        with set (j, l) = data[offsets[j*L+l]:offsets[j*L+l+1]] (sorted)."""
        self = cls.__new__(cls)
        centers = np.ascontiguousarray(centers, np.float64)
        self.K, self.L = centers.shape[0], int(L)
        self.centers = torch.from_numpy(centers).to(device)
        self.offsets = torch.from_numpy(np.ascontiguousarray(offsets, np.int64)).to(device)
        data = np.ascontiguousarray(data, np.uint32)
        self.data = torch.from_numpy(data.view(np.int32)).to(device)
        self.max_set = np.diff(np.asarray(offsets)).reshape(self.K, self.L).max(axis=0)
        self.struct = N.Chunks()
        self.struct.uid = _next_uid()
        self.struct.K, self.struct.L = self.K, self.L
        self.struct.centers_dev = self.centers.data_ptr()
        self.struct.offsets_dev = self.offsets.data_ptr()
        self.struct.data_dev = self.data.data_ptr() if data.size else self.offsets.data_ptr()
        for l in range(self.L):
            self.struct.max_set[l] = int(self.max_set[l])
        return self

    @classmethod
    def from_tensor(cls, centers, offsets, data: torch.Tensor, L: int, device: torch.device):
        """Like from_arrays, with the concatenated sets already a device
        int32 tensor (the uint32 bit patterns), e.g. gathered by load_asset."""
        self = cls.__new__(cls)
        centers = np.ascontiguousarray(centers, np.float64)
        offsets = np.ascontiguousarray(offsets, np.int64)
        self.K, self.L = centers.shape[0], int(L)
        self.centers = torch.from_numpy(centers).to(device)
        self.offsets = torch.from_numpy(offsets).to(device)
        self.data = data
        self.max_set = np.diff(offsets).reshape(self.K, self.L).max(axis=0)
        self.struct = N.Chunks()
        self.struct.uid = _next_uid()
        self.struct.K, self.struct.L = self.K, self.L
        self.struct.centers_dev = self.centers.data_ptr()
        self.struct.offsets_dev = self.offsets.data_ptr()
        self.struct.data_dev = self.data.data_ptr()
        for l in range(self.L):
            self.struct.max_set[l] = int(self.max_set[l])
        return self

    @property
    def union_capacity(self) -> int:
        return int(2 * self.max_set.sum())


class _IdCache:
    """Per-object upload cache keyed by identity (reference dataclasses are
    unhashable), dropped when the host object is collected."""

    def __init__(self, maxlen=16):
        self._d = {}
        self._maxlen = maxlen

    def get(self, obj, key, make):
        k = (id(obj), key)
        hit = self._d.get(k)
        if hit is not None and hit[0]() is obj:
            return hit[1]
        val = make()
        try:
            ref = weakref.ref(obj, lambda _r, k=k: self._d.pop(k, None))
        except TypeError:
            return val
        if len(self._d) >= self._maxlen:
            self._d.pop(next(iter(self._d)))
        self._d[k] = (ref, val)
        return val


_levels = _IdCache()
_plans = _IdCache()


def level_for(scene, device=None, storage="fp64") -> DeviceLevel:
    d = _device(device)
    return _levels.get(scene, (d.index, storage), lambda: DeviceLevel(scene, d, storage))


def plan_for(plan, device=None) -> DevicePlan:
    d = _device(device)
    return _plans.get(plan, d.index, lambda: DevicePlan(plan, d))


class SlabStore:
    """Chunk-slab layout of a resident store (B200 capacity for bandwidth):
    for every chunk j and level l, the records of the set (j, l) copied
    contiguously in set order, so a frame's gather (the union of two sets,
    in index order) reads two streams instead of isolated 48-B records
    scattered over the level -- each Gaussian is stored once per chunk whose
    set holds it (config 3: 3.3x the level store, 25 GB of 180 GB).

    The plan's slab tables (lodge_chunks.slab_geom_dev / slab_sh_dev) point
    lodge_render_frame at the slabs: the union then emits each element's
    position in its owning chunk's set (tags 3/1 primary, 2 other) and the
    projection and payload kernels read that slab -- the values are the
    level store's, so frames are bit-identical to the flat store
    (tests/test_gpu_streaming.py).  Built on the device by an index gather
    from the resident levels (a one-time layout transform at load)."""

    def __init__(self, levels, plan: "DevicePlan"):
        dev = plan.centers.device
        K, L = plan.K, plan.L
        offs = plan.offsets.cpu().numpy()
        data = plan.data.view(torch.int32)
        self.geom, self.sh = [], []
        geom_rows, sh_rows = np.zeros(K * L, np.int64), np.zeros(K * L, np.int64)
        for l, lv in enumerate(levels):
            # positions of level l's sets inside the plan's data, chunk-major
            spans = [(int(offs[j * L + l]), int(offs[j * L + l + 1])) for j in range(K)]
            idx = torch.cat([data[a:b] for a, b in spans]).to(torch.int64) & 0xffffffff
            g = lv.geom.index_select(0, idx).contiguous()
            s = lv.sh.index_select(0, idx).contiguous()
            self.geom.append(g)
            self.sh.append(s)
            start = 0
            for j, (a, b) in enumerate(spans):
                geom_rows[j * L + l] = g.data_ptr() + start * g.shape[1] * g.element_size()
                sh_rows[j * L + l] = s.data_ptr() + start * s[0].numel() * s.element_size()
                start += b - a
        self.geom_tab = torch.from_numpy(geom_rows).to(dev)
        self.sh_tab = torch.from_numpy(sh_rows).to(dev)
        self.levels = levels

    def attach(self, plan: "DevicePlan") -> "DevicePlan":
        plan.struct.slab_geom_dev = self.geom_tab.data_ptr()
        plan.struct.slab_sh_dev = self.sh_tab.data_ptr()
        plan.struct.uid = _next_uid()  # slab unions hold set positions, not indices
        plan._slabs = self  # keep the slabs alive with the plan
        return plan

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.geom + self.sh)
