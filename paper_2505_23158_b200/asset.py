"""Asset loader -> device store.

load_asset reads the reference's asset format (a directory with
manifest.json + data.bin, or a SPLATLOD container; reference
src/assets.py:291-355) straight into the render store on the GPU: the data
section is copied host->device once (pinned staging), every level blob is
split on the device into the fp32 geometry store (n x 12) and SH store
(n x 3 x T) with the value checks of _parse_level_blob
(src/assets.py:257-282) evaluated by the same kernel (lodge_asset_split),
and the chunk plan's index sets are gathered into a DevicePlan and checked
for order and range on the device (lodge_asset_check_sets).  Rotations are
stored raw and normalised in fp64 at projection time (LODGE_GEOM_QNORM),
which reproduces read_asset's load-time normalisation bit for bit.

Restated host code: the manifest, range and count checks below follow
read_asset (reference src/assets.py:358-472) in order and message text --
the AssetError messages are part of the drop-in contract.

The manifest, range and count checks are host logic in read_asset's order
and raise AssetError with its messages (src/assets.py:358-472); the
value and index-set checks raise the same messages from the device results.
"""

from __future__ import annotations

import ctypes as C
import json
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import _native as N
from .device import DeviceLevel, DevicePlan, _device, context

FORMAT_VERSION = 1
CONTAINER_MAGIC = b"SPLATLOD"

_VALUE_CHECKS = [  # (violation bit, message), in _parse_level_blob's order
    (1, "level blob contains non-finite values"),
    (2, "level blob contains non-positive scales"),
    (4, "level blob contains out-of-range opacity"),
    (8, "level blob contains negative filter variance"),
    (16, "level blob contains non-unit rotations"),
]


class AssetError(Exception):
    """Malformed asset (reference src/assets.py:38)."""


@dataclass
class DeviceAsset:
    """A compiled scene resident on the GPU: the render store (one
    DeviceLevel per LOD level, LODGE_GEOM_QNORM set) and the chunk plan, plus
    the host-side metadata read_asset returns (src/assets.py:225-235)."""

    levels: list
    plan: DevicePlan
    sh_degree: int
    reference_focal: float
    filter_scale: float
    gamma: float
    depth_thresholds: list
    provenance: list
    centers: np.ndarray
    radii: np.ndarray
    camera_assignment: np.ndarray
    manifest: dict = field(repr=False, default_factory=dict)

    @property
    def n_levels(self) -> int:
        return len(self.levels)


def _read_bytes(path: Path):
    try:
        if path.is_dir():
            return (path / "manifest.json").read_bytes(), (path / "data.bin").read_bytes()
        raw = path.read_bytes()
        if len(raw) < len(CONTAINER_MAGIC) + 12:
            raise AssetError(f"{path}: container too short")
        if raw[:len(CONTAINER_MAGIC)] != CONTAINER_MAGIC:
            raise AssetError(f"{path}: bad container magic")
        version, mlen = struct.unpack_from("<IQ", raw, len(CONTAINER_MAGIC))
        if version != FORMAT_VERSION:
            raise AssetError(f"{path}: unsupported container version {version}")
        start = len(CONTAINER_MAGIC) + 12
        if start + mlen > len(raw):
            raise AssetError(f"{path}: truncated manifest")
        return raw[start:start + mlen], raw[start + mlen:]
    except OSError as e:
        raise AssetError(f"cannot read asset at {path}: {e}") from e


def _validate_ranges(manifest: dict, data_len: int) -> None:
    ranges = []
    for row in manifest["levels"]:
        ranges.append((row["offset"], row["length"]))
        ranges.append((row["provenance_offset"], row["provenance_length"]))
    for chunk in manifest["chunks"]:
        for s in chunk["index_sets"]:
            ranges.append((s["offset"], s["length"]))
    for off, length in ranges:
        if off < 0 or length < 0 or off + length > data_len:
            raise AssetError(f"blob range [{off}, {off + length}) exceeds data "
                             f"section of {data_len} bytes")
    for (o1, l1), (o2, l2) in zip(sorted(ranges), sorted(ranges)[1:]):
        if o1 + l1 > o2:
            raise AssetError(f"overlapping blob ranges at offset {o2}")


def _upload(data: bytes, dev: torch.device) -> torch.Tensor:
    host = torch.frombuffer(bytearray(data), dtype=torch.uint8) if data else torch.zeros(0, dtype=torch.uint8)
    if dev.type == "cuda" and host.numel():
        host = host.pin_memory()
    return host.to(dev, non_blocking=True)


def load_asset(path, device=None) -> DeviceAsset:
    """read_asset (src/assets.py:374-472) into the device render store."""
    path = Path(path)
    mbytes, data = _read_bytes(path)
    try:
        manifest = json.loads(mbytes.decode("utf-8"))
    except (json.JSONDecodeError, UnicodeDecodeError) as e:
        raise AssetError(f"{path}: manifest is not valid JSON: {e}") from e
    try:
        return _load(path, manifest, data, device)
    except AssetError:
        raise
    except (KeyError, TypeError, ValueError, IndexError, struct.error) as e:
        raise AssetError(f"{path}: malformed asset: {e}") from e


def _load(path: Path, manifest: dict, data: bytes, device) -> DeviceAsset:
    if manifest["format_version"] != FORMAT_VERSION:
        raise AssetError(f"unsupported format_version {manifest['format_version']}")
    sh_degree = int(manifest["sh_degree"])
    if not 0 <= sh_degree <= 3:
        raise AssetError(f"sh_degree {sh_degree} out of range")
    _validate_ranges(manifest, len(data))
    terms = (sh_degree + 1) ** 2
    rec = 4 * (12 + 3 * terms)
    dev = _device(device)
    ctx = context(dev)
    lib = N.lib()
    blob = _upload(data, dev)  # the whole data section, one copy
    levels, thresholds, provenance = [], [], []
    for row in manifest["levels"]:
        count = int(row["gaussian_count"])
        if count * rec != row["length"]:
            raise AssetError(f"level {row['level']}: count {count} disagrees "
                             f"with blob length {row['length']}")
        if count * 4 != row["provenance_length"]:
            raise AssetError(f"level {row['level']}: provenance length mismatch")
        geom = torch.empty((count, 12), dtype=torch.float32, device=dev)
        sh = torch.empty((count, 3, terms), dtype=torch.float32, device=dev)
        bad = C.c_int32(0)
        if count:
            if row["offset"] % 4:
                raise AssetError(f"level {row['level']}: blob offset is not 4-byte aligned")
            N.check(lib.lodge_asset_split(ctx.bind(), C.c_void_p(blob.data_ptr() + row["offset"]),
                                          count, sh_degree, C.c_void_p(geom.data_ptr()),
                                          C.c_void_p(sh.data_ptr()), C.byref(bad)),
                    "lodge_asset_split")
        for bit, msg in _VALUE_CHECKS:
            if bad.value & bit:
                raise AssetError(msg)
        lvl = DeviceLevel.from_tensors(geom, sh, sh_degree)
        lvl.flags |= N.GEOM_QNORM
        lvl.struct = lvl._make_struct()
        levels.append(lvl)
        thresholds.append(float(row["depth_threshold"]))
        off = row["provenance_offset"]
        provenance.append(np.frombuffer(data[off:off + row["provenance_length"]],
                                        dtype="<u4").astype(np.int64))
    if not levels:
        raise AssetError("asset has no levels")
    n0 = levels[0].n
    for row, prov in zip(manifest["levels"], provenance):
        if prov.size and (prov.min() < 0 or prov.max() >= n0):
            raise AssetError(f"level {row['level']}: provenance index out of range")

    L = len(levels)
    chunks = manifest["chunks"]
    centers, radii = [], []
    offsets = [0]
    pieces = []
    for j, chunk in enumerate(chunks):
        if len(chunk["index_sets"]) != L:
            raise AssetError(f"chunk {j}: expected {L} index sets")
        for srow in chunk["index_sets"]:
            n_words = int(srow["length"]) // 4
            pieces.append((int(srow["offset"]), n_words))
            offsets.append(offsets[-1] + n_words)
        centers.append(chunk["center"])
        radii.append(chunk["radius"])
    if not chunks:
        raise AssetError("asset has no chunks")
    # gather the sets out of the uploaded data section (device copies)
    total = offsets[-1]
    flat = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    for (off, n_words), start in zip(pieces, offsets[:-1]):
        if n_words:
            flat[start:start + n_words] = blob[off:off + 4 * n_words].view(torch.int32)
    plan = DevicePlan.from_tensor(np.asarray(centers, np.float64), np.asarray(offsets, np.int64),
                                  flat, L, dev)
    sizes = (C.c_int64 * L)(*[lv.n for lv in levels])
    flags = (C.c_int32 * max(len(chunks) * L, 1))()
    N.check(lib.lodge_asset_check_sets(ctx.bind(), C.byref(plan.struct), sizes, flags),
            "lodge_asset_check_sets")
    for j, chunk in enumerate(chunks):
        for lvl, srow in enumerate(chunk["index_sets"]):
            if srow["count"] * 4 != srow["length"]:
                raise AssetError(f"chunk {j} level {lvl}: count disagrees with length")
            f = flags[j * L + lvl]
            if f & 1:
                raise AssetError(f"chunk {j} level {lvl}: index set not strictly sorted")
            if f & 2:
                raise AssetError(f"chunk {j} level {lvl}: index out of range")
    assignment = np.asarray(manifest.get("camera_assignment", []), dtype=np.int64)
    if assignment.size and (assignment.min() < 0 or assignment.max() >= len(chunks)):
        raise AssetError("camera assignment references unknown chunk")
    torch.cuda.synchronize(dev)
    return DeviceAsset(levels, plan, sh_degree, float(manifest["reference_focal"]),
                       float(manifest["filter_scale"]), float(manifest["gamma"]), thresholds,
                       provenance, np.asarray(centers, float), np.asarray(radii, float),
                       assignment, manifest)
