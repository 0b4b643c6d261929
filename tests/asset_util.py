"""Deterministic corruptions of an asset directory (the reference's format,
src/assets.py:291-355), shared by oracle/make_golden.py (which records the
reference's read_asset message for each) and the asset tests."""

import json
import os
import shutil
import struct

import numpy as np

MAGIC = b"SPLATLOD"


def _load(src):
    m = json.loads(open(os.path.join(src, "manifest.json"), "rb").read().decode())
    data = bytearray(open(os.path.join(src, "data.bin"), "rb").read())
    return m, data


def _write_dir(dst, m, data, mbytes=None):
    os.makedirs(dst, exist_ok=True)
    if mbytes is None:
        mbytes = json.dumps(m, sort_keys=True, separators=(",", ":")).encode()
    open(os.path.join(dst, "manifest.json"), "wb").write(mbytes)
    open(os.path.join(dst, "data.bin"), "wb").write(bytes(data))
    return dst


def container_bytes(m, data, version=1):
    mbytes = json.dumps(m, sort_keys=True, separators=(",", ":")).encode()
    return MAGIC + struct.pack("<IQ", version, len(mbytes)) + mbytes + bytes(data)


def corrupt(src, dst, kind, args):
    """Copy of asset directory `src` at `dst` with one corruption; returns
    the path to read (a directory, or a container file for container kinds)."""
    m, data = _load(src)
    deg = int(m["sh_degree"])
    width = 12 + 3 * (deg + 1) ** 2
    if kind == "f32":
        lv, rec, c, val = args
        row = m["levels"][int(lv[1:])]
        v = float(val) if not isinstance(val, str) else float(val)
        struct.pack_into("<f", data, row["offset"] + (rec * width + c) * 4, v)
    elif kind == "u32swap":
        j, l, k = args
        s = m["chunks"][j]["index_sets"][l]
        a = np.frombuffer(bytes(data[s["offset"]:s["offset"] + s["length"]]), "<u4").copy()
        a[k], a[k + 1] = a[k + 1], a[k]
        data[s["offset"]:s["offset"] + s["length"]] = a.tobytes()
    elif kind == "u32set":
        j, l, k, val = args
        s = m["chunks"][j]["index_sets"][l]
        a = np.frombuffer(bytes(data[s["offset"]:s["offset"] + s["length"]]), "<u4").copy()
        a[k] = val
        data[s["offset"]:s["offset"] + s["length"]] = a.tobytes()
    elif kind == "manifest":
        key, val = args
        m[key] = val
    elif kind == "level_field":
        i, field, val = args
        m["levels"][i][field] = val
    elif kind == "set_field":
        j, l, field, val = args
        m["chunks"][j]["index_sets"][l][field] = val
    elif kind == "drop_set":
        (j,) = args
        m["chunks"][j]["index_sets"].pop()
    elif kind == "manifest_bytes":
        (raw,) = args
        return _write_dir(dst, m, data, mbytes=raw)
    elif kind in ("container", "container_magic", "container_version", "container_truncate"):
        raw = container_bytes(m, data, version=args[0] if kind == "container_version" else 1)
        if kind == "container_magic":
            raw = b"NOTLODGE" + raw[len(MAGIC):]
        if kind == "container_truncate":
            raw = raw[:args[0]]
        os.makedirs(os.path.dirname(dst) or ".", exist_ok=True)
        path = dst.rstrip("/") + ".splatlod"
        open(path, "wb").write(raw)
        return path
    else:
        raise ValueError(kind)
    return _write_dir(dst, m, data)


def clean(dst):
    shutil.rmtree(dst, ignore_errors=True)
    if os.path.exists(dst.rstrip("/") + ".splatlod"):
        os.remove(dst.rstrip("/") + ".splatlod")
