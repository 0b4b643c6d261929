"""ctypes binding of liblodge.so (include/lodge.h).

The library is built in-tree (``paper_2505_23158_b200/liblodge.so``) by
``__graft_entry__.build()``.  There is no fallback: if the library or a CUDA
device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# LODGE_LIB=name loads a diagnostic build liblodge_<name>.so (csrc/Makefile
# VARIANT=name, e.g. the LODGE_VERIFY order checks of the stress test)
_VARIANT = os.environ.get("LODGE_LIB", "")
LIB_PATH = os.path.join(_HERE, f"liblodge_{_VARIANT}.so" if _VARIANT else "liblodge.so")
CSRC = os.path.join(_HERE, "csrc")

MAX_LEVELS = 8
GEOM_FP32 = 1
SH_FP32 = 2
GEOM_QNORM = 4
PREC_FAST = 0
PREC_EXACT = 1
NEED_IMAGE = 1
RECORD_MAX = 2
ACCUMULATE_MAX = 4
FULL_LISTS = 8

ERR = {-1: "BAD_ARG", -2: "CUDA", -3: "OOM", -4: "CAPACITY"}


class LodgeError(RuntimeError):
    pass


class Camera(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("pos", C.c_double * 3), ("fx", C.c_double),
                ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("w", C.c_int32), ("h", C.c_int32), ("near_plane", C.c_double)]


class RasterParams(C.Structure):
    _fields_ = [("alpha_clamp", C.c_double), ("alpha_min", C.c_double),
                ("t_min", C.c_double), ("dilation2d", C.c_double)]


class Level(C.Structure):
    _fields_ = [("n", C.c_int64), ("sh_degree", C.c_int32), ("flags", C.c_int32),
                ("geom_dev", C.c_void_p), ("sh_dev", C.c_void_p)]


class Chunks(C.Structure):
    _fields_ = [("K", C.c_int32), ("L", C.c_int32), ("centers_dev", C.c_void_p),
                ("offsets_dev", C.c_void_p), ("data_dev", C.c_void_p),
                ("max_set", C.c_int64 * MAX_LEVELS), ("slab_geom_dev", C.c_void_p),
                ("slab_sh_dev", C.c_void_p), ("uid", C.c_uint64)]


class FrameOut(C.Structure):
    _fields_ = [("image_dev", C.c_void_p), ("tile_count_dev", C.c_void_p),
                ("visible_dev", C.c_void_p), ("maxw_dev", C.c_void_p),
                ("srgb8_dev", C.c_void_p)]


class FrameStats(C.Structure):
    _fields_ = [("f", C.c_int32), ("o", C.c_int32), ("t_bar", C.c_double), ("t", C.c_double),
                ("U", C.c_uint32), ("U_level", C.c_uint32 * MAX_LEVELS), ("M", C.c_uint32),
                ("P", C.c_uint32), ("overflow", C.c_uint32), ("guard_hits", C.c_uint32),
                ("P_first", C.c_uint32), ("P_second", C.c_uint32), ("fault", C.c_uint32),
                ("M_first", C.c_uint32), ("M_second", C.c_uint32),
                ("comp_members", C.c_uint32), ("block_lists", C.c_uint32),
                ("sorted_first", C.c_uint32)]


class Batch(C.Structure):
    _fields_ = [("src_dev", C.c_void_p), ("mean2d_dev", C.c_void_p),
                ("cov2d_dev", C.c_void_p), ("conic_dev", C.c_void_p),
                ("extent_dev", C.c_void_p), ("depth_dev", C.c_void_p),
                ("opacity_dev", C.c_void_p), ("color_dev", C.c_void_p)]


EXPORTS = {
    "lodge_create": ([C.c_int32, C.POINTER(C.c_void_p)], C.c_int),
    "lodge_set_phase_budget": ([C.c_void_p, C.c_int32], C.c_int),
    "lodge_set_block_lists": ([C.c_void_p, C.c_int32], C.c_int),
    "lodge_set_grid_share": ([C.c_void_p, C.c_int32], C.c_int),
    "lodge_fault_flags": ([C.c_void_p, C.POINTER(C.c_uint32)], C.c_int),
    "lodge_destroy": ([C.c_void_p], None),
    "lodge_last_error": ([], C.c_char_p),
    "lodge_set_stream": ([C.c_void_p, C.c_void_p], C.c_int),
    "lodge_reserve": ([C.c_void_p, C.c_int64, C.c_int64], C.c_int),
    "lodge_set_precision": ([C.c_void_p, C.c_int32], C.c_int),
    "lodge_select": ([C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p,
                      C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "lodge_blend_factor": ([C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p], C.c_int),
    "lodge_compose": ([C.c_void_p, C.POINTER(Chunks), C.c_int32, C.c_int32,
                       C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_int64)],
                      C.c_int),
    "lodge_project": ([C.c_void_p, C.POINTER(Level), C.c_void_p, C.c_int64, C.c_void_p,
                       C.POINTER(Camera), C.POINTER(RasterParams), C.c_int32, C.POINTER(Batch),
                       C.POINTER(C.c_int64)], C.c_int),
    "lodge_rasterize": ([C.c_void_p, C.POINTER(Batch), C.c_int64, C.c_int64, C.POINTER(Camera),
                         C.POINTER(RasterParams), C.c_int32, C.POINTER(FrameOut), C.c_void_p,
                         C.c_void_p, C.c_int64, C.POINTER(FrameStats)], C.c_int),
    "lodge_render_frame": ([C.c_void_p, C.POINTER(Level), C.c_int32, C.POINTER(Chunks),
                            C.c_void_p, C.c_int32, C.c_int32, C.POINTER(RasterParams),
                            C.POINTER(C.c_int32), C.POINTER(C.c_double), C.c_int32,
                            C.POINTER(FrameOut), C.c_void_p], C.c_int),
    "lodge_frame_lists": ([C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64], C.c_int),
    "lodge_frame_union": ([C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64], C.c_int),
    "lodge_profile": ([C.c_void_p, C.c_int32, C.c_int32], C.c_int),
    "lodge_profile_read": ([C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int32)], C.c_int),
    "lodge_to_srgb8": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p], C.c_int),
    "lodge_last_launch_count": ([C.c_void_p], C.c_int32),
    "lodge_debug_counters": ([C.c_void_p, C.POINTER(C.c_uint64)], C.c_int),
    "lodge_frame_report": ([C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_double), C.c_int32,
                            C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_int64, C.c_void_p],
                           C.c_int),
    "lodge_sq_err": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p], C.c_int),
    "lodge_debug_depth_sort": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p,
                                C.c_void_p], C.c_int),
    "lodge_render_lod": ([C.c_void_p, C.POINTER(Level), C.c_int32, C.POINTER(C.c_double),
                          C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.POINTER(RasterParams),
                          C.c_int32, C.POINTER(FrameOut), C.c_void_p], C.c_int),
    "lodge_select_active": ([C.c_void_p, C.POINTER(Level), C.c_int32, C.POINTER(C.c_double),
                             C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "lodge_cover_table": ([C.c_void_p, C.POINTER(Level), C.c_void_p, C.c_int64,
                           C.POINTER(Camera), C.POINTER(RasterParams), C.c_void_p, C.c_void_p,
                           C.POINTER(C.c_int64)], C.c_int),
    "lodge_asset_split": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_void_p,
                           C.POINTER(C.c_int32)], C.c_int),
    "lodge_asset_check_sets": ([C.c_void_p, C.POINTER(Chunks), C.POINTER(C.c_int64),
                                C.POINTER(C.c_int32)], C.c_int),
}
N_STAGES = 10
STAGES = ("select", "union", "project", "depth_sort", "tile_setup", "duplicate", "tile_sort",
          "composite", "second_phase", "composite_b")

_lib = None
_lock = threading.Lock()


# diagnostic variants built next to the product library: name -> nvcc defines
VARIANTS = {
    "verify": "-DLODGE_VERIFY",
}


def build(verbose: bool = False, variants: bool = True) -> str:
    """Compile liblodge.so (and the diagnostic variants) for sm_100a in place
    (make -C csrc)."""
    jobs = [[]]
    if variants:
        jobs += [[f"VARIANT={k}", f"EXTRA={v}"] for k, v in VARIANTS.items()]
    for extra in jobs:
        out = subprocess.run(["make", "-j4", "-C", CSRC] + extra, capture_output=True, text=True)
        if out.returncode != 0:
            raise LodgeError("liblodge build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])
        if verbose:
            print(out.stdout[-2000:])
    return LIB_PATH


def lib():
    """Load liblodge.so; raises LodgeError if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LodgeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                                 "(there is no CPU fallback)")
            L = C.CDLL(LIB_PATH)
            for name, (args, res) in EXPORTS.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = res
            _lib = L
    return _lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = lib().lodge_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(msg)
        raise LodgeError(f"{what}: {ERR.get(rc, rc)}: {msg}")
