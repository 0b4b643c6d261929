"""The C-ABI library loads and exports every symbol include/lodge.h declares
(CPU only: dlopen, no compute calls)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lodge.h")
LIB = os.path.join(ROOT, "paper_2505_23158_b200", "liblodge.so")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^[a-z_][\w \*]*?\b(lodge_\w+)\(", src, re.M)))


def test_header_declares_entry_points():
    names = declared()
    for must in ("lodge_create", "lodge_destroy", "lodge_last_error", "lodge_select",
                 "lodge_compose", "lodge_project", "lodge_rasterize", "lodge_render_frame"):
        assert must in names


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        pytest.skip("liblodge.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_2505_23158_b200 import _native
    assert set(declared()) == set(_native.EXPORTS)


def test_error_string_without_gpu():
    if not os.path.exists(LIB):
        pytest.skip("liblodge.so not built")
    lib = ctypes.CDLL(LIB)
    lib.lodge_last_error.restype = ctypes.c_char_p
    assert isinstance(lib.lodge_last_error(), bytes)
