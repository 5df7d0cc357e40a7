"""The C-ABI library loads without a GPU and exports every declared symbol."""

import ctypes
import os
import re

from paper_2412_15126_b200 import _lib

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "slotrank_b200.h")


def declared():
    text = open(HDR).read()
    return sorted(set(re.findall(r"\b(srk_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared()
    assert "srk_rotate" in names and "srk_keyswitch" in names and len(names) >= 25


def test_library_exports_every_symbol():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2412_15126_b200 import build

        build.build()
    handle = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared() if not hasattr(handle, n)]
    assert not missing, missing
    assert set(declared()) == set(_lib.EXPORTS)
    lib = _lib.lib()
    assert lib.srk_version() == 1


def test_errors_are_reported_not_aborted():
    lib = _lib.lib()
    ctx = ctypes.c_void_p()
    arr = (ctypes.c_uint64 * 2)(3, 5)
    rc = lib.srk_ctx_create(0, 4, arr, arr, 1, 1, 1, ctypes.byref(ctx))
    assert rc != 0 and b"log_n" in lib.srk_last_error()
