"""CPU checks of the C-ABI library: it loads without a GPU and exports every
symbol include/fouroversix.h declares (no compute calls here)."""

import ctypes
import os
import re

from paper_2512_02010_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "fouroversix.h")).read()
    return sorted(set(re.findall(r"\b(f46_[a-z0-9_]+)\s*\(", src)))


def test_header_and_binding_agree():
    assert sorted(_lib.EXPORTS) == header_symbols()


def test_library_exports_every_header_symbol():
    L = ctypes.CDLL(_lib.LIB_PATH)
    for sym in header_symbols():
        assert hasattr(L, sym), sym


def test_size_helpers_match_python():
    L = _lib.load()
    from paper_2512_02010_b200.blockquant import scales_tc_bytes
    for rows, cols in [(1, 16), (5, 7), (128, 64), (129, 4160), (65536, 4096), (3, 1856)]:
        assert L.f46_scales_tc_bytes(rows, cols) == scales_tc_bytes(rows, cols)
        assert L.f46_codes_bytes(rows, cols) == rows * (-(-cols // 16)) * 8
    assert b"sm_100a" in L.f46_build_info()
