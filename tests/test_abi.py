"""The C-ABI library loads and exports every symbol include/hjb200.h declares
(no compute call: this runs on the CPU-only driver container)."""
import ctypes
import os
import re

import pytest

from paper_2411_03501_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "hjb200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hj_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_bound_symbols():
    assert sorted(_lib.EXPORTED_SYMBOLS) == header_functions()


def test_library_exports_every_declared_symbol():
    if not os.path.exists(_lib.library_path()):
        pytest.skip("libhjb200.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(_lib.library_path())
    for name in header_functions():
        assert hasattr(lib, name), name
    typed = _lib.load()
    assert typed.hj_version() == 1


def test_struct_layouts_match_header():
    # offsets of the C structs (x86-64 natural alignment) as declared in include/hjb200.h
    assert ctypes.sizeof(_lib.HjGrid) == 216
    assert _lib.HjGrid.nodes.offset == 152
    assert ctypes.sizeof(_lib.HjHam) == 8 + 128 + 32
    assert ctypes.sizeof(_lib.HjStats) == 88


def test_key_decoding_round_trip():
    import struct

    for x in (0.0, -0.0, 1.5, -1.5, 1e-300, -1e300, float("inf"), float("-inf")):
        k = struct.unpack("<q", struct.pack("<d", x))[0]
        if k < 0:
            k ^= 0x7FFFFFFFFFFFFFFF
        assert struct.pack("<d", _lib.decode_key(k)) == struct.pack("<d", x)
