"""The C-ABI library loads and exports every symbol include/relserve.h declares."""

import re
from pathlib import Path

from paper_2601_11546_b200 import _abi, _native

HEADER = Path(__file__).resolve().parents[1] / "include" / "relserve.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w ]+\*?\s*\**(rs_\w+)\(", text, re.M)))


def test_header_declares_expected_symbols():
    assert set(declared()) == set(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    L = _native.lib()
    for name in declared():
        assert hasattr(L, name), name
    assert b"sm_100a" in L.rs_build_info()


def test_record_layout_matches_header():
    import ctypes

    assert ctypes.sizeof(_abi.IterRecord) == _abi.ITER_RECORD_DTYPE.itemsize == 96
    assert ctypes.sizeof(_abi.Pcg64State) == 40
    assert ctypes.sizeof(_abi.TraceView) == 2 * 8 + 8 * 8
