"""The C-ABI library loads and exports every symbol include/polarsc.h
declares (no compute calls: this runs without a GPU)."""
import ctypes
import os
import re

from paper_1204_5882_b200 import _lib
from paper_1204_5882_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "polarsc.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(pq_[a-z_0-9]+)\s*\(", text, re.M)))


def test_header_symbols_exported():
    build()
    syms = header_symbols()
    assert len(syms) >= 12
    assert set(syms) == set(_lib.EXPORTS)
    L = ctypes.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert hasattr(L, s), s
    assert _lib.load().pq_abi_version() == 1


def test_argument_errors_map_to_valueerror():
    L = _lib.load()
    h = ctypes.c_void_p()
    rc = L.pq_decoder_create(ctypes.byref(h), 0, 1, 0, 0)  # n = 0: rejected before any CUDA call
    assert rc < 0 and b"n must be" in L.pq_last_error()
    rc = L.pq_polar_transform(None, None, 4, 1, None)
    assert rc < 0
    try:
        _lib.check(rc, "pq_polar_transform")
    except ValueError:
        pass
    else:
        raise AssertionError("negative rc must raise ValueError")
