"""The C-ABI library loads, exports every symbol include/pfx.h declares, and rejects
bad arguments with the documented status codes (no GPU work involved)."""
import ctypes
import os
import re

import numpy as np

from paper_2306_16778_b200 import _native
from paper_2306_16778_b200.errors import PFX_BADARG

from .conftest import ROOT


def _declared():
    text = open(os.path.join(ROOT, "include", "pfx.h")).read()
    return sorted(set(re.findall(r"\b(pfx_[a-z_]+)\s*\(", text)))


def test_header_symbols_exported():
    names = _declared()
    assert {"pfx_expm_dense", "pfx_expm_tridiag", "pfx_expm_banded", "pfx_pole_table"} <= set(names)
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_native.SIGNATURES)


def test_version_and_error_string():
    lib = _native.lib()
    assert lib.pfx_version() >= 100
    assert isinstance(lib.pfx_last_error(), bytes)


def _poles(n=16):
    from paper_2306_16778_b200.roots import default_table

    return default_table(n).interleaved()


def test_dense_bad_arguments():
    lib = _native.lib()
    t2, c2 = _poles()
    A = np.zeros((4, 4))
    out = np.zeros(4)
    V = np.ones(4)
    f64 = _native._f64p
    # bad memory kind
    assert lib.pfx_expm_dense(7, A.ctypes.data, 0, 4, 1, V.ctypes.data, 0, 1, 0.0, f64(t2), f64(c2), 8,
                              out.ctypes.data, 0, None, None) == PFX_BADARG
    # out_complex inconsistent with the real path (engine.py:185)
    assert lib.pfx_expm_dense(1, A.ctypes.data, 0, 4, 1, V.ctypes.data, 0, 1, 0.0, f64(t2), f64(c2), 8,
                              out.ctypes.data, 1, None, None) == PFX_BADARG
    assert b"out_complex" in lib.pfx_last_error()
    # non-positive Im(theta)
    bad = t2.copy()
    bad[1] = -1.0
    assert lib.pfx_expm_dense(1, A.ctypes.data, 0, 4, 1, V.ctypes.data, 0, 1, 0.0, f64(bad), f64(c2), 8,
                              out.ctypes.data, 0, None, None) == PFX_BADARG
    # d < 1
    assert lib.pfx_expm_dense(1, A.ctypes.data, 0, 0, 1, V.ctypes.data, 0, 1, 0.0, f64(t2), f64(c2), 8,
                              out.ctypes.data, 0, None, None) == PFX_BADARG
    # infinite shift
    assert lib.pfx_expm_dense(1, A.ctypes.data, 0, 4, 1, V.ctypes.data, 0, 1, float("inf"), f64(t2), f64(c2), 8,
                              out.ctypes.data, 0, None, None) == PFX_BADARG


def test_structured_bad_arguments():
    lib = _native.lib()
    t2, c2 = _poles()
    f64 = _native._f64p
    x = np.zeros(8)
    assert lib.pfx_expm_tridiag(1, x.ctypes.data, x.ctypes.data, 0, x.ctypes.data, 1, 0.0, f64(t2), f64(c2), 8,
                                x.ctypes.data, None, None) == PFX_BADARG
    assert lib.pfx_expm_banded(1, x.ctypes.data, 8, -1, x.ctypes.data, 1, 0.0, f64(t2), f64(c2), 8,
                               x.ctypes.data, None, None) == PFX_BADARG
    assert lib.pfx_pole_table(3, f64(x), f64(x)) == PFX_BADARG


def test_dense_cols_bad_arguments():
    lib = _native.lib()
    t2, c2 = _poles(4)  # two pairs
    A = np.zeros((8, 8))
    out = np.zeros((8, 8))
    f64 = _native._f64p
    i64p = ctypes.POINTER(ctypes.c_int64)

    def call(d, ranges, out_complex=0, a_complex=0, mem=1):
        rg = np.ascontiguousarray(np.asarray(ranges, dtype=np.int64).reshape(-1))
        return lib.pfx_expm_dense_cols(mem, A.ctypes.data, a_complex, d, 0.0, f64(t2), f64(c2), 2,
                                       rg.ctypes.data_as(i64p), out.ctypes.data, out_complex, 0, None)

    # the column split belongs to the blocked large path (d > 512)
    assert call(256, [(0, 256), (0, 256)]) == PFX_BADARG
    assert b"d > 512" in lib.pfx_last_error()
    # ranges: start not a multiple of 64, empty, beyond d
    assert call(1024, [(0, 1024), (32, 1024)]) == PFX_BADARG
    assert call(1024, [(0, 1024), (128, 128)]) == PFX_BADARG
    assert call(1024, [(0, 1024), (0, 1025)]) == PFX_BADARG
    assert b"column ranges" in lib.pfx_last_error()
    # out_complex must follow A
    assert call(1024, [(0, 1024), (0, 1024)], out_complex=1) == PFX_BADARG
    assert call(1024, [(0, 1024), (0, 1024)], mem=9) == PFX_BADARG
