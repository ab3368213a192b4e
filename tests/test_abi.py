"""The C-ABI library loads, exports every symbol include/dk.h declares, fails loudly without
a device (no CPU fallback) and its host-side parts work on any machine."""
from __future__ import annotations

import ctypes as C
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_1510_02148_b200 import _lib


def header_symbols():
    text = (ROOT / "include" / "dk.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(dk_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.EXPORTS) == syms


def test_library_is_sm100a():
    data = _lib.LIB_PATH.read_bytes()
    assert b"sm_100a" in data or b"sm_100" in data


def test_version_and_device_count():
    lib = _lib.load()
    assert lib.dk_version() >= 1
    assert _lib.device_count() >= 0


def test_no_device_means_loud_failure():
    if _lib.device_count() > 0:
        pytest.skip("a device is present")
    import paper_1510_02148_b200 as dk
    A = dk.SparseMatrix.identity(4)
    with pytest.raises(_lib.DeviceUnavailable):
        dk.spmv(A, np.ones(4))
    with pytest.raises(_lib.DeviceUnavailable):
        dk.gmres(A, np.ones(4))
    h = C.c_void_p()
    off = np.zeros(1, dtype=np.int64)
    rc = _lib.load().dk_op_create(C.byref(h), 4, 1, off.ctypes.data_as(C.POINTER(C.c_int64)),
                                  np.ones(4).ctypes.data, None)
    assert rc == _lib.DK_ECUDA and "no CUDA device" in _lib.last_error()


def test_labels_entry_point_validates_then_needs_a_device():
    lib = _lib.load()
    band = np.zeros(8, dtype=np.int64)
    out = np.empty(8, dtype=np.int64)
    cb = np.empty(8, dtype=np.int64)
    n = C.c_int64()
    assert lib.dk_levelset_labels_device(2, 2, 2, band.ctypes.data, 3, 1, 1, out.ctypes.data,
                                         C.byref(n), cb.ctypes.data) == _lib.DK_EINVAL
    if _lib.device_count() == 0:
        assert lib.dk_levelset_labels_device(2, 2, 2, band.ctypes.data, 2, 2, 2,
                                             out.ctypes.data, C.byref(n),
                                             cb.ctypes.data) == _lib.DK_ECUDA
        assert "no CUDA device" in _lib.last_error()
