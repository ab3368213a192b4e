"""ctypes binding of libdk.so, the C ABI declared in include/dk.h.

The product path has no CPU fallback: if the library cannot be loaded, or no CUDA device is
present, every compute call raises DeviceUnavailable (a RuntimeError).
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

from .errors import SingularCoarseMatrix

LIB_PATH = Path(os.environ.get("DK_LIB_PATH") or
                Path(__file__).resolve().parent / "_lib" / "libdk.so")  # override: experiments

DK_OK, DK_EINVAL, DK_ESINGULAR, DK_ECUDA, DK_EUNSUPPORTED = 0, 1, 2, 3, 4
DK_AP_A, DK_AP_AM = 0, 1

#: every symbol include/dk.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "dk_last_error", "dk_version", "dk_device_count", "dk_set_device",
    "dk_op_create", "dk_op_destroy", "dk_op_set_precond", "dk_op_set_stream", "dk_op_spmv", "dk_op_profile",
    "dk_op_profile_read",
    "dk_defl_create", "dk_defl_destroy", "dk_defl_apply_p1", "dk_defl_apply_p2",
    "dk_defl_reconstruct", "dk_defl_x_star", "dk_defl_coarse", "dk_defl_setup_ms",
    "dk_gmres", "dk_gmres_ex", "dk_last_basis_vector", "dk_op_solve_stats",
    "dk_levelset_labels_device", "dk_assemble_tpfa", "dk_defl_create_dense",
    "dk_defl_create_ritz", "dk_defl_coarse_kind", "dk_dense_lu", "dk_lu_solve",
)


class DeviceUnavailable(RuntimeError):
    """The CUDA library or device is missing; the B200 path does not fall back to the CPU."""


class UnsupportedOperator(ValueError):
    """The operator or basis is outside what the device path implements."""


class SolveInfo(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32), ("restarts", C.c_int32), ("cycles", C.c_int32),
        ("converged", C.c_int32), ("warning", C.c_int32), ("last_cols", C.c_int32),
        ("reorths", C.c_int32), ("kernel_launches", C.c_int32),
        ("final_relres", C.c_double), ("solve_seconds", C.c_double),
    ]


class CycleCtl(C.Structure):
    """dk_cycle_ctl: cycle limit and resumable solve state (include/dk.h)."""
    _fields_ = [
        ("max_cycles", C.c_int32), ("resume", C.c_int32), ("iterations", C.c_int32),
        ("cycles", C.c_int32), ("warning", C.c_int32), ("has_prev", C.c_int32),
        ("converged", C.c_int32), ("running", C.c_int32),
        ("denom", C.c_double), ("prev_beta", C.c_double),
    ]


_lock = threading.Lock()
_lib = None

_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I32 = C.POINTER(C.c_int32)
_I64 = C.POINTER(C.c_int64)


def _declare(lib):
    sig = {
        "dk_last_error": (C.c_char_p, []),
        "dk_version": (C.c_int, []),
        "dk_device_count": (C.c_int, [_I32]),
        "dk_set_device": (C.c_int, [C.c_int32]),
        "dk_op_create": (C.c_int, [C.POINTER(_P), C.c_int64, C.c_int32, _I64, _P, _P]),
        "dk_op_destroy": (C.c_int, [_P]),
        "dk_op_set_precond": (C.c_int, [_P, _P]),
        "dk_op_set_stream": (C.c_int, [_P, _P]),
        "dk_op_spmv": (C.c_int, [_P, _P, _P]),
        "dk_op_profile": (C.c_int, [_P, C.c_int32]),
        "dk_op_profile_read": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_char_p), _D, _I64, _D]),
        "dk_defl_create": (C.c_int, [C.POINTER(_P), _P, _P, C.c_int32, C.c_int32, _P]),
        "dk_defl_destroy": (C.c_int, [_P]),
        "dk_defl_apply_p1": (C.c_int, [_P, _P, _P]),
        "dk_defl_apply_p2": (C.c_int, [_P, _P, _P]),
        "dk_defl_reconstruct": (C.c_int, [_P, _P, _P]),
        "dk_defl_x_star": (C.c_int, [_P, _P]),
        "dk_defl_coarse": (C.c_int, [_P, _P, _P]),
        "dk_defl_setup_ms": (C.c_int, [_P, _D]),
        "dk_defl_coarse_kind": (C.c_int, [_P, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
        "dk_gmres": (C.c_int, [_P, _P, _P, _P, C.c_int32, C.c_double, C.c_int32, C.c_int32,
                               _P, _P, _P, _P, C.POINTER(SolveInfo)]),
        "dk_gmres_ex": (C.c_int, [_P, _P, _P, _P, C.c_int32, C.c_double, C.c_int32, C.c_int32,
                                  _P, _P, _P, _P, _P, C.POINTER(SolveInfo), C.POINTER(CycleCtl),
                                  C.POINTER(CycleCtl)]),
        "dk_defl_create_dense": (C.c_int, [C.POINTER(_P), _P, _P, C.c_int32, C.c_int32, _P]),
        "dk_defl_create_ritz": (C.c_int, [C.POINTER(_P), _P, _P, C.c_int32, C.c_int32, C.c_int32,
                                          _P]),
        "dk_last_basis_vector": (C.c_int, [_P, C.c_int32, _P]),
        "dk_op_solve_stats": (C.c_int, [_P, _P, _P]),
        "dk_levelset_labels_device": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, _P, C.c_int32,
                                                C.c_int32, C.c_int32, _P, _I64, _P]),
        "dk_dense_lu": (C.c_int, [C.c_int64, _P, _P, _P, _D]),
        "dk_lu_solve": (C.c_int, [C.c_int64, _P, _P, C.c_int64, _P, _P]),
        "dk_assemble_tpfa": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double,
                                       C.c_double, _P, _P, _P, _P, C.c_int32, _P, _P, C.c_double,
                                       _P, _P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args


def load(build_if_missing: bool = True):
    """Load libdk.so (building it in-tree with nvcc if absent)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists() and build_if_missing:
            from .csrc.build import build
            build()
        if not LIB_PATH.exists():
            raise DeviceUnavailable(f"{LIB_PATH} is missing; run __graft_entry__.build()")
        lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | getattr(os, "RTLD_GLOBAL", 0))
        _declare(lib)
        _lib = lib
        return lib


def last_error() -> str:
    return load().dk_last_error().decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    """Map a dk status to the reference's exception types (errors.py / ValueError)."""
    if rc == DK_OK:
        return
    msg = last_error()
    if rc == DK_EINVAL:
        raise ValueError(msg)
    if rc == DK_ESINGULAR:
        raise SingularCoarseMatrix(msg)
    if rc == DK_EUNSUPPORTED:
        raise UnsupportedOperator(msg)
    raise DeviceUnavailable(f"{what}: {msg}" if what else msg)


def device_count() -> int:
    c = C.c_int32(0)
    load().dk_device_count(C.byref(c))
    return int(c.value)


def require_device() -> None:
    if device_count() < 1:
        raise DeviceUnavailable("no CUDA device: the B200 deflated-GMRES path has no CPU fallback")


def ptr(a) -> int | None:
    """Address of a C-contiguous numpy array or a CUDA torch tensor (None passes NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return int(a.data_ptr())
    raise TypeError(f"unsupported buffer type {type(a)!r}")
