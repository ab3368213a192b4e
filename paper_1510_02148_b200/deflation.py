"""Deflation projectors P1, P2, the coarse matrix E and the coarse solution — on the device.

Reference: defkrylov/deflation.py:19-104.  An indicator (piecewise-constant) basis — the
physics-based PSL basis — is stored as one int32 column label per cell, never as a dense
n x d matrix; E, its factorisation, E^-1 and x* = Z E^-1 Z^T b are built in HBM by
dk_defl_create.  A dense Z whose rows have at most one nonzero equal to 1 is converted to
labels.  Any other (dense) basis with d <= 64 columns — harmonic Ritz vectors (RDGMRES) or a
user basis — is kept as dense rows on the device (dk_defl_create_dense); wider dense bases
raise UnsupportedOperator.
"""
from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _lib
from ._lib import UnsupportedOperator
from .errors import SingularCoarseMatrix
from .sparse import SparseMatrix

_DENSE_LIMIT = 1 << 26  # materialise Z / AZ densely only below this many entries
DENSE_MAX_D = 64        # widest dense (non-indicator) basis of the device path


class DeflationBasis:
    """n x d indicator deflation vectors (deflation.py:19-37), stored as column labels."""

    __slots__ = ("labels", "_n", "_d", "_dense")

    def __init__(self, Z=None, *, labels=None, d=None):
        self._dense = None
        if labels is not None:
            lab = np.ascontiguousarray(np.asarray(labels), dtype=np.int32)
            if lab.ndim != 1:
                raise ValueError("labels must be a vector")
            dd = int(d) if d is not None else int(lab.max(initial=-1)) + 1
            if dd < 1:
                raise ValueError("Z must be n x d with d >= 1")
            if lab.min(initial=-1) < -1 or lab.max(initial=-1) >= dd:
                raise ValueError("labels out of range")
            self.labels, self._n, self._d = lab, len(lab), dd
            return
        Zd = np.asarray(Z, dtype=np.float64)
        if Zd.ndim != 2 or Zd.shape[1] < 1:
            raise ValueError("Z must be n x d with d >= 1")
        self._n, self._d = Zd.shape
        nz = Zd != 0.0
        per_row = nz.sum(axis=1)
        if np.all(per_row <= 1) and np.all(Zd[nz] == 1.0):
            lab = np.full(self._n, -1, dtype=np.int32)
            r, c = np.nonzero(nz)
            lab[r] = c
            self.labels = lab
        else:
            self.labels = None
            self._dense = np.ascontiguousarray(Zd)

    @property
    def n(self) -> int:
        return self._n

    @property
    def d(self) -> int:
        return self._d

    @property
    def Z(self) -> np.ndarray:
        """Dense n x d view (small problems only)."""
        if self._dense is not None:
            return self._dense
        if self._n * self._d > _DENSE_LIMIT:
            raise MemoryError("dense Z of this basis is too large; use .labels")
        Z = np.zeros((self._n, self._d))
        keep = self.labels >= 0
        Z[np.flatnonzero(keep), self.labels[keep]] = 1.0
        return Z

    @property
    def is_indicator(self) -> bool:
        return self.labels is not None


class DeflationContext:
    """Frozen projector state resident on the device (deflation.py:40-68)."""

    def __init__(self, basis: DeflationBasis, A: SparseMatrix, M, A_p_choice: str, h, lib):
        self.basis, self.A, self.M, self.A_p_choice = basis, A, M, A_p_choice
        self.h, self._lib = h, lib
        self._E_lu = None
        self._fin = weakref.finalize(self, lib.dk_defl_destroy, h)

    def close(self) -> None:
        self._fin()

    def _check_operator(self, A: SparseMatrix, M) -> None:
        if A is not self.A:
            raise ValueError("deflation context was built for a different matrix")
        if self.A_p_choice == "AM" and (M is not self.M and not (
                M.kind == "identity" and self.M.kind == "identity")):
            raise UnsupportedOperator("A_p='AM' needs the solve's preconditioner to be the "
                                      "context's")

    def _call(self, fn, v) -> np.ndarray:
        v = np.ascontiguousarray(np.asarray(v, dtype=np.float64))
        if v.shape != (self.A.n,):
            raise ValueError("vector has wrong length")
        self.A.device().set_precond(self.M)
        out = np.empty(self.A.n)
        _lib.check(fn(self.h, _lib.ptr(v), _lib.ptr(out)))
        return out

    def apply_p1(self, v) -> np.ndarray:
        """v - A_p Z E^-1 Z^T v."""
        return self._call(self._lib.dk_defl_apply_p1, v)

    def apply_p2(self, v) -> np.ndarray:
        """v - Z E^-1 Z^T A_p v."""
        return self._call(self._lib.dk_defl_apply_p2, v)

    def reconstruct(self, x_hat) -> np.ndarray:
        """x* + P2 x^."""
        return self._call(self._lib.dk_defl_reconstruct, x_hat)

    @property
    def x_star(self) -> np.ndarray:
        out = np.empty(self.A.n)
        _lib.check(self._lib.dk_defl_x_star(self.h, _lib.ptr(out)))
        return out

    @property
    def d(self) -> int:
        return self.basis.d

    @property
    def E_lu(self):
        """LUFactors of E (deflation.py:46), factorised on the device on first access.

        The solver itself applies E^-1 through its own factor (Cholesky in nested-dissection
        order for a symmetric E, pivoted LU otherwise — dk_defl_coarse_kind); this is the
        reference's getrf-layout view for callers of lu_solve(ctx.E_lu, ...)."""
        if self._E_lu is None:
            from .sparse import dense_lu
            self._E_lu = dense_lu(self.coarse_matrix(inverse=False)[0])
        return self._E_lu

    def coarse_matrix(self, inverse: bool = True):
        """(E, E^-1) copied from the device (d x d); E^-1 is None when inverse=False."""
        d = self.basis.d
        E = np.empty((d, d))
        Einv = np.empty((d, d)) if inverse else None
        _lib.check(self._lib.dk_defl_coarse(self.h, _lib.ptr(E), _lib.ptr(Einv)))
        return E, Einv

    def setup_ms(self) -> dict:
        """Device time of the set-up phases: E assembly, factorisation (Cholesky for an SPD E,
        else pivoted LU), forming E^-1, x*."""
        ms = (C.c_double * 4)()
        _lib.check(self._lib.dk_defl_setup_ms(self.h, ms))
        return {"assemble_E": ms[0], "factor": ms[1], "inverse": ms[2], "x_star": ms[3]}

    _COARSE_KINDS = ("dense_gemv", "packed_symmetric", "nested_dissection_W", "dense_basis")

    def coarse_kind(self) -> tuple:
        """(how E^-1 is applied, 32 x 32 tiles streamed per application) — see include/dk.h."""
        k, t = C.c_int32(), C.c_int64()
        _lib.check(self._lib.dk_defl_coarse_kind(self.h, C.byref(k), C.byref(t)))
        return self._COARSE_KINDS[k.value], int(t.value)

    @property
    def AZ(self) -> np.ndarray:
        """Dense A_p Z (small problems only; the device never forms it)."""
        Z = self.basis.Z
        if self.A.n * Z.shape[1] > _DENSE_LIMIT:
            raise MemoryError("dense AZ is too large")
        cols = [Z[:, j] if self.A_p_choice == "A" else self.M.apply(Z[:, j])
                for j in range(Z.shape[1])]
        from .sparse import spmv
        return np.column_stack([spmv(self.A, c) for c in cols])


def build_context(A: SparseMatrix, M, Z: DeflationBasis, b, A_p_choice: str = "A"
                  ) -> DeflationContext:
    """Assemble E = Z^T A_p Z on the device, factorise it, form x* (deflation.py:71-89).

    Raises SingularCoarseMatrix when the deflation vectors are dependent.
    """
    if A_p_choice not in ("A", "AM"):
        raise ValueError("A_p_choice must be 'A' or 'AM'")
    if Z.n != A.n:
        raise ValueError("deflation basis does not match the matrix dimension")
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    if b.shape != (A.n,):
        raise ValueError("right-hand side has wrong length")
    op = A.device()
    op.set_precond(M)
    h = C.c_void_p()
    ap = _lib.DK_AP_AM if A_p_choice == "AM" else _lib.DK_AP_A
    if Z.is_indicator:
        _lib.check(op._lib.dk_defl_create(C.byref(h), op.h, _lib.ptr(Z.labels), Z.d, ap,
                                          _lib.ptr(b)), "dk_defl_create")
    else:
        if Z.d > DENSE_MAX_D:
            raise UnsupportedOperator(
                f"dense (non-indicator) deflation bases are limited to {DENSE_MAX_D} columns")
        rows = np.ascontiguousarray(Z.Z.T)  # d x n: row k = basis vector k
        _lib.check(op._lib.dk_defl_create_dense(C.byref(h), op.h, _lib.ptr(rows), Z.d, ap,
                                                _lib.ptr(b)), "dk_defl_create_dense")
    return DeflationContext(Z, A, M, A_p_choice, h, op._lib)


class _RitzBasis(DeflationBasis):
    """Z = V_m Y formed on the device from the operator's last Arnoldi cycle; the dense view
    is computed on demand from the cycle data (harmonic.py:91-94)."""

    __slots__ = ("_data", "_Y")

    def __init__(self, data, Y: np.ndarray):
        self._data, self._Y = data, Y
        self.labels = None
        self._n = data._n
        self._d = Y.shape[1]
        self._dense = None

    @property
    def Z(self) -> np.ndarray:
        if self._dense is None:
            self._dense = self._data.V[:self._data.m].T @ self._Y
        return self._dense


def build_ritz_context(A: SparseMatrix, M, data, Y: np.ndarray, b,
                       A_p_choice: str = "A") -> DeflationContext:
    """Deflation context of the harmonic Ritz vectors Z = V_m Y of the last device cycle
    (build_context(A, M, DeflationBasis(V_m Y), b) without moving V to the host)."""
    if A_p_choice not in ("A", "AM"):
        raise ValueError("A_p_choice must be 'A' or 'AM'")
    Y = np.asfortranarray(np.asarray(Y, dtype=np.float64))
    if Y.ndim != 2 or Y.shape[1] < 1:
        raise ValueError("Z must be n x d with d >= 1")
    rows, d = Y.shape
    if d > DENSE_MAX_D:
        raise UnsupportedOperator(
            f"dense (non-indicator) deflation bases are limited to {DENSE_MAX_D} columns")
    if not data.on_device():
        raise RuntimeError("the Arnoldi basis was overwritten by a later solve")
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    op = A.device()
    op.set_precond(M)
    h = C.c_void_p()
    ap = _lib.DK_AP_AM if A_p_choice == "AM" else _lib.DK_AP_A
    _lib.check(op._lib.dk_defl_create_ritz(C.byref(h), op.h, Y.ctypes.data, rows, d, ap,
                                           _lib.ptr(b)), "dk_defl_create_ritz")
    return DeflationContext(_RitzBasis(data, Y), A, M, A_p_choice, h, op._lib)


def apply_p1(ctx: DeflationContext | None, v) -> np.ndarray:
    """P1 v; a missing context is the identity."""
    return v if ctx is None else ctx.apply_p1(v)


def apply_p2(ctx: DeflationContext | None, v) -> np.ndarray:
    """P2 v; a missing context is the identity."""
    return v if ctx is None else ctx.apply_p2(v)


def reconstruct(ctx: DeflationContext | None, x_hat) -> np.ndarray:
    """x = x* + P2 x^ ; a missing context is the identity."""
    return x_hat if ctx is None else ctx.reconstruct(x_hat)
