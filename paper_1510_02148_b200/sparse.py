"""Sparse operator container and the device operator handle.

`SparseMatrix` keeps the reference's CSR interface (defkrylov/sparse.py:21-98: n,
row_offsets, col_indices, values, from_coo / from_dense / identity, diagonal, nnz,
scale_rows) but its working form is DIA: at most 7 diagonals, one fp64 array each, which is
what the B200 stencil kernel streams.  CSR arrays are materialised lazily when a caller asks
for them.  `spmv` runs on the device (sparse.py:101-106 semantics, bit-identical sums).
"""
from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _lib
from ._lib import UnsupportedOperator

MAX_DIAGONALS = 7


def _validate_csr(n: int, ro: np.ndarray, ci: np.ndarray, va: np.ndarray) -> None:
    # same contract and messages as the reference (sparse.py:35-52), vectorised
    if ro.shape != (n + 1,):
        raise ValueError("row_offsets must have length n+1")
    if ro[0] != 0 or ro[-1] != len(va) or np.any(np.diff(ro) < 0):
        raise ValueError("row_offsets must be nondecreasing from 0 to nnz")
    if len(ci) != len(va):
        raise ValueError("col_indices and values must have equal length")
    if len(ci) and (ci.min() < 0 or ci.max() >= n):
        raise ValueError("column index out of range")
    if len(ci) > 1:
        row = np.repeat(np.arange(n), np.diff(ro))
        bad = (row[1:] == row[:-1]) & (np.diff(ci) <= 0)
        if bad.any():
            i = int(row[1:][np.flatnonzero(bad)[0]])
            raise ValueError(f"row {i}: column indices not strictly increasing")


class SparseMatrix:
    """Square real matrix; CSR view for the reference API, DIA storage for the device."""

    __slots__ = ("n", "_ro", "_ci", "_va", "_offsets", "_diags", "_dev", "__weakref__")

    def __init__(self, n: int, row_offsets, col_indices, values):
        self.n = int(n)
        ro = np.asarray(row_offsets, dtype=np.int64)
        ci = np.asarray(col_indices, dtype=np.int64)
        va = np.asarray(values, dtype=np.float64)
        _validate_csr(self.n, ro, ci, va)
        self._ro, self._ci, self._va = ro, ci, va
        self._offsets = None
        self._diags = None
        self._dev = None

    # ---- constructors -----------------------------------------------------------------
    @classmethod
    def from_dia(cls, n: int, offsets, diags) -> "SparseMatrix":
        """Build from diagonals: diags[k, i] = A[i, i + offsets[k]] (zeros are not stored)."""
        offsets = np.asarray(offsets, dtype=np.int64)
        diags = np.ascontiguousarray(np.asarray(diags, dtype=np.float64))
        order = np.argsort(offsets, kind="stable")
        if np.any(order != np.arange(len(order))):  # reorder (copies) only when needed
            offsets, diags = offsets[order], diags[order]
        if diags.shape != (len(offsets), n):
            raise ValueError("diags must be ndiag x n")
        if len(offsets) > MAX_DIAGONALS or len(np.unique(offsets)) != len(offsets):
            raise ValueError("at most 7 distinct diagonals")
        self = cls.__new__(cls)
        self.n = int(n)
        self._ro = self._ci = self._va = None
        self._offsets = offsets
        self._diags = diags
        self._dev = None
        return self

    @classmethod
    def from_coo(cls, n: int, rows, cols, vals) -> "SparseMatrix":
        """Triplets; duplicates are summed (reference sparse.py:54-60)."""
        import scipy.sparse
        m = scipy.sparse.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr()
        m.sum_duplicates()
        m.sort_indices()
        return cls(n, m.indptr, m.indices, m.data)

    @classmethod
    def from_dense(cls, M) -> "SparseMatrix":
        M = np.asarray(M, dtype=np.float64)
        if M.ndim != 2 or M.shape[0] != M.shape[1]:
            raise ValueError("matrix must be square")
        rows, cols = np.nonzero(M)
        n = M.shape[0]
        ro = np.zeros(n + 1, dtype=np.int64)
        np.add.at(ro, rows + 1, 1)
        return cls(n, np.cumsum(ro), cols, M[rows, cols])

    @classmethod
    def identity(cls, n: int) -> "SparseMatrix":
        return cls(n, np.arange(n + 1), np.arange(n), np.ones(n))

    # ---- CSR view (lazy for DIA-built matrices) -----------------------------------------
    def _materialise_csr(self) -> None:
        if self._ro is not None:
            return
        n, off, dg = self.n, self._offsets, self._diags
        i = np.arange(n)
        keep = np.empty((n, len(off)), dtype=bool)
        for k, o in enumerate(off):
            keep[:, k] = (dg[k] != 0.0) | (o == 0)
            keep[:, k] &= (i + o >= 0) & (i + o < n)
        counts = keep.sum(axis=1)
        ro = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(counts, out=ro[1:])
        cols = (i[:, None] + off[None, :])[keep]
        vals = dg.T[keep]
        self._ro, self._ci, self._va = ro, cols.astype(np.int64), vals

    @property
    def row_offsets(self) -> np.ndarray:
        self._materialise_csr()
        return self._ro

    @property
    def col_indices(self) -> np.ndarray:
        self._materialise_csr()
        return self._ci

    @property
    def values(self) -> np.ndarray:
        self._materialise_csr()
        return self._va

    @property
    def nnz(self) -> int:
        return len(self.values)

    # ---- DIA form ------------------------------------------------------------------------
    def dia(self):
        """(offsets ascending, diags ndiag x n); raises UnsupportedOperator past 7 diagonals."""
        if self._offsets is None:
            n, ro, ci, va = self.n, self._ro, self._ci, self._va
            row = np.repeat(np.arange(n, dtype=np.int64), np.diff(ro))
            off = ci - row
            offs = np.unique(off)
            if len(offs) > MAX_DIAGONALS:
                raise UnsupportedOperator(
                    f"the device path stores at most {MAX_DIAGONALS} diagonals (a 7-point "
                    f"stencil); this matrix has {len(offs)} distinct diagonal offsets")
            if len(offs) == 0:
                offs = np.zeros(1, dtype=np.int64)
            diags = np.zeros((len(offs), n))
            diags[np.searchsorted(offs, off), row] = va
            self._offsets, self._diags = offs, diags
        return self._offsets, self._diags

    def diagonal(self) -> np.ndarray:
        off, dg = self.dia()
        k = np.flatnonzero(off == 0)
        return dg[k[0]].copy() if len(k) else np.zeros(self.n)

    def to_dense(self) -> np.ndarray:
        D = np.zeros((self.n, self.n))
        off, dg = self.dia()
        i = np.arange(self.n)
        for k, o in enumerate(off):
            ok = (i + o >= 0) & (i + o < self.n)
            D[i[ok], i[ok] + o] = dg[k][ok]
        return D

    def scale_rows(self, s) -> "SparseMatrix":
        """diag(s) @ self (reference sparse.py:90-98)."""
        s = np.asarray(s, dtype=np.float64)
        if s.shape != (self.n,):
            raise ValueError("scale vector has wrong length")
        off, dg = self.dia()
        out = SparseMatrix.from_dia(self.n, off, dg * s[None, :])
        if self._ro is not None:
            row = np.repeat(np.arange(self.n), np.diff(self._ro))
            out._ro, out._ci, out._va = self._ro, self._ci, self._va * s[row]
        return out

    # ---- device handle ---------------------------------------------------------------------
    def device(self) -> "DeviceOperator":
        if self._dev is None:
            self._dev = DeviceOperator(self)
        return self._dev

    def release_device(self) -> None:
        if self._dev is not None:
            self._dev.close()
            self._dev = None

    def __repr__(self) -> str:
        return f"SparseMatrix(n={self.n})"


class DeviceOperator:
    """A dk_op handle: the DIA operator resident in HBM plus its right preconditioner."""

    def __init__(self, A: SparseMatrix):
        lib = _lib.load()
        _lib.require_device()
        off, dg = A.dia()
        self.n = A.n
        self._lib = lib
        h = C.c_void_p()
        offs = np.ascontiguousarray(off, dtype=np.int64)
        _lib.check(lib.dk_op_create(C.byref(h), A.n, len(offs),
                                    offs.ctypes.data_as(C.POINTER(C.c_int64)),
                                    _lib.ptr(dg), None), "dk_op_create")
        self.h = h
        self._precond_key = None
        self._precond_ref = None
        self._fin = weakref.finalize(self, lib.dk_op_destroy, h)

    def close(self) -> None:
        self._fin()

    def set_precond(self, M) -> None:
        """Install M (identity / Jacobi) unless it is already installed."""
        inv = None if M is None or M.kind == "identity" else M.inv_diag
        key = None if inv is None else id(inv)
        if key == self._precond_key and (inv is None or self._precond_ref is inv):
            return
        if inv is not None:
            inv = np.ascontiguousarray(inv, dtype=np.float64)
            if inv.shape != (self.n,):
                raise ValueError("preconditioner has wrong length")
        _lib.check(self._lib.dk_op_set_precond(self.h, _lib.ptr(inv)), "dk_op_set_precond")
        self._precond_key = key
        self._precond_ref = None if M is None or M.kind == "identity" else M.inv_diag

    def spmv(self, x) -> np.ndarray:
        y = np.empty(self.n)
        _lib.check(self._lib.dk_op_spmv(self.h, _lib.ptr(x), _lib.ptr(y)), "dk_op_spmv")
        return y


def spmv(A: SparseMatrix, x) -> np.ndarray:
    """y = A @ x on the device (reference sparse.py:101-106)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    if x.shape != (A.n,):
        raise ValueError(f"dimension mismatch: matrix is {A.n}, vector is {x.shape}")
    return A.device().spmv(x)


# ---- dense LU helpers (sparse.py:109-145) --------------------------------------------------
class LUFactors:
    """Combined LU storage with pivot permutation, LAPACK getrf layout (sparse.py:109-118):
    `lu` holds unit L strictly below the diagonal and U on and above it, `piv[k]` the 0-based
    row interchanged with row k; `n` the order."""

    __slots__ = ("lu", "piv", "n")

    def __init__(self, lu, piv):
        self.lu = lu
        self.piv = piv
        self.n = lu.shape[0]

    def __repr__(self) -> str:
        return f"LUFactors(n={self.n})"


def dense_lu(M) -> LUFactors:
    """P M = L U with partial pivoting on the device (sparse.py:121-137, dk_dense_lu).

    Raises SingularCoarseMatrix on a pivot below 1e-300, ValueError for a non-square or
    non-finite matrix.
    """
    M = np.asarray(M, dtype=np.float64)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError("matrix must be square")
    if M.size == 0:
        return LUFactors(M.reshape(0, 0), np.zeros(0, dtype=np.int32))
    if not np.isfinite(M).all():  # scipy.linalg.lu_factor(check_finite=True)
        raise ValueError("array must not contain infs or NaNs")
    lib = _lib.load()
    _lib.require_device()
    a = np.ascontiguousarray(M)
    n = a.shape[0]
    lu = np.empty((n, n))
    piv = np.empty(n, dtype=np.int32)
    mp = C.c_double(0.0)
    rc = lib.dk_dense_lu(n, _lib.ptr(a), _lib.ptr(lu), _lib.ptr(piv), C.byref(mp))
    _lib.check(rc, "dk_dense_lu")  # DK_ESINGULAR -> SingularCoarseMatrix
    return LUFactors(lu, piv)


def lu_solve(f: LUFactors, b) -> np.ndarray:
    """Solve M x = b from dense_lu's factors (sparse.py:140-145); b is a vector or stacked
    right-hand sides (n x k).  Triangular solves on the device (dk_lu_solve)."""
    b = np.asarray(b, dtype=np.float64)
    if f.n == 0:
        return np.zeros_like(b)
    if b.shape[0] != f.n or b.ndim not in (1, 2):
        raise ValueError("right-hand side has wrong shape")
    lib = _lib.load()
    _lib.require_device()
    rhs = np.ascontiguousarray(b.reshape(f.n, -1))
    x = np.empty_like(rhs)
    lu = np.ascontiguousarray(f.lu, dtype=np.float64)
    piv = np.ascontiguousarray(f.piv, dtype=np.int32)
    _lib.check(lib.dk_lu_solve(f.n, _lib.ptr(lu), _lib.ptr(piv), rhs.shape[1], _lib.ptr(rhs),
                               _lib.ptr(x)), "dk_lu_solve")
    return x.reshape(b.shape)
