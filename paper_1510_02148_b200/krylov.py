"""Restarted right-preconditioned GMRES(m) — the reference API on the B200 device path.

Signatures, validation, return type and semantics follow defkrylov/krylov.py:22-266.  The
whole cycle loop (Arnoldi, Givens least squares, convergence / breakdown tests, x update)
runs on the device through dk_gmres; the host only converts inputs and builds the report.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .sparse import SparseMatrix


@dataclass(frozen=True)
class Preconditioner:
    """Right preconditioner: identity or Jacobi (inverse diagonal). krylov.py:22-43."""

    kind: str
    inv_diag: np.ndarray | None = None

    @classmethod
    def identity(cls) -> "Preconditioner":
        return cls("identity")

    @classmethod
    def jacobi(cls, A: SparseMatrix) -> "Preconditioner":
        d = A.diagonal()
        if np.any(d == 0):
            raise ValueError("Jacobi preconditioner requires a nonzero diagonal")
        return cls("jacobi", 1.0 / d)

    def apply(self, v: np.ndarray) -> np.ndarray:
        if self.kind == "identity":
            return v
        return v * self.inv_diag


def jacobi_apply(M: Preconditioner, v) -> np.ndarray:
    """Componentwise v_i / a_ii (identity passes v through)."""
    return M.apply(np.asarray(v, dtype=np.float64))


@dataclass
class ArnoldiData:
    """Basis and pristine Hessenberg of the last GMRES cycle (krylov.py:51-62)."""

    V: np.ndarray
    Hbar: np.ndarray
    m: int


class _DeviceArnoldi(ArnoldiData):
    """ArnoldiData whose basis V is copied from HBM on first access."""

    def __init__(self, op, serial: int, n: int, cols: int, Hbar: np.ndarray):
        self._op, self._serial, self._n = op, serial, n
        self._V = None
        self.Hbar = Hbar
        self.m = cols

    @property
    def V(self) -> np.ndarray:  # type: ignore[override]
        if self._V is None:
            if getattr(self._op, "serial", None) != self._serial:
                raise RuntimeError("the device basis was overwritten by a later solve")
            V = np.empty((self.m + 1, self._n))
            for i in range(self.m + 1):
                _lib.check(self._op._lib.dk_last_basis_vector(self._op.h, i, _lib.ptr(V[i])),
                           "dk_last_basis_vector")
            self._V = V
        return self._V

    @V.setter
    def V(self, value) -> None:
        self._V = value


@dataclass
class SolveReport:
    """krylov.py:65-79."""

    x: np.ndarray
    converged: bool
    iterations: int
    restarts: int
    residual_history: np.ndarray
    final_relres: float
    restart_of: np.ndarray
    deflated_flags: np.ndarray
    ritz_trace: list = field(default_factory=list)
    ritz_iter_trace: list = field(default_factory=list)
    arnoldi: ArnoldiData | None = None
    warning: str | None = None
    deflated_from_cycle: int | None = None
    # device-side extras (not in the reference report)
    solve_seconds: float = 0.0
    kernel_launches: int = 0
    reorthogonalisations: int = 0


def ritz_values(data: ArnoldiData) -> np.ndarray:
    """Eigenvalues of H_m sorted by magnitude (krylov.py:82-87)."""
    if data.m < 1:
        raise ValueError("empty Arnoldi data")
    w = np.linalg.eigvals(data.Hbar[:data.m, :data.m])
    return w[np.argsort(np.abs(w))]


def _device_solve(A: SparseMatrix, b, x0, M, m, tol, max_iters, min_iters, ctx) -> SolveReport:
    op = A.device()
    op.set_precond(M)
    if ctx is not None:
        ctx._check_operator(A, M)
    n = A.n
    x = np.empty(n)
    cap = max(int(max_iters), 0) + 1
    hist = np.empty(cap)
    rof = np.empty(cap, dtype=np.int32)
    hbar = np.empty((m, m + 1))  # column-major (m+1) x m == row-major m x (m+1)
    info = _lib.SolveInfo()
    rc = op._lib.dk_gmres(op.h, ctx.h if ctx is not None else None, _lib.ptr(b), _lib.ptr(x0),
                          int(m), float(tol), int(max_iters), int(min_iters), _lib.ptr(x),
                          _lib.ptr(hist), _lib.ptr(rof), _lib.ptr(hbar), C.byref(info))
    _lib.check(rc, "dk_gmres")
    op.serial = getattr(op, "serial", 0) + 1
    it = int(info.iterations)
    Hfull = hbar.T  # (m+1) x m
    cols = int(info.last_cols)
    arnoldi = None
    if info.cycles > 0:
        arnoldi = _DeviceArnoldi(op, op.serial, n, cols, Hfull[:cols + 1, :cols].copy())
        if (cols + 1) * n <= (1 << 22):
            arnoldi.V  # small: copy now so the report outlives later solves
    deflated = ctx is not None
    return SolveReport(
        x=x, converged=bool(info.converged), iterations=it, restarts=int(info.restarts),
        residual_history=hist[:it + 1].copy(), final_relres=float(info.final_relres),
        restart_of=rof[:it + 1].astype(np.int64), deflated_flags=np.full(it + 1, deflated),
        arnoldi=arnoldi, warning="breakdown" if info.warning == 1 else None,
        deflated_from_cycle=0 if deflated else None, solve_seconds=float(info.solve_seconds),
        kernel_launches=int(info.kernel_launches), reorthogonalisations=int(info.reorths))


def gmres(A: SparseMatrix, b, x0=None, M: Preconditioner | None = None, m: int = 30,
          tol: float = 1e-6, max_iters: int = 300, min_iters: int = 0, deflation=None,
          capture_ritz: bool = False) -> SolveReport:
    """Restarted right-preconditioned GMRES(m) (krylov.py:239-266).

    With `deflation` (a DeflationContext) solves P1 A x^ = P1 b and returns x* + P2 x^.
    Hitting max_iters is reported as converged=False, not an error.
    """
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    if b.shape != (A.n,):
        raise ValueError("right-hand side has wrong length")
    if x0 is None:
        x0 = np.zeros(A.n)
    x0 = np.ascontiguousarray(np.asarray(x0, dtype=np.float64))
    if x0.shape != (A.n,):
        raise ValueError("initial guess has wrong length")
    if M is None:
        M = Preconditioner.identity()
    if m < 1:
        raise ValueError("cycle size must be >= 1")
    if tol <= 0:
        raise ValueError("tolerance must be positive")
    if capture_ritz:
        raise NotImplementedError(
            "capture_ritz feeds harmonic-Ritz RDGMRES, which is outside the device hot path")
    return _device_solve(A, b, x0, M, m, tol, max_iters, min_iters, deflation)
