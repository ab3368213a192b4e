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
    """ArnoldiData whose basis V is copied from HBM on first access.  `gram` is the device's
    V^T V_m (the re-orthogonalisation test's Gram matrix), so harmonic Ritz extraction needs
    no copy of V."""

    def __init__(self, op, serial: int, n: int, cols: int, Hbar: np.ndarray,
                 gram: np.ndarray | None = None):
        self._op, self._serial, self._n = op, serial, n
        self._V = None
        self.Hbar = Hbar
        self.m = cols
        self.gram = gram

    def on_device(self) -> bool:
        """The basis of this cycle is still the operator's resident basis."""
        return getattr(self._op, "serial", None) == self._serial

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
    host_syncs: int = 0       # host synchronisations inside the cycle loop (dk_op_solve_stats)
    device_loop: bool = False  # restarts decided on the device (conditional WHILE graph)


def ritz_values(data: ArnoldiData) -> np.ndarray:
    """Eigenvalues of H_m sorted by magnitude (krylov.py:82-87)."""
    if data.m < 1:
        raise ValueError("empty Arnoldi data")
    w = np.linalg.eigvals(data.Hbar[:data.m, :data.m])
    return w[np.argsort(np.abs(w))]


class _Cycles:
    """Runs GMRES(m) cycles through dk_gmres_ex and keeps the resumable device state."""

    def __init__(self, A: SparseMatrix, b, x0, M, m, tol, max_iters, min_iters):
        self.A, self.b, self.x0, self.M = A, b, x0, M
        self.m, self.tol, self.max_iters, self.min_iters = m, tol, max_iters, min_iters
        self.op = A.device()
        self.op.set_precond(M)
        cap = max(int(max_iters), 0) + 1
        self.hist = np.empty(cap)
        self.rof = np.empty(cap, dtype=np.int32)
        self.ctl = None
        self.info = None
        self.x = np.empty(A.n)
        self.arnoldi = None
        self.solve_seconds = 0.0
        self.launches = 0
        self.reorths = 0
        self.host_syncs = 0
        self.device_loop = False

    def run(self, ctx, max_cycles: int = 0, warning: int | None = None):
        """Cycles until convergence / max_iters (or max_cycles of this call) on the current
        deflation context; later calls continue the same solve from the device iterate."""
        op, m = self.op, self.m
        if ctx is not None:
            ctx._check_operator(self.A, self.M)
        hbar = np.empty((m, m + 1))  # column-major (m+1) x m == row-major m x (m+1)
        gram = np.empty((m, m + 1))
        info = _lib.SolveInfo()
        cin = _lib.CycleCtl()
        if self.ctl is not None:
            C.memmove(C.addressof(cin), C.addressof(self.ctl), C.sizeof(cin))
            if warning is not None:
                cin.warning = warning
        cin.max_cycles = int(max_cycles)
        cout = _lib.CycleCtl()
        resume = self.ctl is not None
        rc = op._lib.dk_gmres_ex(op.h, ctx.h if ctx is not None else None, _lib.ptr(self.b),
                                 None if resume or self.x0 is None else _lib.ptr(self.x0),
                                 int(m), float(self.tol),
                                 int(self.max_iters), int(self.min_iters), _lib.ptr(self.x),
                                 _lib.ptr(self.hist), _lib.ptr(self.rof), _lib.ptr(hbar),
                                 _lib.ptr(gram), C.byref(info), C.byref(cin), C.byref(cout))
        _lib.check(rc, "dk_gmres_ex")
        op.serial = getattr(op, "serial", 0) + 1
        self.ctl, self.info = cout, info
        self.solve_seconds += float(info.solve_seconds)
        self.launches += int(info.kernel_launches)
        self.reorths += int(info.reorths)
        hs, dl = C.c_int32(0), C.c_int32(0)
        _lib.check(op._lib.dk_op_solve_stats(op.h, C.byref(hs), C.byref(dl)), "dk_op_solve_stats")
        self.host_syncs += int(hs.value)
        self.device_loop = bool(dl.value)
        cols = int(info.last_cols)
        self.hbar_full = hbar.T.copy()  # (m+1) x m, the cycle's columns before any drop
        if info.cycles > 0:
            Hfull, Gfull = hbar.T, gram.T  # (m+1) x m
            self.arnoldi = _DeviceArnoldi(op, op.serial, self.A.n, cols,
                                          Hfull[:cols + 1, :cols].copy(),
                                          Gfull[:cols + 1, :cols].copy())
        return cout

    def report(self, deflated_flags, warning=None, deflated_from=None, ritz=None) -> SolveReport:
        info = self.info
        it = int(info.iterations)
        if self.arnoldi is not None and (self.arnoldi.m + 1) * self.A.n <= (1 << 22):
            self.arnoldi.V  # small: copy now so the report outlives later solves
        ritz_cycles, ritz_iter = ritz if ritz is not None else ([], [])
        return SolveReport(
            x=self.x, converged=bool(info.converged), iterations=it,
            restarts=int(info.restarts), residual_history=self.hist[:it + 1].copy(),
            final_relres=float(info.final_relres), restart_of=self.rof[:it + 1].astype(np.int64),
            deflated_flags=np.asarray(deflated_flags, dtype=bool)[:it + 1], ritz_trace=ritz_cycles,
            ritz_iter_trace=ritz_iter, arnoldi=self.arnoldi,
            warning=warning if warning is not None else ("breakdown" if info.warning == 1
                                                         else None),
            deflated_from_cycle=deflated_from, solve_seconds=self.solve_seconds,
            kernel_launches=self.launches, reorthogonalisations=self.reorths,
            host_syncs=self.host_syncs, device_loop=self.device_loop)


def _ritz_of_cycle(H: np.ndarray, cols: int, n_iters: int):
    """krylov.py:185-187,208-210: smallest-|.| eigenvalue of H_{j+1} after every iteration of
    the cycle (H: the cycle's pristine Hessenberg), and the sorted Ritz set of H_cols."""
    per_iter = []
    for j in range(n_iters):
        th = np.linalg.eigvals(H[:j + 1, :j + 1])
        per_iter.append(th[np.argmin(np.abs(th))])
    th = np.linalg.eigvals(H[:cols, :cols])
    return th[np.argsort(np.abs(th))], per_iter


def _device_solve(A: SparseMatrix, b, x0, M, m, tol, max_iters, min_iters, ctx,
                  capture_ritz: bool = False) -> SolveReport:
    run = _Cycles(A, b, x0, M, m, tol, max_iters, min_iters)
    deflated = ctx is not None
    if not capture_ritz:
        run.run(ctx)
        it = int(run.info.iterations)
        return run.report(np.full(it + 1, deflated), deflated_from=0 if deflated else None)
    # one cycle per call: the Ritz data of each cycle is read before the next overwrites it
    ritz_cycles, ritz_iter = [], []
    it_before = 0
    while True:
        ctl = run.run(ctx, max_cycles=1)
        if run.info.cycles > len(ritz_cycles) and run.arnoldi is not None and run.arnoldi.m > 0:
            full, per_iter = _ritz_of_cycle(run.hbar_full, run.arnoldi.m,
                                            int(ctl.iterations) - it_before)
            ritz_cycles.append(full)
            ritz_iter.append(per_iter)
        it_before = int(ctl.iterations)
        if not ctl.running:
            break
    it = int(run.info.iterations)
    return run.report(np.full(it + 1, deflated), deflated_from=0 if deflated else None,
                      ritz=(ritz_cycles, ritz_iter))


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
    if x0 is not None:  # None: the device starts from zeros (no upload)
        x0 = np.ascontiguousarray(np.asarray(x0, dtype=np.float64))
    if x0 is not None and x0.shape != (A.n,):
        raise ValueError("initial guess has wrong length")
    if M is None:
        M = Preconditioner.identity()
    if m < 1:
        raise ValueError("cycle size must be >= 1")
    if tol <= 0:
        raise ValueError("tolerance must be positive")
    return _device_solve(A, b, x0, M, m, tol, max_iters, min_iters, deflation, capture_ritz)
