"""Acceptance mirrors: the reference's headline claims for the hot path
(pkg/tests/test_acceptance.py), run through the device solver.

Random operators are drawn on a seven-diagonal band (see test_reference_mirror.py); the
physics cases are the reference's own (sandwich, steam-chamber column), assembled here.
"""
from __future__ import annotations

import time

import numpy as np
import pytest

import paper_1510_02148_b200 as dk

from test_reference_mirror import banded

pytestmark = pytest.mark.gpu


def sandwich_problem(sigma=1e6, nx=7, ny=7, nz=3):
    """High-low-high layers with a corner injector/producer pair, diagonally scaled
    (reference conftest.py:8-18)."""
    grid = dk.Grid(nx, ny, nz)
    field = dk.make_layered_field(grid, [((0, 1), sigma), ((1, 2), 1.0), ((2, 3), sigma)])
    q = np.zeros(grid.n_cells)
    q[0], q[-1] = 1.0, -1.0
    return dk.diagonal_scale(dk.assemble_pressure(field, dk.BoundarySpec(), q)), field


def sagd_case():
    """Steam-chamber-style column (test_acceptance.py:31-43)."""
    grid = dk.Grid(41, 1, 85)
    bands = [((0, 10), 0.0), ((75, 85), 0.0), ((10, 22), 1.0), ((62, 75), 1.0)]
    for i in range(10):
        bands.append(((22 + 4 * i, 26 + 4 * i), (1.0, 1e-3)[i % 2]))
    field = dk.make_sagd_like_field(grid, bands)
    q = np.zeros(grid.n_cells)
    q[grid.index(20, 0, 24)], q[grid.index(20, 0, 23)] = 1.0, -1.0
    return dk.diagonal_scale(dk.assemble_pressure(field, dk.BoundarySpec(), q)), grid


def test_projector_identities_hold_on_random_cases(gpu):
    """Dense-oracle agreement, idempotence, intertwining and annihilation over 100 draws
    (test_acceptance.py:170-201)."""
    rng = np.random.default_rng(11)
    for _ in range(100):
        n = int(rng.integers(8, 25))
        d = int(rng.integers(1, min(6, n // 2 + 1)))
        Ad = banded(rng, n, 2.0)
        Z = rng.standard_normal((n, d))
        A = dk.SparseMatrix.from_dense(Ad)
        b = rng.standard_normal(n)
        ctx = dk.build_context(A, dk.Preconditioner.identity(), dk.DeflationBasis(Z), b)
        Einv = np.linalg.inv(Z.T @ Ad @ Z)
        P1 = np.eye(n) - Ad @ Z @ Einv @ Z.T
        P2 = np.eye(n) - Z @ Einv @ Z.T @ Ad
        v = rng.standard_normal(n)
        s = max(1.0, float(np.linalg.norm(v)))
        p1v, p2v = ctx.apply_p1(v), ctx.apply_p2(v)
        assert np.linalg.norm(p1v - P1 @ v) <= 1e-10 * s
        assert np.linalg.norm(p2v - P2 @ v) <= 1e-10 * s
        assert np.linalg.norm(ctx.apply_p1(p1v) - p1v) <= 1e-10 * s
        assert np.linalg.norm(ctx.apply_p2(p2v) - p2v) <= 1e-10 * s
        assert (np.linalg.norm(ctx.apply_p1(dk.spmv(A, v)) - dk.spmv(A, p2v))
                <= 1e-10 * s * np.linalg.norm(Ad))
        assert np.linalg.norm(Z.T @ p1v) <= 1e-10 * s * np.linalg.norm(Z)
        for j in range(d):
            assert (np.linalg.norm(ctx.apply_p2(Z[:, j]))
                    <= 1e-10 * np.linalg.norm(Z[:, j]) * np.linalg.norm(Ad))


def test_deflated_residuals_dominate_plain_gmres(gpu):
    """Exact eigenvectors as deflation vectors: the deflated residual never exceeds the plain
    one (test_acceptance.py:138-167)."""
    rng = np.random.default_rng(7)
    for _ in range(6):
        n = int(rng.integers(30, 90))
        Ad = banded(rng, n, 2.0)
        A = dk.SparseMatrix.from_dense(Ad)
        b = rng.standard_normal(n)
        w, V = np.linalg.eig(Ad)
        order = np.argsort(np.abs(w))
        for d in (1, 2, 3):
            k = d
            while True:  # widen so conjugate pairs stay whole
                th = w[order[:k]]
                if abs(th[-1].imag) < 1e-12 or any(abs(th[j] - np.conj(th[-1])) < 1e-8
                                                   for j in range(k - 1)):
                    break
                k += 1
            Z = dk.realify(w[order[:k]], V[:, order[:k]])
            ctx = dk.build_context(A, dk.Preconditioner.identity(), dk.DeflationBasis(Z), b)
            plain = dk.gmres(A, b, m=n, tol=1e-14, max_iters=n)
            defl = dk.gmres(A, b, m=n, tol=1e-14, max_iters=n, deflation=ctx)
            L = min(len(plain.residual_history), len(defl.residual_history))
            assert np.all(defl.residual_history[:L]
                          <= plain.residual_history[:L] * (1 + 1e-8))


def test_cycle_size_gates_ritz_deflation(gpu):
    """Contrast 1e8: RDGMRES needs cycle size 40; 20 stalls (test_acceptance.py:204-211)."""
    p, _ = sandwich_problem(1e8)
    short = dk.rdgmres(p.A, p.b, m=20, d=3, tol=1e-6, max_iters=300)
    long = dk.rdgmres(p.A, p.b, m=40, d=3, tol=1e-6, max_iters=300)
    assert not short.converged and long.converged


def test_manual_layer_deflation_halves_sagd_iterations(gpu):
    """Ten manual layer vectors cut iterations to <= 0.6x plain GMRES
    (test_acceptance.py:214-226)."""
    p, grid = sagd_case()
    M = dk.Preconditioner.jacobi(p.A)
    plain = dk.gmres(p.A, p.b, M=M, m=100, tol=1e-6, max_iters=1500)
    basis = dk.partition_to_basis(
        dk.manual_layers(grid, [(22 + 4 * i, 26 + 4 * i) for i in range(10)]))
    defl = dk.pdgmres(p.A, p.b, M=M, m=100, basis=basis, tol=1e-6, max_iters=1500)
    assert plain.converged and defl.converged and basis.d == 10
    assert defl.iterations <= 0.6 * plain.iterations


def test_method_ordering_on_sandwich(gpu):
    """Physics deflation beats self-deflating restarts, which beat plain restarted GMRES
    (test_acceptance.py:229-240)."""
    p, field = sandwich_problem(1e6)
    basis = dk.partition_to_basis(dk.levelset_partition(field))
    pd = dk.pdgmres(p.A, p.b, m=20, basis=basis, tol=1e-6, max_iters=300)
    rd = dk.rdgmres(p.A, p.b, m=40, d=3, tol=1e-6, max_iters=300)
    plain = dk.gmres(p.A, p.b, m=20, tol=1e-6, max_iters=300)
    assert pd.converged and rd.converged
    assert pd.iterations < rd.iterations < plain.iterations


def test_deflation_saves_wall_time(gpu):
    """Physics deflation wins on wall time on the sandwich problem
    (test_acceptance.py:276-...)."""
    p, field = sandwich_problem(1e6)
    basis3 = dk.partition_to_basis(dk.levelset_partition(field))

    def timed(fn):
        fn()
        samples = []
        for _ in range(5):
            t0 = time.perf_counter()
            fn()
            samples.append(time.perf_counter() - t0)
        return sorted(samples)[2]

    t_plain = timed(lambda: dk.gmres(p.A, p.b, m=100, tol=1e-6, max_iters=300))
    t_defl = timed(lambda: dk.pdgmres(p.A, p.b, m=20, basis=basis3, tol=1e-6, max_iters=300))
    assert t_defl < t_plain
