"""Mirrors of the reference's unit tests for the hot path (pkg/tests/test_krylov.py,
test_deflation.py) that the golden-vector tests do not already cover.

The reference draws dense random matrices (np.eye(n) * c + noise); the device path takes at
most seven diagonals (include/dk.h), so the mirrors draw the same distribution restricted to
a seven-diagonal band.  Dense operators themselves raise UnsupportedOperator
(test_device_ops.py::test_more_than_seven_diagonals_is_unsupported).
"""
from __future__ import annotations

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1510_02148_b200 as dk

OFFSETS = (-4, -2, -1, 0, 1, 2, 4)


def banded(rng, n, diag):
    """diag * I + N(0, 1/n) noise on the seven-diagonal band (reference: well_conditioned,
    test_krylov.py:10-12; random_case, test_deflation.py:11-16)."""
    A = np.eye(n) * diag
    for k in OFFSETS:
        if abs(k) < n:
            A += np.diag(rng.standard_normal(n - abs(k)) / np.sqrt(n), k)
    return A


def random_case(seed, n=20, d=3):
    rng = np.random.default_rng(seed)
    Ad = banded(rng, n, 2.0)
    Z = rng.standard_normal((n, d))
    b = rng.standard_normal(n)
    return dk.SparseMatrix.from_dense(Ad), Ad, Z, b


def dense_projectors(Ad, Z):
    Einv = np.linalg.inv(Z.T @ Ad @ Z)
    n = len(Ad)
    return (np.eye(n) - Ad @ Z @ Einv @ Z.T, np.eye(n) - Z @ Einv @ Z.T @ Ad)


def well_conditioned(rng, n):
    return dk.SparseMatrix.from_dense(banded(rng, n, 3.0))


# ---- host-only: basis / context argument checks (test_deflation.py:28-59, :104-109) --------
def test_basis_shape_recorded_and_rejects_empty():
    Z = dk.DeflationBasis(np.ones((6, 2)))
    assert (Z.n, Z.d) == (6, 2)
    with pytest.raises(ValueError):
        dk.DeflationBasis(np.ones((6, 0)))
    with pytest.raises(ValueError):
        dk.DeflationBasis(np.ones(6))


def test_none_context_is_identity():
    v = np.arange(5.0)
    np.testing.assert_array_equal(dk.apply_p1(None, v), v)
    np.testing.assert_array_equal(dk.apply_p2(None, v), v)
    np.testing.assert_array_equal(dk.reconstruct(None, v), v)


def test_context_dimension_and_operator_choice_checks():
    A, _, Z, b = random_case(1)
    I = dk.Preconditioner.identity()
    with pytest.raises(ValueError):
        dk.build_context(A, I, dk.DeflationBasis(Z[:-1]), b)
    with pytest.raises(ValueError):
        dk.build_context(A, I, dk.DeflationBasis(Z), b[:-1])
    with pytest.raises(ValueError):
        dk.build_context(A, I, dk.DeflationBasis(Z), b, A_p_choice="B")


# ---- device: deflation context (test_deflation.py:40-142) ---------------------------------
@pytest.mark.gpu
def test_dependent_columns_raise(gpu):
    A, _, Z, b = random_case(0)
    Z[:, 1] = Z[:, 0]
    with pytest.raises(dk.SingularCoarseMatrix):
        dk.build_context(A, dk.Preconditioner.identity(), dk.DeflationBasis(Z), b)


@pytest.mark.gpu
def test_coarse_solution_in_span(gpu):
    A, _, Z, b = random_case(3)
    ctx = dk.build_context(A, dk.Preconditioner.identity(), dk.DeflationBasis(Z), b)
    resid = ctx.x_star - Z @ np.linalg.lstsq(Z, ctx.x_star, rcond=None)[0]
    assert np.linalg.norm(resid) < 1e-10


@pytest.mark.gpu
@settings(max_examples=25, deadline=None)
@given(st.integers(0, 2**31), st.integers(1, 5))
def test_p1_p2_against_dense_oracle(gpu, seed, d):
    A, Ad, Zfull, b = random_case(seed, n=18, d=5)
    Z = Zfull[:, :d]
    ctx = dk.build_context(A, dk.Preconditioner.identity(), dk.DeflationBasis(Z), b)
    P1, P2 = dense_projectors(Ad, Z)
    v = np.random.default_rng(seed + 1).standard_normal(18)
    np.testing.assert_allclose(ctx.apply_p1(v), P1 @ v, atol=1e-10)
    np.testing.assert_allclose(ctx.apply_p2(v), P2 @ v, atol=1e-10)


@pytest.mark.gpu
def test_idempotence_annihilation_and_commutation(gpu):
    A, _, Z, b = random_case(7)
    ctx = dk.build_context(A, dk.Preconditioner.identity(), dk.DeflationBasis(Z), b)
    v = np.random.default_rng(8).standard_normal(20)
    p1v, p2v = ctx.apply_p1(v), ctx.apply_p2(v)
    np.testing.assert_allclose(ctx.apply_p1(p1v), p1v, atol=1e-10)
    np.testing.assert_allclose(ctx.apply_p2(p2v), p2v, atol=1e-10)
    np.testing.assert_allclose(Z.T @ p1v, 0.0, atol=1e-10)
    for j in range(Z.shape[1]):
        np.testing.assert_allclose(ctx.apply_p2(Z[:, j]), 0.0, atol=1e-10)
    np.testing.assert_allclose(ctx.apply_p1(dk.spmv(A, v)), dk.spmv(A, p2v), atol=1e-10)


@pytest.mark.gpu
def test_helpers_delegate(gpu):
    A, _, Z, b = random_case(11)
    ctx = dk.build_context(A, dk.Preconditioner.identity(), dk.DeflationBasis(Z), b)
    v = np.random.default_rng(12).standard_normal(20)
    np.testing.assert_array_equal(dk.apply_p1(ctx, v), ctx.apply_p1(v))
    np.testing.assert_array_equal(dk.apply_p2(ctx, v), ctx.apply_p2(v))


@pytest.mark.gpu
def test_reconstructed_solution_solves_system(gpu):
    A, _, Z, b = random_case(13)
    ctx = dk.build_context(A, dk.Preconditioner.identity(), dk.DeflationBasis(Z), b)
    rep = dk.gmres(A, b, m=20, tol=1e-12, deflation=ctx)
    assert rep.converged
    assert np.linalg.norm(dk.spmv(A, rep.x) - b) < 1e-9 * np.linalg.norm(b)


@pytest.mark.gpu
def test_am_variant_coincides_with_a_under_identity(gpu):
    A, _, Z, b = random_case(14)
    M = dk.Preconditioner.identity()
    ctx_a = dk.build_context(A, M, dk.DeflationBasis(Z), b, A_p_choice="A")
    ctx_am = dk.build_context(A, M, dk.DeflationBasis(Z), b, A_p_choice="AM")
    v = np.random.default_rng(15).standard_normal(20)
    np.testing.assert_allclose(ctx_am.apply_p1(v), ctx_a.apply_p1(v), atol=1e-12)
    np.testing.assert_allclose(ctx_am.apply_p2(v), ctx_a.apply_p2(v), atol=1e-12)
    rep = dk.gmres(A, b, M=M, m=20, tol=1e-12, deflation=ctx_am)
    assert rep.converged
    assert np.linalg.norm(dk.spmv(A, rep.x) - b) < 1e-9 * np.linalg.norm(b)


# ---- device: GMRES (test_krylov.py:36-175) ------------------------------------------------
@pytest.mark.gpu
def test_solves_to_tolerance(gpu):
    rng = np.random.default_rng(1)
    A = well_conditioned(rng, 40)
    b = rng.standard_normal(40)
    rep = dk.gmres(A, b, m=20, tol=1e-10)
    assert rep.converged and rep.final_relres <= 1e-10
    assert np.linalg.norm(b - dk.spmv(A, rep.x)) <= 1e-9 * np.linalg.norm(b)


@pytest.mark.gpu
def test_restart_counted(gpu):
    rng = np.random.default_rng(3)
    A = well_conditioned(rng, 30)
    b = rng.standard_normal(30)
    rep = dk.gmres(A, b, m=5, tol=1e-12, max_iters=100)
    assert rep.restarts >= 1
    assert rep.iterations + 1 == len(rep.residual_history)


@pytest.mark.gpu
def test_identity_with_min_iters_and_x0_respected(gpu):
    rep = dk.gmres(dk.SparseMatrix.identity(10), np.ones(10), m=10, tol=1e-6, min_iters=3)
    assert rep.iterations >= 1
    rng = np.random.default_rng(5)
    A = well_conditioned(rng, 20)
    xtrue = rng.standard_normal(20)
    rep = dk.gmres(A, dk.spmv(A, xtrue), x0=xtrue, m=20, tol=1e-10)
    assert rep.converged and rep.iterations == 0


@pytest.mark.gpu
def test_right_preconditioning_equivalent_solution(gpu):
    rng = np.random.default_rng(6)
    A = well_conditioned(rng, 30)
    b = rng.standard_normal(30)
    plain = dk.gmres(A, b, m=30, tol=1e-10)
    jac = dk.gmres(A, b, M=dk.Preconditioner.jacobi(A), m=30, tol=1e-10)
    np.testing.assert_allclose(plain.x, jac.x, rtol=1e-6, atol=1e-9)


@pytest.mark.gpu
@settings(max_examples=15, deadline=None)
@given(st.integers(0, 2**31), st.integers(min_value=5, max_value=30))
def test_residual_never_increases_at_cycle_granularity(gpu, seed, n):
    rng = np.random.default_rng(seed)
    A = well_conditioned(rng, n)
    b = rng.standard_normal(n)
    rep = dk.gmres(A, b, m=max(3, n // 3), tol=1e-10, max_iters=6 * n)
    h = rep.residual_history
    for s in np.flatnonzero(np.diff(rep.restart_of)) + 1:
        assert h[s] <= h[s - 1] * (1 + 1e-8)


@pytest.mark.gpu
def test_arnoldi_relation_and_orthonormal_basis(gpu):
    rng = np.random.default_rng(7)
    A = well_conditioned(rng, 20)
    b = rng.standard_normal(20)
    data = dk.gmres(A, b, m=8, tol=1e-16, max_iters=8).arnoldi
    AV = np.column_stack([dk.spmv(A, v) for v in data.V[:data.m]])
    np.testing.assert_allclose(AV, data.V.T @ data.Hbar, atol=1e-10)
    np.testing.assert_allclose(data.V @ data.V.T, np.eye(len(data.V)), atol=1e-8)


@pytest.mark.gpu
def test_ritz_values_match_dense_oracle(gpu):
    rng = np.random.default_rng(9)
    A = well_conditioned(rng, 15)
    b = rng.standard_normal(15)
    data = dk.gmres(A, b, m=15, tol=1e-14, max_iters=15).arnoldi
    if data.m == 15:  # full Krylov space: Ritz values = eigenvalues
        w = np.sort_complex(dk.ritz_values(data))
        true = np.sort_complex(np.linalg.eigvals(A.to_dense()))
        np.testing.assert_allclose(w, true, rtol=1e-8)


@pytest.mark.gpu
def test_capture_ritz_traces_shapes(gpu):
    rng = np.random.default_rng(10)
    A = well_conditioned(rng, 20)
    b = rng.standard_normal(20)
    rep = dk.gmres(A, b, m=6, tol=1e-12, max_iters=30, capture_ritz=True)
    assert len(rep.ritz_trace) >= 1
    assert len(rep.ritz_iter_trace) == len(rep.ritz_trace)
    for per_iter, full in zip(rep.ritz_iter_trace, rep.ritz_trace):
        assert len(full) >= 1 and len(per_iter) >= 1
