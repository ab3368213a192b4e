"""The reference's public LU helpers (sparse.py:109-145) and DeflationContext.E_lu
(deflation.py:46), computed on the device (dk_dense_lu / dk_lu_solve).

Mirrors pkg/tests/test_sparse.py:80-96 and checks the LAPACK getrf layout (lu, piv) against
scipy.linalg.lu_factor — the routine the reference's dense_lu calls — across the device
factorisation's panel edges (32-wide steps, 256-wide outer panels).
"""
from __future__ import annotations

import numpy as np
import pytest
import scipy.linalg

import paper_1510_02148_b200 as dk


# ---- host-side contract (CPU) ------------------------------------------------------------
def test_dense_lu_argument_errors_and_empty():
    with pytest.raises(ValueError):
        dk.dense_lu(np.ones((2, 3)))
    with pytest.raises(ValueError):
        dk.dense_lu(np.ones(4))
    with pytest.raises(ValueError):
        dk.dense_lu(np.array([[1.0, np.nan], [0.0, 1.0]]))
    f = dk.dense_lu(np.zeros((0, 0)))
    assert f.n == 0 and f.lu.shape == (0, 0) and f.piv.dtype == np.int32
    np.testing.assert_array_equal(dk.lu_solve(f, np.zeros(0)), np.zeros(0))


# ---- device (GPU) ------------------------------------------------------------------------
@pytest.mark.gpu
def test_solve_matches_numpy(gpu):
    rng = np.random.default_rng(2)
    E = rng.standard_normal((6, 6)) + 6 * np.eye(6)
    rhs = rng.standard_normal(6)
    lu = dk.dense_lu(E)
    np.testing.assert_allclose(dk.lu_solve(lu, rhs), np.linalg.solve(E, rhs), rtol=1e-12)


@pytest.mark.gpu
def test_singular_raises(gpu):
    with pytest.raises(dk.SingularCoarseMatrix):
        dk.dense_lu(np.zeros((3, 3)))


@pytest.mark.gpu
def test_rank_deficient_raises(gpu):
    E = np.outer(np.arange(1.0, 5.0), np.arange(1.0, 5.0))
    with pytest.raises(dk.SingularCoarseMatrix):
        dk.dense_lu(E)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 255, 256, 257, 300, 530])
def test_getrf_layout_matches_scipy(gpu, n):
    """Same pivots as LAPACK (first row of maximal |a|), same combined factors to rounding."""
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n))
    f = dk.dense_lu(A)
    lu, piv = scipy.linalg.lu_factor(A)
    np.testing.assert_array_equal(f.piv, piv)
    np.testing.assert_allclose(f.lu, lu, rtol=1e-9, atol=1e-9 * np.abs(lu).max())
    # P A = L U
    L = np.tril(f.lu, -1) + np.eye(n)
    U = np.triu(f.lu)
    PA = A.copy()
    for k, p in enumerate(f.piv):
        PA[[k, p]] = PA[[p, k]]
    np.testing.assert_allclose(L @ U, PA, atol=1e-12 * n * np.abs(A).max())


@pytest.mark.gpu
@pytest.mark.parametrize("n,k", [(40, 1), (300, 3), (513, 7)])
def test_lu_solve_vectors_and_stacked(gpu, n, k):
    rng = np.random.default_rng(n + k)
    A = rng.standard_normal((n, n)) + n ** 0.5 * np.eye(n)
    B = rng.standard_normal((n, k))
    f = dk.dense_lu(A)
    X = dk.lu_solve(f, B)
    assert X.shape == (n, k)
    np.testing.assert_allclose(X, scipy.linalg.lu_solve(scipy.linalg.lu_factor(A), B),
                               rtol=1e-10, atol=1e-12)
    x = dk.lu_solve(f, B[:, 0])
    assert x.shape == (n,)
    np.testing.assert_allclose(x, X[:, 0], rtol=1e-13, atol=1e-15)
    # the reference's own factors (scipy) drive the device solve too
    lu, piv = scipy.linalg.lu_factor(A)
    np.testing.assert_allclose(dk.lu_solve(dk.LUFactors(lu, piv), B), X, rtol=1e-10,
                               atol=1e-12)


@pytest.mark.gpu
def test_context_E_lu(gpu, golden):
    """ctx.E_lu: the getrf factors of E = Z^T A Z; lu_solve with them gives E^-1 Z^T b."""
    g = golden("hetero")
    A = dk.SparseMatrix(len(g["b"]), g["ro"], g["ci"], g["va"])
    M = dk.Preconditioner.jacobi(A)
    p = dk.Partition(g["labels"], int(g["d"]), "subdomain_levelset",
                     frozenset(int(e) for e in g["excl"]))
    basis = dk.partition_to_basis(p)
    ctx = dk.build_context(A, M, basis, g["b"])
    try:
        f = ctx.E_lu
        assert isinstance(f, dk.LUFactors) and f.n == basis.d
        lu, piv = scipy.linalg.lu_factor(g["E"])
        np.testing.assert_array_equal(f.piv, piv)
        np.testing.assert_allclose(f.lu, lu, rtol=1e-10, atol=1e-12 * np.abs(lu).max())
        rhs = np.bincount(basis.labels[basis.labels >= 0], weights=g["b"][basis.labels >= 0],
                          minlength=basis.d)
        y = dk.lu_solve(f, rhs)
        np.testing.assert_allclose(y, np.linalg.solve(g["E"], rhs), rtol=1e-9)
    finally:
        ctx.close()
