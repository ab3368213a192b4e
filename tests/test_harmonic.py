"""RDGMRES (harmonic-Ritz self-deflation), harmonic Ritz extraction, capture_ritz and dense
deflation bases — SURVEY §8f item 4.  Golden data: tests/golden/harmonic.npz, produced by the
reference (make_golden.make_harmonic); reference tests mirrored: tests/test_harmonic.py."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1510_02148_b200 as dk
from paper_1510_02148_b200.krylov import ArnoldiData

from conftest import rel


# ---- host-side extraction (no device) ------------------------------------------------------
def test_realify_cases():
    V = np.array([[1.0, 2.0], [3.0, 4.0]])
    np.testing.assert_allclose(dk.realify([1.0, 2.0], V), V)
    u = np.array([1.0 + 2.0j, -1.0j])
    out = dk.realify([0.5 + 1.0j, 0.5 - 1.0j], np.column_stack([u, np.conj(u)]))
    np.testing.assert_allclose(out[:, 0], u.real)
    np.testing.assert_allclose(out[:, 1], -u.imag)
    with pytest.raises(ValueError):
        dk.realify([1.0 + 1.0j], np.array([[1.0 + 1.0j], [0.0j]]))
    rng = np.random.default_rng(0)
    u = rng.standard_normal(6) + 1j * rng.standard_normal(6)
    w = rng.standard_normal(6)
    out = dk.realify([2.0 + 1.0j, 2.0 - 1.0j, 3.0], np.column_stack([u, np.conj(u), w]))
    assert out.shape == (6, 3)
    assert np.linalg.matrix_rank(np.column_stack([out, u.real, u.imag, w])) == 3


@pytest.mark.parametrize("d", [1, 4, 7])
def test_extraction_matches_reference_on_its_cycle(golden, d):
    """Both routes on the reference's own Arnoldi data reproduce its harmonic Ritz sets."""
    g = golden("harmonic")
    data = ArnoldiData(g["ad_V"], g["ad_H"], int(g["ad_m"]))
    hb = dk.harmonic_ritz_b(data, d)
    np.testing.assert_allclose(hb.thetas, g[f"hb{d}_thetas"], rtol=1e-12)
    np.testing.assert_allclose(hb.Y, g[f"hb{d}_Y"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(hb.Zvecs, g[f"hb{d}_Z"], rtol=1e-10, atol=1e-12)
    ha = dk.harmonic_ritz_a(data, d)
    np.testing.assert_allclose(ha.thetas, g[f"ha{d}_thetas"], rtol=1e-10)
    np.testing.assert_allclose(np.sort_complex(ha.thetas), np.sort_complex(hb.thetas),
                               rtol=1e-8, atol=1e-12)


def test_extraction_errors():
    data = ArnoldiData(np.eye(3), np.array([[1.0, 0.0], [1.0, 1.0], [0.0, 1.0]]), 2)
    with pytest.raises(ValueError):
        dk.harmonic_ritz_b(data, 5)
    with pytest.raises(dk.HarmonicRitzFailure):
        dk.harmonic_ritz_b(ArnoldiData(np.eye(3), np.zeros((3, 2)), 2), 1)


def test_rdgmres_invalid_parameters():
    A = dk.SparseMatrix.identity(5)
    b = np.ones(5)
    with pytest.raises(ValueError):
        dk.rdgmres(A, b, d=0)
    with pytest.raises(ValueError):
        dk.rdgmres(A, b, m=2, d=3)


# ---- device -------------------------------------------------------------------------------
def _sandwich(golden):
    g = golden("sandwich")
    return dk.SparseMatrix(len(g["b"]), g["ro"], g["ci"], g["va"]), g["b"]


def _hetero(golden):
    g = golden("hetero")
    return dk.SparseMatrix(len(g["b"]), g["ro"], g["ci"], g["va"]), g["b"]


def _check(rep, g, tag, x_tol=1e-8):
    assert abs(rep.iterations - int(g[f"{tag}_iters"])) <= 2
    assert rep.converged
    assert rel(rep.x, g[f"{tag}_x"]) <= x_tol
    flags = g[f"{tag}_flags"]
    it1 = int(np.argmax(flags)) - 1  # last undeflated history entry of the reference
    assert not rep.deflated_flags[:it1 + 1].any() and rep.deflated_flags[it1 + 1:].all()
    assert (rep.warning or "") == str(g[f"{tag}_warning"])


@pytest.mark.gpu
@pytest.mark.parametrize("tag,kw", [("s3", dict(m=40, d=3, tol=1e-6)),
                                    ("s2", dict(m=40, d=2, tol=1e-8)),
                                    ("s3j", dict(m=40, d=3, tol=1e-6, jacobi=True))])
def test_rdgmres_sandwich_matches_reference(gpu, golden, tag, kw):
    A, b = _sandwich(golden)
    g = golden("harmonic")
    M = dk.Preconditioner.jacobi(A) if kw.pop("jacobi", False) else None
    rep = dk.rdgmres(A, b, M=M, max_iters=300, **kw)
    _check(rep, g, tag, x_tol=1e-6 if kw["tol"] > 1e-8 else 1e-8)
    assert rep.deflated_from_cycle == int(g[f"{tag}_from"]) == 1
    # the first (plain) cycle matches the reference's history up to rounding; its plateau
    # sits at ~1e-9 of the initial residual, where CGS and MGS differ in the last digits
    h_ref = g[f"{tag}_history"]
    np.testing.assert_allclose(rep.residual_history[:41], h_ref[:41], rtol=1e-6,
                               atol=1e-6 * h_ref[0])


@pytest.mark.gpu
@pytest.mark.parametrize("tag,ap", [("h", "A"), ("hAM", "AM")])
def test_rdgmres_hetero_matches_reference(gpu, golden, tag, ap):
    A, b = _hetero(golden)
    g = golden("harmonic")
    rep = dk.rdgmres(A, b, M=dk.Preconditioner.jacobi(A), m=20, d=4, tol=1e-10, max_iters=2000,
                     A_p_choice=ap)
    _check(rep, g, tag)
    # first cycle is plain GMRES: identical to the reference up to rounding
    np.testing.assert_allclose(rep.residual_history[:21], g[f"{tag}_history"][:21], rtol=1e-9)


@pytest.mark.gpu
def test_rdgmres_without_restart_equals_gmres(gpu):
    """Converging inside the first cycle: no hook, identical to plain GMRES."""
    n = 300
    rng = np.random.default_rng(8)
    A = dk.SparseMatrix.from_dia(n, [-1, 0, 1], np.vstack([
        -rng.uniform(0.5, 1.0, n), rng.uniform(3.0, 4.0, n), -rng.uniform(0.5, 1.0, n)]))
    b = rng.standard_normal(n)
    plain = dk.gmres(A, b, m=60, tol=1e-10, max_iters=300)
    r = dk.rdgmres(A, b, m=60, d=2, tol=1e-10, max_iters=300)
    assert plain.iterations <= 60 and r.iterations == plain.iterations
    assert r.deflated_from_cycle is None and not r.deflated_flags.any()
    np.testing.assert_array_equal(r.x, plain.x)


@pytest.mark.gpu
def test_rdgmres_stops_at_max_iters_inside_first_cycle(gpu, golden):
    """max_iters inside cycle 1: the hook still engages and x is reconstructed
    (krylov.py:213-221), as in the reference."""
    A, b = _hetero(golden)
    rep = dk.rdgmres(A, b, M=dk.Preconditioner.jacobi(A), m=20, d=2, tol=1e-12, max_iters=20)
    assert rep.iterations == 20 and not rep.converged
    assert rep.deflated_from_cycle == 1
    assert len(rep.residual_history) == 21


@pytest.mark.gpu
def test_capture_ritz_traces_match_reference(gpu, golden):
    A, b = _hetero(golden)
    g = golden("harmonic")
    rep = dk.gmres(A, b, M=dk.Preconditioner.jacobi(A), m=20, tol=1e-10, max_iters=60,
                   capture_ritz=True)
    assert rep.iterations == int(g["cr_iters"])
    np.testing.assert_array_equal([len(t) for t in rep.ritz_trace], g["cr_cycles"])
    got = np.concatenate(rep.ritz_trace)
    np.testing.assert_allclose(np.abs(got), np.abs(g["cr_trace"]), rtol=1e-7)
    it = np.concatenate([np.asarray(t) for t in rep.ritz_iter_trace])
    np.testing.assert_allclose(np.abs(it), np.abs(g["cr_iter_trace"]), rtol=1e-7)


@pytest.mark.gpu
def test_device_gram_drives_the_same_extraction(gpu, golden):
    """harmonic_ritz_b on device cycle data (device Gram matrix) equals the extraction from the
    copied basis (V V_m^T on the host)."""
    A, b = _hetero(golden)
    rep = dk.gmres(A, b, M=dk.Preconditioner.jacobi(A), m=20, tol=1e-14, max_iters=20)
    dev = rep.arnoldi
    host = ArnoldiData(dev.V, dev.Hbar, dev.m)
    np.testing.assert_allclose(dev.gram, host.V @ host.V[:host.m].T, atol=1e-12)
    for d in (1, 3, 6):
        np.testing.assert_allclose(np.sort_complex(dk.harmonic_ritz_b(dev, d).thetas),
                                   np.sort_complex(dk.harmonic_ritz_b(host, d).thetas),
                                   rtol=1e-9)


@pytest.mark.gpu
def test_dense_basis_context_matches_reference(gpu, golden):
    A, b = _hetero(golden)
    g = golden("harmonic")
    M = dk.Preconditioner.jacobi(A)
    basis = dk.DeflationBasis(g["dz_Z"])
    assert not basis.is_indicator
    ctx = dk.build_context(A, M, basis, b)
    E, _ = ctx.coarse_matrix()
    assert rel(E, g["dz_E"]) < 1e-12
    assert rel(ctx.apply_p1(g["dz_v"]), g["dz_p1v"]) < 1e-10
    assert rel(ctx.apply_p2(g["dz_v"]), g["dz_p2v"]) < 1e-10
    assert rel(ctx.x_star, g["dz_xs"]) < 1e-10
    rep = dk.pdgmres(A, b, M=M, m=20, basis=basis, tol=1e-10, max_iters=2000)
    assert abs(rep.iterations - int(g["dz_iters"])) <= 2
    assert rel(rep.x, g["dz_x"]) <= 1e-8


@pytest.mark.gpu
def test_dense_basis_limits_and_singularity(gpu, golden):
    A, b = _hetero(golden)
    rng = np.random.default_rng(3)
    Z = rng.standard_normal((A.n, 3))
    Z[:, 2] = Z[:, 0]  # dependent columns: E is singular (sparse.py:135-136)
    with pytest.raises(dk.SingularCoarseMatrix):
        dk.build_context(A, dk.Preconditioner.identity(), dk.DeflationBasis(Z), b)
    with pytest.raises(dk.UnsupportedOperator):
        dk.build_context(A, dk.Preconditioner.identity(),
                         dk.DeflationBasis(rng.standard_normal((A.n, 65))), b)
