"""Device building blocks against the reference goldens and the CPU oracle (GPU)."""
from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sp

import paper_1510_02148_b200 as dk
from conftest import rel
from oracle import dk_oracle as O

pytestmark = pytest.mark.gpu


def _hetero(golden):
    g = golden("hetero")
    A = dk.SparseMatrix(len(g["b"]), g["ro"], g["ci"], g["va"])
    return g, A, sp.csr_matrix((g["va"], g["ci"], g["ro"]))


def test_spmv_bit_identical_to_csr(gpu, golden):
    g, A, Ac = _hetero(golden)
    rng = np.random.default_rng(1)
    for _ in range(3):
        x = rng.standard_normal(A.n) * 10.0 ** rng.uniform(-5, 5, A.n)
        np.testing.assert_array_equal(dk.spmv(A, x), Ac @ x)


def test_spmv_linearity_and_shapes(gpu, golden):
    g, A, _ = _hetero(golden)
    rng = np.random.default_rng(2)
    x, y = rng.standard_normal(A.n), rng.standard_normal(A.n)
    np.testing.assert_allclose(dk.spmv(A, 2.0 * x - 3.0 * y),
                               2.0 * dk.spmv(A, x) - 3.0 * dk.spmv(A, y), atol=1e-9)
    with pytest.raises(ValueError):
        dk.spmv(A, np.ones(A.n + 1))


def _ctx(g, A, ap="A"):
    M = dk.Preconditioner.jacobi(A)
    col, dd = O.columns_from_labels(g["labels"], int(g["d"]), g["excl"])
    return dk.build_context(A, M, dk.DeflationBasis(labels=col, d=dd), g["b"], A_p_choice=ap), M


def test_coarse_matrix_and_inverse(gpu, golden):
    g, A, _ = _hetero(golden)
    ctx, _ = _ctx(g, A)
    E, Einv = ctx.coarse_matrix()
    np.testing.assert_allclose(E, g["E"], rtol=1e-12, atol=1e-13 * np.abs(g["E"]).max())
    np.testing.assert_allclose(Einv @ g["E"], np.eye(E.shape[0]), atol=1e-10)


def test_projectors_match_reference(gpu, golden):
    g, A, _ = _hetero(golden)
    ctx, _ = _ctx(g, A)
    scale = np.abs(g["p1v"]).max()
    np.testing.assert_allclose(ctx.apply_p1(g["v"]), g["p1v"], atol=1e-12 * scale)
    np.testing.assert_allclose(ctx.apply_p2(g["v"]), g["p2v"], atol=1e-12)
    np.testing.assert_allclose(ctx.reconstruct(g["v"]), g["rec"], atol=1e-12)
    np.testing.assert_allclose(ctx.x_star, g["x_star"], atol=1e-12)


def test_projector_identities(gpu, golden):
    """Idempotence, Z^T P1 = 0, P2 Z = 0 and P1 A = A P2 (reference test_deflation.py:82-113)."""
    g, A, Ac = _hetero(golden)
    ctx, _ = _ctx(g, A)
    lab = ctx.basis.labels
    keep = lab >= 0
    v = np.random.default_rng(8).standard_normal(A.n)
    p1v = ctx.apply_p1(v)
    np.testing.assert_allclose(ctx.apply_p1(p1v), p1v, atol=1e-10 * np.abs(v).max())
    restr = np.bincount(lab[keep], weights=p1v[keep], minlength=ctx.d)
    assert np.abs(restr).max() < 1e-9 * np.abs(v).max()
    p2v = ctx.apply_p2(v)
    np.testing.assert_allclose(ctx.apply_p2(p2v), p2v, atol=1e-10)
    for j in range(min(ctx.d, 4)):
        zj = (lab == j).astype(float)
        np.testing.assert_allclose(ctx.apply_p2(zj), 0.0, atol=1e-10)
    np.testing.assert_allclose(ctx.apply_p1(Ac @ v), Ac @ ctx.apply_p2(v),
                               atol=1e-9 * np.abs(Ac @ v).max())


def test_am_variant_matches_oracle(gpu, golden):
    g, A, Ac = _hetero(golden)
    ctx, M = _ctx(g, A, ap="AM")
    defl = O.LabelDeflation(Ac, ctx.basis.labels, ctx.d, g["b"], M.inv_diag, ap="AM")
    v = np.random.default_rng(4).standard_normal(A.n)
    np.testing.assert_allclose(ctx.apply_p1(v), defl.apply_p1(v), atol=1e-10 * np.abs(v).max())
    np.testing.assert_allclose(ctx.apply_p2(v), defl.apply_p2(v), atol=1e-10)


def test_singular_coarse_matrix_raises(gpu):
    """An empty indicator column makes E exactly singular (reference sparse.py:135-136)."""
    A = dk.SparseMatrix.from_dia(6, [-1, 0, 1], np.vstack([-np.ones(6), 3 * np.ones(6),
                                                          -np.ones(6)]))
    Z = np.zeros((6, 2))
    Z[:, 0] = 1.0
    with pytest.raises(dk.SingularCoarseMatrix):
        dk.build_context(A, dk.Preconditioner.identity(), dk.DeflationBasis(Z), np.ones(6))
    Zd = np.zeros((6, 2))
    Zd[:3, 0] = Zd[:3, 1] = 1.0   # two equal columns: dependent
    with pytest.raises(dk.SingularCoarseMatrix):
        dk.build_context(A, dk.Preconditioner.identity(), dk.DeflationBasis(Zd), np.ones(6))


def test_context_argument_errors(gpu, golden):
    g, A, _ = _hetero(golden)
    M = dk.Preconditioner.jacobi(A)
    B = dk.DeflationBasis(labels=np.zeros(A.n, dtype=np.int32), d=1)
    with pytest.raises(ValueError):
        dk.build_context(A, M, B, g["b"], A_p_choice="B")
    with pytest.raises(ValueError):
        dk.build_context(A, M, dk.DeflationBasis(labels=np.zeros(A.n - 1, dtype=np.int32), d=1),
                         g["b"])
    with pytest.raises(ValueError):
        dk.build_context(A, M, B, g["b"][:-1])
    with pytest.raises(ValueError):
        dk.DeflationBasis(np.ones((6, 0)))


def test_large_coarse_system_lu_matches_numpy(gpu):
    """d = 1,500 columns (many LU panels): E^-1 against numpy's inverse."""
    from paper_1510_02148_b200 import configs
    c = configs.make_case(3)
    A, b = c.problem()
    p = c.partition()
    basis = dk.partition_to_basis(p)
    # restrict to the first 1500 columns by relabelling the rest to -1
    lab = basis.labels.copy()
    lab[lab >= 1500] = -1
    ctx = dk.build_context(A, dk.Preconditioner.jacobi(A), dk.DeflationBasis(labels=lab, d=1500),
                           b)
    E, Einv = ctx.coarse_matrix()
    ref = np.linalg.inv(E)
    assert rel(Einv, ref) < 1e-10
    np.testing.assert_allclose(E, E.T, rtol=0, atol=1e-12 * np.abs(E).max())
    # the projector through the symmetric packed coarse solve (d >= 256) vs the oracle
    off, dg = A.dia()
    Ac = O.csr_from_dia(A.n, off, dg)
    defl = O.LabelDeflation(Ac, lab, 1500, b, 1.0 / A.diagonal())
    v = np.random.default_rng(3).standard_normal(A.n)
    assert rel(ctx.apply_p1(v), defl.apply_p1(v)) < 1e-10
    assert rel(ctx.apply_p2(v), defl.apply_p2(v)) < 1e-10
    np.testing.assert_allclose(ctx.x_star, defl.x_star, rtol=1e-9, atol=1e-12)


def test_large_nonsymmetric_coarse_system_lu(gpu):
    """A_p = A M (nonsymmetric E, d = 1,500): the pivoted-LU inverse on the tensor-core GEMM."""
    from paper_1510_02148_b200 import configs
    c = configs.make_case(3)
    A, b = c.problem()
    lab = dk.partition_to_basis(c.partition()).labels.copy()
    lab[lab >= 1500] = -1
    ctx = dk.build_context(A, dk.Preconditioner.jacobi(A), dk.DeflationBasis(labels=lab, d=1500),
                           b, A_p_choice="AM")
    E, Einv = ctx.coarse_matrix()
    assert np.abs(E - E.T).max() > 1e-8 * np.abs(E).max()
    assert rel(Einv, np.linalg.inv(E)) < 1e-10


@pytest.mark.parametrize("d", [1, 2, 63, 64, 65, 255, 256, 257, 300, 513, 777])
def test_spd_coarse_inverse_block_edges(gpu, d):
    """Cholesky-based inverse across the diagonal-block (64) and group (256) edges."""
    rng = np.random.default_rng(d)
    n = 4 * d + 7
    main = rng.uniform(2.5, 4.0, n)
    off = -rng.uniform(0.2, 1.0, n)
    A = dk.SparseMatrix.from_dia(n, [-1, 0, 1], np.vstack([np.r_[0.0, off[:-1]], main,
                                                          np.r_[off[:-1], 0.0]]))
    lab = np.sort(rng.integers(0, d, n)).astype(np.int32)
    lab[:d] = np.arange(d)  # every column used
    lab = np.sort(lab)
    ctx = dk.build_context(A, dk.Preconditioner.identity(), dk.DeflationBasis(labels=lab, d=d),
                           np.ones(n))
    E, Einv = ctx.coarse_matrix()
    assert rel(Einv, np.linalg.inv(E)) < 1e-11
    np.testing.assert_array_equal(Einv, Einv.T)


def test_symmetric_indefinite_coarse_system_falls_back_to_lu(gpu):
    """A symmetric but indefinite E fails the Cholesky attempt; the LU path inverts it."""
    n = 3000
    rng = np.random.default_rng(5)
    main = rng.uniform(1.0, 2.0, n) * np.where(np.arange(n) % 3 == 0, -1.0, 1.0) * 4.0
    off = rng.uniform(-0.5, 0.5, n)
    A = dk.SparseMatrix.from_dia(n, [-1, 0, 1], np.vstack([np.r_[0.0, off[:-1]], main,
                                                          np.r_[off[:-1], 0.0]]))
    lab = (np.arange(n) // 2).astype(np.int32)  # 1,500 columns of two cells
    ctx = dk.build_context(A, dk.Preconditioner.identity(), dk.DeflationBasis(labels=lab, d=1500),
                           np.ones(n))
    E, Einv = ctx.coarse_matrix()
    np.testing.assert_array_equal(E, E.T)
    assert np.linalg.eigvalsh(E).min() < 0 < np.linalg.eigvalsh(E).max()
    assert rel(Einv, np.linalg.inv(E)) < 1e-10


@pytest.mark.parametrize("boxes,force", [((12, 10, 6), True), ((24, 20, 12), True)])
def test_nested_dissection_coarse_solve(gpu, boxes, force, monkeypatch):
    """SPD E with hundreds of labels: y = E^-1 s runs as P^T W^T W P s over the nonzero tiles
    of W = L^-1 in nested-dissection order (dk_profile.cu); projectors, x* and the formed
    E^-1 agree with the label oracle's dense solve."""
    grid = dk.Grid(48, 40, 24)
    rng = np.random.default_rng(sum(boxes))
    k = 10.0 ** rng.uniform(-2, 2, grid.n_cells)
    field = dk.PermeabilityField(grid, k, k.copy(), 0.1 * k)
    q = np.zeros(grid.n_cells)
    q[0], q[-1] = 1.0, -1.0
    prob = dk.assemble_pressure(field, dk.BoundarySpec(), q)
    A, b = prob.A, prob.b
    part = dk.subdomain_partition(grid, *boxes)
    basis = dk.partition_to_basis(part)
    M = dk.Preconditioner.jacobi(A)
    if force:  # below the size where it pays: forced (DK_FORCE_ND)
        monkeypatch.setenv("DK_FORCE_ND", "1")
    ctx = dk.build_context(A, M, basis, b)
    kind, tiles = ctx.coarse_kind()
    assert kind == "nested_dissection_W"
    nb = (basis.d + 31) // 32
    assert force or tiles < nb * (nb + 1) // 2
    Ac = sp.csr_matrix((A.values, A.col_indices, A.row_offsets), shape=(A.n, A.n))
    o = O.LabelDeflation(Ac, basis.labels, basis.d, b, M.inv_diag)
    E, Einv = ctx.coarse_matrix()
    np.testing.assert_allclose(Einv @ E, np.eye(basis.d), atol=1e-9)
    v = rng.standard_normal(A.n)
    assert rel(ctx.apply_p1(v), o.apply_p1(v)) < 1e-11
    assert rel(ctx.apply_p2(v), o.apply_p2(v)) < 1e-11
    assert rel(ctx.x_star, o.x_star) < 1e-11
    # deterministic: the same application twice is bit-identical
    np.testing.assert_array_equal(ctx.apply_p1(v), ctx.apply_p1(v))
    rep = dk.gmres(A, b, M=M, m=30, tol=1e-10, max_iters=3000, deflation=ctx)
    ref = O.run_cycles(Ac, b, None, M.inv_diag, 30, 1e-10, 3000, 0, o)
    assert abs(rep.iterations - ref["iterations"]) <= 2
    assert rel(rep.x, ref["x"]) <= 1e-8


@pytest.mark.parametrize("cfg", [3, 4])
def test_full_size_projector_properties(gpu, cfg):
    """BASELINE configs 3 and 4 at full size (1.1 M / 16.8 M cells), where no CPU reference
    finishes in test time: size-independent identities of the deflation projectors through
    the device path — P1 is idempotent and linear, and Zᵀ A_p P2 v = 0 — each to a tolerance
    set by E's conditioning."""
    from paper_1510_02148_b200 import configs
    case = configs.make_case(cfg)
    A, b = case.problem()
    basis = dk.partition_to_basis(case.partition())
    M = dk.Preconditioner.jacobi(A)
    ctx = dk.build_context(A, M, basis, b)
    rng = np.random.default_rng(cfg)
    v = rng.standard_normal(A.n)
    w = rng.standard_normal(A.n)
    p1v = ctx.apply_p1(v)
    scale = np.abs(v).max()
    # config 4's layer contrasts reach 1e6 and cond(E) = 2e18: no fp64 coarse solve
    # reproduces the projector closely there — measured 3e-7 relative on the device, 3.2e-6
    # for the CPU oracle's LU solve on the same inputs; 1e-12 at config 3
    tol = {3: 1e-9, 4: 1e-5}[cfg]
    np.testing.assert_allclose(ctx.apply_p1(p1v), p1v, rtol=0, atol=tol * scale)
    lin = ctx.apply_p1(2.0 * v - 3.0 * w) - (2.0 * p1v - 3.0 * ctx.apply_p1(w))
    assert np.abs(lin).max() <= tol * scale
    # P2 = I - Z E^-1 Z^T A_p: its output has no component left in the deflation space's
    # A_p-coupling, i.e. Z^T A_p P2 v = 0 (restriction of A_p P2 v per column)
    p2v = ctx.apply_p2(v)
    ap = dk.spmv(A, p2v)
    zt = np.bincount(basis.labels[basis.labels >= 0], weights=ap[basis.labels >= 0],
                     minlength=basis.d)
    zt_abs = np.bincount(basis.labels[basis.labels >= 0],
                         weights=np.abs(dk.spmv(A, np.abs(v)))[basis.labels >= 0],
                         minlength=basis.d)
    assert np.all(np.abs(zt) <= 1e3 * tol * (zt_abs + 1.0))
    ctx.close()
