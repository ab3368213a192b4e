"""Operator assembly and containers (CPU): bit-identity with the reference's assembly."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1510_02148_b200 as dk
from paper_1510_02148_b200 import configs
from paper_1510_02148_b200.sparse import SparseMatrix


def _sandwich(sigma=1e6):
    g = dk.Grid(7, 7, 3)
    f = dk.make_layered_field(g, [((0, 1), sigma), ((1, 2), 1.0), ((2, 3), sigma)])
    q = np.zeros(g.n_cells)
    q[0], q[-1] = 1.0, -1.0
    return g, f, q


def test_sandwich_assembly_bit_identical(golden):
    gd = golden("sandwich")
    g, f, q = _sandwich()
    p = dk.diagonal_scale(dk.assemble_pressure(f, dk.BoundarySpec(), q))
    np.testing.assert_array_equal(p.A.row_offsets, gd["ro"])
    np.testing.assert_array_equal(p.A.col_indices, gd["ci"])
    np.testing.assert_array_equal(p.A.values, gd["va"])
    np.testing.assert_array_equal(p.b, gd["b"])


def test_hetero_assembly_bit_identical(golden):
    gd = golden("hetero")
    g = dk.Grid(12, 10, 8, 2.0, 3.0, 0.5)
    f = dk.PermeabilityField(g, gd["kx"], gd["ky"], gd["kz"])
    p = dk.assemble_pressure(f, dk.BoundarySpec(True, 1.5, 0.8), gd["q"])
    np.testing.assert_array_equal(p.A.row_offsets, gd["ro"])
    np.testing.assert_array_equal(p.A.col_indices, gd["ci"])
    np.testing.assert_array_equal(p.A.values, gd["va"])
    np.testing.assert_array_equal(p.b, gd["b"])


def test_csr_dia_roundtrip(golden):
    gd = golden("hetero")
    A = SparseMatrix(len(gd["b"]), gd["ro"], gd["ci"], gd["va"])
    off, dg = A.dia()
    assert len(off) == 7
    B = SparseMatrix.from_dia(A.n, off, dg)
    np.testing.assert_array_equal(B.row_offsets, gd["ro"])
    np.testing.assert_array_equal(B.col_indices, gd["ci"])
    np.testing.assert_array_equal(B.values, gd["va"])
    np.testing.assert_array_equal(A.diagonal(), B.diagonal())


def test_x_face_dirichlet_rule():
    """Ghost half-cell on x faces: T = area / (h/2k + h/2kb) added to the diagonal and b."""
    g = dk.Grid(4, 3, 2, 2.0, 1.0, 1.0)
    k = np.full(g.n_cells, 3.0)
    f = dk.PermeabilityField(g, k, k, k)
    bc = dk.BoundarySpec(top_dirichlet=False, faces=(("xmin", 1.0), ("xmax", 0.0)))
    p = dk.assemble_pressure(f, bc)
    T = (1.0 * 1.0) / (0.5 * 2.0 / 3.0 + 0.5 * 2.0 / 1.0)
    b = p.b.reshape(2, 3, 4)
    np.testing.assert_allclose(b[:, :, 0], T)
    np.testing.assert_allclose(b[:, :, 1:], 0.0)
    assert np.all(p.A.diagonal() > 0)


def test_all_neumann_incompatible_source_raises():
    g = dk.Grid(3, 3, 3)
    f = dk.make_layered_field(g, [((0, 3), 1.0)])
    q = np.zeros(g.n_cells)
    q[0] = 1.0
    with pytest.raises(dk.SingularProblem):
        dk.assemble_pressure(f, dk.BoundarySpec(top_dirichlet=False), q)


def test_dead_cells_get_identity_rows():
    g = dk.Grid(3, 1, 1)
    k = np.array([1.0, 0.0, 1.0])
    f = dk.PermeabilityField(g, k, k, k)
    p = dk.assemble_pressure(f, dk.BoundarySpec(top_dirichlet=True))
    D = p.A.to_dense()
    assert D[1, 1] == 1.0 and D[1, 0] == 0.0 and D[1, 2] == 0.0 and p.b[1] == 0.0


def test_csr_validation_messages():
    with pytest.raises(ValueError, match="n\\+1"):
        SparseMatrix(2, [0, 1], [0], [1.0])
    with pytest.raises(ValueError, match="strictly increasing"):
        SparseMatrix(2, [0, 2, 2], [1, 0], [1.0, 2.0])
    with pytest.raises(ValueError, match="out of range"):
        SparseMatrix(2, [0, 1, 2], [0, 2], [1.0, 2.0])


def test_more_than_seven_diagonals_is_unsupported():
    A = SparseMatrix.from_dense(np.eye(10) + np.triu(np.ones((10, 10)), 1))
    with pytest.raises(dk.UnsupportedOperator):
        A.dia()


@pytest.mark.parametrize("idx", [1, 2, 3])
def test_config_generators_are_deterministic(idx):
    a, b = configs.make_case(idx), configs.make_case(idx)
    np.testing.assert_array_equal(a.field.kx, b.field.kx)
    assert a.grid.n_cells == {1: 32 ** 3, 2: 128 * 128 * 64, 3: 60 * 220 * 85}[idx]


def test_config3_field_statistics():
    c = configs.make_case(3)
    logk = np.log10(c.field.kx).reshape(85, 220, 60)
    top, bot = logk[50:], logk[:50]
    assert abs(top.std() - 1.0) < 0.05 and top.min() >= -3 and top.max() <= 3
    assert set(np.unique(bot)) == {-3.0, 3.0}
    np.testing.assert_array_equal(c.field.kz, 0.1 * c.field.kx)
