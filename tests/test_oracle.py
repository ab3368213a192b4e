"""The CPU oracle against the reference's own outputs (golden fixtures) — pins the checker."""
from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import rel
from oracle import dk_oracle as O


def _csr(g):
    return sp.csr_matrix((g["va"], g["ci"], g["ro"]))


def test_sandwich_dense_context_is_bit_exact(golden):
    g = golden("sandwich")
    A = _csr(g)
    inv = 1.0 / A.diagonal()
    lab = g["labels"]
    d = int(g["d"])
    Z = np.zeros((len(lab), d))
    Z[np.arange(len(lab)), lab] = 1.0
    r = O.run_cycles(A, g["b"], None, inv, 40, 1e-6, 300, 0, O.DenseDeflation(A, Z, g["b"], inv))
    assert r["iterations"] == int(g["pd_iters"]) == 22
    np.testing.assert_array_equal(r["history"], g["pd_history"])
    # the reference frontend's golden CSV (convergence.pdgmres.csv)
    np.testing.assert_array_equal(r["history"], g["fixture_history"])


def test_sandwich_label_context(golden):
    g = golden("sandwich")
    A = _csr(g)
    inv = 1.0 / A.diagonal()
    defl = O.LabelDeflation(A, g["labels"], int(g["d"]), g["b"], inv)
    r = O.run_cycles(A, g["b"], None, inv, 40, 1e-6, 300, 0, defl)
    assert r["iterations"] == int(g["pd_iters"])
    np.testing.assert_allclose(r["history"], g["pd_history"], rtol=1e-6)
    assert rel(r["x"], g["pd_x"]) < 1e-8


def test_sandwich_plain_gmres(golden):
    g = golden("sandwich")
    A = _csr(g)
    inv = 1.0 / A.diagonal()
    r = O.run_cycles(A, g["b"], None, inv, 40, 1e-6, 300, 0, None)
    assert r["iterations"] == int(g["gm_iters"])
    np.testing.assert_array_equal(r["history"], g["gm_history"])


def test_hetero_labels_and_projectors(golden):
    g = golden("hetero")
    lab, d, excl = O.subdomain_levelset_labels(g["kx"], 12, 10, 8, 3, 2, 2, 1.0)
    np.testing.assert_array_equal(lab, g["labels"])
    assert d == int(g["d"]) and sorted(excl) == list(g["excl"])
    A = _csr(g)
    inv = 1.0 / A.diagonal()
    col, dd = O.columns_from_labels(lab, d, excl)
    defl = O.LabelDeflation(A, col, dd, g["b"], inv)
    np.testing.assert_allclose(defl.apply_p1(g["v"]), g["p1v"], atol=1e-12)
    np.testing.assert_allclose(defl.apply_p2(g["v"]), g["p2v"], atol=1e-12)
    np.testing.assert_allclose(defl.reconstruct(g["v"]), g["rec"], atol=1e-12)
    np.testing.assert_allclose(defl.x_star, g["x_star"], atol=1e-12)
    np.testing.assert_allclose(defl.E, g["E"], rtol=1e-12, atol=1e-12 * np.abs(g["E"]).max())


@pytest.mark.parametrize("ap,key", [("A", "pd"), ("AM", "am")])
def test_hetero_pdgmres(golden, ap, key):
    g = golden("hetero")
    A = _csr(g)
    inv = 1.0 / A.diagonal()
    col, dd = O.columns_from_labels(g["labels"], int(g["d"]), g["excl"])
    defl = O.LabelDeflation(A, col, dd, g["b"], inv, ap=ap)
    r = O.run_cycles(A, g["b"], None, inv, 20, 1e-10, 2000, 0, defl)
    assert r["iterations"] == int(g[f"{key}_iters"])
    assert rel(r["x"], g[f"{key}_x"]) < 1e-10


def test_config1_against_reference(golden):
    from paper_1510_02148_b200 import configs
    g = golden("config1")
    case = configs.config1()
    A, b = case.problem()
    off, dg = A.dia()
    Ac = O.csr_from_dia(A.n, off, dg)
    inv = 1.0 / A.diagonal()
    lab, d, excl = O.subdomain_levelset_labels(case.field.kx, 32, 32, 32, 2, 2, 2, 2.0)
    np.testing.assert_array_equal(lab, g["labels"])
    col, dd = O.columns_from_labels(lab, d, excl)
    r = O.run_cycles(Ac, b, None, inv, 50, 1e-8, 20000, 0, O.LabelDeflation(Ac, col, dd, b, inv))
    assert r["iterations"] == int(g["pd_iters"]) == 78
    assert rel(r["x"], g["pd_x"]) < 1e-10
    rp = O.run_cycles(Ac, b, None, inv, 50, 1e-8, 20000, 0, None)
    assert rp["iterations"] == int(g["gm_iters"]) == 218
    assert rel(rp["x"], g["gm_x"]) < 1e-12
