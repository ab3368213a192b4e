"""BASELINE configs 4 and 5 at full size against the CPU oracle (GPU).

The goldens come from oracle/run_case.py on the oracle's own inputs (labels from its box-wise
labeller, pinned to the reference's partition CRCs in tests/test_labels.py):
  config 4 (256^3, d = 960) deflated and plain (`gmres(deflation=None)`, BASELINE's "Z empty"
  run), each bounded to 4 GMRES(50) cycles — the full runs do not reach 1e-8 (see DESIGN.md
  §2 on config 4's stagnation) and the oracle needs ~3 s per iteration at this size;
  config 5 (512x512x256, d = 8,670, GMRES(40)) bounded to 2 cycles (~12 s per oracle
  iteration).
Config 4's coarse matrix has cond(E) ~ 2e18: its diagonal sums nearly cancelling in-label
couplings, and a last-bit difference there moves x by ~3e-5 after 4 cycles.  Device and
oracle therefore assemble E in one fully defined order (row-wise A_p Z first, then sequential
sums over cells; oracle LabelDeflation, dk_coarse.cu build_coarse), which makes the 1e-8 bar
meaningful at this conditioning.
x (16.8 M / 67 M cells) is too large to commit; the golden holds |x|, x[::97] and a 16-row
Johnson-Lindenstrauss sketch S x (oracle.sketch: seeded Rademacher rows).  For any error e,
|S e| / 4 is an unbiased estimate of |e|_2 (within a factor 2 with probability > 0.99), so
the full-vector relative 2-norm difference is checked through it.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_1510_02148_b200 as dk
from conftest import GOLDEN
from oracle import dk_oracle as O
from paper_1510_02148_b200 import configs

pytestmark = pytest.mark.gpu

X_TOL = 1e-8
HIST_RTOL = 1e-6
# Config 4 (cond(E) = 2e18): two oracle runs that differ only in how the coarse system is
# solved (LU of E vs LU of the equilibrated D E D, both backward stable) already differ by
# 2.1e-8 in x after 4 cycles (tools/config4_sensitivity.py); the bar there is that spread.
X_TOL_C4 = 3e-8


def _golden(name):
    path = GOLDEN / f"{name}.npz"
    if not path.exists():
        pytest.fail(f"tests/golden/{name}.npz missing (oracle/run_case.py)")
    return np.load(path)


def _solve(idx, deflate, max_iters):
    case = configs.make_case(idx)
    A, b = case.problem()
    M = dk.Preconditioner.jacobi(A)
    if deflate:
        basis = dk.partition_to_basis(case.partition())
        rep = dk.pdgmres(A, b, M=M, m=case.m, basis=basis, tol=case.tol, max_iters=max_iters)
        return rep, basis.d
    return dk.gmres(A, b, M=M, m=case.m, tol=case.tol, max_iters=max_iters), 0


def _check_x(x, g, tol=X_TOL):
    xn = float(g["x_norm"])
    est = np.linalg.norm(O.sketch(x) - g["x_sketch"]) / np.sqrt(len(g["x_sketch"]))
    xs = x[::97]
    samp = np.linalg.norm(xs - g["x_sample"]) / np.linalg.norm(g["x_sample"])
    assert est <= tol * xn, f"sketched |dx|/|x| = {est / xn:.2e} (sampled {samp:.2e})"
    assert samp <= tol, f"sampled |dx|/|x| = {samp:.2e}"
    assert abs(np.linalg.norm(x) - xn) <= tol * xn


@pytest.mark.parametrize("deflate,name", [(True, "config4_oracle"),
                                          (False, "config4_plain_oracle")])
def test_config4_cycles_match_oracle(gpu, deflate, name):
    g = _golden(name)
    iters = int(g["iters"])
    rep, d = _solve(4, deflate, iters)
    assert d == int(g["d"])
    assert rep.iterations == iters and rep.restarts == int(g["cycles"]) - 1
    np.testing.assert_allclose(rep.residual_history, g["history"], rtol=HIST_RTOL)
    _check_x(rep.x, g, X_TOL_C4 if deflate else X_TOL)
    assert abs(rep.final_relres - float(g["relres"])) <= 1e-6 * float(g["relres"])


def test_config5_cycles_match_oracle(gpu):
    """512x512x256, 4,000 inclusions, d = 8,670, GMRES(40): the first two cycles."""
    g = _golden("config5_oracle")
    iters = int(g["iters"])
    rep, d = _solve(5, True, iters)
    assert d == int(g["d"])
    assert rep.iterations == iters and rep.restarts == int(g["cycles"]) - 1
    np.testing.assert_allclose(rep.residual_history, g["history"], rtol=HIST_RTOL)
    _check_x(rep.x, g)
    assert abs(rep.final_relres - float(g["relres"])) <= 1e-6 * float(g["relres"])
