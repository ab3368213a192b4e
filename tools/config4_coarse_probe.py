"""Accuracy of the device coarse solve at BASELINE config 4 (cond(E) ~ 1e18; diagnostic).

Compares the device E^-1 (dk_defl_coarse) and the device P1 with an equilibrated LU solve
(D E D, D = diag(E)^-1/2) of the same E, and the device x after 4 GMRES(50) cycles with the
equilibrated-oracle run of tools/config4_sensitivity.py (if its npz is given).
"""
import sys
from pathlib import Path

import numpy as np
import scipy.linalg

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1510_02148_b200 as dk  # noqa: E402
from paper_1510_02148_b200 import configs  # noqa: E402
from oracle import dk_oracle as O  # noqa: E402

case = configs.make_case(4)
A, b = case.problem()
M = dk.Preconditioner.jacobi(A)
basis = dk.partition_to_basis(case.partition())
ctx = dk.build_context(A, M, basis, b)
print("coarse kind", ctx.coarse_kind(), "d", basis.d)
E, Einv = ctx.coarse_matrix(inverse=True)
import os
os.makedirs("gpurun_out", exist_ok=True)
np.save("gpurun_out/config4_E_dev.npy", E)
dg = np.abs(np.diag(E))
D = 1.0 / np.sqrt(dg)
Es = D[:, None] * E * D[None, :]
print(f"cond(E) {np.linalg.cond(E):.3e} cond(DED) {np.linalg.cond(Es):.3e}")
lus = scipy.linalg.lu_factor(Es)
lu = scipy.linalg.lu_factor(E)
rng = np.random.default_rng(0)
for trial in range(3):
    s = rng.standard_normal(basis.d) * dg  # a restriction-like right-hand side
    ye = D * scipy.linalg.lu_solve(lus, D * s)
    yl = scipy.linalg.lu_solve(lu, s)
    yd = Einv @ s
    n = np.linalg.norm(ye)
    print(f"|y_dev - y_eq|/|y| {np.linalg.norm(yd - ye) / n:.3e}   |y_lu - y_eq|/|y| "
          f"{np.linalg.norm(yl - ye) / n:.3e}   |E y_dev - s|/|s| "
          f"{np.linalg.norm(E @ yd - s) / np.linalg.norm(s):.3e}  |E y_eq - s|/|s| "
          f"{np.linalg.norm(E @ ye - s) / np.linalg.norm(s):.3e}")
g = np.load(sys.argv[1]) if len(sys.argv) > 1 else None
rep = dk.pdgmres(A, b, M=M, m=case.m, basis=basis, tol=case.tol, max_iters=200)
np.savez("gpurun_out/config4_dev_x.npz", x_sketch=O.sketch(rep.x), x_norm=np.linalg.norm(rep.x),
         x_sample=rep.x[::97], history=rep.residual_history)
for name in ("tests/golden/config4_oracle.npz",) + ((sys.argv[1],) if g is not None else ()):
    gg = np.load(name)
    est = np.linalg.norm(O.sketch(rep.x) - gg["x_sketch"]) / np.sqrt(len(gg["x_sketch"]))
    print(f"device x vs {name}: sketched rel {est / float(gg['x_norm']):.3e}, history max rel "
          f"{np.max(np.abs(rep.residual_history - gg['history']) / gg['history']):.3e}")
