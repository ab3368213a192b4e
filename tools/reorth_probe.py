"""Second Gram-Schmidt passes per solve (diagnostic): fused vs separate launches."""
import os
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1510_02148_b200 as dk
from paper_1510_02148_b200 import configs
g = np.load("tests/golden/hetero.npz")
A = dk.SparseMatrix(len(g["b"]), g["ro"], g["ci"], g["va"])
M = dk.Preconditioner.jacobi(A)
for name, fn in (("hetero gmres", lambda: dk.gmres(A, g["b"], M=M, m=20, tol=1e-10, max_iters=2000)),
                 ("hetero rdgmres", lambda: dk.rdgmres(A, g["b"], M=M, m=20, d=4, tol=1e-10, max_iters=2000))):
    r = fn()
    print(name, r.iterations, "reorths", r.reorthogonalisations, "relres", r.final_relres)
s = np.load("tests/golden/sandwich.npz")
As = dk.SparseMatrix(len(s["b"]), s["ro"], s["ci"], s["va"])
r = dk.gmres(As, s["b"], m=40, tol=1e-6, max_iters=300)
print("sandwich gmres", r.iterations, "reorths", r.reorthogonalisations)
for idx in (1, 3):
    c = configs.make_case(idx); Ac, b = c.problem()
    r = dk.pdgmres(Ac, b, M=dk.Preconditioner.jacobi(Ac), m=c.m,
                   basis=dk.partition_to_basis(c.partition()), tol=c.tol, max_iters=c.max_iters)
    print("config", idx, r.iterations, "reorths", r.reorthogonalisations)
