"""Phase timing of the end-to-end public-API path (diagnostic)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1510_02148_b200 as dk
from paper_1510_02148_b200 import configs
from paper_1510_02148_b200.krylov import _device_solve
c = configs.make_case(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
A, b = c.problem()
off, dg = A.dia()
basis = dk.partition_to_basis(c.partition())
M = dk.Preconditioner.jacobi(A)
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 4):
    t0 = time.perf_counter()
    Ah = dk.SparseMatrix.from_dia(A.n, off, dg)
    op = Ah.device(); t1 = time.perf_counter()
    op.set_precond(M); t2 = time.perf_counter()
    ctx = dk.build_context(Ah, M, basis, b); t3 = time.perf_counter()
    ms = ctx.setup_ms()
    rep = _device_solve(Ah, b, np.zeros(A.n), M, c.m, c.tol, c.max_iters, 0, ctx); t4 = time.perf_counter()
    ctx.close(); t5 = time.perf_counter()
    Ah.release_device(); t6 = time.perf_counter()
    dev_setup = sum(ms.values()) * 1e-3
    print(f"op {t1-t0:.4f} precond {t2-t1:.4f} ctx {t3-t2:.4f} (device {dev_setup:.4f}) "
          f"solve {t4-t3:.4f} (device {rep.solve_seconds:.4f}) ctx.close {t5-t4:.4f} "
          f"release {t6-t5:.4f} total {t6-t0:.4f}", flush=True)
