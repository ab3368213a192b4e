"""Configs 4 and 5 at full size: generation, labels, setup, a bounded solve (diagnostic)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1510_02148_b200 as dk
from paper_1510_02148_b200 import configs
for idx in [int(a) for a in sys.argv[1:]] or [4, 5]:
    t = time.time(); c = configs.make_case(idx); A, b = c.problem(); t1 = time.time()
    p = c.partition(); t2 = time.time()
    B = dk.partition_to_basis(p); M = dk.Preconditioner.jacobi(A)
    print(f"cfg{idx} n={A.n} gen+assemble {t1-t:.1f}s labels {t2-t1:.1f}s d={B.d} excl={len(p.default_exclude)}", flush=True)
    t = time.time(); ctx = dk.build_context(A, M, B, b); print(f"  setup {time.time()-t:.2f}s {ctx.setup_ms()}", flush=True)
    for mi in (100, 300):
        rep = dk.gmres(A, b, M=M, m=c.m, tol=c.tol, max_iters=mi, deflation=ctx)
        print(f"  max_iters={mi}: iters {rep.iterations} conv {rep.converged} relres {rep.final_relres:.3e} hist[-1]/hist[0] {rep.residual_history[-1]/rep.residual_history[0]:.3e} dev {rep.solve_seconds:.3f}s -> {rep.iterations/rep.solve_seconds:.1f} it/s", flush=True)
    ctx.close(); A.release_device()
