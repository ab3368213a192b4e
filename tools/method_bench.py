"""GMRES vs RDGMRES vs PDGMRES on a BASELINE config through the public API (diagnostic).

    python tools/method_bench.py CONFIG [--d 10] [--reps 2]

Prints one JSON line per method: iterations, converged, final relres, device solve time,
wall time of the whole call (host inputs, set-up included) and iterations per second.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_1510_02148_b200 as dk  # noqa: E402
from paper_1510_02148_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", type=int)
ap.add_argument("--d", type=int, default=10)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--max-iters", type=int, default=None)
a = ap.parse_args()
case = configs.make_case(a.config)
A, b = case.problem()
M = dk.Preconditioner.jacobi(A)
basis = dk.partition_to_basis(case.partition())
mi = a.max_iters or case.max_iters
runs = {
    "gmres": lambda: dk.gmres(A, b, M=M, m=case.m, tol=case.tol, max_iters=mi),
    "rdgmres": lambda: dk.rdgmres(A, b, M=M, m=case.m, d=a.d, tol=case.tol, max_iters=mi),
    "pdgmres": lambda: dk.pdgmres(A, b, M=M, m=case.m, basis=basis, tol=case.tol, max_iters=mi),
}
for name, fn in runs.items():
    best = None
    for r in range(a.reps + 1):
        t = time.perf_counter()
        rep = fn()
        wall = time.perf_counter() - t
        if r > 0 and (best is None or wall < best[1]):
            best = (rep, wall)
    rep, wall = best
    print(json.dumps({
        "config": a.config, "method": name, "m": case.m, "d": 0 if name == "gmres" else
        (a.d if name == "rdgmres" else basis.d), "iterations": rep.iterations,
        "converged": rep.converged, "final_relres": rep.final_relres,
        "solve_s": rep.solve_seconds, "wall_s": wall,
        "iters_per_s_device": rep.iterations / max(rep.solve_seconds, 1e-12),
        "iters_per_s_wall": rep.iterations / wall, "warning": rep.warning}), flush=True)
