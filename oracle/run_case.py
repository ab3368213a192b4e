"""Run the CPU oracle on one BASELINE config and store its result (test infrastructure).

    python oracle/run_case.py 3 [--plain] [--max-cycles K] [--out tests/golden/config3_oracle.npz]

Configs 3-5 are too large for the reference's dense-Z context, so their
golden runs come from this label-based restatement, which tests/test_oracle.py pins against
the reference on the sandwich, hetero and config-1/2 goldens.
"""
from __future__ import annotations

import argparse
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import dk_oracle as O  # noqa: E402
from paper_1510_02148_b200 import configs  # noqa: E402
from paper_1510_02148_b200.physics import partition_to_basis  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("--plain", action="store_true", help="no deflation (gmres)")
    ap.add_argument("--max-cycles", type=int, default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    case = configs.make_case(a.config)
    A, b = case.problem()
    off, dg = A.dia()
    Ac = O.csr_from_dia(A.n, off, dg)
    inv = 1.0 / dg[list(off).index(0)]
    t0 = time.time()
    defl = None
    d = 0
    if not a.plain:
        basis = partition_to_basis(case.partition())
        d = basis.d
        defl = O.LabelDeflation(Ac, basis.labels, basis.d, b, inv)
    t1 = time.time()
    r = O.run_cycles(Ac, b, None, inv, case.m, case.tol, case.max_iters, 0, defl,
                     max_cycles=a.max_cycles)
    t2 = time.time()
    print(f"config{a.config} d={d} iters={r['iterations']} converged={r['converged']} "
          f"relres={r['final_relres']:.3e} setup={t1 - t0:.1f}s solve={t2 - t1:.1f}s "
          f"threads={os.environ.get('OPENBLAS_NUM_THREADS', 'default')}")
    if a.out:
        np.savez_compressed(a.out, iters=r["iterations"], history=r["history"],
                            restart_of=r["restart_of"], x_sample=r["x"][::97],
                            x_norm=np.linalg.norm(r["x"]), relres=r["final_relres"],
                            converged=r["converged"], cycles=r["cycles"], d=d,
                            solve_seconds=t2 - t1, setup_seconds=t1 - t0)


if __name__ == "__main__":
    main()
