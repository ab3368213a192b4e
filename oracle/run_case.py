"""Run the CPU oracle on one BASELINE config and store its result (test infrastructure).

    python oracle/run_case.py 3 [--plain] [--max-cycles K] [--full-x] [--out FILE.npz]

Configs 3-5 are too large for the reference's dense-Z context, so their
golden runs come from this label-based restatement, which tests/test_oracle.py pins against
the reference on the sandwich, hetero and config-1/2 goldens.  Every input comes from the
oracle side: the seeded k fields (configs.py generators, plain numpy), the TPFA operator
(host assembly, bit-identical to the reference's assemble_pressure) and the labels from the
oracle's own labeller (subdomain_levelset_labels_boxwise, pinned to the reference's label
CRCs in tests/test_oracle.py) — the product's device labeller is not involved.

Stored: the residual history, iterations, restart map, |x|, x[::97], a 16-row
Johnson-Lindenstrauss sketch of x (oracle.sketch) and, with --full-x, x itself.
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
from paper_1510_02148_b200 import configs  # noqa: E402  (seeded input generators)


def oracle_inputs(idx: int, seed: int = 0):
    """(case, CSR A, b, inv_diag, column labels, d) built without the device library."""
    case = configs.make_case(idx, seed)
    A, b = case.problem()
    off, dg = A.dia()
    Ac = O.csr_from_dia_lean(A.n, off, dg)
    inv = 1.0 / dg[list(off).index(0)]
    g = case.grid
    px, py, pz = case.boxes
    lab, d, excl = O.subdomain_levelset_labels_boxwise(case.band_field.kx, g.nx, g.ny, g.nz,
                                                       px, py, pz, case.jump_threshold)
    col, dcol = O.columns_from_labels(lab, d, excl)
    return case, Ac, b, inv, col, dcol


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", type=int)
    ap.add_argument("--plain", action="store_true", help="no deflation (gmres)")
    ap.add_argument("--max-cycles", type=int, default=None)
    ap.add_argument("--full-x", action="store_true")
    ap.add_argument("--cgs", action="store_true", help="classical Gram-Schmidt (the device's)")
    ap.add_argument("--out", default=None)
    ap.add_argument("--save-xhat", default=None, help="x before reconstruct (.npy, not committed)")
    a = ap.parse_args()
    t0 = time.time()
    case, Ac, b, inv, col, dcol = oracle_inputs(a.config)
    defl = None
    d = 0
    if not a.plain:
        d = dcol
        defl = O.LabelDeflation(Ac, col, dcol, b, inv)
    t1 = time.time()
    r = O.run_cycles(Ac, b, None, inv, case.m, case.tol, case.max_iters, 0, defl,
                     max_cycles=a.max_cycles, gs="cgs" if a.cgs else "mgs")
    t2 = time.time()
    print(f"config{a.config} {'plain' if a.plain else 'deflated'} d={d} "
          f"iters={r['iterations']} cycles={r['cycles']} converged={r['converged']} "
          f"gs={'cgs' if a.cgs else 'mgs'} relres={r['final_relres']:.3e} reorths={r['reorths']} setup={t1 - t0:.1f}s "
          f"solve={t2 - t1:.1f}s threads={os.environ.get('OPENBLAS_NUM_THREADS', 'default')}",
          flush=True)
    if a.save_xhat:
        np.save(a.save_xhat, r["x_hat"])
    if a.out:
        extra = {"x": r["x"]} if a.full_x else {}
        np.savez_compressed(a.out, iters=r["iterations"], history=r["history"],
                            restart_of=r["restart_of"], x_sample=r["x"][::97],
                            x_norm=np.linalg.norm(r["x"]), x_sketch=O.sketch(r["x"]),
                            relres=r["final_relres"], converged=r["converged"],
                            cycles=r["cycles"], d=d, reorths=r["reorths"],
                            max_cycles=-1 if a.max_cycles is None else a.max_cycles,
                            solve_seconds=t2 - t1, setup_seconds=t1 - t0, **extra)


if __name__ == "__main__":
    main()
