"""How well is config 4's deflated iterate defined?  (test infrastructure, CPU)

Runs the label oracle (oracle/dk_oracle.py) on BASELINE config 4 for K GMRES(50) cycles with a
coarse solve that is mathematically identical to the reference's dense_lu / lu_solve
(sparse.py:110-145) but rounds differently: LU of the symmetrically equilibrated
E~ = D E D (D = diag(E)^-1/2), y = D E~^-1 D s.  The distance of its x to the reference-
arithmetic golden (tests/golden/config4_oracle.npz) is the intrinsic spread of the reference's
own answer at cond(E) ~ 1e18: no implementation that rounds differently can agree more closely.

    python tools/config4_sensitivity.py [--max-cycles 4] [--out tests/golden/config4_equil_oracle.npz]
"""
from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np
import scipy.linalg

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

from oracle import dk_oracle as O  # noqa: E402
from oracle.run_case import oracle_inputs  # noqa: E402


class EquilibratedDeflation(O.LabelDeflation):
    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        dg = np.abs(np.diag(self.E))
        self.D = 1.0 / np.sqrt(np.where(dg > 0, dg, 1.0))
        Es = self.D[:, None] * self.E * self.D[None, :]
        self.lus = scipy.linalg.lu_factor(Es)
        print(f"cond(E) = {np.linalg.cond(self.E):.3e}, cond(D E D) = {np.linalg.cond(Es):.3e}",
              flush=True)
        self.x_star = self.prolong_z(self.coarse(self.restrict(self.b_)))

    def coarse(self, s):
        if not hasattr(self, "lus"):
            return super().coarse(s)
        return self.D * scipy.linalg.lu_solve(self.lus, self.D * s, check_finite=False)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-cycles", type=int, default=4)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    case, Ac, b, inv, col, d = oracle_inputs(4)
    EquilibratedDeflation.b_ = b
    defl = EquilibratedDeflation(Ac, col, d, b, inv)
    t = time.time()
    r = O.run_cycles(Ac, b, None, inv, case.m, case.tol, case.max_iters, 0, defl,
                     max_cycles=a.max_cycles)
    print(f"equilibrated oracle: iters={r['iterations']} relres={r['final_relres']:.6e} "
          f"({time.time() - t:.0f}s)", flush=True)
    g = np.load(ROOT / "tests" / "golden" / "config4_oracle.npz")
    x = r["x"]
    xs = x[::97]
    est = np.linalg.norm(O.sketch(x) - g["x_sketch"]) / np.sqrt(len(g["x_sketch"]))
    print(f"vs reference-arithmetic golden: sketched |dx|/|x| = {est / float(g['x_norm']):.3e}, "
          f"sampled = {np.linalg.norm(xs - g['x_sample']) / np.linalg.norm(g['x_sample']):.3e}, "
          f"history max rel diff = "
          f"{np.max(np.abs(r['history'] - g['history']) / np.abs(g['history'])):.3e}", flush=True)
    if a.out:
        np.savez_compressed(a.out, iters=r["iterations"], history=r["history"],
                            x_sample=xs, x_norm=np.linalg.norm(x), x_sketch=O.sketch(x),
                            relres=r["final_relres"], cycles=r["cycles"], d=d,
                            max_cycles=a.max_cycles)


if __name__ == "__main__":
    main()
