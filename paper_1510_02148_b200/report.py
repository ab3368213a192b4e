"""Convergence-CSV and summary-line output, byte-compatible with the reference CLI.

Reference: defkrylov/cli.py:137-142 (_fmt), :294-300 (write_convergence_csv), :312-314
(summary_line).  The CSV schema `iter,resnorm,restart_index,deflated_flag` is what the
reference frontend parses (frontend/src/csv.ts).
"""
from __future__ import annotations

import numpy as np

from .krylov import SolveReport


def _fmt(x) -> str:
    if isinstance(x, (bool, np.bool_)):
        return "1" if x else "0"
    if isinstance(x, (int, np.integer)):
        return str(int(x))
    return repr(float(x))


def write_convergence_csv(path, report: SolveReport) -> None:
    """One row per history entry: iteration, residual estimate, cycle, deflation flag."""
    rows = ["iter,resnorm,restart_index,deflated_flag\n"]
    for i, (r, c, dfl) in enumerate(zip(report.residual_history, report.restart_of,
                                        report.deflated_flags)):
        rows.append(f"{i},{_fmt(r)},{_fmt(c)},{_fmt(dfl)}\n")
    with open(path, "w", newline="") as f:
        f.write("".join(rows))


def summary_line(method: str, m: int, d: int, report: SolveReport, setup_ms: float,
                 solve_ms: float) -> str:
    """`method,m,d,iters,converged,final_relres,setup_ms,solve_ms`."""
    return (f"{method},{m},{d},{report.iterations},{_fmt(report.converged)},"
            f"{_fmt(report.final_relres)},{setup_ms:.3f},{solve_ms:.3f}")
