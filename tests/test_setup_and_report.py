"""Device set-up paths (labels, TPFA assembly) and the reference CSV/summary formats."""
from __future__ import annotations

import numpy as np
import pytest

import paper_1510_02148_b200 as dk
from conftest import GOLDEN
from paper_1510_02148_b200 import configs, report
from paper_1510_02148_b200.krylov import SolveReport


# ---- report formats (CPU) ------------------------------------------------------------------
def test_convergence_csv_bytes_match_reference_cli(tmp_path, golden):
    g = golden("sandwich")
    h = g["fixture_history"]
    rep = SolveReport(x=np.zeros(3), converged=True, iterations=len(h) - 1, restarts=0,
                      residual_history=h, final_relres=0.0,
                      restart_of=np.zeros(len(h), dtype=np.int64),
                      deflated_flags=np.ones(len(h), dtype=bool))
    out = tmp_path / "c.csv"
    report.write_convergence_csv(out, rep)
    assert out.read_bytes() == (GOLDEN / "convergence.pdgmres.ref.csv").read_bytes()


def test_summary_line_format():
    rep = SolveReport(x=np.zeros(1), converged=False, iterations=7, restarts=0,
                      residual_history=np.ones(8), final_relres=0.125,
                      restart_of=np.zeros(8, dtype=np.int64),
                      deflated_flags=np.zeros(8, dtype=bool))
    assert report.summary_line("pdgmres", 40, 3, rep, 1.5, 2.25) == \
        "pdgmres,40,3,7,0,0.125,1.500,2.250"


# ---- device set-up (GPU) ------------------------------------------------------------------
@pytest.mark.gpu
def test_device_assembly_bit_identical(gpu, golden):
    g = golden("hetero")
    grid = dk.Grid(12, 10, 8, 2.0, 3.0, 0.5)
    f = dk.PermeabilityField(grid, g["kx"], g["ky"], g["kz"])
    p = dk.assemble_pressure(f, dk.BoundarySpec(True, 1.5, 0.8), g["q"], backend="device")
    np.testing.assert_array_equal(p.A.row_offsets, g["ro"])
    np.testing.assert_array_equal(p.A.col_indices, g["ci"])
    np.testing.assert_array_equal(p.A.values, g["va"])
    np.testing.assert_array_equal(p.b, g["b"])


@pytest.mark.gpu
@pytest.mark.parametrize("idx", [1, 3])
def test_device_assembly_matches_host_on_configs(gpu, idx):
    c = configs.make_case(idx)
    from paper_1510_02148_b200.testbed import assemble_dia, assemble_dia_device
    o1, d1, b1 = assemble_dia(c.field, c.bc)
    o2, d2, b2 = assemble_dia_device(c.field, c.bc)
    np.testing.assert_array_equal(o1, o2)
    assert d1.tobytes() == d2.tobytes() and b1.tobytes() == b2.tobytes()
