"""Coarse set-up timing (E assembly, factorisation, inverse) for one config (diagnostic)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1510_02148_b200 as dk
from paper_1510_02148_b200 import configs
c = configs.make_case(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
A, b = c.problem()
basis = dk.partition_to_basis(c.partition())
M = dk.Preconditioner.jacobi(A)
for r in range(reps):
    ctx = dk.build_context(A, M, basis, b)
    print("d", basis.d, "setup_ms", ctx.setup_ms(), flush=True)
    ctx.close()
