"""Per-phase time of the persistent small-cycle kernel (diagnostic; -DDK_TIMELINE build):
block 0 sums globaltimer deltas per phase over the cycle and records them at exit."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1510_02148_b200 as dk  # noqa: E402
from paper_1510_02148_b200 import _lib, configs  # noqa: E402

lib = _lib.load()
lib.dk_timeline_enable.argtypes = [C.c_uint32]
lib.dk_timeline_read.argtypes = [C.c_void_p, C.c_uint32]
lib.dk_timeline_read.restype = C.c_int64
case = configs.make_case(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
A, b = case.problem()
M = dk.Preconditioner.jacobi(A)
basis = dk.partition_to_basis(case.partition())
for _ in range(2):
    dk.pdgmres(A, b, M=M, m=case.m, basis=basis, tol=case.tol, max_iters=case.max_iters)
lib.dk_timeline_enable(1 << 16)
rep = dk.pdgmres(A, b, M=M, m=case.m, basis=basis, tol=case.tol, max_iters=case.max_iters)
buf = np.empty(2 << 16, dtype=np.uint64)
n = lib.dk_timeline_read(buf.ctypes.data, 1 << 16)
rec = buf[:2 * n].reshape(n, 2)
kind = (rec[:, 1] >> np.uint64(56)).astype(int)
ph = ((rec[:, 1] >> np.uint64(48)) & np.uint64(0xff)).astype(int)
sel = (kind == 10) & (ph >= 0x80)
names = {1: "stencil + label partials", 2: "barrier 1", 3: "reduce s", 4: "y = E^-1 s",
         5: "prolongation + u_j", 6: "dot partials", 7: "barrier 2", 8: "control (H col, test)",
         9: "GS update + store", 10: "norm partial", 11: "barrier 3", 12: "Givens / flags",
         13: "ctl: reduce", 14: "ctl: h / G column", 15: "ctl: corr", 16: "giv: reduce",
         17: "giv: |H col|"}
tot = {}
for p, v in zip(ph[sel] - 0x80, rec[sel, 0]):
    tot[p] = tot.get(p, 0) + int(v)
its = rep.iterations
print(f"iterations {its}; mean us per step:")
for p in sorted(tot):
    print(f"  {str(names.get(p, p)):28s} {tot[p] / its / 1e3:7.2f}")
print(f"  {'sum':28s} {sum(tot.values()) / its / 1e3:7.2f}")
