"""Phase timeline of the persistent small-cycle kernel (diagnostic; -DDK_TIMELINE build)."""
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
lib.dk_timeline_enable(1 << 20)
rep = dk.pdgmres(A, b, M=M, m=case.m, basis=basis, tol=case.tol, max_iters=case.max_iters)
buf = np.empty(2 << 20, dtype=np.uint64)
n = lib.dk_timeline_read(buf.ctypes.data, 1 << 20)
rec = buf[:2 * n].reshape(n, 2)
t = rec[:, 0].astype(np.int64)
kind = (rec[:, 1] >> np.uint64(56)).astype(int)
ph = ((rec[:, 1] >> np.uint64(48)) & np.uint64(0xff)).astype(int)
sel = kind == 10
t, ph = t[sel], ph[sel]
order = np.argsort(t)
t, ph = t[order], ph[order]
# iterations: phase-0 records come in groups of G blocks
t0 = t[ph == 0]
G = int(np.sum(t0 < t0[0] + 3000))  # blocks per step (records within 3 us)
print("records", len(t), "blocks", G, "iterations", rep.iterations)
starts = t0[::G]
names = ["start", "stencil+restrict", "bar1(y)", "dots", "bar2(ctl)", "gs", "bar3(givens)",
         "lead start", "lead end", "prolong done", "-", "staged", "small_dots"]
acc = np.zeros(13)
cntv = 0
for i in range(5, len(starts) - 1):
    w = (t >= starts[i]) & (t < starts[i + 1])
    row = [np.max(t[w & (ph == p)]) - starts[i] if np.any(w & (ph == p)) else np.nan for p in range(13)]
    acc += np.nan_to_num(row)
    cntv += 1
print("mean of the last block's arrival at each phase end (us after the step's first start):")
for p in range(13):
    print(f"  {names[p]:18s} {acc[p] / cntv / 1e3:7.2f}")
# the three leads of a step, in order
for i in range(5, 8):
    w = (t >= starts[i]) & (t < starts[i + 1])
    print("  step", i, "lead start/end:", ((t[w & (ph == 7)] - starts[i]) / 1e3).round(2),
          ((t[w & (ph == 8)] - starts[i]) / 1e3).round(2))
print(f"step period {np.mean(np.diff(starts)) / 1e3:.2f} us")
