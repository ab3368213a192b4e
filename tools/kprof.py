"""Per-kernel-class device times of one event-profiled solve (diagnostic tool).

    python tools/kprof.py CONFIG [--plain] [--max-iters K]
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1510_02148_b200 as dk  # noqa: E402
from paper_1510_02148_b200 import _lib, configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", type=int)
ap.add_argument("--plain", action="store_true")
ap.add_argument("--max-iters", type=int, default=200)
a = ap.parse_args()
case = configs.make_case(a.config)
A, b = case.problem()
M = dk.Preconditioner.jacobi(A)
op = A.device()
op.set_precond(M)
ctx = None if a.plain else dk.build_context(A, M, dk.partition_to_basis(case.partition()), b)
lib = op._lib
x = np.empty(A.n)
hist = np.empty(a.max_iters + 1)
rof = np.empty(a.max_iters + 1, dtype=np.int32)
info = _lib.SolveInfo()
for prof in (0, 1):
    lib.dk_op_profile(op.h, prof)
    _lib.check(lib.dk_gmres(op.h, ctx.h if ctx else None, _lib.ptr(b), None, case.m, case.tol,
                            a.max_iters, 0, _lib.ptr(x), _lib.ptr(hist), _lib.ptr(rof), None,
                            C.byref(info)))
names = (C.c_char_p * 16)()
ms = (C.c_double * 16)()
nl = (C.c_int64 * 16)()
by = (C.c_double * 16)()
k = lib.dk_op_profile_read(op.h, 16, names, ms, nl, by)
print(f"config {a.config} {'plain' if a.plain else 'deflated'} n={A.n} iters={info.iterations}")
for i in range(k):
    if nl[i]:
        print(f"  {names[i].decode():18s} {1e3 * ms[i] / nl[i]:9.2f} us x {nl[i]:5d}  "
              f"{by[i] / (ms[i] * 1e-3) / 1e9:8.1f} GB/s")
