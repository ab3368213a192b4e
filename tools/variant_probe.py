"""Device-resident solve rate of one config under the current environment (diagnostic tool).

    python tools/variant_probe.py CONFIG [--steps K] [--tag TEXT]

Prints one line: tag, iterations per solve, it/s over K graph-replayed solves (CUDA events on
the solver stream), final relres.  Used to compare DK_* environment knobs run by run.
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1510_02148_b200 as dk  # noqa: E402
from paper_1510_02148_b200 import _lib, configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config", type=int)
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--tag", default="")
ap.add_argument("--plain", action="store_true")
ap.add_argument("--max-iters", type=int, default=0)
a = ap.parse_args()
lib = _lib.load()
case = configs.make_case(a.config)
if a.max_iters:
    case.max_iters = a.max_iters
A, b = case.problem()
M = dk.Preconditioner.jacobi(A)
op = A.device()
stream = torch.cuda.current_stream()
_lib.check(lib.dk_op_set_stream(op.h, C.c_void_p(stream.cuda_stream)))
ctx = None if a.plain else dk.build_context(A, M, dk.partition_to_basis(case.partition()), b)
op.set_precond(M)
b_dev = torch.from_numpy(b).cuda()
x_dev = torch.empty(A.n, dtype=torch.float64, device="cuda")
hist = np.empty(case.max_iters + 1)
rof = np.empty(case.max_iters + 1, dtype=np.int32)
info = _lib.SolveInfo()


def solve():
    _lib.check(lib.dk_gmres(op.h, ctx.h if ctx else None, b_dev.data_ptr(), None, case.m,
                            case.tol, case.max_iters, 0, x_dev.data_ptr(), _lib.ptr(hist),
                            _lib.ptr(rof), None, C.byref(info)))
    return int(info.iterations)


for _ in range(3):
    solve()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
its = sum(solve() for _ in range(a.steps))
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"{a.tag:24s} config {a.config} iters {its // a.steps} it/s {its / (ms * 1e-3):9.1f} "
      f"ms/solve {ms / a.steps:8.2f} relres {info.final_relres:.3e} "
      f"xsum {float(x_dev.sum()):.15e}", flush=True)
