"""Kernel timeline of a graph-replayed config solve (diagnostic; needs the -DDK_TIMELINE build).

    tools/build_all_variant.sh tl -DDK_TIMELINE
    DK_LIB_PATH=build/variants/tl/libdk.so python tools/timeline.py 3 [--window 40] [--at 0.5]

Every block's thread 0 records globaltimer stamps at phase points (0 entry, 1 dependency met,
2 per-cell phase done, 3 sweep done, 4 exit, 5 control block done).  Per launch: first entry,
first / median / last start, last sweep end, last exit; then per-kind means over the solve.
"""
import argparse
import ctypes as C
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1510_02148_b200 as dk  # noqa: E402
from paper_1510_02148_b200 import _lib, configs  # noqa: E402

KIND = {1: "stencil", 2: "restrict", 3: "tgemv1", 4: "tgemv2", 5: "project", 6: "gs",
        9: "dots"}

ap = argparse.ArgumentParser()
ap.add_argument("config", type=int)
ap.add_argument("--window", type=int, default=30)
ap.add_argument("--at", type=float, default=0.5)
ap.add_argument("--cap", type=int, default=1 << 24)
ap.add_argument("--save", default=None)
a = ap.parse_args()
lib = _lib.load()
lib.dk_timeline_enable.argtypes = [C.c_uint32]
lib.dk_timeline_read.argtypes = [C.c_void_p, C.c_uint32]
lib.dk_timeline_read.restype = C.c_int64
case = configs.make_case(a.config)
A, b = case.problem()
M = dk.Preconditioner.jacobi(A)
op = A.device()
stream = torch.cuda.current_stream()
_lib.check(lib.dk_op_set_stream(op.h, C.c_void_p(stream.cuda_stream)))
ctx = dk.build_context(A, M, dk.partition_to_basis(case.partition()), b)
op.set_precond(M)
b_dev = torch.from_numpy(b).cuda()
x_dev = torch.empty(A.n, dtype=torch.float64, device="cuda")
hist = np.empty(case.max_iters + 1)
rof = np.empty(case.max_iters + 1, dtype=np.int32)
info = _lib.SolveInfo()


def solve():
    _lib.check(lib.dk_gmres(op.h, ctx.h, b_dev.data_ptr(), None, case.m, case.tol,
                            case.max_iters, 0, x_dev.data_ptr(), _lib.ptr(hist),
                            _lib.ptr(rof), None, C.byref(info)))


for _ in range(2):
    solve()
torch.cuda.synchronize()
lib.dk_timeline_enable(a.cap)
solve()
torch.cuda.synchronize()
buf = np.empty(2 * a.cap, dtype=np.uint64)
n = lib.dk_timeline_read(buf.ctypes.data, a.cap)
rec = buf[:2 * n].reshape(n, 2)
t = rec[:, 0].astype(np.int64)
t -= t.min()
code = rec[:, 1]
kind = (code >> np.uint64(56)).astype(int)
phase = ((code >> np.uint64(48)) & np.uint64(0xff)).astype(int)
blk = (code & np.uint64(0xffffffffffff)).astype(int)
print(f"{n} records, iterations {info.iterations}")
if a.save:  # a 3 ms window of raw records around --at, for offline analysis
    mid = np.sort(t)[int(n * a.at)]
    w = (t >= mid) & (t < mid + 3_000_000)
    np.savez_compressed(a.save, t=t[w], kind=kind[w], phase=phase[w], blk=blk[w])
order = np.argsort(t, kind="stable")
launch = {}
cnt = defaultdict(int)
L = defaultdict(lambda: defaultdict(list))  # (kind, idx) -> phase -> times
for r in order:
    k, p, bl = kind[r], phase[r], blk[r]
    if p == 0:
        cnt[(k, bl)] += 1
    idx = cnt[(k, bl)] - 1
    L[(k, idx)][p].append(t[r])
rows = []
for (k, idx), ph in L.items():
    if k not in KIND:
        continue
    e = min(ph[0]) if ph[0] else None
    st = np.array(ph[1]) if ph[1] else np.array([e])
    sw = max(ph[3]) if ph[3] else None
    ex = max(ph[4] + ph[5]) if (ph[4] or ph[5]) else None
    fin = max(ph[5]) if ph[5] else None
    p2 = float(np.median(ph[2])) if ph[2] else None
    rows.append((e, k, idx, st.min(), np.median(st), st.max(), p2, sw, ex, fin, len(ph[0])))
rows.sort(key=lambda r: r[0])
i0 = int(len(rows) * a.at)
base = rows[i0][0]
f = lambda v: "      -" if v is None else f"{(v - base) / 1e3:7.2f}"  # noqa: E731
print("kind        idx   entry  start0  startM  startN  cells  sweep   exit  final  blocks (us)")
for r in rows[i0:i0 + a.window]:
    e, k, idx, s0, sm, sn, p2, sw, ex, fin, nb = r
    print(f"{KIND[k]:9s} {idx:5d} {f(e)} {f(s0)} {f(sm)} {f(sn)} {f(p2)} {f(sw)} {f(ex)} {f(fin)} {nb:5d}")
# per-kind averages: busy span (first start -> last exit) and the gap to the next launch
spans = defaultdict(list)
gaps = defaultdict(list)
for i, r in enumerate(rows):
    e, k, idx, s0, sm, sn, p2, sw, ex, fin, nb = r
    if ex is None:
        continue
    spans[KIND[k]].append((ex - s0) / 1e3)
    if i + 1 < len(rows) and rows[i + 1][3] is not None:
        gaps[KIND[k] + "->" + KIND[rows[i + 1][1]]].append((rows[i + 1][3] - ex) / 1e3)
print("\nmean span first start -> last exit (us):")
for k, v in spans.items():
    print(f"  {k:10s} {np.mean(v):7.2f}  (n={len(v)})")
print("mean next launch first start - this launch last exit (us; negative = overlap):")
for k, v in gaps.items():
    if len(v) > 20:
        print(f"  {k:22s} {np.mean(v):7.2f}  (n={len(v)})")
tot = (rows[-1][8] or rows[-1][0]) - rows[0][0]
print(f"\nsolve span {tot / 1e3:.1f} us, {tot / 1e3 / max(info.iterations, 1):.2f} us/iteration")

# per-warp view of the tile GEMV (kinds 7/8): time from the launch's first start to
# 2/3 = finisher's own tiles done (3: block row split over > 32 warps), 4/5 = its output written
for k, name in ((7, "tgemv1"), (8, "tgemv2")):
    sel = kind == k
    if not sel.any():
        continue
    # launches of the block-level kind give the first start of each launch
    starts = sorted(r[3] for r in rows if r[1] == k - 4)
    tt = t[sel]
    ph = phase[sel]
    li = np.searchsorted(np.array(starts), tt, side="right") - 1
    rel = (tt - np.array(starts)[np.clip(li, 0, None)]) / 1e3
    print(f"\n{name} per-warp (us after the launch's first start): ")
    for p_, lab in ((0, "warp entry"), (2, "finisher tiles done, np<=32"),
                    (3, "finisher tiles done, np>32"), (4, "split row written, np<=32"),
                    (5, "split row written, np>32")):
        v = rel[ph == p_]
        if len(v):
            print(f"  {lab:30s} n={len(v):7d} median {np.median(v):6.2f} p90 {np.percentile(v, 90):6.2f} max {v.max():6.2f}")
