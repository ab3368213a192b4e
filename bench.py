"""Benchmark of the deflated-GMRES hot path (BASELINE.json metric) — one JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

A step is one full PDGMRES solve (x0 = 0 to tol 1e-8) of the BASELINE workload: config 3,
60x220x85, subdomain-levelset deflation (d = 10,917 columns), Jacobi, GMRES(50).  Synthetic
seeded inputs (paper_1510_02148_b200/configs.py).

  value     iterations/s over K device-resident solves (operator, basis, E^-1 and b already in
            HBM; CUDA events on the solver's stream; max over ranks)
  e2e       the same metric through the public API `pdgmres` with HOST numpy buffers: operator
            upload, deflation setup (E assembly, LU, E^-1, x*), solve and x download per step
  roofline  the dominant kernel class of an event-profiled solve: algorithmic bytes / time
  cpu_baseline  the reference solver on the host cores (CpuReference), rank 0, N = 1

--impl reference times the reference's own `_run_cycles` (the unmodified package installed
under baseline/_ref) with all host threads, one GMRES(m) cycle per step, on the same
workload, with inputs and labels built without the device library (no libdk.so in the
process; the JSON line lists the repo .so files mapped, which must be none).
Multi-GPU: the path does not shard (BASELINE north_star: one GPU), so N ranks run N
independent replicas (weak scaling, no collective on the data path).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "deflated-GMRES iters/s, time-to-solve, HBM GB/s vs peak @ 60x220x85"
UNIT = "iters/s"


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", "--query-gpu=" + ",".join(self.FIELDS),
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[k] for r in self.rows for k in range(4)
                          if len(r) > 2 + k and r[2 + k].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------------------
def dist_setup(gpus: int):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("DK_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
        pg = dist
    return world, rank, local, pg


def reduce_max(pg, value: float) -> float:
    if pg is None:
        return value
    import torch
    dev = "cuda" if os.environ.get("DK_BENCH_BACKEND", "nccl") == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(pg, value: float) -> float:
    if pg is None:
        return value
    import torch
    dev = "cuda" if os.environ.get("DK_BENCH_BACKEND", "nccl") == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    pg.all_reduce(t, op=pg.ReduceOp.SUM)
    return float(t.item())


def barrier(pg):
    if pg is not None:
        pg.barrier()


# ---------------------------------------------------------------------------------------
def load_reference():
    """The unmodified reference package (`defkrylov`, pure Python) installed under
    baseline/_ref by `pip install --target baseline/_ref`; None if absent."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "defkrylov" / "__init__.py").exists():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import defkrylov
    return defkrylov


def native_libs_loaded():
    """Shared objects of this repo mapped into the process (the reference arm must have none)."""
    try:
        maps = Path("/proc/self/maps").read_text().splitlines()
    except OSError:
        return []
    return sorted({ln.split()[-1] for ln in maps
                   if ln.endswith(".so") and str(ROOT) in ln and "baseline/_ref" not in ln})


def config_dict(case, idx: int, n: int, d: int, seed: int, world: int) -> dict:
    """The workload description; identical in both arms (`same_config`)."""
    vmb = (case.m + 1) * 8.0 * n / 1e6
    return {"workload": case.name, "config_index": idx, "n_cells": n,
            "d": d, "m": case.m, "tol": case.tol, "seed": seed,
            "parallelism": f"replicas{world}" if world > 1 else "single",
            "l2": (f"inputs larger than L2: the basis V alone is {vmb:.0f} MB and every "
                   f"iteration streams hundreds of MB (126 MB L2), no flush needed"
                   if vmb > 126 else
                   f"L2-resident working set (V = {vmb:.0f} MB < 126 MB L2, not flushed): "
                   f"a latency measurement, not the BASELINE workload")}


class CpuReference:
    """The reference solver on the host cores, built without the device library.

    Inputs: the seeded k field (configs.py generator, numpy), the host TPFA assembly
    (bit-identical to the reference's assemble_pressure, tests/test_testbed.py) and labels
    from the oracle's labeller (pinned to the reference's label CRCs).  Solver: the
    reference's own `_run_cycles` (krylov.py:107-236) from baseline/_ref with the
    label-based context of SURVEY.md §0.3 (O.ReferenceLabelContext: R.spmv, R.dense_lu,
    R.lu_solve), or — when baseline/_ref is missing — the oracle port (oracle/dk_oracle.py).
    One step = one GMRES(m) cycle (m iterations) from x0 = 0, plus the reference's
    reconstruct and true-residual epilogue.
    """

    def __init__(self, case, idx: int, A=None, b=None):
        from oracle import dk_oracle as O
        self.O = O
        self.case = case
        self.idx = idx
        t0 = time.perf_counter()
        if A is None:
            A, b = case.problem()
        off, dg = A.dia()
        self.n = A.n
        self.b = b
        Ac = O.csr_from_dia_lean(A.n, off, dg)
        g = case.grid
        px, py, pz = case.boxes
        lab, d, excl = O.subdomain_levelset_labels_boxwise(
            case.band_field.kx, g.nx, g.ny, g.nz, px, py, pz, case.jump_threshold)
        col, self.d = O.columns_from_labels(lab, d, excl)
        self.R = load_reference()
        if self.R is not None:
            R = self.R
            self.kind = "reference"
            self.A = R.SparseMatrix(A.n, Ac.indptr, Ac.indices, Ac.data)
            self.M = R.Preconditioner.jacobi(self.A)
            self.ctx = O.ReferenceLabelContext(R, self.A, col, self.d, b)
            from defkrylov.krylov import _run_cycles
            self._run = _run_cycles
        else:
            self.kind = "port"
            self.A = Ac
            self.inv = 1.0 / dg[list(off).index(0)]
            self.ctx = O.LabelDeflation(Ac, col, self.d, b, self.inv)
        self.setup_s = time.perf_counter() - t0

    def cycle(self) -> int:
        c = self.case
        if self.kind == "reference":
            rep = self._run(self.A, self.b, np.zeros(self.n), self.M, c.m, c.tol, c.m, 0,
                            self.ctx, None, False)
            return int(rep.iterations)
        r = self.O.run_cycles(self.A, self.b, None, self.inv, c.m, c.tol, c.m, 0, self.ctx)
        return int(r["iterations"])

    def sample(self, steps: int) -> str:
        what = ("the reference's own _run_cycles (baseline/_ref defkrylov, krylov.py:107-236)"
                " with a label-based deflation context" if self.kind == "reference" else
                "the oracle port of _run_cycles (baseline/_ref not installed)")
        return (f"{steps} x one GMRES({self.case.m}) cycle ({self.case.m} iterations) of "
                f"config {self.idx} from x0=0: {what}, d={self.d}; set-up "
                f"(operator, labels, E + LU, x*) {self.setup_s:.1f}s excluded")


def run_reference_arm(args, world, rank):
    """--impl reference: the reference solver on the host cores, rank 0 only."""
    if rank != 0:
        return
    threads = host_threads()
    from threadpoolctl import threadpool_limits
    threadpool_limits(threads)
    from paper_1510_02148_b200 import configs
    case = configs.make_case(args.config, seed=args.seed)
    ref = CpuReference(case, args.config)
    for _ in range(args.warmup):
        ref.cycle()
    its = 0
    t = time.perf_counter()
    for _ in range(args.steps):
        its += ref.cycle()
    sec = time.perf_counter() - t
    v = its / sec
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_dict(case, args.config, ref.n, ref.d, args.seed, world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": ref.kind,
                         "sample": ref.sample(args.steps)},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "native_libs_loaded": native_libs_loaded(),
    }), flush=True)


# ---------------------------------------------------------------------------------------
def run_ours(args, world, rank, local, pg):
    import ctypes as C

    import torch

    import paper_1510_02148_b200 as dk
    from paper_1510_02148_b200 import _lib, configs

    lib = _lib.load()
    _lib.check(lib.dk_set_device(local), "dk_set_device")
    torch.cuda.set_device(local)
    case = configs.make_case(args.config, seed=args.seed)
    A, b = case.problem()
    part = case.partition()
    basis = dk.partition_to_basis(part)
    M = dk.Preconditioner.jacobi(A)
    n = A.n
    # ---------------- device-resident solves (value) -------------------------------------
    op = A.device()
    stream = torch.cuda.current_stream()
    _lib.check(lib.dk_op_set_stream(op.h, C.c_void_p(stream.cuda_stream)))
    # set-up timed warm (a first context loads the kernels and fills the buffer pool)
    dk.build_context(A, M, basis, b).close()
    torch.cuda.synchronize()
    t_setup = time.perf_counter()
    ctx = dk.build_context(A, M, basis, b)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    setup_ms = ctx.setup_ms()
    b_dev = torch.from_numpy(b).to(f"cuda:{local}")
    x_dev = torch.empty(n, dtype=torch.float64, device=f"cuda:{local}")
    cap = case.max_iters + 1
    hist = np.empty(cap)
    rof = np.empty(cap, dtype=np.int32)
    info = _lib.SolveInfo()

    def solve():
        rc = lib.dk_gmres(op.h, ctx.h, b_dev.data_ptr(), None, case.m, case.tol, case.max_iters,
                          0, x_dev.data_ptr(), _lib.ptr(hist), _lib.ptr(rof), None,
                          C.byref(info))
        _lib.check(rc, "dk_gmres")
        return int(info.iterations), int(info.kernel_launches)

    for _ in range(args.warmup):
        solve()
    barrier(pg)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    its = launches = 0
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            i, l = solve()
            its += i
            launches += l
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier(pg)
    ms = ev0.elapsed_time(ev1)
    ms_max = reduce_max(pg, ms)
    its_total = reduce_sum(pg, float(its))
    value = its_total / (ms_max * 1e-3)
    iters_per_solve = its // args.steps
    converged = bool(info.converged)
    relres = float(info.final_relres)
    # ---------------- roofline: event-profiled solve -----------------------------------
    lib.dk_op_profile(op.h, 1)
    solve()
    names = (C.c_char_p * 16)()
    pms = (C.c_double * 16)()
    pn = (C.c_int64 * 16)()
    pb = (C.c_double * 16)()
    k = lib.dk_op_profile_read(op.h, 16, names, pms, pn, pb)
    lib.dk_op_profile(op.h, 0)
    prof = {names[i].decode(): {"ms": pms[i], "launches": int(pn[i]), "bytes": pb[i]}
            for i in range(k) if pn[i] > 0}
    peak, peak_kind = peaks()
    dom = max(prof, key=lambda kname: prof[kname]["ms"])
    dk_ = prof[dom]
    avg_s = dk_["ms"] * 1e-3 / dk_["launches"]
    bytes_per_launch = dk_["bytes"] / dk_["launches"]
    achieved = bytes_per_launch / avg_s / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        tr = json.loads(tfile.read_text()).get(str(args.config), {})
        traffic = tr.get(dom)
    tot_bytes = sum(v["bytes"] for v in prof.values())
    tot_s = sum(v["ms"] for v in prof.values()) * 1e-3
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "kernel": dom,
                "peak_source": f"{peak_kind} MEASURED_PEAKS.json hbm_gbs" if peak_kind ==
                "measured" else "fallback 6650 GB/s (B200_PROFILING.md)",
                "bytes_per_launch": bytes_per_launch, "avg_launch_us": avg_s * 1e6}
    bytes_per_iter = tot_bytes / max(iters_per_solve, 1)
    per_rank_rate = value / world
    iteration_roofline = {
        "achieved": bytes_per_iter * per_rank_rate / 1e9, "peak": peak,
        "frac": bytes_per_iter * per_rank_rate / 1e9 / peak,
        "bytes_per_iter": bytes_per_iter,
        "note": "algorithmic bytes of every kernel of an iteration (incl. restart/cycle-end "
                "amortised) x timed iterations/s of the graph-replayed solve (per GPU)",
        "event_profiled": {"achieved": tot_bytes / tot_s / 1e9,
                           "frac": tot_bytes / tot_s / 1e9 / peak,
                           "note": "same bytes over the summed per-kernel CUDA-event times of "
                                   "a non-graph (launch-per-kernel) profiled solve"}}
    share = {kname: v["ms"] / (tot_s * 1e3) for kname, v in prof.items()}
    kernel_avg = {kname: {"us": 1e3 * v["ms"] / v["launches"], "launches": v["launches"],
                          "GB/s": v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["ms"] > 0 else None}
                  for kname, v in prof.items()}
    # ---------------- e2e through the public API with host buffers ----------------------
    off, dg = A.dia()
    e2e_its = 0
    e2e_sec = 0.0
    for s in range(max(1, args.e2e_steps) + 1):
        A_host = dk.SparseMatrix.from_dia(n, off, dg)  # fresh: the operator is uploaded
        torch.cuda.synchronize()
        t = time.perf_counter()
        rep = dk.pdgmres(A_host, b, M=M, m=case.m, basis=basis, tol=case.tol,
                         max_iters=case.max_iters)
        sec = time.perf_counter() - t
        A_host.release_device()
        if os.environ.get("DK_TRACE"):
            print(f"e2e call {s}: {sec:.4f}s", file=sys.stderr, flush=True)
        if s > 0:  # first call warms the library / allocator
            e2e_its += rep.iterations
            e2e_sec += sec
    e2e_v = e2e_its / e2e_sec
    ndiag = len(off)
    h2d = 8 * n * ndiag + 8 * n + 4 * n + 8 * n  # diagonals, M^-1, labels, b (x0 = 0: none)
    d2h = 8 * n + 8 * (case.max_iters + 1) + 4 * (case.max_iters + 1)
    # ---------------- CPU baseline (rank 0, N = 1) ---------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = host_threads()
        from threadpoolctl import threadpool_limits
        with threadpool_limits(threads):
            ref = CpuReference(case, args.config, A, b)
            ref.cycle()  # warm-up
            t = time.perf_counter()
            ci = sum(ref.cycle() for _ in range(args.cpu_cycles))
            cs = time.perf_counter() - t
        cpu = {"value": ci / cs, "unit": UNIT, "cores": threads, "kind": ref.kind,
               "sample": ref.sample(args.cpu_cycles)}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(case, args.config, n, basis.d, args.seed, world),
            "iterations_per_solve": iters_per_solve, "converged": converged,
            "final_relres": relres, "time_to_solve_s": ms_max * 1e-3 / args.steps,
            "setup_s": setup_s, "setup_ms": setup_ms,
            "e2e": {"value": e2e_v, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "time_to_solve_s": e2e_sec / max(1, args.e2e_steps),
                    "path": "paper_1510_02148_b200.pdgmres on host numpy arrays (operator "
                            "upload + E setup + solve + x download)"},
            "roofline": roofline, "iteration_roofline": iteration_roofline,
            "kernel_share": share, "kernel_avg": kernel_avg,
            "cpu_baseline": cpu, "gpu_launches": launches, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-cycles", type=int, default=1)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        # CPU arm: rank 0 alone runs and prints; other ranks exit without work
        world = int(os.environ.get("WORLD_SIZE", "1"))
        run_reference_arm(args, world, int(os.environ.get("RANK", "0")))
        return
    world, rank, local, pg = dist_setup(args.gpus)
    try:
        run_ours(args, world, rank, local, pg)
    finally:
        if pg is not None:
            pg.destroy_process_group()


if __name__ == "__main__":
    main()
