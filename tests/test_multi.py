"""Multi-process plumbing of bench.py on CPU (gloo, world_size 2).

The hot path does not shard (BASELINE north_star: one GPU), so N GPUs run N independent
replicas; the only cross-rank operations are the timing reductions (max of per-rank device
time, sum of iterations), which these tests exercise with the gloo backend.
"""
from __future__ import annotations

import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port),
                       "DK_BENCH_BACKEND": "gloo"})
    sys.path.insert(0, str(ROOT))
    import bench
    w, r, local, pg = bench.dist_setup(world)
    try:
        ms = 100.0 * (r + 1)              # per-rank device time
        its = 761.0                       # iterations per rank (identical replicas)
        bench.barrier(pg)
        q.put((r, bench.reduce_max(pg, ms), bench.reduce_sum(pg, its)))
    finally:
        pg.destroy_process_group()


@pytest.mark.timeout(120)
def test_replica_reductions_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=90) for _ in procs)
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    for r, mx, tot in out:
        assert mx == 200.0 and tot == 1522.0
    # whole-job throughput = iterations of all ranks / slowest rank's time
    assert out[0][2] / (out[0][1] * 1e-3) == pytest.approx(7610.0)


def test_reference_arm_nonzero_ranks_exit_without_work(monkeypatch):
    sys.path.insert(0, str(ROOT))
    import bench
    called = []
    monkeypatch.setattr(bench, "host_threads", lambda: called.append(1) or 1)
    bench.run_reference_arm(type("A", (), {"config": 1})(), 2, 1)
    assert called == []


def test_reference_arm_json_contract():
    """`bench.py --impl reference` prints the driver's JSON line (metric / unit / config of our
    arm, impl, cpu_baseline, e2e with zero transfer bytes) by running the reference's own
    solver on the host, with no repo .so mapped into the process."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "0"], cwd=root,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    assert j["impl"] == "reference" and j["unit"] == "iters/s" and j["value"] > 0
    assert j["higher_is_better"] is True and j["n_gpus"] == 1
    assert j["config"]["config_index"] == 1
    assert j["cpu_baseline"]["kind"] in ("reference", "port") and j["cpu_baseline"]["cores"] >= 1
    assert j["native_libs_loaded"] == []
    assert j["e2e"]["value"] == j["value"]
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["d2h_bytes_per_step"] == 0
