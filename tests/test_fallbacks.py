"""The non-spinning fallbacks reproduce the default device path bit for bit (GPU).

Grids whose blocks wait on other blocks of the same grid (the tile GEMV's split-block
finishers, k_gs's fused second Gram-Schmidt pass) and the early starts across grids each have
a non-waiting fallback, chosen automatically when the grid cannot be co-resident and forced by
environment switches (read once per process, so each variant runs in a subprocess):
  DK_NO_SPIN     tile GEMV pieces all go to slots, k_tg_finish sums them after the grid
  DK_NO_GS_FUSE  the second Gram-Schmidt pass as separate launches
  DK_NO_EARLY    no early start of the stencil / k_gs on published partials
  DK_NO_COOP     the spinning grids launched without the cooperative attribute (by default
                 they are cooperative: all blocks co-resident or the launch fails)
  DK_NO_LOOP_GRAPH     one graph launch and one host read of the state per cycle instead of
                       the conditional WHILE graph (restarts decided on the device)
  DK_RING              (opt-in variant) the persistent bulk-copy ring stencil
                       (k_stencil_sym7_ring) instead of the register-load stencil
                       (k_stencil_sym7); DK_RING_STAGES=2: a 2-stage ring; DK_RING_GROUPS=2: two
                       compute groups per block on alternate tiles
  DK_WPF / DK_PF2      (opt-in) L2 prefetches issued by the ring stencil (W tile store) and a
                       tile pass (the projection's constants): hints only, results unchanged
  DK_FUSE_RESTRICT     (opt-in variant) the column sums inside tile pass 1, behind a grid
                       barrier of the cooperative pass
Config 3 uses the nested-dissection tile streams (the spinning finisher) and its x is
compared bitwise; config 1 checks the small-d coarse paths.
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import hashlib, json, sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_1510_02148_b200 as dk
from paper_1510_02148_b200 import configs
case = configs.make_case({cfg})
A, b = case.problem()
M = dk.Preconditioner.jacobi(A)
basis = dk.partition_to_basis(case.partition())
rep = dk.pdgmres(A, b, M=M, m=case.m, basis=basis, tol=case.tol, max_iters=case.max_iters)
print(json.dumps({{"iters": rep.iterations, "relres": rep.final_relres,
                  "launches": rep.kernel_launches, "syncs": rep.host_syncs,
                  "loop": rep.device_loop,
                  "x": hashlib.sha256(np.ascontiguousarray(rep.x).tobytes()).hexdigest(),
                  "hist": hashlib.sha256(np.asarray(rep.residual_history).tobytes()).hexdigest()}}))
"""


def _run(cfg, env_extra):
    env = {k: v for k, v in os.environ.items() if not k.startswith("DK_")}
    env.update(env_extra)
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=str(ROOT), cfg=cfg)],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("cfg", [1, 3])
def test_fallbacks_bitwise(gpu, cfg):
    ref = _run(cfg, {})
    launches = ref.pop("launches")
    # the default path decides its restarts on the device: one host read for the whole loop
    assert ref.pop("loop") is True and ref.pop("syncs") == 1
    for extra in ({"DK_NO_SPIN": "1"},
                  {"DK_NO_SPIN": "1", "DK_NO_GS_FUSE": "1", "DK_NO_EARLY": "1"},
                  {"DK_NO_COOP": "1"}, {"DK_FUSE_RESTRICT": "1"}, {"DK_NO_LOOP_GRAPH": "1"},
                  {"DK_RING": "1"}, {"DK_RING": "1", "DK_RING_STAGES": "2"},
                  {"DK_RING": "1", "DK_RING_GROUPS": "2"},
                  {"DK_WPF": "1", "DK_PF2": "1"}, {"DK_WPF": "1", "DK_PF2": "2", "DK_WPF_EARLY": "0"}):
        got = _run(cfg, extra)
        got_launches = got.pop("launches")
        loop, syncs = got.pop("loop"), got.pop("syncs")
        if "DK_NO_LOOP_GRAPH" in extra:  # the host reads the state after every cycle
            assert loop is False and syncs >= (16 if cfg == 3 else 2), (loop, syncs)
        assert got == ref, (extra, got, ref)
        if cfg == 3 and "DK_NO_SPIN" in extra:  # the default path spins (one launch a pass)
            assert got_launches > launches, (extra, got_launches, launches)
        if cfg == 3 and "DK_FUSE_RESTRICT" in extra:  # one kernel fewer per coarse solve
            assert got_launches < launches, (extra, got_launches, launches)
