#!/bin/bash
# ring stencil with two compute groups (diagnostic, gpurun): bitwise checks, then it/s of
# two groups / one group / the register-load stencil (default) at configs 3, 2 and 4
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fallbacks.py -m gpu -x -q > gpurun_out/s7_groups_tests.log 2>&1
tail -3 gpurun_out/s7_groups_tests.log
for r in 1 2; do
  for c in 3 2; do
    timeout 120 python tools/variant_probe.py $c --steps 10 --tag default
    DK_RING=1 DK_RING_GROUPS=2 timeout 120 python tools/variant_probe.py $c --steps 10 --tag ring_groups2
    DK_RING=1 timeout 120 python tools/variant_probe.py $c --steps 10 --tag ring_groups1
    DK_RING=1 DK_RING_GROUPS=2 DK_RING_STAGES=2 timeout 120 python tools/variant_probe.py $c --steps 10 --tag ring_groups2_s2
  done
  timeout 200 python tools/variant_probe.py 4 --steps 2 --max-iters 2000 --tag default
  DK_RING=1 DK_RING_GROUPS=2 timeout 200 python tools/variant_probe.py 4 --steps 2 --max-iters 2000 --tag ring_groups2
done 2>&1 | tee gpurun_out/s7_groups_ab.log
for v in "X=1" "DK_RING=1 DK_RING_GROUPS=2" "DK_RING=1"; do
  env $v timeout 250 python bench.py --no-cpu --e2e-steps 1 --steps 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v', round(d['value'],1), {k:round(v['us'],2) for k,v in d['kernel_avg'].items()})
" | tee -a gpurun_out/s7_groups_ab.log
done
