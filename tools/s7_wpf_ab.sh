#!/bin/bash
# L2 prefetches riding on latency-bound kernels (diagnostic, gpurun): the W tile store from the
# ring stencil (DK_NO_WPF / DK_WPF_EARLY) and the projection's constants from a tile pass
# (DK_PF2 / DK_PF2_N): bitwise checks, then it/s of each variant, three rounds
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fallbacks.py tests/test_device_ops.py tests/test_device_solve.py -m gpu -x -q > gpurun_out/s7_wpf_tests.log 2>&1
tail -3 gpurun_out/s7_wpf_tests.log
for r in 1 2 3; do
  timeout 120 python tools/variant_probe.py 3 --steps 10 --tag wpf+pf2_1
  DK_PF2=0 timeout 120 python tools/variant_probe.py 3 --steps 10 --tag wpf
  DK_PF2=0 DK_NO_WPF=1 timeout 120 python tools/variant_probe.py 3 --steps 10 --tag none
  DK_NO_WPF=1 timeout 120 python tools/variant_probe.py 3 --steps 10 --tag pf2_1
  DK_PF2=2 timeout 120 python tools/variant_probe.py 3 --steps 10 --tag wpf+pf2_2
  DK_PF2_N=2 timeout 120 python tools/variant_probe.py 3 --steps 10 --tag wpf+pf2_1_n2
  DK_PF2_N=3 timeout 120 python tools/variant_probe.py 3 --steps 10 --tag wpf+pf2_1_n3
  DK_PF2=0 DK_WPF_EARLY=0 timeout 120 python tools/variant_probe.py 3 --steps 10 --tag wpf_early0
  DK_PF2=0 DK_WPF_EARLY=99 timeout 120 python tools/variant_probe.py 3 --steps 10 --tag wpf_early_all
done 2>&1 | tee gpurun_out/s7_wpf_ab.log
for v in "X=1" "DK_PF2=0" "DK_NO_WPF=1 DK_PF2=0"; do
  env $v timeout 250 python bench.py --no-cpu --e2e-steps 1 --steps 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v', round(d['value'],1), {k:round(v['us'],2) for k,v in d['kernel_avg'].items()})
" | tee -a gpurun_out/s7_wpf_ab.log
done
