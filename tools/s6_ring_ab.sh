#!/bin/bash
# ring stencil A/B (diagnostic, gpurun): bitwise fallback test, then it/s with/without the ring
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fallbacks.py tests/test_device_ops.py -m gpu -x -q > gpurun_out/s6_ring_tests.log 2>&1
tail -5 gpurun_out/s6_ring_tests.log
for r in 1 2; do
  timeout 120 python tools/variant_probe.py 3 --steps 10 --tag ring4
  DK_RING_STAGES=3 timeout 120 python tools/variant_probe.py 3 --steps 10 --tag ring3
  DK_RING_STAGES=2 timeout 120 python tools/variant_probe.py 3 --steps 10 --tag ring2
  DK_NO_RING=1 timeout 120 python tools/variant_probe.py 3 --steps 10 --tag noring
done 2>&1 | tee gpurun_out/s6_ring_ab.log
