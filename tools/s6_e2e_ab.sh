#!/bin/bash
# e2e A/B: loop graph / late graph switches through the public-API phase probe (diagnostic, gpurun)
mkdir -p gpurun_out
for r in 1 2; do
  timeout 200 python tools/e2e_probe.py 3 4 > gpurun_out/s6_e2e_default_$r.log 2>&1
  DK_NO_LOOP_GRAPH=1 timeout 200 python tools/e2e_probe.py 3 4 > gpurun_out/s6_e2e_noloop_$r.log 2>&1
  DK_NO_LATE_GRAPH=1 timeout 200 python tools/e2e_probe.py 3 4 > gpurun_out/s6_e2e_nolate_$r.log 2>&1
done
tail -3 gpurun_out/s6_e2e_*.log
