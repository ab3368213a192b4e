#!/bin/bash
# e2e A/B of the late graph (one-off solves) + set-up kernel launch list (diagnostic, gpurun)
mkdir -p gpurun_out
for r in 1 2; do
  timeout 200 python tools/e2e_probe.py 3 4 > gpurun_out/s4_e2e_late_$r.log 2>&1
  DK_NO_LATE_GRAPH=1 timeout 200 python tools/e2e_probe.py 3 4 > gpurun_out/s4_e2e_eager_$r.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/s4_setup_launches.csv python tools/setup_probe.py 3 1 > gpurun_out/s4_setup_ncu.log 2>&1
tail -2 gpurun_out/s4_e2e_*.log
