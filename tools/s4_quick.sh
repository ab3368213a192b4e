#!/bin/bash
# GPU tests + e2e probe + set-up launch list (diagnostic, gpurun).  $1 = tag
T=${1:-s4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_gputest.log
timeout 200 python tools/e2e_probe.py 3 4 > gpurun_out/${T}_e2e.log 2>&1
DK_NO_SPLITK=1 timeout 200 python tools/e2e_probe.py 3 4 > gpurun_out/${T}_e2e_nosplit.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_setup_launches.csv python tools/setup_probe.py 3 1 > gpurun_out/${T}_setup_ncu.log 2>&1
tail -n 3 gpurun_out/${T}_gputest.log gpurun_out/${T}_e2e.log gpurun_out/${T}_e2e_nosplit.log
