#!/bin/bash
# GPU-box profiling pass of one round (run under gpurun from the repo root): bench lines
# (config 3 + the other BASELINE configs + the reference arm), the ncu launch list (time +
# DRAM bytes per launch) of an event-profiled config-3 solve, one full ncu capture of the
# iteration kernels of a graph-replayed solve.  Outputs under gpurun_out/$TAG*.
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.log
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_reference.log 2>&1
# config 1 solves take 1.7 ms: enough steps that the clock sampler's start-up does not weigh
timeout 600 python bench.py --config 1 --steps 100 --warmup 10 > gpurun_out/${TAG}_bench_config1.log 2>&1
timeout 600 python bench.py --config 2 --steps 20 --warmup 3 > gpurun_out/${TAG}_bench_config2.log 2>&1
timeout 900 python bench.py --config 4 --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_config4.log 2>&1
timeout 1500 python bench.py --config 5 --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/${TAG}_bench_config5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python tools/kprof.py 3 > gpurun_out/${TAG}_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"k_project|k_gs|k_stencil_sym7|k_tgemv|k_restrict" --launch-skip 3000 -c 6 \
  -o gpurun_out/${TAG}_full env DK_NO_LOOP_GRAPH=1 python tools/variant_probe.py 3 --steps 1 > gpurun_out/${TAG}_full.log 2>&1
echo done
