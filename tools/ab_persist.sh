for r in 1 2; do
  DK_NO_W_PERSIST=1 timeout 200 python tools/variant_probe.py 3 --steps 10 --tag evict_last
  timeout 200 python tools/variant_probe.py 3 --steps 10 --tag persist
done > gpurun_out/persist_ab.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --cache-control none --clock-control none -k regex:"k_tgemv" --launch-skip 3000 -c 6 --csv python tools/variant_probe.py 3 --steps 1 > gpurun_out/ncu_tg2.csv 2>&1
