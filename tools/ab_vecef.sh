for r in 1 2; do
  timeout 200 python tools/variant_probe.py 3 --steps 10 --tag cg
  DK_LIB_PATH=build/variants/vecef/libdk.so timeout 200 python tools/variant_probe.py 3 --steps 10 --tag vec_ef
done > gpurun_out/vecef_ab.log 2>&1
DK_LIB_PATH=build/variants/vecef/libdk.so timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --cache-control none --clock-control none -k regex:"k_tgemv" --launch-skip 3000 -c 4 --csv python tools/variant_probe.py 3 --steps 1 > gpurun_out/ncu_tg3.csv 2>&1
