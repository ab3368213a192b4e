# A/B of the current libdk.so against build/variants/base (diagnostic; run under gpurun)
for r in 1 2; do
  DK_LIB_PATH=build/variants/base/libdk.so timeout 300 python tools/kprof.py 3 --max-iters 200 | sed 's/^/base /'
  timeout 300 python tools/kprof.py 3 --max-iters 200 | sed 's/^/new  /'
done > gpurun_out/ab_kprof.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum --cache-control none --clock-control none -k regex:k_tgemv --launch-skip 200 -c 8 --csv python tools/variant_probe.py 3 --steps 1 > gpurun_out/ab_ncu_new.csv 2>&1
DK_LIB_PATH=build/variants/base/libdk.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum --cache-control none --clock-control none -k regex:k_tgemv --launch-skip 200 -c 8 --csv python tools/variant_probe.py 3 --steps 1 > gpurun_out/ab_ncu_base.csv 2>&1
cat gpurun_out/ab_kprof.log
