# full ncu captures of one mid-cycle iteration's K4 (k_project) and K5 (k_gs) (run under gpurun)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02c_gputest.log 2>&1; echo "rc=$?" >> gpurun_out/r02c_gputest.log
timeout 200 python tools/variant_probe.py 3 --steps 10 --tag cur > gpurun_out/r02c_probe.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none \
  -k regex:"k_project|k_gs|k_stencil_sym7" --launch-skip 3075 -c 3 \
  -o gpurun_out/r02c_k4 python tools/variant_probe.py 3 --steps 1 > gpurun_out/r02c_ncu.log 2>&1
