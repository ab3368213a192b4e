# quick A/B of the current build (diagnostic; run under gpurun)
timeout 600 python -m pytest tests/test_device_solve.py tests/test_device_ops.py -x -q 2>&1 | tail -2
for r in 1 2; do timeout 200 python tools/variant_probe.py ${1:-3} --steps 10 --tag cur; done
