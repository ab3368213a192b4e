# timeline + rate of the current build (diagnostic; run under gpurun after tools/build_all_variant.sh tl -DDK_TIMELINE)
TAG=${1:-tl}
DK_LIB_PATH=build/variants/tl/libdk.so timeout 300 python tools/timeline.py 3 --window ${2:-24} --at ${3:-0.5} --save gpurun_out/$TAG.npz > gpurun_out/$TAG.txt 2>&1
for r in 1 2; do timeout 200 python tools/variant_probe.py 3 --steps 10 --tag new; done >> gpurun_out/$TAG.txt 2>&1
