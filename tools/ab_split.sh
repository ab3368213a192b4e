# split iteration A/B (diagnostic; run under gpurun)
for cfg in "DK_NO_SPLIT=1" "DK_TG_CFG=0" "DK_TG_CFG=5" "DK_TG_CFG=5 DK_DOTS_CTAS_PER_SM=3" "DK_TG_CFG=4" "DK_TG_CFG=3"; do
  env $cfg timeout 200 python tools/variant_probe.py 3 --steps 10 --tag "$cfg"
done > gpurun_out/split_ab.log 2>&1
DK_TG_CFG=5 DK_LIB_PATH=build/variants/tl/libdk.so timeout 300 python tools/timeline.py 3 --window 14 --at 0.5 > gpurun_out/tl_split.txt 2>&1
