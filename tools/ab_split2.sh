for cfg in "DK_TG_CFG=2" "DK_SPLIT=1 DK_TG_CFG=6 DK_DOTS_CTAS_PER_SM=2" "DK_SPLIT=1 DK_TG_CFG=7 DK_DOTS_CTAS_PER_SM=2" "DK_SPLIT=1 DK_TG_CFG=6 DK_DOTS_CTAS_PER_SM=3" "DK_TG_CFG=6"; do
  env $cfg timeout 200 python tools/variant_probe.py 3 --steps 10 --tag "$cfg"
done
