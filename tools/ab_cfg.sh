for r in 1 2; do for cfg in 0 1 2 3 4 5; do
  DK_TG_CFG=$cfg timeout 200 python tools/variant_probe.py 3 --steps 10 --tag "cfg$cfg"
done; done > gpurun_out/cfg_ab.log 2>&1
