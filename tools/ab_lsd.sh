for r in 1 2; do
  DK_DENSE_LSD=1 timeout 200 python tools/variant_probe.py 3 --steps 10 --tag dense_lsd
  timeout 200 python tools/variant_probe.py 3 --steps 10 --tag sparse_lsd
done
DK_DENSE_LSD=1 timeout 300 python tools/e2e_probe.py 2>&1 | tail -2
timeout 300 python tools/e2e_probe.py 2>&1 | tail -2
