for r in 1 2 3; do
  DK_LIB_PATH=build/variants/k4single/libdk.so timeout 200 python tools/variant_probe.py 3 --steps 10 --tag single
  timeout 200 python tools/variant_probe.py 3 --steps 10 --tag pair
done
