for r in 1 2 3; do
  DK_LIB_PATH=build/variants/prev/libdk.so timeout 200 python tools/variant_probe.py 3 --steps 10 --tag prev
  timeout 200 python tools/variant_probe.py 3 --steps 10 --tag cur
  DK_LIB_PATH=build/variants/base/libdk.so timeout 200 python tools/variant_probe.py 3 --steps 10 --tag round1
done
