for r in 1 2; do
  for v in prev 821b5d7 338d4f5 53b22e4; do DK_LIB_PATH=build/variants/$v/libdk.so timeout 200 python tools/variant_probe.py 3 --steps 10 --tag $v; done
  timeout 200 python tools/variant_probe.py 3 --steps 10 --tag cur
done
