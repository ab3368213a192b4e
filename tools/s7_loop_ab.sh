#!/bin/bash
# loop graph / ring stencil A/B at the other configs (diagnostic, gpurun)
mkdir -p gpurun_out
for r in 1 2; do
  for c in 1 2; do
    timeout 120 python tools/variant_probe.py $c --steps 20 --tag default
    DK_NO_LOOP_GRAPH=1 timeout 120 python tools/variant_probe.py $c --steps 20 --tag noloop
    DK_NO_RING=1 timeout 120 python tools/variant_probe.py $c --steps 20 --tag noring
    DK_NO_RING=1 DK_NO_LOOP_GRAPH=1 timeout 120 python tools/variant_probe.py $c --steps 20 --tag noloop_noring
  done
  timeout 200 python tools/variant_probe.py 4 --steps 2 --max-iters 2000 --tag default
  DK_NO_LOOP_GRAPH=1 timeout 200 python tools/variant_probe.py 4 --steps 2 --max-iters 2000 --tag noloop
  DK_NO_RING=1 timeout 200 python tools/variant_probe.py 4 --steps 2 --max-iters 2000 --tag noring
  DK_NO_RING=1 DK_NO_LOOP_GRAPH=1 timeout 200 python tools/variant_probe.py 4 --steps 2 --max-iters 2000 --tag noloop_noring
  timeout 120 python tools/variant_probe.py 3 --steps 10 --tag default
  DK_NO_LOOP_GRAPH=1 timeout 120 python tools/variant_probe.py 3 --steps 10 --tag noloop
done 2>&1 | tee gpurun_out/s7_loop_ab.log
