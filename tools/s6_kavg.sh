#!/bin/bash
# per-kernel event times (bench's profiled solve) under the current environment variants
for v in "DK_RING_STAGES=4" "DK_RING_STAGES=3" "DK_RING_STAGES=2" "DK_NO_RING=1"; do
  env $v timeout 250 python bench.py --no-cpu --e2e-steps 1 --steps 3 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v', round(d['value'],1), {k:round(v['us'],2) for k,v in d['kernel_avg'].items()})
"
done
