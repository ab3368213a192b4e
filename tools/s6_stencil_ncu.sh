#!/bin/bash
# kernel-only durations of the stencil variants (ncu launch list of event-profiled solves)
mkdir -p gpurun_out
for v in "X=1" "DK_NO_RING=1" "DK_RING_STAGES=2"; do
  for p in "" "--plain"; do
    env $v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_stencil_sym7" --csv \
      --log-file gpurun_out/s6_st.csv python tools/kprof.py 3 $p --max-iters 60 > /dev/null 2>&1
    python - "$v $p" <<'PY'
import csv,sys,statistics
rows=[r for r in csv.reader(open('gpurun_out/s6_st.csv')) if len(r)>5]
hdr=rows[0]; ix={k:i for i,k in enumerate(hdr)}
vals=[float(r[ix['Metric Value']].replace(',','')) for r in rows[1:] if r[ix['Metric Name']]=='gpu__time_duration.sum']
unit=[r[ix['Metric Unit']] for r in rows[1:]][0] if len(rows)>1 else '?'
print(sys.argv[1], 'n',len(vals),'median',statistics.median(vals) if vals else None, unit, 'min', min(vals) if vals else None)
PY
  done
done
