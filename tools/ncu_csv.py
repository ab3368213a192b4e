"""Pivot an `ncu --csv --metrics ...` log into one line per launch (diagnostic tool)."""
import csv
import sys
from collections import OrderedDict

rows = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]
r = list(csv.reader(rows))
h = r[0]
ki, mi, vi, ii = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
d = OrderedDict()
for x in r[1:]:
    name = x[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")
    d.setdefault((x[ii], name), {})[x[mi]] = x[vi]
for (i, n), v in d.items():
    print(f"{i:>5} {n[:34]:34s} " + " ".join(f"{k.split('__')[1][:26]}={v[k]}" for k in v))
