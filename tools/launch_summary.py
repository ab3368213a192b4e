"""Summarise an ncu --csv launch list (gpu__time_duration.sum): total / count / mean per kernel."""
import csv
import collections
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    seq = []
    for r in rows:
        if hdr is None:
            if "Kernel Name" in r:
                hdr = r
            continue
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
              "msecond": 1e3}.get(d.get("Metric Unit", "ns"), 1e-3)
        seq.append((d["Kernel Name"], v, d.get("Grid Size", "")))
    return seq


if __name__ == "__main__":
    seq = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, v, _ in seq:
        agg[name[:70]][0] += 1
        agg[name[:70]][1] += v
    tot = sum(v for _, v, _ in seq)
    print(f"total {tot / 1e3:.2f} ms over {len(seq)} launches")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
        print(f"{t / 1e3:9.3f} ms {n:6d} x {t / n:9.1f} us  {k}")
