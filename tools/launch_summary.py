"""Summarise an ncu --csv launch list: total / count / mean time per kernel and, when the list
carries dram__bytes_read.sum / dram__bytes_write.sum, the mean DRAM bytes per launch.

    python tools/launch_summary.py LIST.csv [TOP] [--json OUT.json --config 3]

--json merges {config: {class: mean DRAM bytes per launch}} for the iteration kernel classes
bench.py reports (profiles/ncu_traffic.json).
"""
import collections
import csv
import json
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
BYTES = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
# kernel-name prefix -> bench.py / dk_op_profile class
# (a class launch of coarse_gemv is the two tile passes: twice the per-kernel bytes)
CLASSES = {"void dk::k_project<0,": ("prolong_dots", 1), "void dk::k_gs<0>": ("gs_update", 1),
           "void dk::k_stencil_sym7<1, 1, 1>": ("stencil_restrict", 1),
           "void dk::k_stencil_sym7_ring<1, 1, 1>": ("stencil_restrict", 1),
           "void dk::k_stencil<0, 1, 1, 1>": ("stencil_restrict", 1),
           "dk::k_restrict_final": ("restrict_final", 1),
           "void dk::<unnamed>::k_tgemv": ("coarse_gemv", 2)}


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    launches = collections.OrderedDict()
    for r in rows:
        if hdr is None:
            if "Kernel Name" in r:
                hdr = r
            continue
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (d["ID"], d["Kernel Name"])
        rec = launches.setdefault(key, {})
        v = float(d["Metric Value"].replace(",", ""))
        name = d.get("Metric Name")
        if name == "gpu__time_duration.sum":
            rec["us"] = v * UNIT.get(d.get("Metric Unit", "ns"), 1e-3)
        elif name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            rec["bytes"] = rec.get("bytes", 0.0) + v * BYTES.get(d.get("Metric Unit", "byte"), 1.0)
    return [(k[1], rec.get("us", 0.0), rec.get("bytes")) for k, rec in launches.items()]


def main():
    args = sys.argv[1:]
    out_json = cfg = None
    if "--json" in args:
        i = args.index("--json")
        out_json = args[i + 1]
        del args[i:i + 2]
    if "--config" in args:
        i = args.index("--config")
        cfg = args[i + 1]
        del args[i:i + 2]
    seq = load(args[0])
    top = int(args[1]) if len(args) > 1 else 20
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for name, us, by in seq:
        a = agg[name[:70]]
        a[0] += 1
        a[1] += us
        a[2] += by or 0.0
    tot = sum(us for _, us, _ in seq)
    print(f"total {tot / 1e3:.2f} ms over {len(seq)} launches")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        dram = f"  DRAM {b / n / 1e6:8.1f} MB/launch {b / (t * 1e-6) / 1e9:7.0f} GB/s" if b else ""
        print(f"{t / 1e3:9.3f} ms {n:6d} x {t / n:9.1f} us{dram}  {k}")
    if out_json:
        cls = collections.defaultdict(lambda: [0, 0.0])
        for name, us, by in seq:
            for pre, (c, mult) in CLASSES.items():
                if name.startswith(pre) and by is not None:
                    cls[c][0] += 1.0 / mult
                    cls[c][1] += by
        try:
            data = json.load(open(out_json))
        except (OSError, ValueError):
            data = {}
        data.setdefault(cfg or "3", {}).update({c: b / n for c, (n, b) in cls.items()})
        data["note"] = ("mean dram__bytes_read.sum + dram__bytes_write.sum per launch of each "
                        "iteration kernel class over an ncu launch list of an event-profiled "
                        "config-3 solve (tools/profile_round.sh; cold caches between launches)")
        json.dump(data, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main()
