"""Print selected 'details' metrics of an ncu report (diagnostic)."""
import csv
import io
import subprocess
import sys

KEYS = ("Duration", "SM Frequency", "DRAM Throughput", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Executed Ipc Active", "Eligible Warps Per Scheduler",
        "Achieved Occupancy", "Registers Per Thread", "Warp Cycles Per Issued Instruction",
        "Grid Size", "Block Size", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Issue Slots Busy", "No Eligible")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ix = {k: i for i, k in enumerate(hdr)}
cur = None
for r in rows[1:]:
    if len(r) <= ix["Metric Value"]:
        continue
    name = r[ix["Kernel Name"]][:60]
    if name != cur:
        print("==", name, "launch", r[ix["ID"]])
        cur = name
    if r[ix["Metric Name"]] in KEYS:
        print(f"   {r[ix['Section Name']][:28]:28s} {r[ix['Metric Name']]:36s} {r[ix['Metric Value']]:>12s} {r[ix['Metric Unit']]}")
