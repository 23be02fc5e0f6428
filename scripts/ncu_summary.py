"""Key ncu --set full metrics per kernel from `ncu -i rep --page details --csv`."""
import csv
import subprocess
import sys

WANT = ["Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Issue Slots Busy", "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction",
        "L1/TEX Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Memory Throughput", "Block Limit Registers", "Block Limit Shared Mem"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, ii, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
seen = {}
for r in rows[1:]:
    if r[mi] in WANT:
        key = (r[ii], r[ki].split("(")[0])
        seen.setdefault(key, {})[r[mi]] = f"{r[vi]} {r[ui]}"
for (i, k), d in seen.items():
    print(f"== [{i}] {k}")
    for m in WANT:
        if m in d:
            print(f"   {m:36s} {d[m]}")
