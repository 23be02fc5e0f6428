"""Markdown table of the judged metrics per kernel from an ncu --set full report."""
import csv
import subprocess
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
        "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
M = {
    "gpu__time_duration.sum": ("time (us)", None),
    "dram__bytes_read.sum": ("DRAM read (MB)", None),
    "dram__bytes_write.sum": ("DRAM write (MB)", None),
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": ("DRAM % peak", 1),
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": ("FP64 pipe %", 1),
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": ("DMMA pipe %", 1),
    "sm__warps_active.avg.pct_of_peak_sustained_active": ("occupancy %", 1),
    "l1tex__throughput.avg.pct_of_peak_sustained_active": ("L1 %", 1),
    "sm__inst_executed.avg.per_cycle_active": ("IPC", 1),
    "launch__registers_per_thread": ("regs", 1),
}
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
idx = {k: h.index(k) for k in M if k in h}
ki = h.index("Kernel Name")
print("| kernel | " + " | ".join(M[k][0] for k in idx) + " |")
print("|---" * (len(idx) + 1) + "|")
for r in rows[2:]:
    name = r[ki].split("(")[0].replace("void ", "")
    vals = []
    for k, i in idx.items():
        try:
            sc = M[k][1] if M[k][1] is not None else UNIT.get(rows[1][i], 1.0)
            v = float(r[i].replace(",", "")) * sc
            vals.append(f"{v:.1f}" if abs(v) < 1e5 else f"{v:.3g}")
        except ValueError:
            vals.append(r[i])
    print(f"| `{name}` | " + " | ".join(vals) + " |")
