"""Executed-instruction histogram by SASS opcode from an ncu source page
(ncu -i X.ncu-rep --page source --csv --print-source cuda,sass)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = defaultdict(int)
stall = defaultdict(int)
tot = 0
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        si = 3
        ei = hdr.index("Instructions Executed")
        wi = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= ei or not r[si].strip() or not r[2].startswith("0x"):
        continue
    toks = r[si].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    try:
        n = int(r[ei] or 0)
        w = int(r[wi] or 0)
    except ValueError:
        continue
    agg[op] += n
    stall[op] += w
    tot += n
ws = sum(stall.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{k:12s} {100 * v / tot:5.1f}% of instructions  {100 * stall[k] / ws:5.1f}% of stall samples")
print("total warp instructions", tot)
