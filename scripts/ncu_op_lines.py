"""Executed count of one SASS opcode by CUDA source line (ncu source page csv)."""
import csv
import sys
from collections import defaultdict

path, opc = sys.argv[1], sys.argv[2].split(",")
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
rows = list(csv.reader(open(path)))
hdr = None
cur = None
agg = defaultdict(int)
src = {}
fname = ""
tot = 0
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ei = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) <= ei:
        continue
    if r[0].strip():
        cur = (fname, r[0])
        src[cur] = r[1].strip()[:90]
        continue
    if not r[2].startswith("0x"):
        continue
    toks = r[3].split()
    op = (toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
    n = int(r[ei] or 0)
    tot += n
    if op in opc:
        agg[cur] += n
s = sum(agg.values())
print(f"{opc}: {s} of {tot} = {100 * s / tot:.1f}%")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100 * v / tot:5.2f}% {k[0]}:{k[1]} {src[k]}")
