"""Aggregate ncu warp-stall samples by CUDA source line (cuda,sass page)."""
import csv
import sys
from collections import defaultdict

path, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
files = {}
cur_file = None
agg = defaultdict(int)
src = {}
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ws = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= ws:
        continue
    line = r[0]
    if line.strip():
        last = (cur_file, line)
        src[last] = r[1][:100]
    try:
        agg[last] += int(r[ws] or 0)
    except (ValueError, NameError):
        pass
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]} {src.get(k, '').strip()}")
