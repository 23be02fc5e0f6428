import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/launches.csv')))
for i, r in enumerate(rows):
    if 'Kernel Name' in r:
        hdr = r; start = i + 1; break
ki, mi, vi, ui = (hdr.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
idi = hdr.index('ID')
agg = collections.OrderedDict()
for r in rows[start:]:
    name = r[ki].split('(')[0].replace('void ', '')
    v = float(r[vi].replace(',', ''))
    u = r[ui]
    scale = {'nsecond': 1e-3, 'ns': 1e-3, 'usecond': 1.0, 'us': 1.0, 'msecond': 1e3, 'ms': 1e3, 'byte': 1e-6, 'Kbyte': 1e-3, 'Mbyte': 1.0, 'Gbyte': 1e3}.get(u, 1.0)
    agg.setdefault(name, collections.defaultdict(list))[r[mi]].append(v * scale)
for k, d in agg.items():
    t = d.get('gpu__time_duration.sum', [0])
    rd = d.get('dram__bytes_read.sum', [0]); wr = d.get('dram__bytes_write.sum', [0])
    print(f"{k[:48]:48s} n={len(t):3d} mean={sum(t)/len(t):9.1f} us  read={sum(rd)/len(rd):8.1f} MB write={sum(wr)/len(wr):7.1f} MB")
tot = sum(sum(d.get('gpu__time_duration.sum', [0])) for d in agg.values())
print(f"total kernel time {tot / 1e3:.3f} ms over {sum(len(d.get('gpu__time_duration.sum', [])) for d in agg.values())} launches")
