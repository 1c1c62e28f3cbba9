"""Average gpu__time_duration per (kernel, grid) from an ncu --csv launch list."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, iv = h.index('Kernel Name'), h.index('Metric Value')
ig = h.index('Grid Size') if 'Grid Size' in h else None
d = collections.defaultdict(list)
for r in rows[1:]:
    d[(r[ik][:48], r[ig] if ig is not None else '')].append(float(r[iv].replace(',', '')))
for k, v in sorted(d.items()):
    print(f"{k[0]:48s} {k[1]:>14s} n={len(v):3d} avg={sum(v) / len(v) / 1000:8.2f} us")
