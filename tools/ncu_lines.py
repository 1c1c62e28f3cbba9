"""Stall samples per CUDA source line from `ncu -i R --page source --csv --print-source sass,cuda`
(source-line rows carry the aggregated samples of their SASS).  usage: ncu_lines.py CSV [TOP]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], encoding="utf-8", errors="replace")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
data, fname, isamp = [], "", 4
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    elif r and r[0] == "Line No":
        isamp = r.index("Warp Stall Sampling (All Samples)")
    elif r and r[0].isdigit() and len(r) > isamp:
        try:
            data.append((int(r[isamp] or 0), fname, int(r[0]), r[1].strip()[:100]))
        except ValueError:
            pass
tot = sum(d[0] for d in data) or 1
print("total samples", tot)
for n, f, ln, s in sorted(data, reverse=True)[:top]:
    print(f"{n:7d} {100 * n / tot:5.1f}%  {f}:{ln:<5d} {s}")
