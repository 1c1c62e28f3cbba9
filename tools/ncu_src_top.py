"""Top stall SASS lines per kernel from `ncu -i X --page source --csv --print-source sass`."""
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
want = int(sys.argv[2]) if len(sys.argv) > 2 else 0
topn = int(sys.argv[3]) if len(sys.argv) > 3 else 30
secs = [i for i, l in enumerate(lines) if l.startswith('"Kernel Name"')]
secs.append(len(lines))
s, e = secs[want], secs[want + 1]
print(lines[s][:160])
rows = list(csv.reader(lines[s + 1:e]))
hdr = rows[0]
isamp = hdr.index('Warp Stall Sampling (All Samples)')
isrc = hdr.index('Source')
stall_cols = [i for i, h in enumerate(hdr) if h.startswith('stall_') and 'Not Issued' not in h]
data = []
for k, r in enumerate(rows[1:]):
    try:
        n = int(r[isamp])
    except (ValueError, IndexError):
        continue
    top = sorted(((int(r[i]) if r[i].isdigit() else 0, hdr[i]) for i in stall_cols), reverse=True)[:2]
    data.append((n, k, r[isrc].strip()[:60], top))
tot = sum(d[0] for d in data)
print("total samples", tot)
for n, k, src, top in sorted(data, reverse=True)[:topn]:
    print(f"{n:6d} {100*n/tot:5.1f}% #{k:5d} {src:60s} {top}")
