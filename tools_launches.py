"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    i_name, i_val, i_unit = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[1:]:
        v = float(r[i_val].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[r[i_unit]]
        name = r[i_name].split("(")[0].replace("void ", "").replace("skg::", "")
        out.append((name, v))
    return out


if __name__ == "__main__":
    data = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v in data:
        agg[n][0] += 1
        agg[n][1] += v
    tot = sum(v for _, v in data)
    print(f"{len(data)} launches, {tot:.1f} us total")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v:10.1f} us {100 * v / tot:5.1f}%  n={c:4d}  avg={v / c:8.2f}  {k}")
