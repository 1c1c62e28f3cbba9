"""Average DRAM bytes (read + write) and duration per launch for each kernel of one or more
ncu --set full reports -> JSON ({kernel: {"dram_bytes": B, "us": T, "launches": n}}).
bench.py reads profiles/ncu_traffic.json for the roofline's "traffic" field."""
import collections
import csv
import json
import subprocess
import sys

acc = collections.defaultdict(lambda: [0.0, 0.0, 0])
for rep in sys.argv[2:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    col = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    for r in rows[2:]:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("skg::", "").split("<")[0]
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(r[col[k]].replace(",", "")) * scale[units[col[k]]]
        t = float(r[col["gpu__time_duration.sum"]].replace(",", "")) * tscale[units[col["gpu__time_duration.sum"]]]
        a = acc[name]
        a[0] += b
        a[1] += t
        a[2] += 1
out = {k: {"dram_bytes": round(v[0] / v[2]), "us": round(v[1] / v[2], 2), "launches": v[2]} for k, v in sorted(acc.items())}
json.dump(out, open(sys.argv[1], "w"), indent=1, sort_keys=True)
print(json.dumps(out, indent=1))
