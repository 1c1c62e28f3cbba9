"""Per-kernel totals from an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, iv = h.index('Kernel Name'), h.index('Metric Value')
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rows[1:]:
    name = r[ik].split('(')[0].replace('void ', '').replace('skg::', '')
    if '<' in r[ik].split('(')[0]:
        name = r[ik].split('(')[0].replace('void ', '').replace('skg::', '')
    tot[name] += float(r[iv].replace(',', '')) / 1000.0
    cnt[name] += 1
all_us = sum(tot.values())
print(f"{sum(cnt.values())} launches, {all_us:.1f} us total")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v:10.1f} us {100 * v / all_us:5.1f}%  n={cnt[k]:4d}  avg={v / cnt[k]:9.2f}  {k[:150]}")
