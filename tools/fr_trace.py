"""Summarise the range-expand CTA timeline written by bench.py under SKG_FR_TRACE=path:
per phase the mean / max duration over the traced CTAs, and the rounds the CTAs ran in."""
import json
import sys

import numpy as np

a = np.array(json.load(open(sys.argv[1])), dtype=np.float64).reshape(8, 32, 11)
ok = a[:, :, 0] > 0
t = a[ok]
t0 = t[:, 0].min()
names = ["zero", "phase1 (thread 0)", "phase1 barrier", "counts", "look-back", "phase3 (thread 0)", "reductions"]
print(f"{ok.sum()} CTAs traced; span {(t[:, 7].max() - t0) / 1e3:.1f} us")
for i, nm in enumerate(names):
    d = (t[:, i + 1] - t[:, i]) / 1e3
    print(f"  {nm:20s} mean {d.mean():7.2f} us  max {d.max():7.2f}  min {d.min():7.2f}")
tot = (t[:, 7] - t[:, 0]) / 1e3
for nm, a0, a1 in (("count loop (thread 0)", 3, 9), ("count barrier", 9, 4), ("look-back spin", 4, 10), ("fence + barrier", 10, 5)):
    d = (t[:, a1] - t[:, a0]) / 1e3
    print(f"  {nm:20s} mean {d.mean():7.2f} us  max {d.max():7.2f}  min {d.min():7.2f}")
print(f"  {'CTA total':20s} mean {tot.mean():7.2f} us  max {tot.max():7.2f}  min {tot.min():7.2f}")
starts = np.sort((t[:, 0] - t0) / 1e3)
print("  start offsets (us):", np.round(starts[:: max(1, len(starts) // 16)], 1))
