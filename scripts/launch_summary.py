#!/usr/bin/env python
"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name:
  python scripts/launch_summary.py gpurun_out/.../launches.csv [n_runs]
n_runs: divide totals by this many repetitions of the workload (e.g. warmup + steps)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
nrun = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")[:40]
    unit = r[h.index("Metric Unit")]
    v = float(r[h.index("Metric Value")].replace(",", ""))
    v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}.get(unit, 1.0)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(a[1] for a in agg.values())
print(f"| kernel | launches/run | ms/run | share |\n|---|---|---|---|")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| {k} | {a[0] / nrun:.0f} | {a[1] / nrun:.3f} | {a[1] / tot:.3f} |")
print(f"| total | | {tot / nrun:.3f} | 1 |")
