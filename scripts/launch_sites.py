"""Per-launch durations (ncu gpu__time_duration.sum CSV) of the large path's per-site kernels,
last run of the capture: python scripts/launch_sites.py launches.csv [min_us]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
lo = float(sys.argv[2]) if len(sys.argv) > 2 else 200.0
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]
ki, vi, ii = h.index('Kernel Name'), h.index('Metric Value'), h.index('ID')
out = []
for r in rows[hdr + 1:]:
    if len(r) > vi:
        out.append((int(r[ii]), r[ki].split('(')[0].replace('qtt::', ''), float(r[vi].replace(',', '')) / 1e3))
plans = [i for i, x in enumerate(out) if x[1] == 'k_site0_init']
run = out[plans[-1]:] if plans else out
site = -1
for _, name, us in run:
    if name == 'k_plan':
        site += 1
    if us >= lo:
        print(f"site {site:2d} {name:28s} {us:10.1f} us")
