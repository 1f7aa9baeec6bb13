#!/usr/bin/env python
"""Per-kernel table (time-weighted) from an ncu --metrics CSV over many launches:
ncu_kernel_table.py launches.csv > table.md"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
data = collections.defaultdict(lambda: collections.defaultdict(float))
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    key = (r[h.index("ID")], r[h.index("Kernel Name")].split("(")[0].replace("void ", "").replace("qtt::", ""))
    data[key][r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", "") or 0)
    data[key]["unit:" + r[h.index("Metric Name")]] = r[h.index("Metric Unit")]
agg = collections.defaultdict(lambda: collections.defaultdict(float))
for (lid, name), m in data.items():
    t = m.get("gpu__time_duration.sum", 0.0)
    tu = m.get("unit:gpu__time_duration.sum", "ns")
    t_ms = t * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(tu, 1e-6)
    a = agg[name]
    a["n"] += 1
    a["ms"] += t_ms
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        u = m.get("unit:" + k, "byte")
        a[k] += m.get(k, 0.0) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    for k in ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"):
        a[k] += m.get(k, 0.0) * t_ms
tot = sum(a["ms"] for a in agg.values())
print("| kernel | launches | ms | share | DMMA % (time-weighted) | FP64 pipe % | DRAM GB | DRAM GB/s |")
print("|---|---|---|---|---|---|---|---|")
for name, a in sorted(agg.items(), key=lambda x: -x[1]["ms"]):
    gb = (a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) / 1e9
    ms = a["ms"]
    print(f"| {name} | {int(a['n'])} | {ms:.2f} | {ms / tot:.3f} | "
          f"{a['sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active'] / max(ms, 1e-12):.1f} | "
          f"{a['sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'] / max(ms, 1e-12):.1f} | "
          f"{gb:.2f} | {gb / max(ms, 1e-12) * 1e3:.0f} |")
print(f"| total | | {tot:.2f} | 1 | | | | |")
