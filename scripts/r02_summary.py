"""Round-2 evidence summary: copies the evidence of one scripts/r02_final2.sh run (gpurun_out/<dir>)
to profiles/r02/<name>/ and writes ncu_summary.md there (launch list shares of the cfg5 step,
--set full metrics of k_sweep and k_orth, top source lines) plus the cfg5 k_sweep DRAM traffic
per member into profiles/traffic.json (the `traffic` field of bench.py's roofline object).
    python scripts/r02_summary.py gpurun_out/r02final2 final2"""
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src, name = sys.argv[1], sys.argv[2]
dst = os.path.join(ROOT, "profiles", "r02", name)
os.makedirs(dst, exist_ok=True)
for f in sorted(os.listdir(src)):
    if f.endswith((".json", ".log", ".txt", ".csv")) and not f.endswith("_raw.csv") and f != "ncu_full.log":
        shutil.copy(os.path.join(src, f), os.path.join(dst, f))

keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "lts__t_sector_hit_rate.pct",
        "sm__icc_request_hit_rate.pct"]
stall = ["wait", "short_scoreboard", "barrier", "selected", "math_pipe_throttle", "not_selected", "mio_throttle",
         "no_instruction", "long_scoreboard", "branch_resolving", "dispatch_stall"]
rows = list(csv.reader(open(os.path.join(src, "sweep_orth_raw.csv"))))
h, u = rows[0], rows[1]
kern = []
for r in rows[2:]:
    d = {"name": r[h.index("Kernel Name")].split("(")[0], "grid": r[h.index("Grid Size")]}
    for k in keys:
        if k in h:
            d[k] = (r[h.index(k)], u[h.index(k)])
    d["stall"] = {}
    for s in stall:
        k = "smsp__average_warps_issue_stalled_%s_per_issue_active.ratio" % s
        if k in h:
            d["stall"][s] = float(r[h.index(k)])
    kern.append(d)


def gbytes(v):
    val, unit = v
    return float(val) * {"Gbyte": 1.0, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9}.get(unit, 1.0)


bench = json.load(open(os.path.join(src, "bench_cfg5.json")))
members = bench["config"]["members_per_gpu"]
sweep = [k for k in kern if k["name"] == "k_sweep"][0]
traffic = (gbytes(sweep["dram__bytes_read.sum"]) + gbytes(sweep["dram__bytes_write.sum"])) * 1e9
tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
tj["cfg5"] = {"kernel": "k_sweep", "bytes_per_member": round(traffic / members),
              "source": "profiles/r02/%s/ncu_summary.md: ncu --set full, %d members, dram__bytes_read.sum + "
                        "dram__bytes_write.sum" % (name, members)}
json.dump(tj, open(os.path.join(ROOT, "profiles", "traffic.json"), "w"), indent=1)

launch = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "launch_summary.py"),
                         os.path.join(src, "launches_cfg5.csv"), "5"], capture_output=True, text=True).stdout
lines = open(os.path.join(src, "sweep_orth_lines.txt")).read().splitlines()[:30]
out = ["# ncu evidence, round 2 (%s)" % name, "",
       "Commands (B200, one GPU, `scripts/r02_final2.sh`): every bench line first ran plain (exit 0);",
       "launch list `ncu --metrics gpu__time_duration.sum --clock-control none -c 400` of",
       "`python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e` (cfg5, 512 members; 5 runs of the",
       "step: cold-cache, serialised launches -- compare shares); `ncu --set full --clock-control none",
       "--import-source on -k regex:\"k_sweep|k_orth\" -s 6 -c 3` of `bench.py --steps 1 --warmup 3`.", "",
       "## Launch list per cfg5 step", "", launch.strip(), "",
       "(k_dmma / k_dfma are the FP64 peak probes bench.py runs once per process.)", "",
       "## Per-kernel metrics (--set full)", "",
       "| metric | " + " | ".join("%s %s" % (k["name"], k["grid"]) for k in kern) + " |",
       "|---|" + "---|" * len(kern)]
for key in keys:
    if all(key in k for k in kern):
        out.append("| %s | %s |" % (key, " | ".join("%s %s" % k[key] for k in kern)))
out.append("| DRAM bytes per member (read + write) | %s |" % " | ".join(
    "%.2f MB" % ((gbytes(k["dram__bytes_read.sum"]) + gbytes(k["dram__bytes_write.sum"])) * 1e3 / members)
    for k in kern))
out += ["", "Warp stall reasons, cycles per issued instruction:", "",
        "| reason | " + " | ".join(k["name"] for k in kern) + " |", "|---|" + "---|" * len(kern)]
for s in stall:
    out.append("| %s | %s |" % (s, " | ".join("%.3f" % k["stall"].get(s, 0.0) for k in kern)))
out += ["", "## Top source lines (warp-stall samples of the captured launches, `scripts/ncu_lines.py`)", "", "```"]
out += lines
out += ["```", ""]
open(os.path.join(dst, "ncu_summary.md"), "w").write("\n".join(out))
print("wrote", os.path.join(dst, "ncu_summary.md"), "traffic/member", round(traffic / members))
