"""profiles/r01_ncu_member.md from gpurun_out/prof_{qft,var,w2}.ncu-rep (scripts/prof_member.sh)."""
import csv, io, os, subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
KEYS = ["Grid Size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]
out = ["# ncu evidence: the per-member kernels (round 1)", "",
       "Commands (B200, 1 GPU, `scripts/prof_member.sh`; each run plain first, exit 0):",
       "`bench.py --workload qft` (f2), `--workload variational` (f3), `--window 2` (f4);",
       "`ncu --set full --clock-control none --import-source on`, one launch each.", ""]
for tag, what in (("qft", "k_zipup<complex>: one zip-up of the 2^13 Fourier chain (one member)"),
                  ("var", "k_variational: one sweep over 512 cfg5 members"),
                  ("w2", "k_zipup<double>: one window-2 zip-up of 512 cfg5 members")):
    rep = os.path.join(G, f"prof_{tag}.ncu-rep")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, r = rows[0], rows[1], rows[2]
    out += [f"## {what}", "", "| metric | value |", "|---|---|"]
    for k in KEYS:
        if k in h:
            out.append(f"| {k} | {r[h.index(k)]} {u[h.index(k)]} |")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    top = subprocess.run(["python", os.path.join(ROOT, "scripts", "ncu_lines.py"), "6"], input=src,
                         capture_output=True, text=True).stdout
    out += ["", "Top source lines (share of stall samples, dominant reasons):", "", "```", top.rstrip(), "```", ""]
open(os.path.join(ROOT, "profiles", "r01_ncu_member.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
