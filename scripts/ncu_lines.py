"""Aggregate ncu warp-stall samples per CUDA source line from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass` output (stdin)."""
import csv, sys, collections
rows = list(csv.reader(sys.stdin))
cur = None; hdr = None; tot = 0.0
per = collections.Counter(); stall = collections.defaultdict(collections.Counter); text = {}
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; si = hdr.index("Warp Stall Sampling (All Samples)"); sc = [i for i, n in enumerate(hdr) if n.startswith("stall_") and "Not Issued" not in n]; continue
    if hdr is None or r[0] == "" or len(r) <= si: continue
    if r[2] not in ("", "-"): continue    # sass row
    try: s = float(r[si] or 0)
    except ValueError: continue
    key = (cur, int(r[0])); per[key] += s; tot += s; text[key] = r[1].strip()[:70]
    for c in sc:
        try: stall[key][hdr[c][6:]] += float(r[c] or 0)
        except ValueError: pass
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for k, v in per.most_common(n):
    top = ",".join(f"{a}:{b/v*100:.0f}%" for a, b in stall[k].most_common(2)) if v else ""
    print(f"{v/tot*100:5.1f}% {k[0]}:{k[1]:<5d} {text[k]:70s} {top}")
