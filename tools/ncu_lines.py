"""Aggregate ncu warp-stall samples by CUDA source line (needs -lineinfo).
usage: python tools/ncu_lines.py REPORT.ncu-rep [top]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = defaultdict(lambda: defaultdict(int))
text = {}
cur_file = None
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    line = r[0]
    key = (cur_file, int(line)) if line.isdigit() else (cur_file, -1)
    text[key] = r[1].strip()
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    v = r[iss]
    if v.isdigit():
        agg[key]["all"] += int(v)
        for i, c in enumerate(hdr):
            if c.startswith("stall_") and r[i].isdigit():
                agg[key][c] += int(r[i])
tot = sum(a["all"] for a in agg.values())
print(f"# stall samples {tot}")
for key, a in sorted(agg.items(), key=lambda t: -t[1]["all"])[:top]:
    reasons = sorted(((k, v) for k, v in a.items() if k != "all"), key=lambda t: -t[1])[:2]
    rs = " ".join(f"{k[6:]}:{100 * v / max(a['all'], 1):.0f}%" for k, v in reasons)
    print(f"{key[0]}:{key[1]:<5d} {a['all']:8d} {100 * a['all'] / tot:5.1f}%  {rs:32s} {text.get(key, '')[:80]}")
