"""Aggregate ncu 'Instructions Executed' (warp-level) by CUDA source line (needs -lineinfo):
where the issue slots go. usage: python tools/ncu_inst_lines.py REPORT.ncu-rep [top]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, text = defaultdict(int), {}
cur_file, hdr = None, None
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
    key = (cur_file, int(r[0])) if r[0].isdigit() else (cur_file, -1)
    text[key] = r[1].strip()
    v = r[hdr.index("Instructions Executed")]
    if v.isdigit():
        agg[key] += int(v)
tot = sum(agg.values())
print(f"# warp instructions executed {tot}")
for key, v in sorted(agg.items(), key=lambda t: -t[1])[:top]:
    print(f"{key[0]}:{key[1]:<5} {v:12d} {100 * v / max(tot, 1):5.1f}%  {text.get(key, '')[:80]}")
