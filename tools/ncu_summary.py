"""Summarise an ncu --set full report (raw metrics + top SASS stall lines) into text.
usage: python tools/ncu_summary.py REPORT.ncu-rep [label] > profiles/...txt"""
import csv, io, subprocess, sys

rep = sys.argv[1]
label = sys.argv[2] if len(sys.argv) > 2 else rep
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
print(f"# ncu --set full summary: {label}")
print(f"# source report: {rep}")
vals = {}
for i, k in enumerate(h):
    if k in want:
        vals[k] = (v[i], u[i])
        print(f"{k:70s} {v[i]:>20s} {u[i]}")


def to_bytes(val, unit):
    f = float(val.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


rd = to_bytes(*vals["dram__bytes_read.sum"])
wr = to_bytes(*vals["dram__bytes_write.sum"])
print(f"{'dram bytes read+write (traffic per launch)':70s} {rd + wr:20.0f} byte")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
hh = srows[1]
data = srows[2:]
iss = hh.index("Warp Stall Sampling (All Samples)")
isrc = hh.index("Source")
cols = [c for c in hh if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(r[iss]) for r in data if r[iss].isdigit())
agg = {c: 0 for c in cols}
for r in data:
    for c in cols:
        x = r[hh.index(c)]
        if x.isdigit():
            agg[c] += int(x)
print(f"\n# warp-stall samples: {tot}; by reason (share)")
for c, x in sorted(agg.items(), key=lambda t: -t[1])[:10]:
    print(f"  {c:28s} {x:10d}  {100.0 * x / max(tot, 1):5.1f}%")
print("\n# top 15 SASS lines by stall samples")
for r in sorted(data, key=lambda r: -int(r[iss]) if r[iss].isdigit() else 0)[:15]:
    top = max(cols, key=lambda c: int(r[hh.index(c)]) if r[hh.index(c)].isdigit() else 0)
    print(f"  {r[iss]:>8s}  {r[isrc].strip()[:60]:60s} {top}")
print(f"\nTRAFFIC_BYTES {rd + wr:.0f}")
