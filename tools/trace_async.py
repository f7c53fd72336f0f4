"""GI_TRACE build of libgi.so: where the async drain's time goes (per phase and per item).
usage: python tools/trace_async.py cfg1|cfg2|path [delta] [drain: async|bsp] [max_ctas]"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import gen  # noqa: E402

# TRACE_W=1024: the 1024-thread build is the primary one (the trace buffers live there)
W = int(os.environ.get("TRACE_W", "512"))
so = os.environ.get("TRACE_SO", f"/tmp/libgi_trace{W}.so")
CS = os.path.join(ROOT, "paper_1911_07260_b200/csrc")
if not os.path.exists(so) or os.environ.get("REBUILD"):
    nv = ["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-DGI_TRACE", "-Xcompiler",
          "-fPIC", "-I", os.path.join(ROOT, "include")]
    objs = []
    units = [(f"{CS}/gi_kernels.cu", ["-DGI_BLOCK=512", "-DGI_VARIANT=v512", f"-DGI_PRIMARY={int(W == 512)}"], "k512"),
             (f"{CS}/gi_kernels.cu", ["-DGI_BLOCK=1024", "-DGI_VARIANT=v1024", f"-DGI_PRIMARY={int(W == 1024)}"], "k1024")]
    units += [(f"{CS}/{f}", [], f[:-3]) for f in sorted(os.listdir(CS)) if f.endswith(".cu") and f != "gi_kernels.cu"]
    for src, defs, tag in units:
        obj = f"/tmp/trace{W}_{tag}.o"
        subprocess.check_call(nv + defs + ["-c", src, "-o", obj])
        objs.append(obj)
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", so] + objs)
if len(sys.argv) > 1 and sys.argv[1] == "build":  # prebuild here (TRACE_SO in-tree ships to the box)
    sys.exit(0)
lib = ctypes.CDLL(so)
vp, i64, i32, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
lib.gi_debug_trace.argtypes = [vp, ctypes.c_int]
lib.gi_debug_trace2.argtypes = [vp, vp, ctypes.c_int]
lib.gi_graph_create.argtypes = [i64, i64, vp, vp, vp, ctypes.c_int, ctypes.POINTER(vp)]
from paper_1911_07260_b200.gi import gi_options, gi_stats  # noqa: E402  (struct layouts only)
lib.gi_sssp_delta_ex.argtypes = [vp, i32, u32, ctypes.POINTER(gi_options), vp, ctypes.POINTER(gi_stats)]
lib.gi_options_default.argtypes = [ctypes.POINTER(gi_options)]

what = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
delta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
drain = sys.argv[3] if len(sys.argv) > 3 else "async"
max_ctas = int(sys.argv[4]) if len(sys.argv) > 4 else 0
if what == "path":
    g = gen.path(20000); src_v = 0; delta = delta or 10**9
elif what == "path1":  # one bucket per vertex: the per-phase cost
    g = gen.path(5000); src_v = 0; delta = 1
elif what == "cfg4":
    g = gen.config_graph(4); src_v = gen.config_source(4, g); delta = delta or 2
elif what == "cfg3":
    g = gen.config_graph(3); src_v = gen.config_source(3, g); delta = delta or 1
elif what == "cfg1":
    g = gen.config_graph(1); src_v = 0; delta = delta or 1000
else:
    g = gen.config_graph(2); src_v = gen.config_source(2, g); delta = delta or 32768
h = vp()
assert lib.gi_graph_create(g.n, g.m, g.offsets.ctypes.data, g.cols.ctypes.data, g.w.ctypes.data, 0,
                           ctypes.byref(h)) == 0
import torch  # noqa: E402

out = torch.empty(g.n, dtype=torch.int32, device="cuda")
opt = gi_options()
lib.gi_options_default(ctypes.byref(opt))
opt.max_ctas = max_ctas
opt.cta_threads = W  # the trace buffers live in the primary build
opt.drain = {"async": 2, "bsp": 1, "unfused": 1}[drain]
opt.fusion = 0 if drain == "unfused" else 1
st = gi_stats()
buf = np.zeros(64, np.uint64)
ph = np.zeros((7, 16384), np.uint64)
it = np.zeros(16, np.uint64)
for rep in range(2):
    lib.gi_debug_trace(buf.ctypes.data, 1)
    lib.gi_debug_trace2(ph.ctypes.data, it.ctypes.data, 1)
    rc = lib.gi_sssp_delta_ex(h, src_v, delta, ctypes.byref(opt), out.data_ptr(), ctypes.byref(st))
    if rc != 0:
        lib.gi_last_error.restype = ctypes.c_char_p
        print('rc', rc, lib.gi_last_error())
        sys.exit(1)
    lib.gi_debug_trace(buf.ctypes.data, 0)
    lib.gi_debug_trace2(ph.ctypes.data, it.ctypes.data, 0)
print(what, "delta", delta, "drain", drain, "max_ctas", max_ctas, "gpu_ms %.3f" % st.gpu_ms, "subrounds",
      st.fused_subrounds, "critical", st.critical_subrounds, "buckets", st.buckets, "kind", st.kernel_kind)
clk = 1.965e3  # cycles per µs at the max SM clock
names = {0: "bsp drain loop top", 2: "slot load", 3: "relax", 4: "rest", 5: "decision", 6: "feed (async) / extract",
         7: "phase work end", 8: "far flush + fmin", 9: "group barrier", 11: "drain (async, CTA 0)",
         12: "stage B scan", 13: "stage B edge loop", 14: "ROUND claim+staging", 15: "hub slices (after B)",
         16: "B iter: search + edge-load issue", 17: "B iter: relax_batch (waits)", 18: "expand relax tail", 19: "expand: collection barrier", 20: "expand: scan + barrier + S", 21: "expand it: pre-read issue + next map/load", 22: "expand it: consume (waits pre-reads) + pushes", 23: "expand it: far flush", 24: "E1 collect (reserve + copy)", 25: "ROUND next claim", 26: "EXTRACT chunk loads + classify", 27: "EXTRACT keep append", 28: "EXTRACT bins + frontier append",
         29: "relax: slot wait (in relax)", 30: "relax: atomic wait"}
tot = 0
for k in range(32):
    c = int(buf[32 + k])
    if c:
        tot += int(buf[k])
        print(f"CTA0 {k:2d} {names.get(k, '?'):28s} calls={c:8d} cyc/call={int(buf[k]) / c:9.1f} "
              f"total={int(buf[k]) / clk / 1e3:8.3f} ms")
print(f"CTA0 traced total {tot / clk / 1e3:.3f} ms")
dr, dep = ph[0].astype(np.float64), ph[1].astype(np.float64)
m = dr > 0
if m.any():
    print(f"phases traced {int(m.sum())}; sum over phases of max-CTA feed+drain = {dr[m].sum() / clk / 1e3:.3f} ms; "
          f"sum max depth = {int(dep[m].sum())}; cycles per depth level = {dr[m].sum() / max(dep[m].sum(), 1):.0f}")
    q = np.percentile(dr[m] / np.maximum(dep[m], 1), [10, 50, 90])
    print("per-phase cycles/level p10/p50/p90:", q.round(0))
if it[8]:
    nb = it[8]
    print(f"items: warp-iterations={int(nb)} entries={int(it[9])} (avg {it[9] / nb:.2f}/iter, "
          f"continuation {it[10] / max(it[9], 1):.1%}); idle polls={int(it[7])}")
mx, sm = ph[2].astype(np.float64), ph[3].astype(np.float64)
m2 = mx > 0
if m2.any():
    G = st.ctas
    print(f"phases {int(m2.sum())}: sum of max-CTA busy {mx[m2].sum() / clk / 1e3:.3f} ms, sum of mean-CTA busy "
          f"{sm[m2].sum() / G / clk / 1e3:.3f} ms (imbalance {mx[m2].sum() / max(sm[m2].sum() / G, 1):.2f}x); "
          f"gpu_ms {st.gpu_ms:.3f}")
    for md, name in ((0, "ROUND"), (1, "EXTRACT")):
        sel = m2 & (ph[4] == md)
        print(f"  {name} phases {int(sel.sum())}: sum of max-CTA busy {mx[sel].sum() / clk / 1e3:.3f} ms")
    top = np.argsort(-mx)[:10]
    print("  heaviest phases: (phase, us max, us mean, mode 0=ROUND/1=EXTRACT, cnt, hubs)")
    for i in top:
        print("   ", int(i), round(mx[i] / clk, 1), round(sm[i] / G / clk, 1), int(ph[4][i]), int(ph[5][i]), int(ph[6][i]))
