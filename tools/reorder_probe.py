"""Would a degree-descending vertex relabelling help the RMAT configs? Relabels an RMAT graph
on the host (numpy), runs SSSP on the original or on the relabelled CSR from the same
(mapped) source, and prints the times; with both arms in one process it also checks that the
distances agree after un-permuting.
usage: python tools/reorder_probe.py SCALE [DELTA] [orig|sorted|both]
SCALE 22 / 26 use configs 3 / 4 exactly (one arm per process avoids the config-4 placement
effect)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gen
from paper_1911_07260_b200 import gi

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
delta = int(sys.argv[2]) if len(sys.argv) > 2 else 2
arms = sys.argv[3] if len(sys.argv) > 3 else "both"
g = {22: lambda: gen.config_graph(3), 26: lambda: gen.config_graph(4)}.get(
    scale, lambda: gen.rmat(scale, 16, 1, scale, 3 + scale))()
src = gen.max_degree_vertex(g)
todo = {}
if arms in ("orig", "both"):
    todo["orig"] = (g.offsets, g.cols, g.w, src)
if arms in ("sorted", "both"):
    t0 = time.time()
    deg = np.diff(g.offsets)
    new2old = np.argsort(-deg, kind="stable").astype(np.int64)
    old2new = np.empty_like(new2old)
    old2new[new2old] = np.arange(g.n)
    noff = np.zeros(g.n + 1, np.int64)
    np.cumsum(deg[new2old], out=noff[1:])
    starts = g.offsets[new2old]
    idx = np.repeat(starts - noff[:-1], deg[new2old])
    idx += np.arange(g.m)
    ncols = old2new[g.cols[idx]].astype(np.int32)
    nw = g.w[idx]
    del idx
    print("relabel s", round(time.time() - t0, 1), flush=True)
    todo["degree-sorted"] = (noff, ncols, nw, int(old2new[src]))
res = {}
for name, (off, cols, w, s) in todo.items():
    G = gi.Graph(off, cols, w)
    ts = []
    for i in range(6):
        d, st = gi.sssp(G, s, delta)
        ts.append(st["gpu_ms"])
    if arms == "both":
        res[name] = gi.as_uint32(d).copy()
    print(name, "ms", [round(t, 2) for t in ts], "median", round(float(np.median(ts[1:])), 3),
          "edges", st["edges_relaxed"], "launches", st.get("kernel_launches"), flush=True)
    G.close()
if arms == "both":
    assert np.array_equal(res["orig"], res["degree-sorted"][old2new]), "relabelled distances differ"
    print("distances identical after un-permuting")
