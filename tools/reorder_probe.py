"""Would a degree-descending vertex relabelling help the RMAT configs? Relabels an RMAT graph
on the host (numpy), runs SSSP on the original and on the relabelled CSR from the same
(mapped) source, checks the distances agree after un-permuting, and prints both times.
usage: python tools/reorder_probe.py SCALE [DELTA]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gen
from paper_1911_07260_b200 import gi

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
delta = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g = gen.config_graph(3) if scale == 22 else gen.rmat(scale, 16, 1, scale, 3 + scale)
src = gen.max_degree_vertex(g)
deg = np.diff(g.offsets)
new2old = np.argsort(-deg, kind="stable").astype(np.int64)
old2new = np.empty_like(new2old)
old2new[new2old] = np.arange(g.n)
noff = np.zeros(g.n + 1, np.int64)
np.cumsum(deg[new2old], out=noff[1:])
# gather edges of each new vertex (vectorised: edge index map)
starts = g.offsets[new2old]
idx = np.repeat(starts - noff[:-1], deg[new2old]) + np.arange(g.m)
ncols = old2new[g.cols[idx]].astype(np.int32)
nw = g.w[idx]
del idx
res = {}
for name, (off, cols, w, s) in {"orig": (g.offsets, g.cols, g.w, src),
                                "degree-sorted": (noff, ncols, nw, int(old2new[src]))}.items():
    G = gi.Graph(off, cols, w)
    ts = []
    for i in range(5):
        d, st = gi.sssp(G, s, delta)
        ts.append(st["gpu_ms"])
    res[name] = gi.as_uint32(d)
    print(name, "ms", round(float(np.median(ts[1:])), 3), "edges", st["edges_relaxed"], flush=True)
    G.close()
assert np.array_equal(res["orig"], res["degree-sorted"][old2new]), "relabelled distances differ"
print("distances identical after un-permuting")
