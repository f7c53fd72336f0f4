"""Would a DensePull round do less work than push on the
RMAT configs? Per bucket b of Δ-stepping, push reads the out-edges of the bucket's vertices;
pull reads the in-edges of every vertex not yet settled (bucket >= b) and, for SSSP, cannot
stop early (it needs the minimum over all frontier in-neighbours). Buckets are taken from the
final distances (scipy's Dijkstra, not the oracle: tools/ must not use oracle/), which is a
lower bound on push work (re-relaxations are ignored).
usage: python tools/pull_estimate.py [CONFIG] [DELTA ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import dijkstra
import gen

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
deltas = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
g = gen.config_graph(cfg)
src = gen.config_source(cfg, g)
A = sp.csr_matrix((g.w.astype(np.float64), g.cols, g.offsets), shape=(g.n, g.n))
d = dijkstra(A, indices=src)
deg = np.diff(g.offsets)
reach = np.isfinite(d)
d = np.where(reach, d, 0).astype(np.int64)
print(f"config {cfg}: n {g.n} m {g.m} reached {int(reach.sum())}")
for delta in deltas:
    b = d[reach] // delta
    push = np.bincount(b, weights=deg[reach])
    pull = np.cumsum(push[::-1])[::-1]
    r = pull / np.maximum(push, 1)
    heavy = int(np.argmax(push))
    print(f"delta {delta}: {len(push)} buckets; heaviest bucket {heavy}: push {push[heavy] / 1e6:.1f}M edges, "
          f"pull {pull[heavy] / 1e6:.1f}M; min pull/push over buckets {r.min():.2f}; "
          f"total push {push.sum() / 1e6:.1f}M, total pull if pulled where cheaper {np.minimum(push, pull).sum() / 1e6:.1f}M")
