"""Latency micro-benchmarks on the path graph (unit weights), through the C ABI.
* Δ >= n, fusion on:  one bucket, the CTA drains a chain of n vertices -> per-sub-round latency
* Δ = 1:              n buckets of one vertex -> one group barrier + one level per vertex
"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen
from paper_1911_07260_b200 import gi

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
g = gen.path(n)
G = gi.Graph.from_csr(g)
res = {}
for name, delta, opts in [("chain_fused_148", n + 1, dict(fusion=True)),
                          ("chain_fused_1cta", n + 1, dict(fusion=True, max_ctas=1)),
                          ("chain_unfused_148", n + 1, dict(fusion=False)),
                          ("delta1_fused_148", 1, dict(fusion=True)),
                          ("delta1_fused_16", 1, dict(fusion=True, max_ctas=16)),
                          ("delta1_fused_1", 1, dict(fusion=True, max_ctas=1))]:
    best = None
    for _ in range(3):
        d, st = gi.sssp(G, 0, delta, **opts)
        best = st if best is None or st["gpu_ms"] < best["gpu_ms"] else best
    res[name] = dict(gpu_ms=best["gpu_ms"], us_per_vertex=best["gpu_ms"] * 1e3 / n, rounds=best["rounds"],
                     grid_syncs=best["grid_syncs"], subrounds=best["fused_subrounds"], ctas=best["ctas"])
    print(name, json.dumps(res[name]))
