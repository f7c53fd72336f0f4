"""Per-sub-round cost vs frontier width: R x C unit-weight grid, source at the corner,
one bucket (Δ huge), fused. Critical sub-rounds ≈ R + C - 1; time / critical = cost of
one sub-round carrying ~R entries."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen
from paper_1911_07260_b200 import gi

for R, C, ctas in [(1, 40000, 1), (8, 20000, 1), (40, 20000, 1), (128, 8000, 1), (512, 4000, 1),
                   (40, 20000, 148), (512, 4000, 148)]:
    g = gen.grid(R, C, 1, 2, 0)
    G = gi.Graph.from_csr(g)
    best = None
    for _ in range(3):
        d, st = gi.sssp(G, 0, 1 << 30, max_ctas=ctas)
        best = st if best is None or st["gpu_ms"] < best["gpu_ms"] else best
    print(json.dumps(dict(R=R, C=C, ctas=ctas, gpu_ms=round(best["gpu_ms"], 3), crit=best["critical_subrounds"],
                          us_per_crit=round(best["gpu_ms"] * 1e3 / max(best["critical_subrounds"], 1), 3),
                          entries_per_sub=round(best["vertices_processed"] / max(best["fused_subrounds"], 1), 1))))
