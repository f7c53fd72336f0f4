"""Run a few queries of one config (for ncu / compute-sanitizer captures).
usage: python tools/profile_run.py --config 2 --delta 65536 --reps 2 [--no-fusion]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen
from paper_1911_07260_b200 import gi

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2, help="0 = path graph of 20000 vertices (one chain)")
ap.add_argument("--delta", type=int, default=1 << 16)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--no-fusion", action="store_true")
ap.add_argument("--threshold", type=int, default=0)
ap.add_argument("--max-ctas", type=int, default=0)
ap.add_argument("--pre-read", type=int, default=0)
ap.add_argument("--drain", default="auto")
ap.add_argument("--kcore", action="store_true", help="run k-core instead of SSSP")
a = ap.parse_args()
g = gen.config_graph(a.config) if a.config else gen.path(20000)
G = gi.Graph.from_csr(g)
src = gen.config_source(a.config, g) if a.config else 0
if a.kcore:
    for i in range(a.reps):
        core, st = gi.kcore(G)
        print(i, "kcore", {k: st[k] for k in ("gpu_ms", "buckets", "rounds", "grid_syncs", "fused_subrounds",
                                              "critical_subrounds", "spills")})
    sys.exit(0)
if a.config == 5:  # the 64-source batch
    srcs = gen.config_sources(5, g, 64)
    for i in range(a.reps):
        d, sts = gi.sssp_batch(G, srcs, a.delta)
        print(i, "batch gpu_ms", sts[0]["gpu_ms"] if isinstance(sts, list) else sts)
    sys.exit(0)
for i in range(a.reps):
    d, st = gi.sssp(G, src, a.delta, fusion=not a.no_fusion, threshold=a.threshold, max_ctas=a.max_ctas, pre_read=a.pre_read,
                     drain=a.drain)
    print(i, {k: st[k] for k in ("gpu_ms", "buckets", "rounds", "grid_syncs", "fused_subrounds", "critical_subrounds", "spills", "ctas", "edges_relaxed")})
