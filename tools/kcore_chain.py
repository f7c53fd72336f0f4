"""Per-level latency of the k-core drain: k-core of a path (every coreness 1; the peel
cascades from both ends, one vertex per level), time / critical sub-rounds; SSSP on the
same path for comparison. usage: python tools/kcore_chain.py [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen
from paper_1911_07260_b200 import gi

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
G = gi.Graph.from_csr(gen.path(n))  # symmetric path
for i in range(3):
    core, st = gi.kcore(G)
print("kcore path", n, "ms", round(st["gpu_ms"], 3), "critical", st["critical_subrounds"], "us/level",
      round(st["gpu_ms"] * 1e3 / max(st["critical_subrounds"], 1), 2), "rounds", st["rounds"], "buckets", st["buckets"])
for i in range(3):
    d, st = gi.sssp(G, 0, 10**9)
print("sssp path", n, "ms", round(st["gpu_ms"], 3), "critical", st["critical_subrounds"], "us/level",
      round(st["gpu_ms"] * 1e3 / max(st["critical_subrounds"], 1), 2))
