"""Eager vs fully-lazy bucket maintenance (PAPER.md Fig. alg:lazy_delta_stepping):
device time, rounds, buckets, grid syncs and far-pile entries scanned per (config, Δ), median
of 5 after 2 warm-ups, through the product library. Prints a markdown table (committed as
profiles/r02_lazy_table.md).
usage: python tools/lazy_table.py [configs...]   (default 1 2 3 4)"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import gen  # noqa: E402
from paper_1911_07260_b200 import gi  # noqa: E402

CASES = {1: [100, 1000], 2: [1 << 13, 1 << 16], 3: [1, 2, 4], 4: [2]}
ARMS = [("eager fused", dict()), ("eager unfused", dict(fusion=False)), ("lazy", dict(fusion=False, lazy=True))]
cfgs = [int(x) for x in sys.argv[1:]] or [1, 2, 3, 4]
print("| config | Δ | arm | ms | rounds | buckets | grid syncs | far scanned |")
print("|---|---|---|---|---|---|---|---|")
for cfg in cfgs:
    g = gen.config_graph(cfg)
    G = gi.Graph.from_csr(g)
    src = gen.config_source(cfg, g)
    out = torch.empty(g.n, dtype=torch.int32, device="cuda")
    for delta in CASES[cfg]:
        for name, o in ARMS:
            ts, st = [], None
            for i in range(7):
                st = gi.gi_sssp_delta(G, src, delta, out, gi.make_options(**o))
                if i >= 2:
                    ts.append(st.gpu_ms)
            print(f"| {cfg} | {delta} | {name} | {statistics.median(ts):.2f} | {st.rounds} | {st.buckets} | "
                  f"{st.grid_syncs} | {st.far_scanned} |", flush=True)
    G.close()
    del g
