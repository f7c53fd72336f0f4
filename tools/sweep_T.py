"""Fusion threshold sweep (the "measured threshold" of north_star; R2): device
time of one query per (config, Δ, T), median of 5 after 2 warm-ups, through the product
library. Prints a markdown table (committed as profiles/r02_T_sweep.md).
usage: python tools/sweep_T.py [configs...]   (default 1 2 3)"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import gen  # noqa: E402
from paper_1911_07260_b200 import gi  # noqa: E402

CASES = {1: [1000], 2: [1 << 14, 1 << 16], 3: [2]}
TS = [1, 16, 64, 256, 1024, 2048, 4096]
cfgs = [int(x) for x in sys.argv[1:]] or [1, 2, 3]
print("| config | Δ | " + " | ".join(f"T={t}" for t in TS) + " | unfused |")
print("|---|---|" + "---|" * (len(TS) + 1))
for cfg in cfgs:
    g = gen.config_graph(cfg)
    G = gi.Graph.from_csr(g)
    src = gen.config_source(cfg, g)
    out = torch.empty(g.n, dtype=torch.int32, device="cuda")
    for delta in CASES[cfg]:
        row = []
        for t in TS + [None]:
            o = dict(fusion=False) if t is None else dict(threshold=t)
            ts, st = [], None
            for i in range(7):
                st = gi.gi_sssp_delta(G, src, delta, out, gi.make_options(**o))
                if i >= 2:
                    ts.append(st.gpu_ms)
            row.append(f"{statistics.median(ts):.2f} ms ({st.spills} sp, {st.rounds} r)")
        print(f"| {cfg} | {delta} | " + " | ".join(row) + " |", flush=True)
    G.close()
