"""Config-5 batch: is a 2-CTA group's query bound by its chain (the source's eccentricity)
or by its work (the whole grid, the same for every source)? Times the 64-source batch as
seeded, and 64 copies of its nearest-to-centre and of its farthest-from-centre source.
usage: python tools/batch_ecc.py   (prints one JSON line per arm; device ms, median of 3)"""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import gen  # noqa: E402
import torch  # noqa: E402
from paper_1911_07260_b200 import gi  # noqa: E402

g = gen.config_graph(2)
G = gi.Graph.from_csr(g)
srcs = gen.config_sources(5, g)
side = 4096
r, c = srcs // side, srcs % side
ecc = np.maximum(r, side - 1 - r) + np.maximum(c, side - 1 - c)  # lattice hops to the farthest corner
lo, hi = int(srcs[np.argmin(ecc)]), int(srcs[np.argmax(ecc)])
out = torch.empty((len(srcs), g.n), dtype=torch.int32, device="cuda")
for name, s in (("seeded", srcs), ("min_ecc_x64", np.full(64, lo, np.int32)),
                ("max_ecc_x64", np.full(64, hi, np.int32)), ("seeded_again", srcs)):
    ts = []
    for i in range(4):
        st = gi.gi_sssp_batch(G, s, 8192, out, None)
        if i:
            ts.append(st[0].gpu_ms)
    b = [int(st[i].buckets) for i in range(len(s))]
    print(json.dumps({"arm": name, "ms_median": statistics.median(ts), "buckets_min": min(b),
                      "buckets_max": max(b), "buckets_mean": sum(b) / len(b),
                      "ecc_hops": [int(ecc.min()), int(ecc.max())]}), flush=True)
