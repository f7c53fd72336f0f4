"""Does buffer placement change config-4 kernel time? Creates the graph after a padding
allocation of PAD MB (torch), times the fused query, destroys it; repeats for several pads.
usage: python tools/placement_probe.py [pads...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import gen
from paper_1911_07260_b200 import gi

g = gen.config_graph(4)
src = gen.config_source(4, g)
out = torch.empty(g.n, dtype=torch.int32, device="cuda")
pads = [int(x) for x in sys.argv[1:]] or [0, 0, 256, 512, 1024, 2048, 4096]
for pad in pads:
    p = torch.empty(max(pad, 1) << 20, dtype=torch.uint8, device="cuda") if pad else None
    G = gi.Graph.from_csr(g)
    ts = []
    for i in range(5):
        d, st = gi.sssp(G, src, 2, out=out)
        ts.append(st["gpu_ms"])
    print(f"pad {pad:5d} MB: {np.median(ts[1:]):.2f} ms  (all {[round(t, 1) for t in ts]})", flush=True)
    G.close()
    del p
    torch.cuda.empty_cache()
