"""Placement effect on config 4, part 4: two graphs alive at once, and a dummy block before
the graph. usage: python tools/placement_probe4.py two|dummy"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import gen
from paper_1911_07260_b200 import gi

g = gen.config_graph(4)
src = gen.config_source(4, g)
out = torch.empty(g.n, dtype=torch.int32, device="cuda")


def timed(G, reps=4):
    ts = []
    for _ in range(reps):
        _, st = gi.sssp(G, src, 2, out=out)
        ts.append(st["gpu_ms"])
    return round(float(np.median(ts[1:])), 2)


mode = sys.argv[1]
if mode == "two":
    G1 = gi.Graph.from_csr(g)
    print("G1", timed(G1), flush=True)
    G2 = gi.Graph.from_csr(g)
    print("G2 (G1 alive)", timed(G2), flush=True)
    print("G1 again", timed(G1), flush=True)
elif mode == "dummy":
    d = torch.empty(24 << 30, dtype=torch.uint8, device="cuda")
    G = gi.Graph.from_csr(g)
    del d
    torch.cuda.empty_cache()
    print("after 24 GB dummy", timed(G), flush=True)
elif mode == "dummy_alive":   # a 24 GB block alive while the graph AND its workspace are made
    d = torch.empty(24 << 30, dtype=torch.uint8, device="cuda")
    G = gi.Graph.from_csr(g)
    print("dummy alive, first", timed(G), flush=True)
    del d
    torch.cuda.empty_cache()
    print("dummy freed", timed(G), flush=True)
elif mode == "two_free":      # second graph after the first is freed
    G1 = gi.Graph.from_csr(g)
    print("G1", timed(G1), flush=True)
    G1.close()
    G2 = gi.Graph.from_csr(g)
    print("G2 (G1 freed)", timed(G2), flush=True)
elif mode == "dummy_touched":  # the 24 GB block written (physically backed) before the graph
    d = torch.zeros(24 << 30, dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    G = gi.Graph.from_csr(g)
    print("dummy touched, alive", timed(G), flush=True)
    del d
    torch.cuda.empty_cache()
    print("dummy touched, freed", timed(G), flush=True)
elif mode == "small_dummy":    # how much has to be in front? 4 / 8 / 12 GB touched
    for gb in (4, 8, 12):
        d = torch.zeros(gb << 30, dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()
        G = gi.Graph.from_csr(g)
        print(f"{gb} GB touched in front", timed(G), flush=True)
        G.close()
        del d
        torch.cuda.empty_cache()
