"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
SSSP (bsp, unfused, async drains; 512 and 1024 threads), batch, PPSP, A*, k-core, on a
64x64 road-like grid and a small RMAT."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gen
import oracle
from paper_1911_07260_b200 import gi

g = gen.grid(64, 64, 1, 100, 3, p_del=0.05, p_diag=0.05)
r = gen.rmat(12, 8, 1, 12, 4)
for graph, s in ((g, 100), (r, gen.max_degree_vertex(r))):
    G = gi.Graph.from_csr(graph)
    ref, _ = oracle.dijkstra(graph, s)
    for o in (dict(), dict(fusion=False), dict(cta_threads=1024), dict(cta_threads=512, threshold=4),
              dict(hub_min=256)):
        d, _ = gi.sssp(G, s, 50, **o)
        assert np.array_equal(gi.as_uint32(d), ref), o
    if graph is g:
        d, _ = gi.sssp(G, s, 50, drain="async")
        assert np.array_equal(gi.as_uint32(d), ref)
        h = gen.grid_heuristic(64, 64, 7, 1)
        assert gi.astar(G, s, 7, 50, h)[0] == int(ref[7])
    out, _ = gi.sssp_batch(G, np.array([s, 0, 5], np.int32), 50)
    many = np.arange(10, dtype=np.int32)  # >= 8 sources: the throughput configuration (1024 threads, big bins)
    outm, _ = gi.sssp_batch(G, many, 50)
    import torch
    mats = [torch.zeros((3, graph.n), dtype=torch.int32, device="cuda") for _ in range(2)]
    for rr, (lo, hi) in enumerate(((0, 2), (2, 3))):  # the fused gather, two ranks in one process
        gi.gi_sssp_batch_peers(G, np.array([s, 0, 5], np.int32)[lo:hi], 50,
                               [m.data_ptr() + lo * graph.n * 4 for m in mats], rr)
    torch.cuda.synchronize()
    assert all(np.array_equal(gi.as_uint32(m), gi.as_uint32(out)) for m in mats)
    assert gi.ppsp(G, s, 3, 50)[0] == int(ref[3])
    core, _ = gi.kcore(G)
    assert np.array_equal(gi.as_uint32(core), oracle.kcore(graph))
    G.close()
print("sanitize_run OK")
