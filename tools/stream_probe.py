"""Does the query's stream matter? Same graph, same process: cuda_stream = torch's current
stream vs the library's own workspace stream (NULL), alternating.
usage: GI_GEN_CACHE=/tmp/gcache python tools/stream_probe.py CONFIG DELTA"""
import ctypes, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
from paper_1911_07260_b200 import gi

cfg, delta = int(sys.argv[1]), int(sys.argv[2])
g = gen.config_graph(cfg)
G = gi.Graph.from_csr(g)
src = gen.config_source(cfg, g)
out = torch.empty(g.n, dtype=torch.int32, device="cuda")
lib = gi.lib()
side = torch.cuda.Stream()
res = {}
for rep in range(4):
    for name, stream in (("torch-current", torch.cuda.current_stream().cuda_stream), ("library", 0),
                         ("torch-side", side.cuda_stream)):
        o = gi.make_options()
        o.cuda_stream = stream
        st = gi.gi_stats()
        ts = []
        for i in range(5):
            rc = lib.gi_sssp_delta_ex(G.handle, src, delta, ctypes.byref(o), out.data_ptr(), ctypes.byref(st))
            assert rc == 0
            ts.append(st.gpu_ms)
        res.setdefault(name, []).append(statistics.median(ts[1:]))
for k, v in res.items():
    print(k, [round(x, 3) for x in v], flush=True)
