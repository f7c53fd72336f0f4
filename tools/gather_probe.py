"""Config-4 gather ceiling (tools/gather_probe.cu): G edges/s of cols -> dist[col] reads.
usage: GI_GEN_CACHE=/tmp/gcache python tools/gather_probe.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import gen

so = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ab", "libprobe.so")
lib = ctypes.CDLL(so)
lib.probe_gather.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                             ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
g = gen.config_graph(int(os.environ.get("CFG", "4")))
pad_mb = int(os.environ.get("PAD_MB", "-1"))  # >= 0: dist allocated first, after a pad of that size
if pad_mb >= 0:
    pad = torch.empty(max(pad_mb, 0) << 20, dtype=torch.uint8, device="cuda") if pad_mb else None
    dist = torch.zeros(g.n, dtype=torch.int32, device="cuda")
cols = torch.from_numpy(np.array(g.cols)).cuda()
m = g.m
if pad_mb < 0:
    dist = torch.zeros(g.n, dtype=torch.int32, device="cuda")
print("PAD_MB", pad_mb, "dist at", hex(dist.data_ptr()))
sink = torch.zeros(4, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
CASES = [(0, "u32 dist U=8", 148, 1024), (4, "u32 dist U=4", 148, 1024), (11, "u8 mirror U=8", 148, 1024),
         (13, "u8 mirror U=16", 148, 1024), (12, "u16 mirror U=8", 148, 1024), (2, "edge stream only", 148, 1024),
         (20, "red.min all U=8", 148, 1024), (22, "red.min all U=4", 148, 1024), (21, "atomicMin ret U=8", 148, 1024),
         (20, "red.min all 296x1024", 296, 1024), (0, "u32 dist 296x1024", 296, 1024)]
for mode, name, blocks, threads in CASES:
    if True:
        ts = []
        for r in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            rc = lib.probe_gather(mode, cols.data_ptr(), m, dist.data_ptr(), sink.data_ptr(), blocks, threads,
                                  ctypes.c_void_p(st.cuda_stream))
            assert rc == 0, rc
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = min(ts[1:])
        print(f"{name:24s} grid {blocks}x{threads}: {t:.3f} ms  {m / t / 1e6:.1f} G edges/s", flush=True)

# the distances a config-4 query produces: does a 1-byte saturated mirror hold them exactly?
if os.environ.get("DIST_HIST", "0") == "1":
    from paper_1911_07260_b200 import gi
    del dist
    G = gi.Graph.from_csr(g)
    src = gen.config_source(int(os.environ.get("CFG", "4")), g)
    out = torch.empty(g.n, dtype=torch.int32, device="cuda")
    gi.sssp(G, src, gen.CONFIG_DELTAS[int(os.environ.get("CFG", "4"))][0], out=out)
    d = out.cpu().numpy().view(np.uint32)
    fin = d[d != 0xFFFFFFFF]
    print("reached", fin.size, "max dist", int(fin.max()), "p99", int(np.percentile(fin, 99)),
          "frac < 255", float((fin < 255).mean()))
    print("hist (x10)", np.bincount(np.minimum(fin // 10, 40)).tolist())
