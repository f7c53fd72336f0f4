"""Config-4 placement effect: which condition makes a query fast?
usage: GI_GEN_CACHE=/tmp/gcache python tools/placement_test.py MODE   (one mode per process)
  single      one library (tools/ab/libgi_cs.so), nothing else loaded
  two         the product libgi.so loaded (ctypes, never called), then libgi_cs.so runs
  two_called  libgi.so creates+destroys a tiny graph, then libgi_cs.so runs
  tiny_same   libgi_cs.so creates+destroys a tiny graph, then runs config 4
  torch_pre   a 22 GB torch block written and freed (empty_cache), then libgi_cs.so runs
  out_first   the torch output tensor is allocated before the graph (as tools/ab_time.py does)
  torch_tiny  torch allocates a 4-byte tensor first (its CUDA state initialised), out after the graph"""
import ctypes, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import gen

vp = ctypes.c_void_p


class Opt(ctypes.Structure):  # gi_options (include/gi.h)
    _fields_ = [("struct_size", ctypes.c_uint32), ("fusion", ctypes.c_int32), ("fusion_threshold", ctypes.c_uint32),
                ("max_ctas", ctypes.c_int32), ("hub_min", ctypes.c_uint32), ("drain", ctypes.c_uint32),
                ("group_ctas", ctypes.c_int32), ("pre_read", ctypes.c_int32), ("cuda_stream", ctypes.c_void_p),
                ("cta_threads", ctypes.c_int32), ("expand", ctypes.c_int32), ("lazy", ctypes.c_int32),
                ("rung", ctypes.c_int32)]


class St(ctypes.Structure):  # gi_stats
    _fields_ = [(k, ctypes.c_uint64) for k in ("buckets", "rounds", "grid_syncs", "kernel_launches", "fused_subrounds",
                                               "spills", "vertices_processed", "edges_relaxed", "empty_extractions",
                                               "far_scanned", "critical_subrounds")] + [
        ("gpu_ms", ctypes.c_float), ("ctas", ctypes.c_int32), ("threads_per_cta", ctypes.c_int32),
        ("groups", ctypes.c_int32), ("kernel_kind", ctypes.c_int32), ("rung", ctypes.c_int32)]


def load(path):
    lib = ctypes.CDLL(path)
    lib.gi_graph_create.argtypes = [ctypes.c_int64, ctypes.c_int64, vp, vp, vp, ctypes.c_int, ctypes.POINTER(vp)]
    lib.gi_sssp_delta_ex.argtypes = [vp, ctypes.c_int32, ctypes.c_uint32, ctypes.POINTER(Opt), vp, ctypes.POINTER(St)]
    lib.gi_options_default.argtypes = [ctypes.POINTER(Opt)]
    lib.gi_graph_destroy.argtypes = [vp]
    return lib


def create(lib, g):
    h = vp()
    assert lib.gi_graph_create(g.n, g.m, g.offsets.ctypes.data, g.cols.ctypes.data, g.w.ctypes.data, 0,
                               ctypes.byref(h)) == 0
    return h


root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
mode = sys.argv[1]
tiny = gen.config_graph(1)
if mode in ("two", "two_called"):
    a = load(os.path.join(root, "paper_1911_07260_b200", "libgi.so"))
    if mode == "two_called":
        a.gi_graph_destroy(create(a, tiny))
if mode == "torch_pre":
    x = torch.empty(22 << 30, dtype=torch.uint8, device="cuda"); x.fill_(1); del x; torch.cuda.empty_cache()
b = load(os.path.join(root, "tools", "ab", "libgi_cs.so"))
if mode == "tiny_same":
    b.gi_graph_destroy(create(b, tiny))
g = gen.config_graph(4)
src = gen.config_source(4, g)
if mode == "out_first":
    out = torch.empty(g.n, dtype=torch.int32, device="cuda")
if mode == "torch_tiny":
    tiny_t = torch.zeros(1, device="cuda")
if mode.startswith("torch_mb_"):  # torch_mb_<X>[_free]: an X MB torch block first (freed + cache emptied with _free)
    parts = mode.split("_")
    blk = torch.empty(int(parts[2]) << 20, dtype=torch.uint8, device="cuda")
    if len(parts) > 3:
        del blk
        torch.cuda.empty_cache()
h = create(b, g)
if mode != "out_first":
    out = torch.empty(g.n, dtype=torch.int32, device="cuda")
o = Opt(); b.gi_options_default(ctypes.byref(o))
st = St(); ts = []
for i in range(8):
    assert b.gi_sssp_delta_ex(h, src, 2, ctypes.byref(o), out.data_ptr(), ctypes.byref(st)) == 0
    ts.append(st.gpu_ms)
print(os.environ.get("PYTORCH_CUDA_ALLOC_CONF"), torch._C._cuda_getAllocatorBackend() if hasattr(torch._C, "_cuda_getAllocatorBackend") else "?")
print(mode, "median ms", round(statistics.median(ts[2:]), 3), [round(t, 2) for t in ts], flush=True)
