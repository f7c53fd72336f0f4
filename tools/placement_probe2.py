"""Placement effect on config 4, part 2: is the second library instance fast because of its
module, or because a graph was created and destroyed before? usage: python tools/placement_probe2.py MODE
MODE: createonly | createsmall | nothing | bigalloc | runonly | = lib a only creates/destroys a graph; runonly = lib a runs queries on a tiny graph"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import gen
from paper_1911_07260_b200.gi import gi_options as Opt, gi_stats as St  # noqa: E402 (struct layouts only)

mode = sys.argv[1] if len(sys.argv) > 1 else "createonly"
g = gen.config_graph(4)
src = gen.config_source(4, g)
out = torch.empty(g.n, dtype=torch.int32, device="cuda")
here = os.path.dirname(os.path.abspath(__file__))
vp = ctypes.c_void_p


def load(name):
    lib = ctypes.CDLL(os.path.join(here, "ab", name))
    lib.gi_graph_create.argtypes = [ctypes.c_int64, ctypes.c_int64, vp, vp, vp, ctypes.c_int, ctypes.POINTER(vp)]
    lib.gi_sssp_delta_ex.argtypes = [vp, ctypes.c_int32, ctypes.c_uint32, ctypes.POINTER(Opt), vp, ctypes.POINTER(St)]
    lib.gi_options_default.argtypes = [ctypes.POINTER(Opt)]
    return lib


def run(lib, gg, s, reps=5):
    h = vp()
    assert lib.gi_graph_create(gg.n, gg.m, gg.offsets.ctypes.data, gg.cols.ctypes.data, gg.w.ctypes.data, 0,
                               ctypes.byref(h)) == 0
    o = Opt(); lib.gi_options_default(ctypes.byref(o))
    st = St(); ts = []
    o2 = torch.empty(gg.n, dtype=torch.int32, device="cuda")
    for _ in range(reps):
        assert lib.gi_sssp_delta_ex(h, s, 2, ctypes.byref(o), o2.data_ptr(), ctypes.byref(st)) == 0
        ts.append(st.gpu_ms)
    lib.gi_graph_destroy(h)
    return np.median(ts[1:]) if reps > 1 else ts[0]


a = load("libgi_a.so")
if mode == "createonly":
    h = vp()
    assert a.gi_graph_create(g.n, g.m, g.offsets.ctypes.data, g.cols.ctypes.data, g.w.ctypes.data, 0, ctypes.byref(h)) == 0
    a.gi_graph_destroy(h)
    print("lib a: create+destroy only")
elif mode == "createsmall":  # lib a creates/destroys a tiny graph: modules loaded, little memory
    t = gen.config_graph(1)
    h = vp()
    assert a.gi_graph_create(t.n, t.m, t.offsets.ctypes.data, t.cols.ctypes.data, t.w.ctypes.data, 0, ctypes.byref(h)) == 0
    a.gi_graph_destroy(h)
    print("lib a: tiny create+destroy only")
elif mode == "nothing":  # lib a loaded, never called
    print("lib a: loaded only")
elif mode == "bigalloc":  # a plain 22 GB cudaMalloc/cudaFree through torch before lib b
    x = torch.empty(22 << 30, dtype=torch.uint8, device="cuda"); x.fill_(1); del x; torch.cuda.empty_cache()
    print("torch 22 GB touched and freed")
elif mode == "runonly":
    t = gen.config_graph(1)
    print("lib a on config 1:", run(a, t, 0))
else:
    print("lib a on config 4:", run(a, g, src))
b = load("libgi_b.so")
print(f"lib b on config 4 ({mode}): {run(b, g, src):.2f} ms")
print(f"lib a again on config 4: {run(a, g, src):.2f} ms")
