"""A/B timing of libgi.so builds in tools/ab/ on a config (fused / unfused) through the bare C ABI.
usage: python tools/ab_time.py CONFIG DELTA"""
import ctypes, glob, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gen
import torch

class Opt(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("fusion", ctypes.c_int32), ("fusion_threshold", ctypes.c_uint32),
                ("max_ctas", ctypes.c_int32), ("hub_min", ctypes.c_uint32), ("drain", ctypes.c_uint32),
                ("group_ctas", ctypes.c_int32), ("pre_read", ctypes.c_int32), ("cuda_stream", ctypes.c_void_p)]
class St(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint64) for k in ("buckets", "rounds", "grid_syncs", "kernel_launches", "fused_subrounds",
                "spills", "vertices_processed", "edges_relaxed", "empty_extractions", "far_scanned", "critical_subrounds")] + \
               [("gpu_ms", ctypes.c_float), ("ctas", ctypes.c_int32), ("tpc", ctypes.c_int32), ("groups", ctypes.c_int32),
                ("kind", ctypes.c_int32), ("pad", ctypes.c_int32 * 8)]
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
delta = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
g = gen.config_graph(cfg)
src = gen.config_source(cfg, g)
out = torch.empty(g.n, dtype=torch.int32, device="cuda")
for so in sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ab", "libgi_*.so"))):
    lib = ctypes.CDLL(so)
    vp = ctypes.c_void_p
    lib.gi_graph_create.argtypes = [ctypes.c_int64, ctypes.c_int64, vp, vp, vp, ctypes.c_int, ctypes.POINTER(vp)]
    lib.gi_sssp_delta_ex.argtypes = [vp, ctypes.c_int32, ctypes.c_uint32, ctypes.POINTER(Opt), vp, ctypes.POINTER(St)]
    lib.gi_options_default.argtypes = [ctypes.POINTER(Opt)]
    h = vp()
    assert lib.gi_graph_create(g.n, g.m, g.offsets.ctypes.data, g.cols.ctypes.data, g.w.ctypes.data, 0, ctypes.byref(h)) == 0
    res = []
    for fusion in (1, 0):
        o = Opt(); lib.gi_options_default(ctypes.byref(o)); o.fusion = fusion
        st = St(); ts = []
        for i in range(6):
            assert lib.gi_sssp_delta_ex(h, src, delta, ctypes.byref(o), out.data_ptr(), ctypes.byref(st)) == 0
            ts.append(st.gpu_ms)
        res.append(round(float(np.median(ts[2:])), 3))
    print(os.path.basename(so), "fused/unfused ms", res, flush=True)
    lib.gi_graph_destroy(h)
