"""A/B timing of libgi.so builds in tools/ab/ on a config (fused / unfused) through the bare C ABI.
usage: python tools/ab_time.py CONFIG DELTA"""
import ctypes, glob, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gen
import torch

from paper_1911_07260_b200.gi import gi_options as Opt, gi_stats as St  # noqa: E402 (struct layouts only)
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
delta = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
g = gen.config_graph(cfg)
src = gen.config_source(cfg, g)
srcs = gen.config_sources(5, g, 64).astype(np.int32) if cfg == 5 else None
out = torch.empty((64 if cfg == 5 else 1) * g.n, dtype=torch.int32, device="cuda")
libs = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ.get("AB_DIR", "ab"), "libgi_*.so")))
if os.environ.get("AB_ONLY"):  # one library per process: no second-instance placement effect
    libs = [x for x in libs if os.path.basename(x) == f"libgi_{os.environ['AB_ONLY']}.so"]
for so in libs:
    lib = ctypes.CDLL(so)
    vp = ctypes.c_void_p
    lib.gi_graph_create.argtypes = [ctypes.c_int64, ctypes.c_int64, vp, vp, vp, ctypes.c_int, ctypes.POINTER(vp)]
    lib.gi_sssp_delta_ex.argtypes = [vp, ctypes.c_int32, ctypes.c_uint32, ctypes.POINTER(Opt), vp, ctypes.POINTER(St)]
    lib.gi_options_default.argtypes = [ctypes.POINTER(Opt)]
    lib.gi_sssp_batch_ex.argtypes = [vp, vp, ctypes.c_int32, ctypes.c_uint32, ctypes.POINTER(Opt), vp, vp]
    h = vp()
    assert lib.gi_graph_create(g.n, g.m, g.offsets.ctypes.data, g.cols.ctypes.data, g.w.ctypes.data, 0, ctypes.byref(h)) == 0
    res = []
    for fusion in ((1,) if cfg == 5 else (1, 0)):
        o = Opt(); lib.gi_options_default(ctypes.byref(o)); o.fusion = fusion
        for kv in os.environ.get("AB_OPTS", "").split(","):  # e.g. AB_OPTS=cta_threads=512,expand=1
            if kv:
                k_, v_ = kv.split("=")
                setattr(o, k_, int(v_))
        st = St(); ts = []
        for i in range(6):
            if cfg == 5:  # batch: every entry's gpu_ms is the whole batch's device time
                sts = (St * 64)()
                assert lib.gi_sssp_batch_ex(h, srcs.ctypes.data, 64, delta, ctypes.byref(o), out.data_ptr(), sts) == 0
                st = sts[0]
            else:
                assert lib.gi_sssp_delta_ex(h, src, delta, ctypes.byref(o), out.data_ptr(), ctypes.byref(st)) == 0
            ts.append(st.gpu_ms)
        res.append(round(float(np.median(ts[2:])), 3))
    print(os.path.basename(so), "fused/unfused ms", res, "ctas", st.ctas, "threads", st.threads_per_cta, "kind",
          st.kernel_kind, "rounds", st.rounds, "spills", st.spills, "edges", st.edges_relaxed, flush=True)
    lib.gi_graph_destroy(h)
