"""Parity of a variant build (tools/ab/libgi_<AB_ONLY>.so) on a 512x512 grid against scipy's
Dijkstra, over single-CTA and small-group launches — for builds that shrink buffers to force
the overflow paths (e.g. -DGI_FARSTAGE=512). usage: AB_ONLY=name python tools/ab_parity.py"""
import ctypes, glob, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import dijkstra
import torch
import gen
from paper_1911_07260_b200.gi import gi_options as Opt, gi_stats as St  # noqa: E402 (struct layouts only)

g = gen.grid(512, 512, 1, 100, 21, p_del=0.05, p_diag=0.02)
A = sp.csr_matrix((g.w.astype(np.float64), g.cols, g.offsets), shape=(g.n, g.n))
ref = dijkstra(A, indices=0)
ref = np.where(np.isfinite(ref), ref, 2**32 - 1).astype(np.uint64)
so = glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ab", f"libgi_{os.environ['AB_ONLY']}.so"))[0]
lib = ctypes.CDLL(so)
vp = ctypes.c_void_p
lib.gi_graph_create.argtypes = [ctypes.c_int64, ctypes.c_int64, vp, vp, vp, ctypes.c_int, ctypes.POINTER(vp)]
lib.gi_sssp_delta_ex.argtypes = [vp, ctypes.c_int32, ctypes.c_uint32, ctypes.POINTER(Opt), vp, ctypes.POINTER(St)]
lib.gi_options_default.argtypes = [ctypes.POINTER(Opt)]
h = vp()
assert lib.gi_graph_create(g.n, g.m, g.offsets.ctypes.data, g.cols.ctypes.data, g.w.ctypes.data, 0, ctypes.byref(h)) == 0
out = torch.empty(g.n, dtype=torch.int32, device="cuda")
for mc, T, delta, thr in ((1, 2048, 10**9, 0), (1, 0, 64, 0), (2, 2048, 16, 0), (1, 0, 10**9, 1024), (148, 0, 50, 0)):
    o = Opt(); lib.gi_options_default(ctypes.byref(o)); o.max_ctas = mc; o.fusion_threshold = T; o.cta_threads = thr
    st = St()
    assert lib.gi_sssp_delta_ex(h, 0, delta, ctypes.byref(o), out.data_ptr(), ctypes.byref(st)) == 0
    d = out.cpu().numpy().view(np.uint32).astype(np.uint64)
    print(os.path.basename(so), "ctas", mc, "T", T, "delta", delta, "threads", thr, "spills", st.spills,
          "parity", bool(np.array_equal(d, ref)), flush=True)
