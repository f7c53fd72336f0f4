"""Build a GI_TRACE variant of libgi.so into /tmp and report cycle breakdowns of CTA 0 / thread 0.
usage: python tools/trace_run.py path|cfg1|cfg2 [delta] [max_ctas]"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import gen  # noqa: E402

so = "/tmp/libgi_trace.so"
src = [os.path.join(ROOT, "paper_1911_07260_b200/csrc", f) for f in ("gi_kernels.cu", "gi_capi.cu")]
subprocess.check_call(["nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-DGI_TRACE",
                       "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"), "-o", so] + src)
lib = ctypes.CDLL(so)
vp, i64, i32, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
lib.gi_debug_trace.argtypes = [vp, ctypes.c_int]
lib.gi_graph_create.argtypes = [i64, i64, vp, vp, vp, ctypes.c_int, ctypes.POINTER(vp)]
from paper_1911_07260_b200.gi import gi_options, gi_stats  # noqa: E402  (struct layouts only)
lib.gi_sssp_delta_ex.argtypes = [vp, i32, u32, ctypes.POINTER(gi_options), vp, ctypes.POINTER(gi_stats)]
lib.gi_options_default.argtypes = [ctypes.POINTER(gi_options)]

what = sys.argv[1] if len(sys.argv) > 1 else "path"
delta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
max_ctas = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if what == "path":
    g = gen.path(20000); src_v = 0; delta = delta or 10**9
elif what == "cfg1":
    g = gen.config_graph(1); src_v = 0; delta = delta or 1000
else:
    g = gen.config_graph(2); src_v = gen.config_source(2, g); delta = delta or 65536
h = vp()
assert lib.gi_graph_create(g.n, g.m, g.offsets.ctypes.data, g.cols.ctypes.data, g.w.ctypes.data, 0,
                           ctypes.byref(h)) == 0
import torch  # noqa: E402

out = torch.empty(g.n, dtype=torch.int32, device="cuda")
opt = gi_options()
lib.gi_options_default(ctypes.byref(opt))
opt.max_ctas = max_ctas
st = gi_stats()
buf = np.zeros(32, np.uint64)
for rep in range(2):
    lib.gi_debug_trace(buf.ctypes.data, 1)
    rc = lib.gi_sssp_delta_ex(h, src_v, delta, ctypes.byref(opt), out.data_ptr(), ctypes.byref(st))
    assert rc == 0, rc
    lib.gi_debug_trace(buf.ctypes.data, 0)
print(what, "delta", delta, "max_ctas", max_ctas, "gpu_ms %.3f" % st.gpu_ms, "subrounds", st.fused_subrounds,
      "buckets", st.buckets)
names = {0: "drain loop top (since previous point)", 1: "swap+reset syncs", 2: "slot load",
         3: "relax_k (atomics+push)", 4: "rest of relax_wave", 5: "decision", 6: "extract scan",
         7: "phase work end", 8: "far flush + fmin", 9: "group barrier", 10: "relax_k: nd compute",
         11: "relax_k: atomics issued", 12: "relax_k: atomics returned", 13: "slot (before stale check)"}
for k in range(14):
    c = int(buf[16 + k])
    print(f"{k} {names[k]:40s} calls={c:8d} cycles/call={int(buf[k]) / max(c, 1):9.1f} total={int(buf[k]):12d}")
