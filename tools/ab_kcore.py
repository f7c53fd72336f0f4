"""A/B timing of k-core across libgi builds in tools/ab/ (one library per process with AB_ONLY).
usage: AB_ONLY=name python tools/ab_kcore.py CONFIG"""
import ctypes, glob, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import gen
from paper_1911_07260_b200.gi import gi_options as Opt, gi_stats as St  # noqa: E402 (struct layouts only)

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g = gen.config_graph(cfg)
out = torch.empty(g.n, dtype=torch.int32, device="cuda")
libs = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ.get("AB_DIR", "ab"),
                                     "libgi_*.so")))
if os.environ.get("AB_ONLY"):
    libs = [x for x in libs if os.path.basename(x) == f"libgi_{os.environ['AB_ONLY']}.so"]
vp = ctypes.c_void_p
for so in libs:
    lib = ctypes.CDLL(so)
    lib.gi_graph_create.argtypes = [ctypes.c_int64, ctypes.c_int64, vp, vp, vp, ctypes.c_int, ctypes.POINTER(vp)]
    lib.gi_kcore_ex.argtypes = [vp, ctypes.POINTER(Opt), vp, ctypes.POINTER(St)]
    h = vp()
    assert lib.gi_graph_create(g.n, g.m, g.offsets.ctypes.data, g.cols.ctypes.data, g.w.ctypes.data, 0, ctypes.byref(h)) == 0
    ts = []
    st = St()
    for i in range(5):
        assert lib.gi_kcore_ex(h, None, out.data_ptr(), ctypes.byref(st)) == 0
        ts.append(st.gpu_ms)
    core = out.cpu().numpy().view(np.uint32)
    print(os.path.basename(so), "kcore ms", round(float(np.median(ts[1:])), 3), "rounds", st.rounds, "critical",
          st.critical_subrounds, "spills", st.spills, "max core", int(core.max()),
          "checksum", int((core.astype(np.uint64) * np.arange(1, g.n + 1, dtype=np.uint64)).sum() % (1 << 61)), flush=True)
    lib.gi_graph_destroy(h)
