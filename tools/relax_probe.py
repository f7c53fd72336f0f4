"""Ingredient costs of the expand relaxation on config 4 (tools/relax_probe.cu).
usage: GI_GEN_CACHE=/tmp/gcache python tools/relax_probe.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import gen

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ab", "librelax.so"))
vp = ctypes.c_void_p
lib.probe_relax.argtypes = [ctypes.c_int, vp, ctypes.c_int64, vp, vp, vp, vp, ctypes.c_uint32, ctypes.c_int, ctypes.c_int, vp]
g = gen.config_graph(4)
colbits = 26
pe = torch.from_numpy((np.asarray(g.w, np.uint32) << np.uint32(colbits)) | np.asarray(g.cols).view(np.uint32)).cuda()
m, n = g.m, g.n
bits = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
lst = torch.zeros(1 << 26, dtype=torch.int32, device="cuda")
counts = torch.zeros(148 * 32 * 4, dtype=torch.int32, device="cuda")
init = (torch.arange(n, device="cuda", dtype=torch.int64) * 2654435761 % 97).to(torch.int32)  # dist in [0, 97)
st = torch.cuda.current_stream()
names = ["R0 gather+compare", "R1 +red.min", "R2 +smem push", "R3 +flush (1 global counter)", "R4 +flush (per-CTA counters)"]
for mode in []:
    for blocks, threads in ((148, 1024), (148, 512)):
        ts = []
        for r in range(3):
            dist = init.clone(); bits.zero_(); counts.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            rc = lib.probe_relax(mode, pe.data_ptr(), m, dist.data_ptr(), bits.data_ptr(), lst.data_ptr(),
                                 counts.data_ptr(), colbits, blocks, threads, vp(st.cuda_stream))
            e1.record(st)
            torch.cuda.synchronize()
            assert rc == 0, rc
            ts.append(e0.elapsed_time(e1))
        imp = int((dist != init).sum())
        print(f"{names[mode]:32s} {blocks}x{threads}: {min(ts[1:]):.3f} ms  {m / min(ts[1:]) / 1e6:.1f} G edges/s "
              f"(targets lowered {imp})", flush=True)

# MODE 5: the expand mapping over X = every vertex of degree > 8 (its whole edge list)
lib.probe_relax_x.argtypes = [ctypes.c_int, vp, vp, vp, ctypes.c_uint32, ctypes.c_uint64, vp, vp, vp, vp,
                              ctypes.c_uint32, ctypes.c_int, ctypes.c_int, vp]
deg = np.diff(np.asarray(g.offsets))
big = np.nonzero(deg > 8)[0]
Xh = np.zeros(big.shape[0], dtype=[("beg", "<i8"), ("deg", "<u4"), ("du", "<u4")])
Xh["beg"] = np.asarray(g.offsets)[big]
Xh["deg"] = deg[big]
Xh["du"] = (big.astype(np.uint64) * 2654435761 % 32).astype(np.uint32)
pre = np.zeros(big.shape[0], np.uint64)
pre[1:] = np.cumsum(deg[big].astype(np.uint64))[:-1]
E = int(deg[big].sum())
X = torch.from_numpy(Xh.view(np.uint8)).cuda()
xpre = torch.from_numpy(pre.view(np.int64)).cuda()
# the same list in a random order (the frontier order of a real phase): prefix recomputed
perm = np.random.default_rng(1).permutation(big.shape[0])
Xp = Xh[perm]
prep = np.zeros(big.shape[0], np.uint64)
prep[1:] = np.cumsum(Xp["deg"].astype(np.uint64))[:-1]
Xr = torch.from_numpy(Xp.view(np.uint8)).cuda()
xprer = torch.from_numpy(prep.view(np.int64)).cuda()
for K, Xd, xp, tag in ((4, X, xpre, "id order"), (8, X, xpre, "id order"), (4, Xr, xprer, "random order"), (8, Xr, xprer, "random order")):
    X_, xpre_ = Xd, xp
    for blocks, threads in ((148, 1024), (148, 512)):
        ts = []
        for r in range(3):
            dist = init.clone(); bits.zero_(); counts.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            rc = lib.probe_relax_x(K, pe.data_ptr(), X_.data_ptr(), xpre_.data_ptr(), big.shape[0], E, dist.data_ptr(),
                                   bits.data_ptr(), lst.data_ptr(), counts.data_ptr(), colbits, blocks, threads,
                                   vp(st.cuda_stream))
            e1.record(st)
            torch.cuda.synchronize()
            assert rc == 0, rc
            ts.append(e0.elapsed_time(e1))
        print(f"R5 expand mapping K={K} {tag:12s} {blocks}x{threads}: {min(ts[1:]):.3f} ms  {E / min(ts[1:]) / 1e6:.1f} G edges/s "
              f"(E={E})", flush=True)

# MODE 5 on a real phase list dumped by GI_DUMP_X (entries {beg, deg, du}) with the real dist
import glob
for fn in sorted(glob.glob(os.environ.get("XDUMP", "/tmp/xdump") + "_*_E*.bin")):
    Xh2 = np.fromfile(fn, dtype=[("beg", "<i8"), ("deg", "<u4"), ("du", "<u4")])
    dd = np.fromfile(fn.split("_p")[0] + "_dist.bin", dtype=np.int32)
    pre2 = np.zeros(Xh2.shape[0], np.uint64)
    pre2[1:] = np.cumsum(Xh2["deg"].astype(np.uint64))[:-1]
    E2 = int(Xh2["deg"].astype(np.uint64).sum())
    X2 = torch.from_numpy(Xh2.view(np.uint8)).cuda()
    xpre2 = torch.from_numpy(pre2.view(np.int64)).cuda()
    dist0 = torch.from_numpy(dd).cuda()
    for K in (4, 8):
        ts = []
        for r in range(3):
            dist = dist0.clone(); bits.zero_(); counts.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            rc = lib.probe_relax_x(K, pe.data_ptr(), X2.data_ptr(), xpre2.data_ptr(), Xh2.shape[0], E2, dist.data_ptr(),
                                   bits.data_ptr(), lst.data_ptr(), counts.data_ptr(), colbits, 148, 1024, vp(st.cuda_stream))
            e1.record(st)
            torch.cuda.synchronize()
            assert rc == 0, rc
            ts.append(e0.elapsed_time(e1))
        imp = int((dist != dist0).sum())
        print(f"R5 on {os.path.basename(fn)} K={K}: entries {Xh2.shape[0]} {min(ts[1:]):.3f} ms  {E2 / min(ts[1:]) / 1e6:.1f} G edges/s, lowered {imp}", flush=True)
