"""Window probe (tools/window_probe.cu): G edges/s of random dist[col] gathers / red.min's
with the column ids confined to a window of n/R vertices (n = 2^26, config 4's size), R = 1..16.
usage: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC
           tools/window_probe.cu -o tools/ab/libwprobe.so && python tools/window_probe.py"""
import ctypes, os
import torch

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ab", "libwprobe.so"))
lib.probe_window.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                             ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
n, m = 1 << 26, 1 << 30
g = torch.Generator(device="cuda").manual_seed(7)
raw = torch.randint(0, 1 << 31, (m,), dtype=torch.int64, device="cuda", generator=g)
dist = torch.full((n,), -1, dtype=torch.int32, device="cuda")
sink = torch.zeros(4, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
for R in (1, 2, 4, 8, 16):
    win = n // R
    # R passes, each over m/R ids confined to window r (total m ids, same as R = 1)
    cols = [((raw[r * (m // R):(r + 1) * (m // R)] % win) + r * win).to(torch.int32) for r in range(R)]
    for mode, name in ((0, "read"), (1, "red.min"), (2, "pre-read+red.min")):
        ts = []
        for rep in range(4):
            dist.fill_(-1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for c in cols:
                assert lib.probe_window(mode, c.data_ptr(), c.numel(), dist.data_ptr(), sink.data_ptr(), 148, 1024,
                                        ctypes.c_void_p(st.cuda_stream)) == 0
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t = min(ts[1:])
        print(f"R={R:2d} window {win * 4 >> 20:4d} MB {name:18s}: {t:.3f} ms  {m / t / 1e6:.1f} G edges/s", flush=True)
    del cols
