"""Windows of one allocation: random read / atomic rate per 256 MiB window offset.
usage: python tools/placement_bench.py"""
import ctypes, os, sys
import torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ab", "libplace.so"))
lib.place_rnd.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
buf = torch.zeros(6 << 30, dtype=torch.uint8, device="cuda")
sink = torch.zeros(4, dtype=torch.int32, device="cuda")
st = torch.cuda.current_stream()
W = 256 << 20
iters = 64
ops = 148 * 2 * 1024 * 8 * iters
for atom in (0, 1):
    for off_mb in list(range(0, 1024 + 1, 64)) + [2048, 2048 + 128, 4096, 4096 + 128]:
        ts = []
        for r in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            rc = lib.place_rnd(atom, buf.data_ptr() + (off_mb << 20), W // 4, iters, sink.data_ptr(), ctypes.c_void_p(st.cuda_stream))
            e1.record(st)
            torch.cuda.synchronize()
            assert rc == 0
            ts.append(e0.elapsed_time(e1))
        print(f"{'atomic' if atom else 'read  '} window @ {off_mb:5d} MiB: {ops / min(ts[1:]) / 1e6:7.1f} G ops/s", flush=True)
print("base address", hex(buf.data_ptr()))
