"""paper_1911_07260_b200 — B200-native Δ-stepping SSSP (lazy far-bucket updates + bucket fusion).

The hot path lives in ``libgi.so`` (sm_100a CUDA kernels behind the C ABI in
``include/gi.h``); ``gi`` is the ctypes binding, ``dist`` the torch.distributed batch
sharding. Importing ``gi`` fails loudly if the library has not been built.
"""
__all__ = ["gi", "dist"]
