"""Thin ctypes binding over libgi.so (include/gi.h): argument marshalling only.

Every step of the SSSP path runs in the library's sm_100a kernels; this module only
converts torch tensors / numpy arrays to pointers. There is no CPU fallback: if the
shared library is missing the import fails loudly.

torch has no full uint32 support, so distances are returned as int32 tensors holding
the uint32 bit pattern (UINT32_MAX reads as -1); ``as_uint32`` converts on the host.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_PKG, "libgi.so")

if not os.path.exists(_SO):
    raise ImportError(f"libgi.so not built at {_SO}: run __graft_entry__.build() "
                      "(the CUDA path has no fallback)")
_lib = ctypes.CDLL(_SO)

GI_OK = 0
STATUS = {0: "GI_OK", 1: "GI_ERR_INVALID_ARGUMENT", 2: "GI_ERR_OUT_OF_RANGE", 3: "GI_ERR_INVALID_GRAPH",
          4: "GI_ERR_OUT_OF_MEMORY", 5: "GI_ERR_CUDA", 6: "GI_ERR_OVERFLOW", 7: "GI_ERR_UNSUPPORTED"}
EXPORTS = ["gi_graph_create", "gi_graph_destroy", "gi_graph_info", "gi_sssp_delta", "gi_sssp_batch",
           "gi_options_default", "gi_sssp_delta_ex", "gi_sssp_batch_ex", "gi_last_error",
           "gi_status_string", "gi_version", "gi_ppsp_delta", "gi_ppsp_delta_ex", "gi_astar_delta",
           "gi_astar_delta_ex", "gi_kcore", "gi_kcore_ex", "gi_sssp_batch_peers", "gi_ipc_get_handle",
           "gi_ipc_open_handle", "gi_ipc_close_handle", "gi_probe_floors"]


class GiError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status
        self.name = STATUS.get(status, str(status))


class OverflowDistance(GiError):
    pass


class gi_options(ctypes.Structure):
    _fields_ = [("struct_size", ctypes.c_uint32), ("fusion", ctypes.c_int32),
                ("fusion_threshold", ctypes.c_uint32), ("max_ctas", ctypes.c_int32),
                ("hub_min", ctypes.c_uint32), ("drain", ctypes.c_uint32),
                ("group_ctas", ctypes.c_int32), ("pre_read", ctypes.c_int32), ("cuda_stream", ctypes.c_void_p),
                ("cta_threads", ctypes.c_int32), ("expand", ctypes.c_int32), ("lazy", ctypes.c_int32),
                ("rung", ctypes.c_int32), ("window", ctypes.c_int32)]


class gi_stats(ctypes.Structure):
    _fields_ = [("buckets", ctypes.c_uint64), ("rounds", ctypes.c_uint64), ("grid_syncs", ctypes.c_uint64),
                ("kernel_launches", ctypes.c_uint64), ("fused_subrounds", ctypes.c_uint64),
                ("spills", ctypes.c_uint64), ("vertices_processed", ctypes.c_uint64),
                ("edges_relaxed", ctypes.c_uint64), ("empty_extractions", ctypes.c_uint64),
                ("far_scanned", ctypes.c_uint64), ("critical_subrounds", ctypes.c_uint64),
                ("gpu_ms", ctypes.c_float), ("ctas", ctypes.c_int32),
                ("threads_per_cta", ctypes.c_int32), ("groups", ctypes.c_int32),
                ("kernel_kind", ctypes.c_int32), ("rung", ctypes.c_int32)]

    def to_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class gi_floors(ctypes.Structure):
    _fields_ = [("t_sync_us", ctypes.c_float), ("t_hop_us", ctypes.c_float), ("t_launch_us", ctypes.c_float),
                ("sm_clock_mhz", ctypes.c_float), ("ctas", ctypes.c_int32)]

    def to_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


_vp, _i64, _i32, _u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32
_lib.gi_graph_create.argtypes = [_i64, _i64, _vp, _vp, _vp, ctypes.c_int, ctypes.POINTER(_vp)]
_lib.gi_graph_destroy.argtypes = [_vp]
_lib.gi_graph_destroy.restype = None
_lib.gi_graph_info.argtypes = [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64), ctypes.POINTER(_i32)]
_lib.gi_sssp_delta.argtypes = [_vp, _i32, _u32, _vp]
_lib.gi_sssp_batch.argtypes = [_vp, _vp, _i32, _u32, _vp]
_lib.gi_options_default.argtypes = [ctypes.POINTER(gi_options)]
_lib.gi_options_default.restype = None
_lib.gi_sssp_delta_ex.argtypes = [_vp, _i32, _u32, ctypes.POINTER(gi_options), _vp, ctypes.POINTER(gi_stats)]
_lib.gi_sssp_batch_ex.argtypes = [_vp, _vp, _i32, _u32, ctypes.POINTER(gi_options), _vp, ctypes.POINTER(gi_stats)]
_lib.gi_sssp_batch_peers.argtypes = [_vp, _vp, _i32, _u32, ctypes.POINTER(gi_options), ctypes.POINTER(_vp), _i32,
                                     _i32, ctypes.POINTER(gi_stats)]
_lib.gi_ipc_get_handle.argtypes = [_vp, _vp, ctypes.POINTER(ctypes.c_uint64)]
_lib.gi_ipc_open_handle.argtypes = [_vp, ctypes.c_uint64, _i32, ctypes.POINTER(_vp)]
_lib.gi_ipc_close_handle.argtypes = [_vp, ctypes.c_uint64, _i32]
_lib.gi_ppsp_delta.argtypes = [_vp, _i32, _i32, _u32, _vp]
_lib.gi_ppsp_delta_ex.argtypes = [_vp, _i32, _i32, _u32, ctypes.POINTER(gi_options), _vp, ctypes.POINTER(gi_stats)]
_lib.gi_astar_delta.argtypes = [_vp, _i32, _i32, _u32, _vp, _vp]
_lib.gi_kcore.argtypes = [_vp, _vp]
_lib.gi_kcore_ex.argtypes = [_vp, ctypes.POINTER(gi_options), _vp, ctypes.POINTER(gi_stats)]
_lib.gi_astar_delta_ex.argtypes = [_vp, _i32, _i32, _u32, _vp, ctypes.POINTER(gi_options), _vp,
                                   ctypes.POINTER(gi_stats)]
_lib.gi_probe_floors.argtypes = [_i32, _i32, ctypes.POINTER(gi_floors)]
_lib.gi_last_error.restype = ctypes.c_char_p
_lib.gi_status_string.argtypes = [ctypes.c_int]
_lib.gi_status_string.restype = ctypes.c_char_p
_lib.gi_version.restype = _i32
for _f in ("gi_graph_create", "gi_graph_info", "gi_sssp_delta", "gi_sssp_batch", "gi_sssp_delta_ex",
           "gi_sssp_batch_ex", "gi_ppsp_delta", "gi_ppsp_delta_ex", "gi_astar_delta", "gi_astar_delta_ex", "gi_kcore",
           "gi_kcore_ex", "gi_sssp_batch_peers", "gi_ipc_get_handle", "gi_ipc_open_handle", "gi_ipc_close_handle",
           "gi_probe_floors"):
    getattr(_lib, _f).restype = ctypes.c_int


def _check(rc):
    if rc != GI_OK:
        msg = (_lib.gi_last_error() or b"").decode()
        if rc == 6:
            raise OverflowDistance(rc, msg)
        raise GiError(rc, msg)


def lib():
    return _lib


def version() -> int:
    return int(_lib.gi_version())


def _ptr(x):
    """data pointer of a torch tensor / numpy array (must be contiguous)."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return x.ctypes.data
    raise TypeError(type(x))


def _is_torch(x):
    return hasattr(x, "data_ptr") and hasattr(x, "dtype") and not isinstance(x, np.ndarray)


def _as_index_array(x, dtype, what):
    """Validate / coerce an index array to a contiguous `dtype` (np.int32 or np.int64) array or
    tensor of the same kind; values must fit the target type. Lists become numpy arrays."""
    import torch
    if _is_torch(x):
        want = torch.int32 if dtype == np.int32 else torch.int64
        if x.dtype == want:
            return x.contiguous()
        if x.dtype in (torch.int8, torch.int16, torch.int32, torch.int64, torch.uint8):
            info = np.iinfo(dtype)
            if x.numel() and (int(x.min()) < info.min or int(x.max()) > info.max):
                raise ValueError(f"{what}: values do not fit {np.dtype(dtype).name}")
            return x.to(want).contiguous()
        raise TypeError(f"{what}: integer tensor required, got {x.dtype}")
    a = np.asarray(x)
    if a.dtype.kind not in "iu":
        raise TypeError(f"{what}: integer array required, got {a.dtype}")
    if a.dtype != dtype:
        info = np.iinfo(dtype)
        if a.size and (int(a.min()) < info.min or int(a.max()) > info.max):
            raise ValueError(f"{what}: values do not fit {np.dtype(dtype).name}")
    return np.ascontiguousarray(a, dtype=dtype)


def _as_u32_bits(x, what):
    """uint32 data (weights, heuristics): numpy uint32 (int32 reinterpreted; other integer
    dtypes range-checked and converted) or a 4-byte integer torch tensor (int32 holds the bits)."""
    import torch
    if _is_torch(x):
        if x.dtype in (torch.int32, getattr(torch, "uint32", torch.int32)):
            return x.contiguous()
        if x.dtype in (torch.int64, torch.int16, torch.uint8, torch.int8):
            if x.numel() and (int(x.min()) < 0 or int(x.max()) > 0xFFFFFFFF):
                raise ValueError(f"{what}: values outside [0, 2^32)")
            return _u32_tensor(x)
        raise TypeError(f"{what}: 32-bit integer tensor required, got {x.dtype}")
    a = np.asarray(x)
    if a.dtype == np.uint32:
        return np.ascontiguousarray(a)
    if a.dtype == np.int32:
        return np.ascontiguousarray(a).view(np.uint32)
    if a.dtype.kind not in "iu":
        raise TypeError(f"{what}: integer array required, got {a.dtype}")
    if a.size and (int(a.min()) < 0 or int(a.max()) > 0xFFFFFFFF):
        raise ValueError(f"{what}: values outside [0, 2^32)")
    return np.ascontiguousarray(a, dtype=np.uint32)


def _u32_tensor(x):
    """integer tensor with values in [0, 2^32) -> int32 tensor holding the uint32 bits."""
    import torch
    y = x.to(torch.int64)
    y = torch.where(y >= 2 ** 31, y - 2 ** 32, y)
    return y.to(torch.int32).contiguous()


def _check_out(x, count, what):
    """A result buffer: 4-byte elements, contiguous, exactly `count` of them."""
    if _is_torch(x):
        if x.element_size() != 4 or x.dtype.is_floating_point:
            raise TypeError(f"{what}: int32/uint32 tensor required, got {x.dtype}")
        if not x.is_contiguous():
            raise ValueError(f"{what}: tensor must be contiguous")
        if x.numel() != count:
            raise ValueError(f"{what}: {x.numel()} elements, need {count}")
        return
    if not isinstance(x, np.ndarray):
        raise TypeError(f"{what}: numpy array or torch tensor required")
    if x.dtype not in (np.uint32, np.int32):
        raise TypeError(f"{what}: uint32/int32 array required, got {x.dtype}")
    if not x.flags["C_CONTIGUOUS"] or not x.flags["WRITEABLE"]:
        raise ValueError(f"{what}: array must be C-contiguous and writeable")
    if x.size != count:
        raise ValueError(f"{what}: {x.size} elements, need {count}")


def _default_stream(options, *tensors):
    """Options with cuda_stream = torch's current stream of the tensors' device when the
    caller gave none and some argument is a CUDA tensor, so that the query is ordered after
    the torch work that produced its inputs and before the work that reads its output."""
    dev = None
    for t in tensors:
        if _is_torch(t) and t.is_cuda:
            dev = t.device
            break
    if dev is None:
        return options
    if options is None:
        options = make_options()
    if not options.cuda_stream:
        import torch
        options.cuda_stream = torch.cuda.current_stream(dev).cuda_stream
    return options


def make_options(fusion=True, threshold=0, max_ctas=0, group_ctas=0, pre_read=0, hub_min=0,
                 drain=0, stream=None, cta_threads=0, expand=0, lazy=False, rung=0, window=0) -> gi_options:
    o = gi_options()
    _lib.gi_options_default(ctypes.byref(o))
    o.fusion = 1 if fusion else 0
    o.fusion_threshold = threshold
    o.max_ctas = max_ctas
    o.group_ctas = group_ctas
    o.pre_read = pre_read
    o.hub_min = hub_min
    o.drain = {"auto": 0, "bsp": 1, "async": 2}.get(drain, drain)
    o.cta_threads = cta_threads
    o.expand = {"auto": 0, "on": 1, "off": 2}.get(expand, expand)
    o.lazy = 1 if lazy else 0
    o.rung = {"auto": 0, "cta": 1, "cluster": 2, "grid": 3}.get(rung, rung)
    o.window = window
    if stream is not None:
        o.cuda_stream = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    return o


class Graph:
    """Device-resident CSR graph (gi_graph_create). Arrays may be numpy (host) or torch
    (host or CUDA) — int64 offsets[n+1], int32 cols[m], uint32/int32 weights[m]."""

    def __init__(self, offsets, cols, weights, device: int = 0):
        offsets = _as_index_array(offsets, np.int64, "offsets")
        cols = _as_index_array(cols, np.int32, "cols")
        weights = _as_u32_bits(weights, "weights")
        n = int(offsets.shape[0]) - 1
        m = int(cols.shape[0])
        if int(weights.shape[0]) != m:
            raise ValueError(f"weights: {int(weights.shape[0])} elements, cols has {m}")
        h = _vp()
        _check(_lib.gi_graph_create(n, m, _ptr(offsets), _ptr(cols) if m else None,
                                    _ptr(weights) if m else None, device, ctypes.byref(h)))
        self._h = h
        self.n, self.m, self.device = n, m, device

    @classmethod
    def from_csr(cls, csr, device: int = 0):
        return cls(csr.offsets, csr.cols, csr.w, device)

    @property
    def handle(self):
        return self._h

    def info(self):
        n, m, d = _i64(), _i64(), _i32()
        _check(_lib.gi_graph_info(self._h, ctypes.byref(n), ctypes.byref(m), ctypes.byref(d)))
        return n.value, m.value, d.value

    def close(self):
        if getattr(self, "_h", None):
            _lib.gi_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gi_sssp_delta(g: Graph, src: int, delta: int, dist_out, options: gi_options | None = None,
                  want_stats: bool = True):
    """C-ABI gi_sssp_delta_ex. dist_out: torch int32/uint32 CUDA tensor [n] or numpy uint32 [n]."""
    _check_out(dist_out, g.n, "dist_out")
    options = _default_stream(options, dist_out)
    st = gi_stats() if want_stats else None
    _check(_lib.gi_sssp_delta_ex(g.handle, int(src), int(delta), ctypes.byref(options) if options else None,
                                 _ptr(dist_out), ctypes.byref(st) if st is not None else None))
    return st


def gi_sssp_batch(g: Graph, srcs, delta: int, dist_out, options: gi_options | None = None,
                  want_stats: bool = True):
    """C-ABI gi_sssp_batch_ex. srcs: int32 array/tensor [k]; dist_out [k, n]."""
    srcs = _as_index_array(srcs, np.int32, "srcs")
    k = int(srcs.shape[0])
    _check_out(dist_out, k * g.n, "dist_out")
    options = _default_stream(options, dist_out, srcs)
    st = (gi_stats * max(k, 1))() if want_stats else None
    _check(_lib.gi_sssp_batch_ex(g.handle, _ptr(srcs), k, int(delta),
                                 ctypes.byref(options) if options else None, _ptr(dist_out), st))
    return st


def gi_sssp_batch_peers(g: Graph, srcs, delta: int, peer_rows, self_index: int,
                        options: gi_options | None = None, want_stats: bool = True):
    """C-ABI gi_sssp_batch_peers. peer_rows: device addresses (ints) of this block's first
    row inside every rank's result matrix; rows are computed in peer_rows[self_index]."""
    srcs = _as_index_array(srcs, np.int32, "srcs")
    k = int(srcs.shape[0])
    if options is None or not options.cuda_stream:
        import torch
        options = options if options is not None else make_options()
        options.cuda_stream = torch.cuda.current_stream(g.device).cuda_stream
    st = (gi_stats * max(k, 1))() if want_stats else None
    arr = (_vp * len(peer_rows))(*[int(p) for p in peer_rows])
    _check(_lib.gi_sssp_batch_peers(g.handle, _ptr(srcs), k, int(delta), ctypes.byref(options) if options else None,
                                    arr, len(peer_rows), int(self_index), st))
    return st


def ipc_handle(t) -> tuple[bytes, int]:
    """(64-byte IPC handle of the allocation holding tensor t, byte offset of t in it)."""
    h = (ctypes.c_uint8 * 64)()
    off = ctypes.c_uint64()
    _check(_lib.gi_ipc_get_handle(_vp(t.data_ptr()), h, ctypes.byref(off)))
    return bytes(h), off.value


def ipc_open(handle: bytes, offset: int, device: int) -> int:
    """Map another process's allocation; returns the device address of base + offset."""
    h = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    p = _vp()
    _check(_lib.gi_ipc_open_handle(h, int(offset), int(device), ctypes.byref(p)))
    return int(p.value)


def ipc_close(addr: int, offset: int, device: int) -> None:
    _check(_lib.gi_ipc_close_handle(_vp(addr), int(offset), int(device)))


def sssp(g: Graph, src: int, delta: int, out=None, **opts):
    """Single-source Δ-stepping on the graph's device. Returns (dist int32 tensor [n]
    holding uint32 bits, stats dict)."""
    import torch
    if out is None:
        out = torch.empty(g.n, dtype=torch.int32, device=f"cuda:{g.device}")
    st = gi_sssp_delta(g, src, delta, out, make_options(**opts) if opts else None)
    return out, st.to_dict()


def sssp_batch(g: Graph, srcs, delta: int, out=None, **opts):
    import torch
    srcs = _as_index_array(srcs, np.int32, "srcs")
    k = int(srcs.shape[0])
    if out is None:
        out = torch.empty((k, g.n), dtype=torch.int32, device=f"cuda:{g.device}")
    st = gi_sssp_batch(g, srcs, delta, out, make_options(**opts) if opts else None)
    return out, [st[i].to_dict() for i in range(k)]


def gi_ppsp_delta(g: Graph, src: int, dst: int, delta: int, dist_st, options: gi_options | None = None,
                  want_stats: bool = True):
    """C-ABI gi_ppsp_delta_ex. dist_st: one-element uint32 (or int32) array/tensor."""
    _check_out(dist_st, 1, "dist_st")
    options = _default_stream(options, dist_st)
    st = gi_stats() if want_stats else None
    _check(_lib.gi_ppsp_delta_ex(g.handle, int(src), int(dst), int(delta),
                                 ctypes.byref(options) if options else None, _ptr(dist_st),
                                 ctypes.byref(st) if st is not None else None))
    return st


def ppsp(g: Graph, src: int, dst: int, delta: int, **opts):
    """Point-to-point Δ-stepping with the paper's early stop. Returns (δ(src, dst) as a
    Python int, UINT32_MAX if unreachable; stats dict)."""
    out = np.zeros(1, np.uint32)
    st = gi_ppsp_delta(g, src, dst, delta, out, make_options(**opts) if opts else None)
    return int(out[0]), st.to_dict()


def gi_astar_delta(g: Graph, src: int, dst: int, delta: int, h, dist_st, options: gi_options | None = None,
                   want_stats: bool = True):
    """C-ABI gi_astar_delta_ex. h: uint32 (or int32 bits) [n] array/tensor, host or device."""
    h = _as_u32_bits(h, "h")
    if int(h.shape[0]) != g.n:
        raise ValueError(f"h: {int(h.shape[0])} elements, need {g.n}")
    _check_out(dist_st, 1, "dist_st")
    options = _default_stream(options, dist_st, h)
    st = gi_stats() if want_stats else None
    _check(_lib.gi_astar_delta_ex(g.handle, int(src), int(dst), int(delta), _ptr(h),
                                  ctypes.byref(options) if options else None, _ptr(dist_st),
                                  ctypes.byref(st) if st is not None else None))
    return st


def astar(g: Graph, src: int, dst: int, delta: int, h, **opts):
    """A* (Δ-stepping on the priority dist + h, PPSP stop). Returns (distance, stats dict)."""
    out = np.zeros(1, np.uint32)
    st = gi_astar_delta(g, src, dst, delta, h, out, make_options(**opts) if opts else None)
    return int(out[0]), st.to_dict()


def gi_kcore(g: Graph, core_out, options: gi_options | None = None, want_stats: bool = True):
    """C-ABI gi_kcore_ex. core_out: uint32/int32 [n], host or device."""
    _check_out(core_out, g.n, "core_out")
    options = _default_stream(options, core_out)
    st = gi_stats() if want_stats else None
    _check(_lib.gi_kcore_ex(g.handle, ctypes.byref(options) if options else None, _ptr(core_out),
                            ctypes.byref(st) if st is not None else None))
    return st


def kcore(g: Graph, out=None, **opts):
    """Coreness of every vertex (bucketed peel on the GPU). Returns (int32 tensor [n]
    holding uint32 values, stats dict)."""
    import torch
    if out is None:
        out = torch.empty(g.n, dtype=torch.int32, device=f"cuda:{g.device}")
    st = gi_kcore(g, out, make_options(**opts) if opts else None)
    return out, st.to_dict()


def probe_floors(device: int = 0, iters: int = 2000) -> dict:
    """C-ABI gi_probe_floors: t_sync / t_hop / t_launch (µs) measured on `device`."""
    f = gi_floors()
    _check(_lib.gi_probe_floors(int(device), int(iters), ctypes.byref(f)))
    return f.to_dict()


def as_uint32(t) -> np.ndarray:
    """int32 tensor/array holding uint32 bits -> numpy uint32 (host)."""
    if hasattr(t, "cpu"):
        t = t.cpu().numpy()
    return np.asarray(t).view(np.uint32)
