"""Seeded synthetic CSR graphs — the one input module shared by oracle/ and the CUDA path.

Holds none of the method's arithmetic (no relaxation, no bucketing): it builds
inputs only. The recipe is SURVEY.md §8(d) ("Generator (proposed exact
recipe)"), standing in for the paper's datasets (PAPER.md:885-904,
table:datasets), which are not available: large-diameter road networks
(RD/GE) and skewed social graphs with weights [1, log n)
(PAPER.md:910).

CSR layout everywhere: ``offsets`` int64[n+1], ``cols`` int32[m], ``w`` uint32[m];
rows by source id, neighbours ascending (SPEC.md:30-35 invariants).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libgigen.so")
_SRC = os.path.join(_HERE, "gigen.cpp")

INF = 0xFFFFFFFF  # unreached sentinel

TAG_W, TAG_DEL, TAG_DIAG, TAG_RMAT, TAG_SRC = 1, 2, 3, 4, 5


def build(force: bool = False) -> str:
    """Compile libgigen.so (host C++/OpenMP)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["g++", "-O3", "-march=x86-64-v2", "-std=c++17", "-fopenmp", "-fPIC", "-shared",
               _SRC, "-o", _SO + ".tmp"]
        subprocess.check_call(cmd)
        os.replace(_SO + ".tmp", _SO)
    return _SO


class _CSR(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("m", ctypes.c_int64),
                ("offsets", ctypes.POINTER(ctypes.c_int64)),
                ("cols", ctypes.POINTER(ctypes.c_int32)),
                ("w", ctypes.POINTER(ctypes.c_uint32))]


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.gigen_grid.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint32,
                                    ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32,
                                    ctypes.POINTER(_CSR)]
        _lib.gigen_rmat.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, ctypes.c_uint32,
                                    ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint64,
                                    ctypes.POINTER(_CSR)]
        _lib.gigen_from_undirected.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                               ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32,
                                               ctypes.c_uint64, ctypes.POINTER(_CSR)]
        _lib.gigen_uniform.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint32,
                                       ctypes.c_uint64, ctypes.POINTER(_CSR)]
        _lib.gigen_sources.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64, ctypes.c_void_p]
        _lib.gigen_free.argtypes = [ctypes.POINTER(_CSR)]
        _lib.gigen_mix64.argtypes = [ctypes.c_uint64]
        _lib.gigen_mix64.restype = ctypes.c_uint64
        _lib.gigen_u32.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        _lib.gigen_u32.restype = ctypes.c_uint32
        for f in ("gigen_grid", "gigen_rmat", "gigen_from_undirected", "gigen_uniform", "gigen_sources"):
            getattr(_lib, f).restype = ctypes.c_int
    return _lib


class _Owner:
    """Keeps C-allocated CSR buffers alive for the numpy views that alias them."""

    def __init__(self, c: _CSR):
        self.c = c

    def __del__(self):
        try:
            _L().gigen_free(ctypes.byref(self.c))
        except Exception:
            pass


@dataclass
class CSR:
    """Canonical CSR graph. ``w`` is uint32; ``cols`` int32; ``offsets`` int64."""
    offsets: np.ndarray
    cols: np.ndarray
    w: np.ndarray
    name: str = ""
    meta: dict = field(default_factory=dict)
    _owner: object = None

    @property
    def n(self) -> int:
        return int(self.offsets.shape[0] - 1)

    @property
    def m(self) -> int:
        return int(self.cols.shape[0])

    def degrees(self) -> np.ndarray:
        return np.diff(self.offsets)


def _wrap(c: _CSR, name: str, meta: dict) -> CSR:
    n, m = int(c.n), int(c.m)
    own = _Owner(c)
    off = np.ctypeslib.as_array(c.offsets, shape=(n + 1,))
    cols = np.ctypeslib.as_array(c.cols, shape=(max(m, 1),))[:m]
    w = np.ctypeslib.as_array(c.w, shape=(max(m, 1),))[:m]
    return CSR(off, cols, w, name, meta, own)


def _check(rc: int, what: str):
    if rc != 0:
        raise RuntimeError(f"gigen {what} failed rc={rc}")


def bernoulli_threshold(p: float) -> int:
    """floor(p * 2^32): 0.05 -> 214,748,364; 0.01 -> 42,949,672."""
    return int(p * (1 << 32))


def u32(seed: int, tag: int, x: int) -> int:
    return int(_L().gigen_u32(seed, tag, x))


def mix64(z: int) -> int:
    return int(_L().gigen_mix64(z & 0xFFFFFFFFFFFFFFFF))


def grid(rows: int, cols: int, w_lo: int, w_hi: int, seed: int, p_del: float = 0.0,
         p_diag: float = 0.0, name: str = "grid") -> CSR:
    c = _CSR()
    _check(_L().gigen_grid(rows, cols, w_lo, w_hi, seed, bernoulli_threshold(p_del),
                           bernoulli_threshold(p_diag), ctypes.byref(c)), "grid")
    return _wrap(c, name, dict(kind="grid", rows=rows, cols=cols, w_lo=w_lo, w_hi=w_hi,
                               seed=seed, p_del=p_del, p_diag=p_diag))


RMAT_T = (2448131358, 3264175144, 4080218931)  # floor(.57, .76, .95 * 2^32)


def rmat(scale: int, edge_factor: int, w_lo: int, w_hi: int, seed: int, name: str = "rmat") -> CSR:
    c = _CSR()
    _check(_L().gigen_rmat(scale, edge_factor, *RMAT_T, w_lo, w_hi, seed, ctypes.byref(c)), "rmat")
    return _wrap(c, name, dict(kind="rmat", scale=scale, edge_factor=edge_factor, w_lo=w_lo,
                               w_hi=w_hi, seed=seed))


def from_undirected(n: int, edges, w_lo: int = 1, w_hi: int = 2, seed: int = 0, name="undirected") -> CSR:
    e = np.asarray(edges, dtype=np.int32).reshape(-1, 2)
    us = np.ascontiguousarray(e[:, 0])
    vs = np.ascontiguousarray(e[:, 1])
    c = _CSR()
    _check(_L().gigen_from_undirected(n, e.shape[0], us.ctypes.data, vs.ctypes.data, w_lo, w_hi,
                                      seed, ctypes.byref(c)), "from_undirected")
    return _wrap(c, name, dict(kind="undirected"))


def uniform_random(n: int, m: int, w_lo: int, w_hi: int, seed: int, name="uniform") -> CSR:
    """SPEC.md:58-66 uniform_random (directed, with replacement, parallel edges kept)."""
    c = _CSR()
    _check(_L().gigen_uniform(n, m, w_lo, w_hi, seed, ctypes.byref(c)), "uniform")
    return _wrap(c, name, dict(kind="uniform", n=n, m=m, w_lo=w_lo, w_hi=w_hi, seed=seed))


def from_edges(n: int, edges) -> CSR:
    """Directed edge list [(u, v, w), ...] -> CSR, keeping parallel edges and self-loops
    (SPEC.md:93, :103). Rows sorted by (col, w) for a canonical order."""
    e = np.asarray(list(edges), dtype=np.int64).reshape(-1, 3)
    if e.shape[0] and (e[:, :2].min() < 0 or e[:, :2].max() >= n or e[:, 2].min() < 0
                       or e[:, 2].max() > 0xFFFFFFFF):
        raise ValueError("edge out of range")
    order = np.lexsort((e[:, 2], e[:, 1], e[:, 0])) if e.shape[0] else np.zeros(0, np.int64)
    e = e[order]
    off = np.zeros(n + 1, np.int64)
    np.add.at(off, e[:, 0] + 1, 1)
    off = np.cumsum(off).astype(np.int64)
    return CSR(off, e[:, 1].astype(np.int32), e[:, 2].astype(np.uint32), "edges", {})


def path(n: int, w: int = 1) -> CSR:
    """Symmetric path 0-1-...-(n-1), all weights w ("path")."""
    edges = [(i, i + 1, w) for i in range(n - 1)] + [(i + 1, i, w) for i in range(n - 1)]
    return from_edges(n, edges)


def sources(n: int, k: int, seed: int = 5) -> np.ndarray:
    out = np.zeros(k, np.int32)
    _check(_L().gigen_sources(n, k, seed, out.ctypes.data), "sources")
    return out


def grid_heuristic(rows: int, cols: int, target: int, scale: int) -> np.ndarray:
    """A* input for a row-major rows x cols grid (id = r*cols + c): h(v) = scale x the
    Chebyshev distance from v to target. With scale <= the smallest edge weight it is
    admissible and consistent on 4-neighbour grids with diagonals (an edge changes the
    Chebyshev distance by at most 1). Coordinates only; no shortest-path arithmetic."""
    r = np.arange(rows * cols, dtype=np.int64) // cols
    c = np.arange(rows * cols, dtype=np.int64) % cols
    tr, tc = divmod(int(target), cols)
    h = np.maximum(np.abs(r - tr), np.abs(c - tc)) * int(scale)
    return np.minimum(h, 0xFFFFFFFE).astype(np.uint32)


def max_degree_vertex(g: CSR) -> int:
    """Highest out-degree vertex, ties -> smallest id."""
    return int(np.argmax(g.degrees()))


# ---- BASELINE.json configs --------------------------------------------

CONFIG_DELTAS = {
    1: [1000],
    2: [1 << k for k in range(10, 17)],
    3: [1, 2, 4, 8],
    4: [2],
    5: [1 << 13],
}


def config_graph(cfg: int) -> CSR:
    """The config's canonical graph. With GI_GEN_CACHE=<dir> set (measurement tools only),
    the CSR is kept there as .npy files and memory-mapped on later calls."""
    cache = os.environ.get("GI_GEN_CACHE")
    if cache:
        base = os.path.join(cache, f"cfg{2 if cfg == 5 else cfg}")
        names = ("offsets", "cols", "w")
        if all(os.path.exists(f"{base}_{k}.npy") for k in names):
            arrs = [np.load(f"{base}_{k}.npy", mmap_mode="r") for k in names]
            g = _config_graph(cfg, meta_only=True)
            return CSR(arrs[0], arrs[1], arrs[2], g.name, g.meta)
        g = _config_graph(cfg)
        os.makedirs(cache, exist_ok=True)
        for k in names:
            np.save(f"{base}_{k}.npy", getattr(g, k))
        return g
    return _config_graph(cfg)


_CONFIG_META = {
    1: ("cfg1_grid256", dict(kind="grid", rows=256, cols=256, w_lo=1, w_hi=1000, seed=1, p_del=0.0, p_diag=0.0)),
    2: ("cfg2_road4096", dict(kind="grid", rows=4096, cols=4096, w_lo=1, w_hi=10000, seed=2, p_del=0.05,
                              p_diag=0.01)),
    3: ("cfg3_rmat22", dict(kind="rmat", scale=22, edge_factor=16, w_lo=1, w_hi=22, seed=3)),
    4: ("cfg4_rmat26", dict(kind="rmat", scale=26, edge_factor=16, w_lo=1, w_hi=26, seed=4)),
}


def _config_graph(cfg: int, meta_only: bool = False) -> CSR:
    if meta_only:
        name, meta = _CONFIG_META[2 if cfg == 5 else cfg]
        e = np.zeros(0, np.int32)
        return CSR(np.zeros(1, np.int64), e, e.view(np.uint32), name, dict(meta))
    if cfg == 1:
        return grid(256, 256, 1, 1000, 1, name="cfg1_grid256")
    if cfg in (2, 5):
        return grid(4096, 4096, 1, 10000, 2, p_del=0.05, p_diag=0.01, name="cfg2_road4096")
    if cfg == 3:
        return rmat(22, 16, 1, 22, 3, name="cfg3_rmat22")
    if cfg == 4:
        return rmat(26, 16, 1, 26, 4, name="cfg4_rmat26")
    raise ValueError(cfg)


def config_source(cfg: int, g: CSR) -> int:
    if cfg == 1:
        return 0
    if cfg in (2, 5):
        return (4096 // 2) * 4096 + 4096 // 2  # centre = 8,390,656
    return max_degree_vertex(g)


def config_sources(cfg: int, g: CSR, k: int = 64) -> np.ndarray:
    if cfg == 5:
        return sources(g.n, k, 5)
    return np.array([config_source(cfg, g)], np.int32)


# ---- .wel loader and binary cache -----------------------------------------

def load_wel(path_: str, symmetrize: bool = False) -> CSR:
    """Weighted edge list: lines 'src dst weight'; '#' comments; optional '# n <count>'."""
    n_decl = None
    rows = []
    with open(path_) as f:
        for ln, line in enumerate(f, 1):
            s = line.strip()
            if not s:
                continue
            if s.startswith("#"):
                t = s[1:].split()
                if len(t) == 2 and t[0] == "n":
                    n_decl = int(t[1])
                continue
            t = s.split()
            if len(t) != 3:
                raise ValueError(f"parse error at line {ln}")
            try:
                u, v, w = int(t[0]), int(t[1]), int(t[2])
            except ValueError:
                raise ValueError(f"parse error at line {ln}") from None
            if u < 0 or v < 0:
                raise ValueError(f"parse error at line {ln}")
            if w < 0:
                raise ValueError(f"domain error (negative weight) at line {ln}")
            rows.append((u, v, w))
            if symmetrize:
                rows.append((v, u, w))
    mx = max((max(r[0], r[1]) for r in rows), default=-1) + 1
    n = max(n_decl or 0, mx, 1)
    return from_edges(n, rows)


def save_bin(g: CSR, path_: str) -> None:
    np.savez(path_, offsets=g.offsets, cols=g.cols, w=g.w)


def load_bin(path_: str) -> CSR:
    z = np.load(path_)
    return CSR(z["offsets"], z["cols"], z["w"], os.path.basename(path_), {})
