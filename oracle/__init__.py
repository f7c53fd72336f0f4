"""CPU oracle for Δ-stepping SSSP — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. It shares no code with the CUDA
path (``paper_1911_07260_b200/``); the only common dependency is the input module
``gen/`` (seeded graph generators, no method arithmetic).

Functions and what they follow:

* ``dijkstra`` — plain C binary-heap Dijkstra (oracle.c). The Δ-stepping result has a
  plain definition, the SSSP distance vector (§1), so
  the oracle is that definition computed by the textbook algorithm.
* ``bellman_ford`` — brute force, n-1 passes; pins ``dijkstra``.
* ``certificate`` — C0–C2 (north_star's "two invariants over every edge").
* ``bucket_count`` — closed form of the number of non-empty buckets processed: the number
  of distinct ⌊δ(v)/Δ⌋ over reached v (bucket i holds [iΔ,(i+1)Δ), PAPER.md:969;
  p' = ⌊p/Δ⌋).
* ``delta_stepping_lazy`` — pure-Python, step-by-step transcription of the paper's lazy
  Δ-stepping (Fig. alg:lazy_delta_stepping) for small graphs, reporting
  buckets / rounds / updates; pinned by the Bellman-Ford-vs-Δ-stepping "10 vs 7 updates"
  claim on the hand example Ex5.
* ``frontier_bellman_ford`` — pure-Python frontier Bellman-Ford (PAPER.md:157-161,
  :1555-1562) counting updates, for the same pin.
* ``kcore`` — coreness by the textbook serial min-degree peel (oracle.c; Matula & Beck,
  Batagelj & Zaversnik), the definition of; pinned by
  ``kcore_bruteforce`` (the k-core definition by repeated deletion, every k, tiny graphs)
  and closed forms (clique, cycle, star, path, full grid).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")

INF = 0xFFFFFFFF
OK, OVERFLOW, BAD_INPUT, NOMEM = 0, 1, -1, -2


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc). Building the checker is not using it."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", _SRC, "-o", _SO + ".tmp"])
        os.replace(_SO + ".tmp", _SO)
    return _SO


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        _lib.oracle_dijkstra.argtypes = [i64, vp, vp, vp, ctypes.c_int32, vp]
        _lib.oracle_dijkstra_budget.argtypes = [i64, vp, vp, vp, ctypes.c_int32, vp, ctypes.c_double,
                                                ctypes.POINTER(i64), ctypes.POINTER(i64)]
        _lib.oracle_bellman_ford.argtypes = [i64, vp, vp, vp, ctypes.c_int32, vp]
        _lib.oracle_transpose.argtypes = [i64, i64, vp, vp, vp, vp, vp, vp]
        _lib.oracle_certificate.argtypes = [i64, vp, vp, vp, vp, vp, vp, ctypes.c_int32, vp, vp]
        _lib.oracle_kcore.argtypes = [i64, vp, vp, vp]
        for f in ("oracle_dijkstra", "oracle_dijkstra_budget", "oracle_bellman_ford", "oracle_transpose", "oracle_certificate",
                  "oracle_kcore"):
            getattr(_lib, f).restype = ctypes.c_int
    return _lib


def _arrs(g):
    off = np.ascontiguousarray(g.offsets, dtype=np.int64)
    col = np.ascontiguousarray(g.cols, dtype=np.int32)
    w = np.ascontiguousarray(g.w, dtype=np.uint32)
    return off, col, w


def dijkstra(g, src: int):
    """Returns (dist uint32[n], status). status OVERFLOW if a finite δ >= UINT32_MAX."""
    off, col, w = _arrs(g)
    dist = np.empty(g.n, np.uint32)
    rc = _L().oracle_dijkstra(g.n, off.ctypes.data, col.ctypes.data, w.ctypes.data, int(src),
                              dist.ctypes.data)
    if rc < 0:
        raise ValueError(f"oracle_dijkstra rc={rc}")
    return dist, rc


def dijkstra_budget(g, src: int, budget_s: float):
    """Timing only (bench.py's bounded CPU baseline): the same Dijkstra, stopped after
    budget_s seconds of wall time. Returns (vertices settled, out-edges scanned, status)."""
    off, col, w = _arrs(g)
    dist = np.empty(g.n, np.uint32)
    settled, scanned = ctypes.c_int64(), ctypes.c_int64()
    rc = _L().oracle_dijkstra_budget(g.n, off.ctypes.data, col.ctypes.data, w.ctypes.data, int(src),
                                     dist.ctypes.data, float(budget_s) * 1e3, ctypes.byref(settled),
                                     ctypes.byref(scanned))
    return int(settled.value), int(scanned.value), rc


def bellman_ford(g, src: int):
    off, col, w = _arrs(g)
    dist = np.empty(g.n, np.uint32)
    rc = _L().oracle_bellman_ford(g.n, off.ctypes.data, col.ctypes.data, w.ctypes.data, int(src),
                                  dist.ctypes.data)
    if rc < 0:
        raise ValueError(f"oracle_bellman_ford rc={rc}")
    return dist, rc


def transpose(g):
    off, col, w = _arrs(g)
    toff = np.empty(g.n + 1, np.int64)
    tcol = np.empty(max(g.m, 1), np.int32)
    tw = np.empty(max(g.m, 1), np.uint32)
    rc = _L().oracle_transpose(g.n, g.m, off.ctypes.data, col.ctypes.data, w.ctypes.data,
                               toff.ctypes.data, tcol.ctypes.data, tw.ctypes.data)
    if rc != 0:
        raise ValueError(f"oracle_transpose rc={rc}")
    return toff, tcol[:g.m], tw[:g.m]


def certificate(g, src: int, dist, symmetric: bool = False):
    """(code, bad_vertex): code 0 = C0∧C1∧C2 hold; 1/2/3 = first failing check."""
    off, col, w = _arrs(g)
    if symmetric:
        toff, tcol, tw = off, col, w
    else:
        toff, tcol, tw = transpose(g)
    d = np.ascontiguousarray(dist, dtype=np.uint32)
    bad = ctypes.c_int64(-1)
    rc = _L().oracle_certificate(g.n, off.ctypes.data, col.ctypes.data, w.ctypes.data,
                                 toff.ctypes.data, tcol.ctypes.data, tw.ctypes.data, int(src),
                                 d.ctypes.data, ctypes.byref(bad))
    if rc < 0:
        raise ValueError(f"oracle_certificate rc={rc}")
    return rc, int(bad.value)


def dijkstra_many(g, srcs, threads: int | None = None):
    """One Dijkstra per source on a thread pool over host cores (ctypes drops the GIL).
    Returns (dist uint32[len(srcs), n], statuses, threads_used)."""
    srcs = [int(s) for s in srcs]
    threads = threads or os.cpu_count() or 1
    out = np.empty((len(srcs), g.n), np.uint32)
    off, col, w = _arrs(g)

    def one(i):
        return _L().oracle_dijkstra(g.n, off.ctypes.data, col.ctypes.data, w.ctypes.data, srcs[i],
                                    out[i].ctypes.data)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        rcs = list(ex.map(one, range(len(srcs))))
    return out, rcs, threads


def bucket_count(dist, delta: int) -> int:
    """Closed form: number of distinct ⌊δ(v)/Δ⌋ over reached v."""
    d = np.asarray(dist, dtype=np.uint64)
    d = d[d != INF]
    return int(np.unique(d // np.uint64(delta)).size)


def checksum(dist) -> int:
    """Σ_v dist[v]·(v+1) mod 2^64 (SURVEY §8(d) fingerprint; unreached counts as 2^32-1)."""
    d = np.asarray(dist, dtype=np.uint64)
    v = np.arange(1, d.size + 1, dtype=np.uint64)
    return int(np.sum(d * v, dtype=np.uint64))


# ---- pure-Python small-graph transcriptions (paper order) ---------------------------------

def delta_stepping_lazy(g, src: int, delta: int):
    """Fig. alg:lazy_delta_stepping, one step per pseudocode line.

    * Dist = {inf}; B = LazyBucket(Dist, Δ, startV); Dist[startV] = 0   (l.413-416)
    * while B non-empty: minBucket = B.getMinBucket()                   (l.417-418)
    *   for src in minBucket, for e in out-edges:                      (l.420-421)
    *     Dist[dst] = min(Dist[dst], Dist[src] + w)                    (l.422)
    *     buffer.syncAppend(dst, ⌊Dist[dst]/Δ⌋)  — only when Dist[dst] changed: the
    *       generated code appends only on a priority change (tracking var)
    *   buffer.reduceBucketUpdates() — one final update per vertex     (l.427, :446)
    *   B.bulkUpdateBuckets(buffer)                                    (l.428)
    The parallel-for is executed sequentially in vertex-id order (a valid schedule).
    Returns dict(dist, buckets, rounds, updates). Small graphs only.
    """
    n = g.n
    off, col, w = g.offsets, g.cols, g.w
    dist = [INF] * n
    dist[src] = 0
    bucket_of = {src: 0}               # vertex -> bucket id (live membership)
    buckets = {0: {src}}
    rounds = updates = 0
    seen_buckets = set()
    while buckets:
        b = min(buckets)
        min_bucket = sorted(buckets.pop(b))
        for v in min_bucket:
            del bucket_of[v]
        seen_buckets.add(b)
        rounds += 1
        buffer = []
        for s in min_bucket:
            for e in range(int(off[s]), int(off[s + 1])):
                d = int(col[e])
                nd = dist[s] + int(w[e])
                if nd < dist[d]:
                    dist[d] = nd
                    updates += 1
                    buffer.append((d, nd // delta))
        reduced = {}
        for d, bk in buffer:             # reduceBucketUpdates: keep the final (smallest) bucket
            reduced[d] = min(bk, reduced.get(d, bk))
        for d, bk in reduced.items():   # bulkUpdateBuckets
            old = bucket_of.get(d)
            if old is not None:
                buckets[old].discard(d)
                if not buckets[old]:
                    del buckets[old]
            bucket_of[d] = bk
            buckets.setdefault(bk, set()).add(d)
    out = np.array([x if x < INF else INF for x in dist], dtype=np.uint64)
    if np.any((out >= INF) & (out != INF)):
        raise OverflowError("distance not representable in uint32")
    return dict(dist=out.astype(np.uint32), buckets=len(seen_buckets), rounds=rounds, updates=updates)


def frontier_bellman_ford(g, src: int):
    """Frontier Bellman-Ford: each round relaxes the out-edges
    of every vertex updated in the previous round, reading distances at the round start.
    Returns dict(dist, rounds, updates)."""
    n = g.n
    off, col, w = g.offsets, g.cols, g.w
    dist = [INF] * n
    dist[src] = 0
    frontier = [src]
    rounds = updates = 0
    while frontier:
        rounds += 1
        snap = list(dist)
        nxt = set()
        for s in frontier:
            for e in range(int(off[s]), int(off[s + 1])):
                d = int(col[e])
                nd = snap[s] + int(w[e])
                if nd < dist[d]:
                    dist[d] = nd
                    updates += 1
                    nxt.add(d)
        frontier = sorted(nxt)
    return dict(dist=np.array(dist, dtype=np.uint64), rounds=rounds, updates=updates)


def kcore(g):
    """Coreness of every vertex (uint32[n]) by the serial min-degree peel (oracle.c)."""
    off, col, _ = _arrs(g)
    core = np.zeros(g.n, np.uint32)
    rc = _L().oracle_kcore(g.n, off.ctypes.data, col.ctypes.data, core.ctypes.data)
    if rc != 0:
        raise ValueError(f"oracle_kcore rc={rc}")
    return core


def kcore_bruteforce(g):
    """The definition, for tiny graphs: for each k, delete vertices whose degree inside the
    remaining set is < k until none is left to delete (the k-core); coreness[v] = the
    largest k whose k-core contains v. Degrees count CSR entries."""
    off = np.asarray(g.offsets)
    col = np.asarray(g.cols)
    n = g.n
    core = np.zeros(n, np.uint32)
    maxdeg = int(np.diff(off).max(initial=0))
    for k in range(1, maxdeg + 1):
        alive = np.ones(n, bool)
        changed = True
        while changed:
            changed = False
            for v in range(n):
                if alive[v] and sum(1 for e in range(off[v], off[v + 1]) if alive[col[e]]) < k:
                    alive[v] = False
                    changed = True
        core[alive] = k
    return core
