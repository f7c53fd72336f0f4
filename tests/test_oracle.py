"""Pins for the CPU oracle (oracle/) against things other than itself.

* hand-worked examples (tests/golden/hand_examples.json, each with its citation);
* the paper's "Bellman-Ford needs 10 updates, whereas Δ-stepping needs only 7"
   on Ex5;
* brute-force Bellman-Ford on tiny graphs, every source;
* scipy.sparse.csgraph.dijkstra (independent library routine);
* closed forms: Manhattan distances on a uniform-weight grid, the path graph;
* the certificate accepting the truth and rejecting corruptions.
"""
import json
import os

import numpy as np
import pytest

import gen
import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "hand_examples.json")))["examples"]
INF = oracle.INF


def _graph(ex):
    return gen.from_edges(ex["n"], ex["edges"])


@pytest.mark.parametrize("ex", GOLDEN, ids=[e["name"] for e in GOLDEN])
def test_hand_examples(ex):
    g = _graph(ex)
    d, rc = oracle.dijkstra(g, ex["src"])
    bf, rc_bf = oracle.bellman_ford(g, ex["src"])
    if ex.get("status") == "overflow":
        assert rc == oracle.OVERFLOW and rc_bf == oracle.OVERFLOW
        return
    assert rc == oracle.OK and rc_bf == oracle.OK
    assert d.tolist() == ex["dist"]
    assert bf.tolist() == ex["dist"]
    assert oracle.bucket_count(d, ex["delta"]) == ex["buckets"]
    lz = oracle.delta_stepping_lazy(g, ex["src"], ex["delta"])
    assert lz["dist"].tolist() == ex["dist"]
    assert lz["buckets"] == ex["buckets"]


def test_paper_updates_10_vs_7():
    """PAPER.md:1551 (fig:delta_stepping_demo caption): BF 10 updates, Δ-stepping (Δ=30) 7."""
    ex = next(e for e in GOLDEN if e["name"].startswith("Ex5"))
    g = _graph(ex)
    assert oracle.frontier_bellman_ford(g, 0)["updates"] == 10
    assert oracle.delta_stepping_lazy(g, 0, 30)["updates"] == 7


def test_spec_corpus_dijkstra_equals_bellman_ford_all_sources():
    """SPEC.md:508 corpus shape (uniform_random n=64, m=512, [1,1000)); every source."""
    for seed in range(100):
        g = gen.uniform_random(64, 512, 1, 1000, seed)
        for s in range(64):
            d, rc = oracle.dijkstra(g, s)
            b, rcb = oracle.bellman_ford(g, s)
            assert rc == rcb == 0
            assert np.array_equal(d, b), (seed, s)


def test_brute_force_tiny_with_zero_weights_and_loops():
    rng = np.random.default_rng(1)
    for t in range(200):
        n = int(rng.integers(1, 9))
        m = int(rng.integers(0, 20))
        edges = [(int(rng.integers(0, n)), int(rng.integers(0, n)), int(rng.integers(0, 4))) for _ in range(m)]
        g = gen.from_edges(n, edges)
        for s in range(n):
            d, _ = oracle.dijkstra(g, s)
            b, _ = oracle.bellman_ford(g, s)
            assert np.array_equal(d, b)
            # paper-order lazy Δ-stepping reaches the same fixed point for any Δ
            for delta in (1, 2, 5, 1000):
                assert np.array_equal(oracle.delta_stepping_lazy(g, s, delta)["dist"], d)


def _scipy_dist(g, src):
    import scipy.sparse as sp
    from scipy.sparse.csgraph import dijkstra as sdij
    # scipy treats explicit zeros as missing edges; corpora here have w >= 1
    A = sp.csr_matrix((g.w.astype(np.float64), g.cols, g.offsets), shape=(g.n, g.n))
    d = sdij(A, directed=True, indices=src)
    out = np.where(np.isinf(d), INF, d).astype(np.uint64)
    return out.astype(np.uint32)


def test_scipy_cross_check_uniform_and_grid():
    for seed in range(10):
        g = gen.uniform_random(200, 1500, 1, 1000, 100 + seed)
        for s in (0, 17, 199):
            assert np.array_equal(oracle.dijkstra(g, s)[0], _scipy_dist(g, s))
    g = gen.grid(40, 50, 1, 10000, 5, p_del=0.1, p_diag=0.05)
    assert np.array_equal(oracle.dijkstra(g, 123)[0], _scipy_dist(g, 123))


def test_config1_scipy_and_fingerprint(config_graph):
    g = config_graph(1)
    d, rc = oracle.dijkstra(g, 0)
    assert rc == 0
    assert np.array_equal(d, _scipy_dist(g, 0))
    # SURVEY §8(d) fingerprints (scipy-computed there)
    assert int(d.max()) == 117722
    assert int(d.astype(np.uint64).sum()) == 4250305769
    assert oracle.checksum(d) == 160211844129846
    for delta, b in ((250, 470), (500, 236), (1000, 118), (2000, 59), (4000, 30)):
        assert oracle.bucket_count(d, delta) == b
    assert oracle.certificate(g, 0, d, symmetric=True)[0] == 0


@pytest.mark.slow
def test_config2_fingerprint(config_graph):
    g = config_graph(2)
    d, rc = oracle.dijkstra(g, 8390656)
    assert rc == 0
    reached = d != INF
    assert int(reached.sum()) == 16777113
    assert int(d[reached].max()) == 9804213
    assert int(d[reached].astype(np.uint64).sum()) == 88054548793581
    assert oracle.checksum(d) == 3787979249957408387
    exp = [9562, 4785, 2394, 1197, 599, 300, 150]
    assert [oracle.bucket_count(d, 1 << k) for k in range(10, 17)] == exp


@pytest.mark.slow
def test_config3_fingerprint(config_graph):
    g = config_graph(3)
    d, rc = oracle.dijkstra(g, 0)
    assert rc == 0
    reached = d != INF
    assert int(reached.sum()) == 2394029
    assert int(d[reached].max()) == 56
    assert int(d[reached].astype(np.uint64).sum()) == 17886599
    assert oracle.checksum(d) == 8744335342905669924
    assert [oracle.bucket_count(d, k) for k in (1, 2, 4, 8)] == [49, 25, 13, 7]


def test_closed_form_uniform_grid_manhattan():
    """Uniform weight w0 on a 4-neighbour grid: δ = w0·(|r-rs|+|c-cs|)."""
    R = C = 64
    g = gen.grid(R, C, 3, 4, 0)  # all weights 3
    assert np.all(g.w == 3)
    s = 32 * C + 32
    d, _ = oracle.dijkstra(g, s)
    r, c = np.divmod(np.arange(R * C), C)
    assert np.array_equal(d.astype(np.int64), 3 * (np.abs(r - 32) + np.abs(c - 32)))
    assert [oracle.bucket_count(d, x) for x in (1, 3, 7, 100)] == [65, 65, 28, 2]


def test_closed_form_path():
    """Path, unit weights, source 0: dist[i] = i; buckets = ⌈n/Δ⌉; paper-order lazy
    Δ-stepping takes exactly n BSP rounds (one vertex per round)."""
    for n, delta in ((1000, 100), (257, 16), (50, 1), (10, 1000)):
        g = gen.path(n)
        d, _ = oracle.dijkstra(g, 0)
        assert d.tolist() == list(range(n))
        assert oracle.bucket_count(d, delta) == -(-n // delta)
        lz = oracle.delta_stepping_lazy(g, 0, delta)
        assert lz["rounds"] == n and lz["buckets"] == -(-n // delta)


def test_certificate_rejects_corruptions(config_graph):
    g = config_graph(1)
    d, _ = oracle.dijkstra(g, 0)
    rng = np.random.default_rng(0)
    for t in range(60):
        v = int(rng.integers(1, g.n))
        bad = d.copy()
        delta = [1, -1, 7, -7, 1000][t % 5]
        bad[v] = np.uint32(int(bad[v]) + delta)
        assert oracle.certificate(g, 0, bad, symmetric=True)[0] in (2, 3)
    bad = d.copy(); bad[5] = INF
    assert oracle.certificate(g, 0, bad, symmetric=True)[0] in (2, 3)
    bad = d.copy(); bad[0] = 1
    assert oracle.certificate(g, 0, bad, symmetric=True)[0] == 1


def test_certificate_directed_uses_transpose():
    g = gen.uniform_random(64, 512, 1, 1000, 3)
    d, _ = oracle.dijkstra(g, 0)
    assert oracle.certificate(g, 0, d)[0] == 0
    bad = d.copy()
    v = int(np.argmax(np.where(d != INF, d, 0)))
    bad[v] += 1
    assert oracle.certificate(g, 0, bad)[0] in (2, 3)


def test_dijkstra_many_threads():
    g = gen.grid(30, 30, 1, 100, 1)
    srcs = [0, 5, 899, 450]
    out, rcs, th = oracle.dijkstra_many(g, srcs, threads=3)
    assert th == 3 and rcs == [0] * 4
    for i, s in enumerate(srcs):
        assert np.array_equal(out[i], oracle.dijkstra(g, s)[0])
    # symmetric graph: δ(si, sj) == δ(sj, si) (SURVEY §8c c4 batch symmetry)
    for i, a in enumerate(srcs):
        for j, b in enumerate(srcs):
            assert out[i][b] == out[j][a]


# ---- k-core oracle pins ----

def _sym(n, und):
    edges = []
    for u, v in und:
        edges += [(u, v, 1), (v, u, 1)]
    return gen.from_edges(n, edges)


def test_kcore_closed_forms():
    tri = _sym(3, [(0, 1), (1, 2), (0, 2)])
    assert oracle.kcore(tri).tolist() == [2, 2, 2]
    star = _sym(5, [(0, i) for i in range(1, 5)])
    assert oracle.kcore(star).tolist() == [1] * 5
    for n in (1, 2, 5, 9):
        k = _sym(n, [(i, j) for i in range(n) for j in range(i + 1, n)])
        assert oracle.kcore(k).tolist() == [n - 1] * n  # clique K_n
    cyc = _sym(7, [(i, (i + 1) % 7) for i in range(7)])
    assert oracle.kcore(cyc).tolist() == [2] * 7
    path = _sym(6, [(i, i + 1) for i in range(5)])
    assert oracle.kcore(path).tolist() == [1] * 6
    grid = gen.grid(20, 30, 1, 2, 0)  # full 4-neighbour grid: its 2-core is everything, no 3-core
    assert set(oracle.kcore(grid).tolist()) == {2}
    iso = gen.from_edges(4, [])
    assert oracle.kcore(iso).tolist() == [0] * 4
    # two cliques K5 and K3 joined by a bridge: 4 on the K5, 2 on the K3
    und = [(i, j) for i in range(5) for j in range(i + 1, 5)] + [(5, 6), (6, 7), (5, 7), (4, 5)]
    assert oracle.kcore(_sym(8, und)).tolist() == [4] * 5 + [2] * 3


def test_kcore_matches_definition_bruteforce():
    rng = np.random.default_rng(5)
    for t in range(60):
        n = int(rng.integers(1, 30))
        und = [(int(rng.integers(0, n)), int(rng.integers(0, n))) for _ in range(int(rng.integers(0, 4 * n)))]
        g = _sym(n, und)  # includes parallel edges and self-loops (a self-loop stores 2 entries)
        assert np.array_equal(oracle.kcore(g), oracle.kcore_bruteforce(g)), t
    g = gen.uniform_random(64, 512, 1, 2, 7)  # SPEC.md:370 corpus shape, symmetrised
    src = np.repeat(np.arange(g.n), np.diff(g.offsets))
    und = list(zip(src.tolist(), g.cols.tolist()))
    s = _sym(64, und)
    assert np.array_equal(oracle.kcore(s), oracle.kcore_bruteforce(s))


def test_dijkstra_budget_is_the_same_loop():
    """The bounded-sample entry point (bench.py's CPU baseline) with no budget settles every
    reached vertex once and scans exactly their out-edges; its distances equal dijkstra's."""
    g = gen.grid(40, 40, 1, 100, 3, p_del=0.2)
    ref, _ = oracle.dijkstra(g, 5)
    settled, scanned, rc = oracle.dijkstra_budget(g, 5, 0.0)
    reached = ref != oracle.INF
    assert rc == 0 and settled == int(reached.sum())
    assert scanned == int(np.diff(g.offsets)[reached].sum())
    s2, e2, _ = oracle.dijkstra_budget(g, 5, 1e-9)  # a budget stops early but never before one pop
    assert 1 <= s2 <= settled and e2 <= scanned
