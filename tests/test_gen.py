"""Input generators (gen/): recipe fingerprints, determinism, CSR invariants, loaders.

Fingerprints are SURVEY.md §8(d) "Fingerprints of this exact recipe" (computed there
from an independent numpy implementation of the same recipe).
"""
import numpy as np
import pytest

import gen


def _check_csr(g, symmetric):
    off, cols, w = g.offsets, g.cols, g.w
    assert off[0] == 0 and off[-1] == g.m
    assert np.all(np.diff(off) >= 0)
    assert g.m == 0 or (cols.min() >= 0 and cols.max() < g.n)
    # rows sorted ascending, no duplicates (canonical)
    for v in range(min(g.n, 2000)):
        r = cols[off[v]:off[v + 1]]
        assert np.all(np.diff(r) > 0)
    if symmetric:
        # (u,v,w) present <=> (v,u,w) present
        u = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(off))
        a = np.stack([u, cols.astype(np.int64), w.astype(np.int64)], 1)
        b = np.stack([cols.astype(np.int64), u, w.astype(np.int64)], 1)
        a = a[np.lexsort(a.T[::-1])]
        b = b[np.lexsort(b.T[::-1])]
        assert np.array_equal(a, b)


def test_mix64_splitmix_reference_values():
    # SplitMix64 finalizer (Steele, Lea & Flood 2014) on 0 is 0; on 1 it is the
    # well-known constant below (first output of splitmix64 seeded with
    # 1 - 0x9E3779B97F4A7C15, i.e. finalizer(1)).
    assert gen.mix64(0) == 0
    z = 1
    z ^= z >> 30; z = (z * 0xBF58476D1CE4E5B9) & (2**64 - 1)
    z ^= z >> 27; z = (z * 0x94D049BB133111EB) & (2**64 - 1)
    z ^= z >> 31
    assert gen.mix64(1) == z


def test_bernoulli_thresholds():
    assert gen.bernoulli_threshold(0.05) == 214748364
    assert gen.bernoulli_threshold(0.01) == 42949672
    assert gen.RMAT_T == (int(0.57 * 2**32), int(0.76 * 2**32), int(0.95 * 2**32))


def test_config1_fingerprint(config_graph):
    g = config_graph(1)
    assert (g.n, g.m) == (65536, 261120)
    assert int(g.w.astype(np.uint64).sum()) == 130761856
    deg = g.degrees()
    assert (deg == 2).sum() == 4 and (deg == 3).sum() == 1016 and (deg == 4).sum() == 64516
    assert g.w.min() >= 1 and g.w.max() < 1000
    _check_csr(g, symmetric=True)


@pytest.mark.slow
def test_config2_fingerprint(config_graph):
    g = config_graph(2)
    assert (g.n, g.m) == (16777216, 64407462)
    assert int(g.w.astype(np.uint64).sum()) == 322056043522
    assert int((g.degrees() == 0).sum()) == 103
    assert g.degrees().max() <= 8
    assert gen.config_source(2, g) == 8390656
    s = gen.config_sources(5, g)
    assert list(s[:8]) == [4199085, 1879102, 11836061, 3746776, 4627827, 5576377, 9660751, 11448549]
    assert int(s.astype(np.int64).sum()) == 579338766 and s.min() == 159028 and s.max() == 16760123
    assert len(set(s.tolist())) == 64


@pytest.mark.slow
def test_config3_fingerprint(config_graph):
    g = config_graph(3)
    assert (g.n, g.m) == (4194304, 128308946)
    assert int(g.w.astype(np.uint64).sum()) == 1411516956
    deg = g.degrees()
    assert int((deg == 0).sum()) == 1798755
    assert int(deg.max()) == 163329 and gen.config_source(3, g) == 0
    assert g.w.min() >= 1 and g.w.max() < 22


def test_determinism_and_symmetry_small():
    a = gen.grid(37, 53, 1, 100, 9, p_del=0.2, p_diag=0.3)
    b = gen.grid(37, 53, 1, 100, 9, p_del=0.2, p_diag=0.3)
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.cols, b.cols) and np.array_equal(a.w, b.w)
    _check_csr(a, symmetric=True)
    r = gen.rmat(10, 8, 1, 10, 11)
    _check_csr(r, symmetric=True)
    assert not np.any(r.cols == np.repeat(np.arange(r.n), r.degrees()))  # no self-loops


def test_uniform_random_determinism():
    a = gen.uniform_random(64, 512, 1, 1000, 7)
    b = gen.uniform_random(64, 512, 1, 1000, 7)
    assert a.m == 512 and np.array_equal(a.cols, b.cols) and np.array_equal(a.w, b.w)
    u = np.repeat(np.arange(64), a.degrees())
    assert not np.any(u == a.cols)  # self-loops rejected


def test_path_and_grid_spec_examples():
    p = gen.path(3)
    assert p.m == 4 and list(p.cols) == [1, 0, 2, 1]
    g = gen.grid(2, 2, 1, 2, 0)
    assert g.m == 8  # SPEC.md: grid(2,2) -> 8 directed edges


def test_wel_loader(tmp_path):
    f = tmp_path / "a.wel"
    f.write_text("# comment\n0 1 5\n1 2 3\n")
    g = gen.load_wel(str(f))
    assert (g.n, g.m) == (3, 2) and list(g.cols[g.offsets[0]:g.offsets[1]]) == [1]
    gs = gen.load_wel(str(f), symmetrize=True)
    assert gs.m == 4
    r = gs.offsets[1], gs.offsets[2]
    assert sorted(zip(gs.cols[r[0]:r[1]].tolist(), gs.w[r[0]:r[1]].tolist())) == [(0, 5), (2, 3)]
    bad = tmp_path / "b.wel"
    bad.write_text("0 -1 5\n")
    with pytest.raises(ValueError, match="line 1"):
        gen.load_wel(str(bad))


def test_bin_cache_roundtrip(tmp_path):
    g = gen.grid(9, 7, 1, 50, 3)
    p = str(tmp_path / "g.npz")
    gen.save_bin(g, p)
    h = gen.load_bin(p)
    assert np.array_equal(g.offsets, h.offsets) and np.array_equal(g.cols, h.cols) and np.array_equal(g.w, h.w)


def test_grid_heuristic_admissible_and_consistent():
    """A* input: w_min x Chebyshev distance on the road-like grid recipe
    (deletions + diagonals) never exceeds the true remaining distance (admissible, checked
    against the Dijkstra oracle from the target on the symmetric graph) and drops by at most
    w(u,v) along every edge (consistent)."""
    import oracle
    rows, cols = 48, 40
    g = gen.grid(rows, cols, 3, 50, 9, p_del=0.05, p_diag=0.2)
    t = 17 * cols + 23
    h = gen.grid_heuristic(rows, cols, t, 3).astype(np.int64)
    assert h[t] == 0
    d, rc = oracle.dijkstra(g, t)
    reach = d != 0xFFFFFFFF
    assert np.all(h[reach] <= d[reach].astype(np.int64))
    src = np.repeat(np.arange(g.n), np.diff(g.offsets))
    assert np.all(h[src] <= g.w.astype(np.int64) + h[g.cols])
