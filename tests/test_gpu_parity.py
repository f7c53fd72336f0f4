"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, element by element.

Bar (north_star): bit-exact uint32 distances for every vertex, unreached = UINT32_MAX.
Counters are checked only where a closed form pins them.
"""
import json
import os

import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "hand_examples.json")))["examples"]
INF = 0xFFFFFFFF


@pytest.fixture(scope="module")
def gi():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1911_07260_b200 import _build
    _build.build_lib()
    from paper_1911_07260_b200 import gi as m
    return m


def run(gi, G, src, delta, **opts):
    d, st = gi.sssp(G, src, delta, **opts)
    return gi.as_uint32(d), st


# drain: default bsp (CTA barrier per sub-round); "async" = barrier-free ring (out-degree <= 8)
OPTS = [dict(fusion=True), dict(fusion=False), dict(fusion=True, threshold=2),
        dict(fusion=True, drain="async"), dict(fusion=True, drain="async", threshold=2),
        dict(fusion=True, max_ctas=1), dict(fusion=True, max_ctas=1, drain="async"),
        dict(fusion=False, max_ctas=3), dict(fusion=True, threshold=1, max_ctas=5),
        dict(fusion=True, pre_read=1), dict(fusion=False, pre_read=2)]


@pytest.mark.parametrize("ex", GOLDEN, ids=[e["name"] for e in GOLDEN])
def test_hand_examples(gi, ex):
    g = gen.from_edges(ex["n"], ex["edges"])
    G = gi.Graph.from_csr(g)
    for o in OPTS:
        if ex.get("status") == "overflow":
            with pytest.raises(gi.OverflowDistance):
                run(gi, G, ex["src"], ex["delta"], **o)
            continue
        d, st = run(gi, G, ex["src"], ex["delta"], **o)
        assert d.tolist() == ex["dist"], o
        assert st["buckets"] == ex["buckets"], (o, st)


def test_spec_corpus(gi):
    """SPEC.md:508 acceptance corpus: 100 uniform_random graphs n=64, m=512, [1,1000), 3 sources."""
    for seed in range(100):
        g = gen.uniform_random(64, 512, 1, 1000, seed)
        G = gi.Graph.from_csr(g)
        for s in (0, 31, 63):
            ref, _ = oracle.dijkstra(g, s)
            for o, delta in ((dict(fusion=True), 100), (dict(fusion=False), 100), (dict(fusion=True), 1),
                             (dict(fusion=True, threshold=4), 2000)):
                d, _ = run(gi, G, s, delta, **o)
                assert np.array_equal(d, ref), (seed, s, o, delta)


def test_random_small_with_zero_weights_multi_edges(gi):
    rng = np.random.default_rng(7)
    for t in range(60):
        n = int(rng.integers(1, 300))
        m = int(rng.integers(0, 2000))
        edges = [(int(rng.integers(0, n)), int(rng.integers(0, n)), int(rng.integers(0, 50))) for _ in range(m)]
        g = gen.from_edges(n, edges)
        G = gi.Graph.from_csr(g)
        s = int(rng.integers(0, n))
        ref, _ = oracle.dijkstra(g, s)
        for delta in (1, 7, 10**6):
            d, _ = run(gi, G, s, delta, fusion=bool(t % 2), max_ctas=int(rng.integers(1, 40)))
            assert np.array_equal(d, ref), (t, delta)


def test_config1_delta_sweep(gi, config_graph):
    g = config_graph(1)
    G = gi.Graph.from_csr(g)
    ref, _ = oracle.dijkstra(g, 0)
    for delta in (250, 500, 1000, 2000, 4000, 1, 10**9):
        for o in OPTS:
            d, st = run(gi, G, 0, delta, **o)
            assert np.array_equal(d, ref), (delta, o)
            assert st["buckets"] == oracle.bucket_count(ref, delta), (delta, o, st)


def test_host_output_buffer(gi, config_graph):
    g = config_graph(1)
    G = gi.Graph.from_csr(g)
    out = np.zeros(g.n, np.uint32)
    gi.gi_sssp_delta(G, 0, 1000, out)
    assert np.array_equal(out, oracle.dijkstra(g, 0)[0])
    srcs = np.array([5, 700, 65535, 5], np.int32)
    outb = np.zeros((4, g.n), np.uint32)
    gi.gi_sssp_batch(G, srcs, 1000, outb)
    assert np.array_equal(outb, oracle.dijkstra_many(g, srcs)[0])


def test_device_csr_input(gi, config_graph):
    import torch
    g = config_graph(1)
    G = gi.Graph(torch.from_numpy(g.offsets).cuda(), torch.from_numpy(g.cols).cuda(),
                 torch.from_numpy(g.w.view(np.int32)).cuda())
    d, _ = run(gi, G, 0, 1000)
    assert np.array_equal(d, oracle.dijkstra(g, 0)[0])


def test_path_closed_form_rounds(gi):
    """Path, unit weights: rounds without fusion = n; with fusion = ⌈n/Δ⌉ = buckets."""
    for n, delta in ((1000, 100), (4096, 1024), (300, 1)):
        g = gen.path(n)
        G = gi.Graph.from_csr(g)
        d, st = run(gi, G, 0, delta, fusion=False)
        assert d.tolist() == list(range(n))
        assert st["rounds"] == n and st["buckets"] == -(-n // delta)
        d, st = run(gi, G, 0, delta, fusion=True)
        assert d.tolist() == list(range(n))
        assert st["rounds"] == -(-n // delta) == st["buckets"], st
        assert st["spills"] == 0


def test_lazy_schedule(gi, config_graph):
    """The fully lazy schedule (gi_options.lazy, Fig. alg:lazy_delta_stepping):
    exact distances; path closed form (rounds = n, buckets = ⌈n/Δ⌉, the round counts of the
    oracle's step-by-step transcription); Δ <= w_min gives one round per bucket; a skewed graph
    and a road grid; lazy with fusion is an argument error."""
    for n, delta in ((1000, 100), (257, 1)):
        g = gen.path(n)
        G = gi.Graph.from_csr(g)
        d, st = run(gi, G, 0, delta, fusion=False, lazy=True)
        lz = oracle.delta_stepping_lazy(g, 0, delta)
        assert d.tolist() == list(range(n))
        assert st["rounds"] == n == lz["rounds"] and st["buckets"] == -(-n // delta) == lz["buckets"], st
    g = gen.grid(48, 48, 3, 40, 5)  # w >= 3
    G = gi.Graph.from_csr(g)
    ref, _ = oracle.dijkstra(g, 0)
    for delta in (1, 3):
        d, st = run(gi, G, 0, delta, fusion=False, lazy=True)
        assert np.array_equal(d, ref)
        assert st["rounds"] == st["buckets"] == oracle.bucket_count(ref, delta), st
    rng = np.random.default_rng(17)
    for t in range(8):
        n = int(rng.integers(50, 4000))
        m = int(rng.integers(n, 8 * n))
        g = gen.uniform_random(n, m, 0 if t % 2 else 1, int(rng.choice([5, 1000])), 40 + t)
        G = gi.Graph.from_csr(g)
        s = int(rng.integers(0, n))
        ref, _ = oracle.dijkstra(g, s)
        for delta in (1, 7, 1 << 20):
            for o in (dict(), dict(max_ctas=3), dict(pre_read=1)):
                d, st = run(gi, G, s, delta, fusion=False, lazy=True, **o)
                assert np.array_equal(d, ref), (t, delta, o)
                assert st["buckets"] == oracle.bucket_count(ref, delta) and st["rounds"] >= st["buckets"]
    g = config_graph(1)
    G = gi.Graph.from_csr(g)
    ref, _ = oracle.dijkstra(g, 0)
    d, st = run(gi, G, 0, 1000, fusion=False, lazy=True)
    assert np.array_equal(d, ref) and st["buckets"] == oracle.bucket_count(ref, 1000)
    with pytest.raises(gi.GiError):
        run(gi, G, 0, 1000, fusion=True, lazy=True)


def test_execution_group_rungs(gi, config_graph):
    """The execution-group ladder: one CTA per group (CTA barrier), one
    thread-block cluster per group (hardware cluster barrier; 2..16 CTAs) and the grid give
    the same exact distances, single and batch, fused / unfused / lazy / async drain; the
    rung is reported."""
    rng = np.random.default_rng(5)
    graphs = [config_graph(1), gen.from_edges(1, []),
              gen.uniform_random(3000, 20000, 0, 50, 9)]
    for g in graphs:
        G = gi.Graph.from_csr(g)
        s = 0 if g.n < 3 else int(rng.integers(0, g.n))
        ref, _ = oracle.dijkstra(g, s)
        for o, want in ((dict(rung="cta"), 1), (dict(rung="cluster", group_ctas=2), 2),
                        (dict(rung="cluster"), 2), (dict(rung="cluster", group_ctas=16), 2),
                        (dict(rung="grid"), 3), (dict(rung="cta", fusion=False), 1),
                        (dict(rung="cluster", group_ctas=4, fusion=False, lazy=True), 2),
                        (dict(rung="cta", threshold=1), 1)):
            for delta in (7, 1000):
                d, st = run(gi, G, s, delta, **o)
                assert np.array_equal(d, ref), (g.n, o, delta)
                assert st["rung"] == want and st["buckets"] == oracle.bucket_count(ref, delta)
        if g.n > 100:
            srcs = rng.integers(0, g.n, 13).astype(np.int32)
            refs, _, _ = oracle.dijkstra_many(g, srcs)
            for o in (dict(rung="cta"), dict(rung="cluster", group_ctas=4), dict(rung="grid")):
                out, sts = gi.sssp_batch(G, srcs, 100, **o)
                assert np.array_equal(gi.as_uint32(out), refs), o
    g = config_graph(1)
    if max(np.diff(g.offsets)) <= 8:
        G = gi.Graph.from_csr(g)
        ref, _ = oracle.dijkstra(g, 0)
        d, st = run(gi, G, 0, 1000, rung="cluster", drain="async")
        assert np.array_equal(d, ref) and st["rung"] == 2


def test_delta_le_wmin_processes_each_vertex_once(gi):
    """Δ <= w_min: every reached vertex is processed exactly once."""
    g = gen.grid(64, 64, 3, 4, 0)
    G = gi.Graph.from_csr(g)
    s = 32 * 64 + 32
    for delta in (1, 3):
        for fusion in (True, False):
            d, st = run(gi, G, s, delta, fusion=fusion)
            assert np.array_equal(d, oracle.dijkstra(g, s)[0])
            assert st["vertices_processed"] == g.n and st["edges_relaxed"] == g.m


def test_errors(gi):
    g = gen.path(5)
    G = gi.Graph.from_csr(g)
    with pytest.raises(gi.GiError) as e:
        run(gi, G, 5, 1)
    assert e.value.status == 2
    with pytest.raises(gi.GiError) as e:
        run(gi, G, -1, 1)
    assert e.value.status == 2
    with pytest.raises(gi.GiError) as e:
        run(gi, G, 0, 0)
    assert e.value.status == 1
    bad_off = np.array([0, 2, 1, 3], np.int64)
    with pytest.raises(gi.GiError) as e:
        gi.Graph(bad_off, np.zeros(3, np.int32), np.ones(3, np.uint32))
    assert e.value.status == 3
    with pytest.raises(gi.GiError) as e:
        gi.Graph(np.array([0, 1], np.int64), np.array([1], np.int32), np.ones(1, np.uint32))
    assert e.value.status == 3
    with pytest.raises(gi.GiError) as e:
        gi.Graph(np.array([0, 1, 3], np.int64), np.zeros(2, np.int32), np.ones(2, np.uint32))
    assert e.value.status == 3
    # nsrc = 0 is a no-op
    import torch
    out = torch.empty((0, 5), dtype=torch.int32, device="cuda")
    gi.gi_sssp_batch(G, np.zeros(0, np.int32), 1, out)


@pytest.mark.slow
def test_config2_full(gi, config_graph):
    g = config_graph(2)
    G = gi.Graph.from_csr(g)
    src = gen.config_source(2, g)
    ref, _ = oracle.dijkstra(g, src)
    for delta, o in ((1 << 13, dict()), (1 << 16, dict()), (1 << 10, dict(fusion=False)),
                     (1 << 15, dict(drain="async")), (1 << 15, dict(threshold=64)), (1 << 20, dict())):
        d, st = run(gi, G, src, delta, **o)
        assert np.array_equal(d, ref), (delta, o)
        assert st["buckets"] == oracle.bucket_count(ref, delta)
    assert oracle.certificate(g, src, d, symmetric=True)[0] == 0


@pytest.mark.slow
def test_config3_full(gi, config_graph):
    g = config_graph(3)
    G = gi.Graph.from_csr(g)
    ref, _ = oracle.dijkstra(g, 0)
    for delta in (1, 2, 4, 8):
        for fusion in (True, False):
            d, st = run(gi, G, 0, delta, fusion=fusion)
            assert np.array_equal(d, ref), (delta, fusion)
            assert st["buckets"] == oracle.bucket_count(ref, delta)
    d, st = run(gi, G, 0, 1)
    assert st["edges_relaxed"] == int(np.diff(g.offsets)[ref != INF].sum())  # Δ=1 <= w_min


@pytest.mark.slow
def test_config5_batch(gi, config_graph):
    g = config_graph(5)
    G = gi.Graph.from_csr(g)
    srcs = gen.config_sources(5, g)
    out, st = gi.sssp_batch(G, srcs, 1 << 13)
    got = gi.as_uint32(out)
    # batch symmetry on a symmetric graph: δ(si,sj) == δ(sj,si) for all 64x64 pairs
    M = got[:, srcs.astype(np.int64)]
    assert np.array_equal(M, M.T)
    # element-wise parity on every row (oracle ~5 s per source, threaded over host cores)
    refs, _, _ = oracle.dijkstra_many(g, srcs)
    assert np.array_equal(got, refs)
    for i in range(64):
        assert st[i]["buckets"] > 0


@pytest.mark.slow
def test_config5_batch_peers_two_ranks(gi, config_graph):
    """The multi-GPU product path at full size (config 5: 64 sources on the 4096^2 road grid),
    two 'ranks' in one process: each computes its contiguous block of 32 sources with
    gi_sssp_batch_peers into its own [64, n] matrix and the kernel writes every finished row
    into the other rank's matrix. Both matrices must equal the oracle on every row."""
    import torch
    from paper_1911_07260_b200.dist import peer_row_addresses, shard_bounds
    g = config_graph(5)
    G = gi.Graph.from_csr(g)
    srcs = gen.config_sources(5, g).astype(np.int32)
    mats = [torch.full((64, g.n), 7, dtype=torch.int32, device="cuda") for _ in range(2)]
    bases = [m.data_ptr() for m in mats]
    for r in range(2):
        lo, hi = shard_bounds(64, r, 2)
        gi.gi_sssp_batch_peers(G, srcs[lo:hi], 1 << 13, peer_row_addresses(bases, lo, g.n), r)
    torch.cuda.synchronize()
    refs, _, _ = oracle.dijkstra_many(g, srcs)
    for m in mats:
        assert np.array_equal(gi.as_uint32(m), refs)


@pytest.mark.slow
def test_stress_repeated_full_size(gi, config_graph):
    """Race stress at full size (compute-sanitizer is closed on this pool): 20 runs each of
    config 3 at Δ=8 (skewed; pre-read / red.min protocol, R11; the late staleness gate, R12)
    and config 2 with the async drain (ring protocol, R10), with random CTA counts,
    thresholds and pre-read settings, every run compared with the oracle element by element.
    GI_STRESS_SEED / GI_STRESS_ITERS lengthen it into a soak (tools/r02_runs.sh arm aw)."""
    rng = np.random.default_rng(int(os.environ.get("GI_STRESS_SEED", "2024")))
    iters = int(os.environ.get("GI_STRESS_ITERS", "20"))
    for cfg, delta, base in ((3, 8, dict()), (2, 1 << 14, dict(drain="async"))):
        g = config_graph(cfg)
        G = gi.Graph.from_csr(g)
        src = gen.config_source(cfg, g)
        ref, _ = oracle.dijkstra(g, src)
        for it in range(iters):
            o = dict(base)
            o["max_ctas"] = int(rng.choice([0, 0, 1, 7, 64, 147]))
            o["threshold"] = int(rng.choice([0, 1, 16, 256, 1000]))
            if cfg == 3:
                o["pre_read"] = int(rng.choice([0, 1, 2]))
                o["expand"] = str(rng.choice(["auto", "on", "off"]))
            d, st = run(gi, G, src, delta, **o)
            assert np.array_equal(d, ref), (cfg, it, o)
            assert st["buckets"] == oracle.bucket_count(ref, delta), (cfg, it, o)


@pytest.mark.slow
def test_ppsp_astar_config2(gi, config_graph):
    """PPSP and A* at full size on the road grid (config 2): δ(s, t) equal to the oracle's
    dist[t] for the centre source and seeded targets, and never more buckets than SSSP."""
    g = config_graph(2)
    G = gi.Graph.from_csr(g)
    src = gen.config_source(2, g)
    ref, _ = oracle.dijkstra(g, src)
    full = run(gi, G, src, 1 << 16)[1]
    for t in [int(x) for x in gen.sources(g.n, 6, 7)] + [src]:
        d, st = gi.ppsp(G, src, t, 1 << 16)
        assert d == int(ref[t]), t
        assert st["buckets"] <= full["buckets"]
        h = gen.grid_heuristic(4096, 4096, t, int(g.w.min()))
        assert gi.astar(G, src, t, 1 << 16, h)[0] == int(ref[t]), t


def test_async_drain_low_degree_random(gi):
    """Random directed graphs with out-degree <= 8 (the async drain's domain): zero weights,
    self-loops, parallel edges, unreachable parts; every drain / threshold / CTA count."""
    rng = np.random.default_rng(23)
    for t in range(40):
        n = int(rng.integers(1, 3000))
        deg = rng.integers(0, 9, size=n)
        wmax = int(rng.choice([1, 3, 50, 10000]))
        edges = [(u, int(rng.integers(0, n)), int(rng.integers(0, wmax))) for u in range(n) for _ in range(deg[u])]
        g = gen.from_edges(n, edges)
        G = gi.Graph.from_csr(g)
        s = int(rng.integers(0, n))
        ref, _ = oracle.dijkstra(g, s)
        for delta in (1, 5, 64, 10**6, 2**31):
            for o in (dict(drain="async"), dict(drain="async", threshold=1), dict(drain="async", threshold=3, max_ctas=2),
                      dict(drain="async", max_ctas=1), dict(drain="bsp")):
                d, st = run(gi, G, s, delta, **o)
                assert np.array_equal(d, ref), (t, delta, o)
                assert st["kernel_kind"] == (2 if o["drain"] == "async" else 1)
                assert st["buckets"] == oracle.bucket_count(ref, delta), (t, delta, o, st)


def test_drain_selection_and_unsupported(gi):
    g = gen.grid(16, 16, 1, 10, 0)
    G = gi.Graph.from_csr(g)
    assert run(gi, G, 0, 8)[1]["kernel_kind"] == 1
    assert run(gi, G, 0, 8, drain="async")[1]["kernel_kind"] == 2
    assert run(gi, G, 0, 8, fusion=False)[1]["kernel_kind"] == 0
    star = gen.from_edges(20, [(0, v, 1) for v in range(1, 20)])
    S = gi.Graph.from_csr(star)
    assert run(gi, S, 0, 1)[1]["kernel_kind"] == 1
    with pytest.raises(gi.GiError) as e:
        run(gi, S, 0, 1, drain="async")
    assert e.value.status == 7


def test_hubs_and_mixed_degrees(gi):
    """High-degree vertices (deg > 8) take the CTA-wide edge-balanced path; a hub of
    degree 120,000 and many medium vertices exercise prefix sums and the search."""
    rng = np.random.default_rng(11)
    n = 150_000
    edges = [(0, int(v), int(rng.integers(1, 100))) for v in rng.choice(np.arange(1, n), 120_000, replace=False)]
    for _ in range(300_000):
        u, v = int(rng.integers(0, n)), int(rng.integers(0, n))
        edges.append((u, v, int(rng.integers(0, 30))))
    g = gen.from_edges(n, edges)
    G = gi.Graph.from_csr(g)
    for s in (0, 7):
        ref, _ = oracle.dijkstra(g, s)
        for o, delta in ((dict(fusion=True), 1), (dict(fusion=True), 64), (dict(fusion=False), 8),
                         (dict(fusion=True, pre_read=2), 3), (dict(fusion=True, max_ctas=2), 1 << 20),
                         (dict(fusion=True, hub_min=1024), 2), (dict(fusion=False, hub_min=1 << 30), 5),
                         (dict(fusion=True, max_ctas=7, hub_min=1024), 1)):
            d, _ = run(gi, G, s, delta, **o)
            assert np.array_equal(d, ref), (s, o, delta)


def test_expand_edge_balanced(gi):
    """Expand (skewed graphs): ROUND phases collect every frontier vertex of degree > 8 into
    one group list and split the concatenation of their edges evenly over all warps. Random
    power-law-like graphs; packed (weights fit the spare bits) and unpacked edges; groups of
    1..7 CTAs and the whole grid; expand forced on / off; fusion on / off; several Δ."""
    rng = np.random.default_rng(41)
    for t in range(6):
        n = int(rng.integers(2_000, 60_000))
        # degrees: a few hubs, a body of medium vertices, many tiny ones (max degree > 32)
        deg = np.minimum(rng.zipf(1.7, size=n), n - 1)
        deg[rng.integers(0, n, 3)] = rng.integers(2_000, max(2_001, n // 2), 3)
        wmax = int(rng.choice([3, 30, 1 << 20]))  # 1 << 20: too wide to pack beside the ids
        edges = [(u, int(v), int(w)) for u in range(n) for v, w in
                 zip(rng.integers(0, n, deg[u]), rng.integers(0, wmax, deg[u]))]
        g = gen.from_edges(n, edges)
        G = gi.Graph.from_csr(g)
        s = int(np.argmax(deg)) if t % 2 == 0 else int(rng.integers(0, n))
        ref, _ = oracle.dijkstra(g, s)
        for o, delta in ((dict(expand="on"), 1), (dict(expand="on"), 7), (dict(expand="off"), 7),
                         (dict(expand="on", fusion=False), 3), (dict(expand="on", max_ctas=1), 5),
                         (dict(expand="on", max_ctas=2, threshold=1), 2), (dict(expand="on", max_ctas=7), 1 << 30),
                         (dict(expand="on", fusion=False, max_ctas=3), 1), (dict(expand="on", pre_read=2), 4),
                         (dict(expand="on", cta_threads=512), 2)):
            d, st = run(gi, G, s, delta, **o)
            assert np.array_equal(d, ref), (t, o, delta)
            assert st["buckets"] == oracle.bucket_count(ref, delta), (t, o, delta)
        srcs = rng.integers(0, n, 5).astype(np.int32)
        out, _ = gi.sssp_batch(G, srcs, 4)
        refs, _, _ = oracle.dijkstra_many(g, srcs)
        assert np.array_equal(gi.as_uint32(out), refs), t


def test_expand_split_segments(gi, monkeypatch):
    """Split expand (single queries on skewed graphs): every list of >= GI_SPLIT_MIN edges is
    relaxed by expand_kernel between two segments of the persistent kernel, which saves and
    restores its phase-loop state (KState). With GI_SPLIT_MIN=1 every expand phase splits;
    PPSP and A* (whose stop test runs at phase ends) and a one-CTA group included."""
    monkeypatch.setenv("GI_SPLIT_MIN", "1")  # every list but the smallest goes to expand_kernel
    rng = np.random.default_rng(43)
    for t in range(4):
        n = int(rng.integers(3_000, 40_000))
        deg = np.minimum(rng.zipf(1.6, size=n), n - 1)
        deg[rng.integers(0, n, 2)] = rng.integers(1_000, max(1_001, n // 3), 2)
        wmax = int(rng.choice([5, 1 << 22]))
        edges = [(u, int(v), int(w)) for u in range(n) for v, w in
                 zip(rng.integers(0, n, deg[u]), rng.integers(1, wmax, deg[u]))]
        g = gen.from_edges(n, edges)
        G = gi.Graph.from_csr(g)
        s = int(np.argmax(deg))
        ref, _ = oracle.dijkstra(g, s)
        for o, delta in ((dict(expand="on"), 1), (dict(expand="on"), 9), (dict(expand="on", fusion=False), 4),
                         (dict(expand="on", max_ctas=1), 3), (dict(expand="on", cta_threads=512), 2)):
            d, st = run(gi, G, s, delta, **o)
            assert np.array_equal(d, ref), (t, o, delta)
            assert st["buckets"] == oracle.bucket_count(ref, delta), (t, o, delta)
            assert st["kernel_launches"] >= 1
        tgt = int(rng.integers(0, n))
        assert gi.ppsp(G, s, tgt, 3, expand="on")[0] == int(ref[tgt]), t


def test_expand_mirror_filter(gi, monkeypatch):
    """expand_kernel's pre-read filter (KArgs.mirror, a 1-byte saturated copy of dist):
    distances that straddle the byte's range (some below 255, some above, 0xFF = unknown),
    zero-weight edges, and the mirror switched off (GI_MIRROR=0) — all equal to the oracle."""
    monkeypatch.setenv("GI_SPLIT_MIN", "1")
    rng = np.random.default_rng(53)
    for t, wmax in enumerate((30, 200, 3000)):
        n = int(rng.integers(5_000, 30_000))
        deg = np.minimum(rng.zipf(1.7, size=n), n - 1)
        deg[rng.integers(0, n, 3)] = rng.integers(1_000, max(1_001, n // 4), 3)
        edges = [(u, int(v), int(w)) for u in range(n) for v, w in
                 zip(rng.integers(0, n, deg[u]), rng.integers(0 if t == 0 else 1, wmax, deg[u]))]
        g = gen.from_edges(n, edges)
        G = gi.Graph.from_csr(g)
        s = int(np.argmax(deg))
        ref, _ = oracle.dijkstra(g, s)
        fin = ref[ref != 0xFFFFFFFF]
        if t == 2:  # distances on both sides of the byte's range
            assert (fin < 255).sum() > 1 and fin.max() >= 255, (int(fin.min()), int(fin.max()))
        for mv in ("1", "0"):
            monkeypatch.setenv("GI_MIRROR", mv)
            for o, delta in ((dict(expand="on"), 1), (dict(expand="on"), 7), (dict(expand="on", fusion=False), 3)):
                d, st = run(gi, G, s, delta, **o)
                assert np.array_equal(d, ref), (t, mv, o, delta)
                assert st["buckets"] == oracle.bucket_count(ref, delta), (t, mv, o, delta)
    monkeypatch.delenv("GI_MIRROR")


def test_bucket_window(gi, monkeypatch, config_graph):
    """The bucket window of expand queries (gi_options.window buckets): far entries
    beyond the open window wait in the later pile and are rescanned only when the window
    advances. Widths 1 (an advance per bucket), 2, 8 and off; extractions in the persistent
    kernel and in extract_kernel; fused / unfused / lazy; PPSP (its stop clears the later
    pile's bits) and A*; config 3 at full size. Exact distances and bucket counts."""
    rng = np.random.default_rng(59)
    for t in range(3):
        n = int(rng.integers(4_000, 30_000))
        deg = np.minimum(rng.zipf(1.6, size=n), n - 1)
        deg[rng.integers(0, n, 2)] = rng.integers(1_000, max(1_001, n // 3), 2)
        wmax = int(rng.choice([9, 300]))
        edges = [(u, int(v), int(w)) for u in range(n) for v, w in
                 zip(rng.integers(0, n, deg[u]), rng.integers(1, wmax, deg[u]))]
        g = gen.from_edges(n, edges)
        G = gi.Graph.from_csr(g)
        s = int(np.argmax(deg))
        ref, _ = oracle.dijkstra(g, s)
        tgt = int(rng.integers(0, n))
        for win in (1, 2, 8, 0):
            for split_min, xsplit_min in (("1", "1"), ("1", str(1 << 30)), (str(1 << 40), "1")):
                monkeypatch.setenv("GI_SPLIT_MIN", split_min)
                monkeypatch.setenv("GI_XSPLIT_MIN", xsplit_min)
                for o, delta in ((dict(expand="on"), 1), (dict(expand="on"), 5), (dict(expand="on", fusion=False), 2),
                                 (dict(expand="on", fusion=False, lazy=True), 3), (dict(expand="on", max_ctas=3), 1)):
                    d, st = run(gi, G, s, delta, window=win, **o)
                    assert np.array_equal(d, ref), (t, win, split_min, xsplit_min, o, delta)
                    assert st["buckets"] == oracle.bucket_count(ref, delta), (t, win, o, delta)
                assert gi.ppsp(G, s, tgt, 2, expand="on", window=win)[0] == int(ref[tgt]), (t, win)
                h = np.zeros(n, np.uint32)
                assert gi.astar(G, s, tgt, 2, h, expand="on", window=win)[0] == int(ref[tgt]), (t, win)
                # the workspace ends clean after the PPSP stop: a full query still matches
                d, _ = run(gi, G, s, 1, expand="on", window=win)
                assert np.array_equal(d, ref), (t, win, "after ppsp")
    monkeypatch.setenv("GI_SPLIT_MIN", str(1 << 20))
    monkeypatch.setenv("GI_XSPLIT_MIN", "4096")
    g = config_graph(3)
    G = gi.Graph.from_csr(g)
    src = gen.config_source(3, g)
    ref, _ = oracle.dijkstra(g, src)
    for win in (1, 4):
        for delta in (1, 2):
            d, st = run(gi, G, src, delta, expand="on", window=win)
            assert np.array_equal(d, ref), (win, delta)
            assert st["buckets"] == oracle.bucket_count(ref, delta), (win, delta)
    # the window opened late (GI_WINDOW_PILE: at the first extraction of a pile that small)
    for pile in ("1000000", "50000"):
        monkeypatch.setenv("GI_WINDOW_PILE", pile)
        for win, delta in ((2, 1), (4, 2)):
            d, st = run(gi, G, src, delta, expand="on", window=win)
            assert np.array_equal(d, ref), (pile, win, delta)
            assert st["buckets"] == oracle.bucket_count(ref, delta), (pile, win, delta)
        assert gi.ppsp(G, src, int(np.argmax(ref != INF)), 1, expand="on", window=2)[0] == int(
            ref[int(np.argmax(ref != INF))])
    monkeypatch.delenv("GI_WINDOW_PILE")
    with pytest.raises(gi.GiError):
        run(gi, G, src, 1, window=-1)


def test_extract_split_segments(gi, monkeypatch, config_graph):
    """Split extraction (single queries on skewed graphs with expand): an EXTRACT phase whose
    far pile holds >= GI_XSPLIT_MIN entries stops the persistent kernel (KState, pending 2);
    extract_kernel partitions the pile (bucket b -> the global frontier, later buckets kept,
    earlier ones dropped) and the kernel resumes at the same phase. With GI_XSPLIT_MIN=1 every
    extraction splits, mixed with split expands; fused / unfused / lazy, PPSP and A*; and
    config 3 at full size."""
    monkeypatch.setenv("GI_XSPLIT_MIN", "1")
    rng = np.random.default_rng(47)
    for t in range(3):
        n = int(rng.integers(3_000, 40_000))
        deg = np.minimum(rng.zipf(1.6, size=n), n - 1)
        deg[rng.integers(0, n, 2)] = rng.integers(1_000, max(1_001, n // 3), 2)
        wmax = int(rng.choice([5, 1 << 22]))
        edges = [(u, int(v), int(w)) for u in range(n) for v, w in
                 zip(rng.integers(0, n, deg[u]), rng.integers(1, wmax, deg[u]))]
        g = gen.from_edges(n, edges)
        G = gi.Graph.from_csr(g)
        s = int(np.argmax(deg))
        ref, _ = oracle.dijkstra(g, s)
        for split_min in ("1", str(1 << 40)):  # with / without split expands
            monkeypatch.setenv("GI_SPLIT_MIN", split_min)
            for o, delta in ((dict(expand="on"), 1), (dict(expand="on"), 9), (dict(expand="on", fusion=False), 4),
                             (dict(expand="on", fusion=False, lazy=True), 2), (dict(expand="on", max_ctas=3), 3)):
                d, st = run(gi, G, s, delta, **o)
                assert np.array_equal(d, ref), (t, split_min, o, delta)
                assert st["buckets"] == oracle.bucket_count(ref, delta), (t, split_min, o, delta)
                assert st["kernel_launches"] > 2, (t, split_min, o, delta)  # it did split
        tgt = int(rng.integers(0, n))
        assert gi.ppsp(G, s, tgt, 3, expand="on")[0] == int(ref[tgt]), t
        h = np.zeros(n, np.uint32)
        assert gi.astar(G, s, tgt, 3, h, expand="on")[0] == int(ref[tgt]), t
    monkeypatch.setenv("GI_SPLIT_MIN", str(1 << 20))
    monkeypatch.setenv("GI_XSPLIT_MIN", "4096")
    g = config_graph(3)
    G = gi.Graph.from_csr(g)
    src = gen.config_source(3, g)
    ref, _ = oracle.dijkstra(g, src)
    for delta in (1, 2, 8):
        d, st = run(gi, G, src, delta, expand="on")
        assert np.array_equal(d, ref), delta
        assert st["buckets"] == oracle.bucket_count(ref, delta), delta


@pytest.mark.slow
@pytest.mark.skipif(os.environ.get("GI_SKIP_CFG4") == "1",
                    reason="config 4 (RMAT-26, 2.1 B edges): ~2 min and ~25 GB of host RAM (GI_SKIP_CFG4=1)")
def test_config4_full(gi):
    """RMAT-26 at Δ=2: the certificate over every edge (exact for w >= 1),
    the bucket closed form, and the full Dijkstra oracle element by element."""
    g = gen.config_graph(4)
    G = gi.Graph.from_csr(g)
    src = gen.config_source(4, g)
    d, st = run(gi, G, src, 2)
    assert oracle.certificate(g, src, d, symmetric=True)[0] == 0
    assert st["buckets"] == oracle.bucket_count(d, 2)
    ref, rc = oracle.dijkstra(g, src)
    assert rc == 0 and np.array_equal(d, ref)


def test_ppsp_matches_oracle_and_stops_early(gi, config_graph):
    """PPSP: δ(s,t) equals the Dijkstra oracle's
    dist[t] on random triples; it never runs more buckets/rounds than SSSP
    (SPEC.md:353); target == source costs one bucket; unreachable -> UINT32_MAX."""
    rng = np.random.default_rng(31)
    g = config_graph(1)
    G = gi.Graph.from_csr(g)
    for _ in range(20):
        s, t = (int(x) for x in rng.integers(0, g.n, 2))
        ref, _ = oracle.dijkstra(g, s)
        for delta, o in ((1000, dict()), (250, dict(fusion=False)), (4000, dict(drain="async")), (7, dict())):
            d, st = gi.ppsp(G, s, t, delta, **o)
            assert d == int(ref[t]), (s, t, delta, o)
            _, full = gi.sssp(G, s, delta, **o)
            assert st["buckets"] <= full["buckets"] and st["rounds"] <= full["rounds"]
    d, st = gi.ppsp(G, 77, 77, 1000)
    assert d == 0 and st["buckets"] == 1
    # random small graphs with unreachable targets, zero weights, parallel edges
    for trial in range(30):
        n = int(rng.integers(2, 400))
        edges = [(int(rng.integers(0, n)), int(rng.integers(0, n)), int(rng.integers(0, 20)))
                 for _ in range(int(rng.integers(0, 3 * n)))]
        h = gen.from_edges(n, edges)
        H = gi.Graph.from_csr(h)
        s, t = int(rng.integers(0, n)), int(rng.integers(0, n))
        ref, _ = oracle.dijkstra(h, s)
        for delta in (1, 5, 1 << 20):
            assert gi.ppsp(H, s, t, delta)[0] == int(ref[t]), (trial, s, t, delta)
    # device scalar output and error codes
    import torch
    out = torch.zeros(1, dtype=torch.int32, device="cuda")
    gi.gi_ppsp_delta(G, 0, 65535, 1000, out)
    assert int(out.item()) == int(oracle.dijkstra(g, 0)[0][65535])
    with pytest.raises(gi.GiError) as e:
        gi.ppsp(G, 0, g.n, 1000)
    assert e.value.status == 2
    with pytest.raises(gi.GiError) as e:
        gi.ppsp(G, 0, -1, 1000)
    assert e.value.status == 2


def test_ppsp_overflow_only_for_the_target(gi):
    """Ex7-like: 0->1 (2^32-2), 1->2 (1). PPSP to 1 is fine; PPSP to 2 overflows."""
    g = gen.from_edges(3, [(0, 1, 2**32 - 2), (1, 2, 1)])
    G = gi.Graph.from_csr(g)
    assert gi.ppsp(G, 0, 1, 1)[0] == 2**32 - 2
    with pytest.raises(gi.OverflowDistance):
        gi.ppsp(G, 0, 2, 1)


def test_astar_matches_oracle(gi, config_graph):
    """A* (PAPER.md:979-982): priority dist + h, PPSP stop. With an
    admissible h (consistent: w_min x Chebyshev; inconsistent: random fractions of the true
    remaining distance; perfect: the true remaining distance) the result equals the Dijkstra
    oracle's dist[t]; h = 0 reproduces PPSP; an inadmissible h (x10) never
    returns less than the true distance (documents the non-guarantee)."""
    rng = np.random.default_rng(41)
    rows, cols = 256, 256
    g = config_graph(1)
    G = gi.Graph.from_csr(g)
    wmin = int(g.w.min())
    for _ in range(12):
        s, t = (int(x) for x in rng.integers(0, g.n, 2))
        ref, _ = oracle.dijkstra(g, s)
        to_t, _ = oracle.dijkstra(g, t)  # symmetric graph: δ(v, t) = δ(t, v)
        hc = gen.grid_heuristic(rows, cols, t, wmin)
        hr = (to_t.astype(np.float64) * rng.random(g.n)).astype(np.uint32)
        for delta, o in ((1000, dict()), (250, dict(fusion=False)), (64, dict(threshold=4))):
            for h in (hc, hr, to_t):
                d, st = gi.astar(G, s, t, delta, h, **o)
                assert d == int(ref[t]), (s, t, delta, o)
            d0, st0 = gi.astar(G, s, t, delta, np.zeros(g.n, np.uint32), **o)
            dp, stp = gi.ppsp(G, s, t, delta, **o)
            assert d0 == dp == int(ref[t]) and st0["buckets"] == stp["buckets"]
            d10, _ = gi.astar(G, s, t, delta, np.minimum(to_t.astype(np.uint64) * 10, 2**32 - 2).astype(np.uint32))
            assert d10 >= int(ref[t])
    # road-like recipe with diagonals, device-resident h, and the async drain rejected
    import torch
    h = gen.grid_heuristic(rows, cols, 5, wmin)
    hd = torch.from_numpy(h.view(np.int32)).cuda()
    out = torch.zeros(1, dtype=torch.int32, device="cuda")
    gi.gi_astar_delta(G, 60000, 5, 1000, hd, out)
    assert int(out.item()) == int(oracle.dijkstra(g, 60000)[0][5])
    with pytest.raises(gi.GiError) as e:
        gi.astar(G, 0, 5, 1000, h, drain="async")
    assert e.value.status == 7


def test_astar_random_symmetric_graphs(gi):
    rng = np.random.default_rng(43)
    for trial in range(25):
        n = int(rng.integers(2, 500))
        und = [(int(rng.integers(0, n)), int(rng.integers(0, n))) for _ in range(int(rng.integers(0, 4 * n)))]
        edges = []
        for u, v in und:
            w = int(rng.integers(0, 30))
            edges += [(u, v, w), (v, u, w)]
        g = gen.from_edges(n, edges)
        G = gi.Graph.from_csr(g)
        s, t = int(rng.integers(0, n)), int(rng.integers(0, n))
        ref, _ = oracle.dijkstra(g, s)
        to_t, _ = oracle.dijkstra(g, t)
        h = np.where(to_t == 0xFFFFFFFF, 0, (to_t * rng.random(n)).astype(np.uint32)).astype(np.uint32)
        for delta in (1, 4, 1 << 20):
            assert gi.astar(G, s, t, delta, h)[0] == int(ref[t]), (trial, s, t, delta)


def _sym_graph(n, und):
    edges = []
    for u, v in und:
        edges += [(u, v, 1), (v, u, 1)]
    return gen.from_edges(n, edges)


def test_kcore_matches_oracle(gi, config_graph):
    """k-core (Fig. 10): coreness of every vertex equals
    the serial peeling oracle, element by element — closed forms, random symmetric
    multigraphs (parallel edges, self-loops, isolated vertices), every CTA count, the full
    grid of config 1 (all 2) and RMAT-22 (config 3: skewed degrees, hubs)."""
    tri = gi.Graph.from_csr(_sym_graph(3, [(0, 1), (1, 2), (0, 2)]))
    assert gi.as_uint32(gi.kcore(tri)[0]).tolist() == [2, 2, 2]
    star = gi.Graph.from_csr(_sym_graph(5, [(0, i) for i in range(1, 5)]))
    assert gi.as_uint32(gi.kcore(star)[0]).tolist() == [1] * 5
    rng = np.random.default_rng(47)
    for t in range(40):
        n = int(rng.integers(1, 2000))
        und = [(int(rng.integers(0, n)), int(rng.integers(0, n))) for _ in range(int(rng.integers(0, 6 * n)))]
        g = _sym_graph(n, und)
        G = gi.Graph.from_csr(g)
        ref = oracle.kcore(g)
        for o in (dict(), dict(max_ctas=1), dict(max_ctas=7)):
            got, st = gi.kcore(G, **o)
            assert np.array_equal(gi.as_uint32(got), ref), (t, o)
            assert st["vertices_processed"] == n and st["buckets"] == len(set(ref.tolist()))
    g1 = config_graph(1)
    c1, _ = gi.kcore(gi.Graph.from_csr(g1))
    assert set(gi.as_uint32(c1).tolist()) == {2}
    host = np.zeros(g1.n, np.uint32)
    gi.gi_kcore(gi.Graph.from_csr(g1), host)
    assert set(host.tolist()) == {2}
    g3 = config_graph(3)
    G3 = gi.Graph.from_csr(g3)
    ref3 = oracle.kcore(g3)
    for _ in range(4):  # repeated: a vertex finished twice (a race) would show up as a mismatch
        c3, st3 = gi.kcore(G3)
        assert np.array_equal(gi.as_uint32(c3), ref3)
        assert st3["edges_relaxed"] == g3.m  # every vertex is peeled once: each CSR entry is scanned once


def test_batch_peers_fused_gather_one_process(gi, config_graph):
    """gi_sssp_batch_peers (north_star multi-GPU batch) emulated in one
    process: two 'ranks' each compute a block of sources into their own matrix, and the
    kernel writes every finished row into the other matrix too. Both matrices must equal
    the oracle row for row (n % 4 == 0: 16-byte copies; n % 4 != 0: element copies)."""
    import torch
    for g in (config_graph(1), gen.uniform_random(1001, 6000, 1, 100, 3)):
        G = gi.Graph.from_csr(g)
        srcs = gen.sources(g.n, 9, 11).astype(np.int32)
        ref, _ = oracle.dijkstra_many(g, srcs)[:2]
        mats = [torch.full((9, g.n), 7, dtype=torch.int32, device="cuda") for _ in range(2)]
        bases = [m.data_ptr() for m in mats]
        from paper_1911_07260_b200.dist import peer_row_addresses, shard_bounds
        for r in range(2):
            lo, hi = shard_bounds(9, r, 2)
            gi.gi_sssp_batch_peers(G, srcs[lo:hi], 50 if g.n == 1001 else 1000,
                                   peer_row_addresses(bases, lo, g.n), r)
        torch.cuda.synchronize()
        for m in mats:
            assert np.array_equal(gi.as_uint32(m), ref)
        with pytest.raises(gi.GiError):
            gi.gi_sssp_batch_peers(G, srcs[:2], 10, bases, 2)  # self out of range
        with pytest.raises(gi.GiError):
            gi.gi_sssp_batch_peers(G, srcs[:2], 10, [bases[0], 0], 0)  # NULL peer row


def _peers_worker(rank, world, port, q):
    import socket  # noqa: F401
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_1911_07260_b200 import gi as m
    from paper_1911_07260_b200.dist import sssp_batch_fused_gather
    g = gen.config_graph(1)
    G = m.Graph.from_csr(g)
    srcs = gen.sources(g.n, 10, 5).astype(np.int32)
    full = sssp_batch_fused_gather(G, srcs, 1000)
    torch.cuda.synchronize()
    q.put((rank, m.as_uint32(full)))
    dist.barrier()
    dist.destroy_process_group()


def test_batch_peers_ipc_two_processes(gi):
    """The fused gather across processes (CUDA IPC handles exchanged over a gloo group):
    two ranks on this one GPU — their kernels do not wait on each other, each only writes
    its finished rows into the other's matrix — and both end with all 10 rows."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_peers_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    g = gen.config_graph(1)
    srcs = gen.sources(g.n, 10, 5).astype(np.int32)
    ref, _ = oracle.dijkstra_many(g, srcs)[:2]
    for r in (0, 1):
        assert np.array_equal(res[r], ref), r


def test_concurrent_host_threads_one_graph(gi, config_graph):
    """SURVEY §8(b) semantics: the graph is immutable and each call takes its own workspace
    (and stream), so queries from several host threads on one graph may overlap — their
    persistent kernels are cooperative launches, each co-resident as a whole. Every result
    must still be bit-exact."""
    import threading
    g = config_graph(1)
    G = gi.Graph.from_csr(g)
    srcs = [0, 777, 31337, 65535, 4242, 12]
    refs = {s: oracle.dijkstra(g, s)[0] for s in srcs}
    errors = []

    def worker(i):
        try:
            for rep in range(3):
                s = srcs[(i + rep) % len(srcs)]
                d, _ = run(gi, G, s, 1000, fusion=bool((i + rep) % 2))
                if not np.array_equal(d, refs[s]):
                    errors.append((i, rep, s))
            out, _ = gi.sssp_batch(G, np.array(srcs[:3], np.int32), 1000)
            if not np.array_equal(gi.as_uint32(out), np.stack([refs[s] for s in srcs[:3]])):
                errors.append((i, "batch"))
        except Exception as e:  # noqa: BLE001
            errors.append((i, repr(e)))

    ts = [threading.Thread(target=worker, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in ts), "a query did not finish"
    assert not errors, errors


def test_single_cta_overflow_paths(gi):
    """One or two CTAs on a 512x512 grid: a sub-round pushes more vertices than a bin holds
    (the per-lane full-bin fallback to the global frontier) and a warp stages more far-pile
    entries in one phase than its segment holds (the per-lane fallback to the global pile).
    Distances must still be bit-exact."""
    g = gen.grid(512, 512, 1, 100, 21, p_del=0.05, p_diag=0.02)
    G = gi.Graph.from_csr(g)
    ref, _ = oracle.dijkstra(g, 0)
    for o, delta in ((dict(max_ctas=1, threshold=2048), 10**9), (dict(max_ctas=1), 64),
                     (dict(max_ctas=2, threshold=2048), 16), (dict(max_ctas=1, cta_threads=1024), 10**9)):
        d, _ = run(gi, G, 0, delta, **o)
        assert np.array_equal(d, ref), (o, delta)
