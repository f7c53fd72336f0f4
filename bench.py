#!/usr/bin/env python
"""Benchmark: Δ-stepping SSSP on B200 (BASELINE.json metric: time/source and GTEPS = m/time;
achieved HBM GB/s vs peak; bucket / launch / grid-sync counts with and without fusion).

Default workload (N=1): BASELINE.json configs[1] — the 4096x4096 road-like grid (config 2),
centre source, one single-source query per step. With --gpus N (torchrun, one rank per GPU)
every rank runs its own replica of the same query (single-source SSSP does not shard:
DESIGN.md "Multi-GPU"), value = N*m / max-over-ranks time ("scaling": "weak").
--config 5: the 64-source batch, sources sharded over ranks, rows gathered with NCCL.

--impl reference: the oracle (CPU Dijkstra, oracle/) timed on the host on the same
workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import gen  # noqa: E402

METRIC = "Δ-stepping SSSP GTEPS (m / time per source)"
UNIT = "GTEPS"
DEFAULT_DELTA = {1: 1000, 2: 1 << 16, 3: 2, 4: 2, 5: 1 << 13}
WORKLOAD = {
    1: "cfg1: 256x256 4-neighbour grid, w~U[1,1000) seed 1, src 0",
    2: "cfg2: road-like 4096x4096 grid (5% lattice edges deleted, 1% diagonals), w~U[1,10000) seed 2, "
       "centre source 8390656",
    3: "cfg3: RMAT-22 ef16 (.57,.19,.19,.05) symmetrized, w~U[1,22) seed 3, max-degree source",
    4: "cfg4: RMAT-26 ef16 symmetrized, w~U[1,26) seed 4, max-degree source",
    5: "cfg5: 64 sources (seed 5) on the cfg2 road-like grid, sharded over GPUs, rows gathered",
}


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        j = json.load(open(p))
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 6 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows if len(r) >= 6 for k in range(4)
                          if r[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def reached_stats(g, dist_u32):
    reached = dist_u32 != 0xFFFFFFFF
    n_r = int(reached.sum())
    m_r = int(np.diff(g.offsets)[reached].sum())
    return n_r, m_r


def b_alg(g, n_r, m_r, nsrc=1):
    """B_alg = 12·m_r + 16·n_r + 4·n per source (col 4 + w 4 + dist[v] 4 per
    reached edge; offsets 8 + dist[u] 4 + one improving write 4 per reached vertex; init/output)."""
    return nsrc * (12 * m_r + 16 * n_r + 4 * g.n)


def load_traffic(cfg, delta):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        j = json.load(open(p))
        return j.get(f"cfg{cfg}_delta{delta}")
    except Exception:
        return None


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import oracle
    cfg = args.config
    g = gen.config_graph(cfg)
    srcs = gen.config_sources(cfg, g, 64) if cfg == 5 else [gen.config_source(cfg, g)]
    src = int(srcs[0])
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        d, rc = oracle.dijkstra(g, src)
        t1 = time.perf_counter()
        if i >= args.warmup:
            times.append(t1 - t0)
    t = statistics.mean(times)
    v = g.m / t / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong" if cfg == 5 else "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": WORKLOAD[cfg], "source": src, "n": g.n, "m": g.m},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"one full binary-heap Dijkstra per step from source {src} "
                                       f"(single-threaded C, oracle/oracle.c)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(g, src, budget_s=12.0):
    """Oracle timed on the host (rank 0, N=1 only): whole Dijkstra queries from the same
    source until ~budget_s of CPU work (at least one)."""
    import oracle
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        oracle.dijkstra(g, src)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s or len(times) >= 5:
            break
    t = statistics.mean(times)
    return {"value": g.m / t / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{len(times)} full single-threaded Dijkstra queries from source {src} "
                      f"(oracle/oracle.c), mean {t:.3f} s each"}


def run_kcore(args, g, G, opts, rank, world):
    """k-core on the config's symmetric graph: coreness of every vertex,
    checked element by element against the serial peeling oracle; the oracle is timed on
    the host beside it (one full peel)."""
    import torch
    import oracle
    from paper_1911_07260_b200 import gi
    out = torch.empty(g.n, dtype=torch.int32, device="cuda")
    o = gi.make_options(**{k: v for k, v in opts.items() if k in ("max_ctas", "stream")})
    for _ in range(max(args.warmup, 3)):
        gi.gi_kcore(G, out, o)
    stream = opts["stream"]
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    sts = [gi.gi_kcore(G, out, o) for _ in range(args.steps)]
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    if rank != 0:
        return 0
    got = gi.as_uint32(out)
    if args.no_cpu_baseline:  # the oracle runs only as the cpu_baseline leg (and parity reference)
        ref, t_or = None, None
    else:
        t0 = time.perf_counter()
        ref = oracle.kcore(g)
        t_or = time.perf_counter() - t0
    st = sts[-1]
    line = {"metric": "k-core time per full peel (and m / time)", "value": g.m / (ms * 1e-3) / 1e9, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "dtype": "u32", "data": "synthetic",
            "config": {"workload": WORKLOAD[args.config], "app": "kcore", "n": g.n, "m": g.m},
            "parity": bool(np.array_equal(got, ref)) if ref is not None else None,
            "max_core": int(got.max()) if got.size else 0,
            "cpu_baseline": None if ref is None else {
                "value": g.m / t_or / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
                "sample": f"one serial peel (oracle/oracle.c), {t_or:.3f} s"},
            "counters": {k: getattr(st, k) for k in ("buckets", "rounds", "grid_syncs", "vertices_processed",
                                                      "edges_relaxed", "empty_extractions", "fused_subrounds",
                                                      "critical_subrounds", "spills", "kernel_kind")}}
    print(json.dumps(line), flush=True)
    return 0 if line["parity"] is not False else 1


def run_app(args, g, G, delta, opts, rank, world):
    """PPSP / A* on the config's source and a seeded target; checked
    against the Dijkstra oracle's dist[target] (rank 0) and timed with CUDA events."""
    import torch
    import oracle
    from paper_1911_07260_b200 import gi
    cfg = args.config
    if args.app == "kcore":
        return run_kcore(args, g, G, opts, rank, world)
    src = gen.config_source(cfg, g)
    tgt = int(gen.sources(g.n, 1, seed=7)[0])
    out = torch.zeros(1, dtype=torch.int32, device="cuda")
    h = None
    if args.app == "astar":
        if g.meta.get("kind") != "grid":
            raise SystemExit("--app astar needs a grid config (1, 2): the heuristic uses grid coordinates")
        hh = gen.grid_heuristic(g.meta["rows"], g.meta["cols"], tgt, int(g.w.min()))
        h = torch.from_numpy(hh.view(np.int32)).cuda()

    def step():
        o = gi.make_options(**opts)
        if h is None:
            return gi.gi_ppsp_delta(G, src, tgt, delta, out, o)
        return gi.gi_astar_delta(G, src, tgt, delta, h, out, o)
    for _ in range(max(args.warmup, 3)):
        step()
    stream = opts["stream"]
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    sts = [step() for _ in range(args.steps)]
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    if rank != 0:
        return 0
    got = int(out.item()) & 0xFFFFFFFF
    # cpu_baseline leg: one full oracle Dijkstra from the source, timed on the host; its
    # dist[target] is also the parity reference for this line
    ref, cpu = None, None
    if not args.no_cpu_baseline:
        t0 = time.perf_counter()
        ref = int(oracle.dijkstra(g, src)[0][tgt])
        t_or = time.perf_counter() - t0
        cpu = {"value": g.m / t_or / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"one full Dijkstra from source {src} (oracle/oracle.c), {t_or:.3f} s"}
    st = sts[-1]
    line = {"metric": f"{args.app} time per query (and m / time)", "value": g.m / (ms * 1e-3) / 1e9, "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "dtype": "u32", "data": "synthetic",
            "config": {"workload": WORKLOAD[cfg], "app": args.app, "source": src, "target": tgt, "delta": delta},
            "result": got, "oracle": ref, "parity": (got == ref) if ref is not None else None,
            "cpu_baseline": cpu,
            "counters": {k: getattr(st, k) for k in ("buckets", "rounds", "grid_syncs", "vertices_processed",
                                                      "edges_relaxed", "critical_subrounds", "kernel_kind")}}
    print(json.dumps(line), flush=True)
    return 0 if ref is None or got == ref else 1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--delta", type=int, default=0)
    ap.add_argument("--threshold", type=int, default=0)
    ap.add_argument("--no-fusion", action="store_true")
    ap.add_argument("--max-ctas", type=int, default=0)
    ap.add_argument("--group-ctas", type=int, default=0)
    ap.add_argument("--hub-min", type=int, default=0)
    ap.add_argument("--pre-read", type=int, default=0, help="0 auto, 1 on, 2 off")
    ap.add_argument("--cta-threads", type=int, default=0, choices=[0, 512, 1024],
                    help="threads per persistent CTA (0 = auto: 1024 on skewed graphs)")
    ap.add_argument("--drain", default="auto", choices=["auto", "bsp", "async"],
                    help="fused drain: per-sub-round CTA barriers (default) or the barrier-free async ring")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--app", default="sssp", choices=["sssp", "ppsp", "astar", "kcore"],
                    help="next rows (SURVEY §8(f)): point-to-point Δ-stepping, A* to a seeded target (grids), "
                         "k-core (coreness of every vertex)")
    ap.add_argument("--no-compare", action="store_true", help="skip the fusion on/off counter comparison")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_1911_07260_b200 import gi

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = args.config
    delta = args.delta or DEFAULT_DELTA[cfg]
    g = gen.config_graph(cfg)
    t0 = time.perf_counter()
    G = gi.Graph.from_csr(g, device=local)
    torch.cuda.synchronize()
    t_upload = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    opts = dict(fusion=not args.no_fusion, threshold=args.threshold, max_ctas=args.max_ctas,
                group_ctas=args.group_ctas, hub_min=args.hub_min, pre_read=args.pre_read, drain=args.drain,
                stream=stream, cta_threads=args.cta_threads)

    if cfg == 5:
        from paper_1911_07260_b200.dist import exchange_handles, peer_row_addresses, shard_bounds
        srcs_all = gen.config_sources(5, g, 64)
        lo, hi = shard_bounds(len(srcs_all), rank, world)  # contiguous block of the 64 sources
        srcs = torch.from_numpy(srcs_all[lo:hi].copy())
        # every rank holds the whole [64, n] result; the kernel writes each finished row
        # into every rank's copy over NVLink (gi_sssp_batch_peers): the gather is fused into
        # the compute, no collective moves data
        full = torch.empty((len(srcs_all), g.n), dtype=torch.int32, device="cuda")
        bases, opened = exchange_handles(full, rank, world, local) if world > 1 else ([full.data_ptr()], [])
        peers = peer_row_addresses(bases, lo, g.n)
        out = full[lo:hi]

        def step():
            return gi.gi_sssp_batch_peers(G, srcs, delta, peers, rank, gi.make_options(**opts))
        units_per_step = len(srcs_all) * g.m  # whole job: all 64 sources
        launches_per_step = 1
    elif args.app != "sssp":
        return run_app(args, g, G, delta, opts, rank, world)
    else:
        src = gen.config_source(cfg, g)
        out = torch.empty(g.n, dtype=torch.int32, device="cuda")

        def step():
            return gi.gi_sssp_delta(G, src, delta, out, gi.make_options(**opts))
        units_per_step = world * g.m
        launches_per_step = 1

    for _ in range(max(args.warmup, 3) if args.warmup >= 3 else args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    kernel_ms = []
    stats = []
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0.record(stream)
    for _ in range(args.steps):
        st = step()
        s0 = st if cfg != 5 else st[0]
        kernel_ms.append(s0.gpu_ms)
        stats.append(st)
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    kms = statistics.mean(kernel_ms)
    if world > 1:
        t = torch.tensor([ms, kms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kms = float(t[0]), float(t[1])
    value = units_per_step / (ms * 1e-3) / 1e9

    if cfg == 5:
        for addr, off in opened:  # every rank is past the final barrier: no peer writes remain
            gi.ipc_close(addr, off, local)
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant (only) kernel: sssp_persistent ----
    d_host = gi.as_uint32(out if cfg != 5 else out[0])
    n_r, m_r = reached_stats(g, d_host)
    nsrc_local = 1 if cfg != 5 else out.shape[0]
    if cfg == 5:
        rows = gi.as_uint32(out)
        bytes_alg = sum(b_alg(g, *reached_stats(g, rows[i])) for i in range(rows.shape[0]))
    else:
        bytes_alg = b_alg(g, n_r, m_r)
    peak, peak_src = measured_peak()
    achieved = bytes_alg / (kms * 1e-3) / 1e9
    traffic = load_traffic(cfg, delta)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": "sssp_persistent", "kernel_ms": kms,
                "bytes_alg_per_launch": bytes_alg, "peak_source": peak_src,
                "note": "latency/sync-bound on road graphs: see DESIGN.md sync floor"}

    s_last = stats[-1] if cfg != 5 else stats[-1][0]
    # the dependent chain that bounds road graphs: levels a CTA had to run
    # one after another, the time per level, and the bare hop (atomicMin ∥ slot load,
    # tools/hop_bench.cu: ~650 cycles = 0.33 µs at 1,965 MHz) as its floor
    chain = None
    if cfg != 5 and s_last.critical_subrounds:
        hop_us = 650 / 1965.0
        chain = {"critical_subrounds": s_last.critical_subrounds, "phases": s_last.grid_syncs,
                 "us_per_level": kms * 1e3 / s_last.critical_subrounds, "hop_floor_us": hop_us,
                 "chain_floor_ms": s_last.critical_subrounds * hop_us / 1e3,
                 "frac_of_chain_floor": (s_last.critical_subrounds * hop_us / 1e3) / kms}
    counters = {k: getattr(s_last, k) for k in ("buckets", "rounds", "grid_syncs", "kernel_launches",
                                                  "fused_subrounds", "spills", "vertices_processed",
                                                  "edges_relaxed", "empty_extractions", "far_scanned", "critical_subrounds",
                                                  "ctas", "threads_per_cta", "groups", "kernel_kind")}

    # ---- fusion on vs off (untimed comparison run, same Δ) ----
    compare = None
    if not args.no_compare and cfg != 5:
        compare = {}
        variants = [("fused", dict(fusion=True)), ("unfused", dict(fusion=False))]
        if int(np.diff(g.offsets).max(initial=0)) <= 8:  # both drains run on low-degree graphs
            variants = [("fused", dict(fusion=True, drain="bsp")), ("fused_async_drain", dict(fusion=True, drain="async")),
                        ("unfused", dict(fusion=False))]
        for name, ov in variants:
            o2 = dict(opts)
            o2.update(ov)
            sts = [gi.gi_sssp_delta(G, src, delta, out, gi.make_options(**o2)) for _ in range(3)]
            s = sts[-1]
            compare[name] = {
                "gpu_ms": statistics.median([x.gpu_ms for x in sts]), "buckets": s.buckets,
                "rounds": s.rounds, "grid_syncs": s.grid_syncs, "kernel_launches": s.kernel_launches,
                "fused_subrounds": s.fused_subrounds, "spills": s.spills,
                "critical_subrounds": s.critical_subrounds, "kernel_kind": s.kernel_kind}

    # ---- e2e through the public C ABI with HOST buffers (pinned), copies inside ----
    e2e = None
    if cfg != 5:
        host_out = torch.empty(g.n, dtype=torch.int32, pin_memory=True)
        host_src = torch.tensor([src], dtype=torch.int32).pin_memory()
        times = []
        o_e2e = dict(opts)
        o_e2e.pop("stream")
        for i in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s_val = int(host_src[0])  # source id read from pinned host memory (4 bytes H2D inside the call)
            gi.gi_sssp_delta(G, s_val, delta, host_out.numpy(), gi.make_options(**o_e2e))
            t1 = time.perf_counter()
            if i >= args.warmup:
                times.append(t1 - t0)
        te = statistics.mean(times)
        e2e = {"value": world * g.m / te / 1e9, "unit": UNIT, "h2d_bytes_per_step": 4,
               "d2h_bytes_per_step": 4 * g.n, "ms_per_step": te * 1e3,
               "api": "gi_sssp_delta_ex with a pinned host dist_out (library stages + copies back)"}
        assert np.array_equal(host_out.numpy().view(np.uint32), d_host)

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(g, int(src if cfg != 5 else srcs_all[0]))

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if cfg == 5 else "weak",  # cfg5: 64 sources in total, split over the ranks
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": WORKLOAD[cfg], "config": cfg, "delta": delta, "fusion": not args.no_fusion,
                   "threshold": args.threshold or "default", "n": g.n, "m": g.m, "n_reached": n_r,
                   "m_reached": m_r, "time_per_source_ms": ms / (64 / world if cfg == 5 else 1),
                   "l2": f"inputs larger than L2 (CSR {(g.offsets.nbytes + 8 * g.m) / 1e6:.0f} MB > 126 MB); "
                         "dist re-initialised every step",
                   "parallelism": f"{'sources sharded' if cfg == 5 else 'replica'} x{world}",
                   "graph_upload_s": t_upload},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clocks, "counters": counters, "fusion_compare": compare, "chain": chain,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
