#!/usr/bin/env python
"""Benchmark: Δ-stepping SSSP on B200 (BASELINE.json metric: time/source and GTEPS = m/time;
achieved HBM GB/s vs peak; bucket / launch / grid-sync counts with and without fusion).

Workload of a step:
- N=1 (default): config 4, BASELINE.json's largest single-GPU config — RMAT-26, 2.1 B
  directed edges, Δ=2, highest-degree source; one single-source query per step. The line
  also carries config 2 (the large-diameter road grid where bucket fusion matters) and the
  config-5 batch at one GPU as secondary keys.
- N>1 (torchrun, one rank per GPU): config 5, the 64-source batch on the road grid, sources
  sharded over the ranks, every finished row written into every rank's result matrix by the
  kernel (fused gather, "scaling": "strong"); `--gather nccl` times the compute-then-NCCL
  all-gather baseline beside it.
Other configs with --config 1..5; next rows with --app ppsp|astar|kcore.

--impl reference: the oracle (CPU Dijkstra, oracle/) timed on the host on the same workload,
each step a bounded sample; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

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
    4: "cfg4: RMAT-26 ef16 (.57,.19,.19,.05) symmetrized (2.1B directed edges), w~U[1,26) seed 4, "
       "max-degree source, one B200",
    5: "cfg5: 64 sources (seed 5) on the cfg2 road-like grid, sharded over GPUs, rows gathered",
}
# CPU baseline sample sizes (seconds of oracle work): a bounded sample of the workload
CPU_BUDGET_S = 15.0
REF_STEP_BUDGET_S = 2.0


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def host_info():
    """Host the oracle runs on: cores, CPU model, RAM (BASELINE.md:109)."""
    model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    ram = None
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal"):
                ram = round(int(line.split()[1]) / 2 ** 20, 1)
                break
    except OSError:
        pass
    return {"host_cores": os.cpu_count(), "cpu_model": model, "host_ram_gib": ram}


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


# ---------------------------------------------------------------------------------------
# CPU oracle legs (the only places bench.py runs oracle/)
# ---------------------------------------------------------------------------------------

def oracle_sample_single(g, src, budget_s):
    """One Dijkstra from src, stopped after budget_s (a bounded sample; a query that ends
    sooner is complete). Returns (GTEPS = out-edges scanned / time, description)."""
    import oracle
    t0 = time.perf_counter()
    settled, scanned, _ = oracle.dijkstra_budget(g, src, budget_s)
    t = time.perf_counter() - t0
    full = settled >= int(g.n) or t < budget_s
    desc = (f"{'one full' if full else 'a ' + format(budget_s, 'g') + ' s prefix of a'} binary-heap Dijkstra from "
            f"source {src} (single-threaded C, oracle/oracle.c): {settled} vertices settled, {scanned} out-edges "
            f"scanned in {t:.2f} s; GTEPS = edges scanned / time")
    return scanned / t / 1e9, desc, t


def oracle_sample_batch(g, srcs, budget_s):
    """One bounded Dijkstra per source, all host cores in parallel (ctypes drops the GIL).
    Returns (aggregate GTEPS = edges scanned / wall time, cores used, description)."""
    import oracle
    cores = os.cpu_count() or 1
    use = [int(s) for s in srcs[:cores]]
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=len(use)) as ex:
        res = list(ex.map(lambda s: oracle.dijkstra_budget(g, s, budget_s), use))
    t = time.perf_counter() - t0
    scanned = sum(r[1] for r in res)
    desc = (f"{len(use)} binary-heap Dijkstras (the first {len(use)} batch sources, one per host core, each "
            f"stopped after {budget_s:g} s if unfinished; oracle/oracle.c): {scanned} out-edges scanned in "
            f"{t:.2f} s wall; GTEPS = edges scanned / wall time")
    return scanned / t / 1e9, len(use), desc


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    cfg = args.config or (4 if world == 1 else 5)
    g = gen.config_graph(cfg)
    srcs = gen.config_sources(cfg, g, 64) if cfg == 5 else [gen.config_source(cfg, g)]
    vals, times, desc, cores = [], [], "", 1
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        if cfg == 5:
            v, cores, desc = oracle_sample_batch(g, srcs, REF_STEP_BUDGET_S)
        else:
            v, desc, _ = oracle_sample_single(g, int(srcs[0]), REF_STEP_BUDGET_S)
        t1 = time.perf_counter()
        if i >= args.warmup:
            vals.append(v)
            times.append(t1 - t0)
    v = statistics.mean(vals)
    info = host_info()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(times) * 1e3,
            "higher_is_better": True, "scaling": "strong" if cfg == 5 else "weak", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic",
            "config": {"workload": WORKLOAD[cfg], "config": cfg, "sources": [int(s) for s in srcs[:cores]],
                       "n": g.n, "m": g.m},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"per step: {desc}", **info},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------------------

def floors_from(fl, st, kms):
    """Sync floor: grid_syncs x t_sync + launches x t_launch; chain floor:
    the dependent levels (critical_subrounds, and one level per phase) x t_hop."""
    sync_ms = (st.grid_syncs * fl["t_sync_us"] + st.kernel_launches * fl["t_launch_us"]) / 1e3
    levels = st.critical_subrounds + st.grid_syncs
    chain_ms = levels * fl["t_hop_us"] / 1e3
    return {"t_sync_us": fl["t_sync_us"], "t_hop_us": fl["t_hop_us"], "t_launch_us": fl["t_launch_us"],
            "grid_syncs": st.grid_syncs, "dependent_levels": levels,
            "sync_floor_ms": sync_ms, "chain_floor_ms": chain_ms,
            "us_per_level": kms * 1e3 / max(levels, 1),
            "frac_of_chain_floor": chain_ms / kms if kms else None,
            "source": "gi_probe_floors, measured in this run"}


def time_single(gi, torch, G, src, delta, out, opts, steps, warmup, stream):
    """W untimed queries, then K timed ones (CUDA events on the launching stream)."""
    for _ in range(warmup):
        gi.gi_sssp_delta(G, src, delta, out, gi.make_options(**opts))
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats = []
    ev0.record(stream)
    for _ in range(steps):
        stats.append(gi.gi_sssp_delta(G, src, delta, out, gi.make_options(**opts)))
    ev1.record(stream)
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / steps, stats


def counters_of(s):
    return {k: getattr(s, k) for k in ("buckets", "rounds", "grid_syncs", "kernel_launches", "fused_subrounds",
                                       "spills", "vertices_processed", "edges_relaxed", "empty_extractions",
                                       "far_scanned", "critical_subrounds", "ctas", "threads_per_cta", "groups",
                                       "kernel_kind")}


def compare_variants(gi, G, src, delta, out, opts, variants):
    """Counters and device time of option variants (same Δ), 3 runs each (median time)."""
    res = {}
    for name, ov in variants:
        o2 = dict(opts)
        o2.update(ov)
        sts = [gi.gi_sssp_delta(G, src, delta, out, gi.make_options(**o2)) for _ in range(3)]
        s = sts[-1]
        res[name] = {"gpu_ms": statistics.median([x.gpu_ms for x in sts]), **{
            k: getattr(s, k) for k in ("buckets", "rounds", "grid_syncs", "kernel_launches", "fused_subrounds",
                                       "spills", "critical_subrounds", "kernel_kind")}}
    return res


def secondary_cfg2(gi, torch, local, stream, floors, opts):
    """Config 2 (road grid, Δ=2^16): the large-diameter case bucket fusion targets."""
    g = gen.config_graph(2)
    G = gi.Graph.from_csr(g, device=local)
    src, delta = gen.config_source(2, g), DEFAULT_DELTA[2]
    out = torch.empty(g.n, dtype=torch.int32, device="cuda")
    o = {k: v for k, v in opts.items() if k in ("stream",)}
    ms, stats = time_single(gi, torch, G, src, delta, out, o, 10, 3, stream)
    kms = statistics.mean(s.gpu_ms for s in stats)
    d = gi.as_uint32(out)
    n_r, m_r = reached_stats(g, d)
    peak, _ = measured_peak()
    ba = b_alg(g, n_r, m_r)
    # the GPU analogue of table:eager_lazy_perf_impact and table:fusion_perf_impact (PAPER.md
    # :1105-1138): eager + fusion (default), eager without fusion, fully lazy
    comp = compare_variants(gi, G, src, delta, out, o, [("fused", dict(drain="bsp")),
                                                        ("fused_async_drain", dict(drain="async")),
                                                        ("unfused", dict(fusion=False)),
                                                        ("lazy", dict(fusion=False, lazy=True))])
    res = {"workload": WORKLOAD[2], "delta": delta, "ms_per_step": ms, "kernel_ms": kms,
           "value": g.m / (ms * 1e-3) / 1e9, "unit": UNIT,
           "roofline": {"bound": "hbm", "achieved": ba / (kms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": ba / (kms * 1e-3) / 1e9 / peak, "traffic": load_traffic(2, delta),
                        "bytes_alg_per_launch": ba},
           "counters": counters_of(stats[-1]), "fusion_compare": comp,
           "floors": floors_from(floors, stats[-1], kms)}
    G.close()
    return res


def run_single(args, gi, torch, rank, world, local):
    cfg = args.config
    delta = args.delta or DEFAULT_DELTA[cfg]
    t0 = time.perf_counter()
    g = gen.config_graph(cfg)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    G = gi.Graph.from_csr(g, device=local)
    torch.cuda.synchronize()
    t_upload = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    opts = dict(fusion=not args.no_fusion, threshold=args.threshold, max_ctas=args.max_ctas,
                group_ctas=args.group_ctas, hub_min=args.hub_min, pre_read=args.pre_read, drain=args.drain,
                stream=stream, cta_threads=args.cta_threads, expand=args.expand)
    floors = gi.probe_floors(local)
    src = gen.config_source(cfg, g)
    out = torch.empty(g.n, dtype=torch.int32, device="cuda")

    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    ms, stats = time_single(gi, torch, G, src, delta, out, opts, args.steps, max(args.warmup, 0), stream)
    clocks = clk.stop()
    kms = statistics.mean(s.gpu_ms for s in stats)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms, kms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, kms = float(t[0]), float(t[1])
    value = world * g.m / (ms * 1e-3) / 1e9
    if rank != 0:
        return 0

    d_host = gi.as_uint32(out)
    n_r, m_r = reached_stats(g, d_host)
    bytes_alg = b_alg(g, n_r, m_r)
    peak, peak_src = measured_peak()
    achieved = bytes_alg / (kms * 1e-3) / 1e9
    traffic = load_traffic(cfg, delta)
    launches = stats[-1].kernel_launches
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic,
                "kernel": "sssp_persistent" if launches == 1 else
                          f"sssp_persistent segments + expand_kernel + extract_kernel ({launches} launches per query)",
                "kernel_ms": kms,
                "bytes_alg_per_launch": bytes_alg, "peak_source": peak_src,
                "bytes_alg_formula": "12*m_r + 16*n_r + 4*n (SURVEY §8(d))",
                "traffic_source": "profiles/ncu_traffic.json (ncu dram__bytes_read.sum + dram__bytes_write.sum of the "
                                  "query's launches)",
                "note": "achieved = algorithmic bytes / the query's device time (CUDA events around every launch)"}
    s_last = stats[-1]

    compare = None
    if not args.no_compare:
        variants = [("fused", dict(fusion=True)), ("unfused", dict(fusion=False))]
        if int(np.diff(g.offsets).max(initial=0)) <= 8:  # both drains run on low-degree graphs
            variants = [("fused", dict(fusion=True, drain="bsp")),
                        ("fused_async_drain", dict(fusion=True, drain="async")), ("unfused", dict(fusion=False))]
        else:
            variants += [("fused_expand", dict(fusion=True, expand="on")),
                         ("fused_no_expand", dict(fusion=True, expand="off"))]
        variants.append(("lazy", dict(fusion=False, lazy=True)))
        compare = compare_variants(gi, G, src, delta, out, opts, variants)

    # ---- e2e through the public C ABI with HOST buffers (pinned), copies inside ----
    host_out = torch.empty(g.n, dtype=torch.int32, pin_memory=True)
    host_src = torch.tensor([src], dtype=torch.int32).pin_memory()
    o_e2e = dict(opts)
    o_e2e.pop("stream")
    times = []
    for i in range(args.warmup + args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s_val = int(host_src[0])  # source id read from pinned host memory (4 bytes H2D inside the call)
        gi.gi_sssp_delta(G, s_val, delta, host_out.numpy(), gi.make_options(**o_e2e))
        t1 = time.perf_counter()
        if i >= args.warmup:
            times.append(t1 - t0)
    te = statistics.mean(times)
    e2e = {"value": world * g.m / te / 1e9, "unit": UNIT, "h2d_bytes_per_step": 4, "d2h_bytes_per_step": 4 * g.n,
           "ms_per_step": te * 1e3, "api": "gi_sssp_delta_ex with a pinned host dist_out (library stages + copies back)"}
    assert np.array_equal(host_out.numpy().view(np.uint32), d_host)

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, desc, _ = oracle_sample_single(g, src, CPU_BUDGET_S)
        cpu = {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc, **host_info()}

    secondary = None
    if cfg == 4 and world == 1 and not args.no_secondary:
        secondary = {"cfg2": secondary_cfg2(gi, torch, local, stream, floors, opts),
                     "cfg5_one_gpu": run_batch_anchor(gi, torch, local, stream)}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": WORKLOAD[cfg], "config": cfg, "delta": delta, "source": src,
                   "fusion": not args.no_fusion, "threshold": args.threshold or "default", "n": g.n, "m": g.m,
                   "n_reached": n_r, "m_reached": m_r, "time_per_source_ms": ms,
                   "l2": f"inputs larger than L2 (CSR {(g.offsets.nbytes + 8 * g.m) / 1e6:.0f} MB > 126 MB); "
                         "dist re-initialised every step",
                   "parallelism": f"replica x{world}" if world > 1 else "one GPU",
                   "graph_gen_s": round(t_gen, 1), "graph_upload_s": round(t_upload, 2)},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": stats[-1].kernel_launches * args.steps,
        "clocks": clocks, "counters": counters_of(s_last), "fusion_compare": compare,
        "floors": floors_from(floors, s_last, kms), "secondary": secondary,
    }
    print(json.dumps(line), flush=True)
    return 0


def run_batch_anchor(gi, torch, local, stream):
    """Config 5 on one GPU (the N=1 point of the batch scaling curve): 64 sources through
    the fused-gather entry point with one peer (this GPU's own matrix)."""
    g = gen.config_graph(5)
    G = gi.Graph.from_csr(g, device=local)
    srcs_all = gen.config_sources(5, g, 64)
    full = torch.empty((64, g.n), dtype=torch.int32, device="cuda")
    srcs = torch.from_numpy(srcs_all.copy())
    delta = DEFAULT_DELTA[5]
    o = gi.make_options(stream=stream)
    gi.gi_sssp_batch_peers(G, srcs, delta, [full.data_ptr()], 0, o)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    sts = [gi.gi_sssp_batch_peers(G, srcs, delta, [full.data_ptr()], 0, o) for _ in range(3)]
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / 3
    G.close()
    return {"workload": WORKLOAD[5], "delta": delta, "ms_per_step": ms, "time_per_source_ms": ms / 64,
            "kernel_ms": sts[-1][0].gpu_ms, "value": 64 * g.m / (ms * 1e-3) / 1e9, "unit": UNIT}


def run_batch(args, gi, torch, rank, world, local):
    """Config 5: 64 sources sharded over the ranks (contiguous blocks), graph replicated."""
    import torch.distributed as dist
    from paper_1911_07260_b200.dist import (exchange_handles, peer_row_addresses, shard_bounds,
                                            sssp_batch_multi_gpu)
    delta = args.delta or DEFAULT_DELTA[5]
    g = gen.config_graph(5)
    G = gi.Graph.from_csr(g, device=local)
    stream = torch.cuda.current_stream()
    srcs_all = gen.config_sources(5, g, 64)
    k = len(srcs_all)
    lo, hi = shard_bounds(k, rank, world)
    srcs = torch.from_numpy(srcs_all[lo:hi].copy())
    # every rank holds the whole [64, n] result; the kernel writes each finished row into
    # every rank's copy over NVLink (gi_sssp_batch_peers): the gather is fused into compute
    full = torch.empty((k, g.n), dtype=torch.int32, device="cuda")
    bases, opened = exchange_handles(full, rank, world, local) if world > 1 else ([full.data_ptr()], [])
    peers = peer_row_addresses(bases, lo, g.n)
    o = gi.make_options(stream=stream)

    def step_fused():
        return gi.gi_sssp_batch_peers(G, srcs, delta, peers, rank, o)

    def barrier():
        if world > 1:
            dist.barrier()

    def timed(step, steps, warmup):
        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        kms = []
        for _ in range(steps):
            st = step()
            barrier()  # the job's step ends when every rank's rows are in every matrix
            if st is not None:
                kms.append(st[0].gpu_ms)
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ms = ev0.elapsed_time(ev1) / steps
        km = statistics.mean(kms) if kms else None
        if world > 1:
            t = torch.tensor([ms, km or 0.0], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms, km = float(t[0]), float(t[1])
        return ms, km

    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    ms, kms = timed(step_fused, args.steps, max(args.warmup, 0))
    clocks = clk.stop()
    gather = {"fused_peer_stores": {"ms_per_step": ms, "max_rank_kernel_ms": kms}}
    if args.gather in ("nccl", "both") and world > 1:
        def step_nccl():
            sssp_batch_multi_gpu(G, srcs_all, delta, stream=stream)
            return None
        ms_n, _ = timed(step_nccl, args.steps, 1)
        gather["nccl_all_gather"] = {"ms_per_step": ms_n,
                                     "api": "gi.sssp_batch on the rank's block, then all_gather_into_tensor"}
    value = k * g.m / (ms * 1e-3) / 1e9

    # e2e: the public batch API with HOST buffers — this rank's sources from pinned memory,
    # its rows copied back to pinned host memory inside the timed region
    host_rows = torch.empty((hi - lo, g.n), dtype=torch.int32, pin_memory=True)
    host_srcs = torch.from_numpy(srcs_all[lo:hi].copy()).pin_memory()
    te_list = []
    for i in range(max(args.warmup, 1) + args.steps):
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        if hi > lo:
            gi.gi_sssp_batch(G, host_srcs.numpy(), delta, host_rows.numpy(), gi.make_options())
        barrier()
        t1 = time.perf_counter()
        if i >= max(args.warmup, 1):
            te_list.append(t1 - t0)
    te = statistics.mean(te_list)
    if world > 1:
        t = torch.tensor([te], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        te = float(t[0])
    for addr, off in opened:  # every rank is past the last barrier: no peer writes remain
        gi.ipc_close(addr, off, local)
    if rank != 0:
        dist.destroy_process_group()
        return 0

    rows = gi.as_uint32(full)
    # parity sample (not timed): the 64x64 symmetry of the gathered matrix (a symmetric
    # graph has δ(si, sj) == δ(sj, si)), and one row per rank against the oracle
    M = rows[:, srcs_all.astype(np.int64)]
    parity = {"symmetry_64x64": bool(np.array_equal(M, M.T))}
    if not args.no_cpu_baseline:
        import oracle
        check = [shard_bounds(k, r, world)[0] for r in range(world) if shard_bounds(k, r, world)[1] >
                 shard_bounds(k, r, world)[0]]
        refs, _, _ = oracle.dijkstra_many(g, srcs_all[check])
        parity["rows_vs_oracle"] = {"rows": check, "bit_exact": bool(np.array_equal(rows[check], refs))}
    bytes_alg = sum(b_alg(g, *reached_stats(g, rows[i])) for i in range(lo, hi))
    peak, peak_src = measured_peak()
    achieved = bytes_alg / (kms * 1e-3) / 1e9 if kms else None
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, cores, desc = oracle_sample_batch(g, srcs_all, CPU_BUDGET_S)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc, **host_info()}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": WORKLOAD[5], "config": 5, "delta": delta, "nsrc": k, "n": g.n, "m": g.m,
                   "time_per_source_ms": ms / k, "rank0_block": [lo, hi],
                   "l2": "inputs larger than L2 (CSR 649 MB > 126 MB); dist re-initialised every step",
                   "parallelism": f"sources sharded x{world}, rows gathered by peer stores"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if achieved else None, "traffic": load_traffic(5, delta),
                     "kernel": "sssp_persistent", "kernel_ms_max_rank": kms, "bytes_alg_per_launch": bytes_alg,
                     "peak_source": peak_src, "note": "rank 0's rows over the slowest rank's kernel time"},
        "cpu_baseline": cpu,
        "e2e": {"value": k * g.m / te / 1e9, "unit": UNIT, "h2d_bytes_per_step": 4 * k,
                "d2h_bytes_per_step": 4 * k * g.n, "ms_per_step": te * 1e3,
                "api": "gi_sssp_batch_ex per rank with pinned host sources and rows"},
        "gpu_launches": args.steps, "clocks": clocks, "gather": gather, "parity": parity,
        "per_rank": {"wall_ms_per_step": ms, "kernel_ms_max_rank": kms},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0 if parity["symmetry_64x64"] and parity.get("rows_vs_oracle", {}).get("bit_exact", True) else 1


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
                "sample": f"one serial peel (oracle/oracle.c), {t_or:.3f} s", **host_info()},
            "counters": {k: getattr(st, k) for k in ("buckets", "rounds", "grid_syncs", "vertices_processed",
                                                      "edges_relaxed", "empty_extractions", "fused_subrounds",
                                                      "critical_subrounds", "spills", "kernel_kind")}}
    print(json.dumps(line), flush=True)
    return 0 if line["parity"] is not False else 1


def run_app(args, gi, torch, rank, world, local):
    """PPSP / A* on the config's source and a seeded target; checked
    against the Dijkstra oracle's dist[target] (rank 0) and timed with CUDA events."""
    import oracle
    cfg = args.config
    delta = args.delta or DEFAULT_DELTA[cfg]
    g = gen.config_graph(cfg)
    G = gi.Graph.from_csr(g, device=local)
    stream = torch.cuda.current_stream()
    opts = dict(fusion=not args.no_fusion, threshold=args.threshold, max_ctas=args.max_ctas,
                group_ctas=args.group_ctas, hub_min=args.hub_min, pre_read=args.pre_read, drain=args.drain,
                stream=stream, cta_threads=args.cta_threads, expand=args.expand)
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
               "sample": f"one full Dijkstra from source {src} (oracle/oracle.c), {t_or:.3f} s", **host_info()}
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
    ap.add_argument("--config", type=int, default=0, choices=[0, 1, 2, 3, 4, 5],
                    help="0 = default: config 4 on one GPU, config 5 (sharded batch) with N > 1")
    ap.add_argument("--delta", type=int, default=0)
    ap.add_argument("--threshold", type=int, default=0)
    ap.add_argument("--no-fusion", action="store_true")
    ap.add_argument("--max-ctas", type=int, default=0)
    ap.add_argument("--group-ctas", type=int, default=0)
    ap.add_argument("--hub-min", type=int, default=0)
    ap.add_argument("--pre-read", type=int, default=0, help="0 auto, 1 on, 2 off")
    ap.add_argument("--expand", default="auto", choices=["auto", "on", "off"],
                    help="edge-balanced expansion of high-degree frontier vertices in expand_kernel (skewed graphs)")
    ap.add_argument("--cta-threads", type=int, default=0, choices=[0, 512, 1024],
                    help="threads per persistent CTA (0 = auto: 1024 on skewed graphs)")
    ap.add_argument("--drain", default="auto", choices=["auto", "bsp", "async"],
                    help="fused drain: per-sub-round CTA barriers (default) or the barrier-free async ring")
    ap.add_argument("--gather", default="both", choices=["fused", "nccl", "both"],
                    help="config 5 with N > 1: time the fused peer-store gather, the NCCL all-gather arm, or both")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="config 4: skip the config-2 / config-5 keys")
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
    if not args.config:
        args.config = 4 if world == 1 else 5
    if args.app != "sssp":
        return run_app(args, gi, torch, rank, world, local)
    if args.config == 5:
        return run_batch(args, gi, torch, rank, world, local)
    rc = run_single(args, gi, torch, rank, world, local)
    if world > 1:
        dist.destroy_process_group()
    return rc


if __name__ == "__main__":
    sys.exit(main())
