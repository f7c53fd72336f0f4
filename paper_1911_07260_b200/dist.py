"""Multi-GPU batch of independent sources (north_star: "Batches of
independent sources are split across GPUs, with the graph replicated per GPU and results
gathered over NCCL/NVLink. A single-source query runs on one GPU.").

One process per GPU (torchrun). Every rank holds a replica of the graph (generated
deterministically, so no broadcast is needed) and computes a contiguous block of sources.

Two ways to assemble the [k, n] result on every rank:
- ``sssp_batch_fused_gather`` (the product path): every rank's result matrix is mapped into
  every other rank (CUDA IPC handles exchanged once over the process group), and the
  kernel itself writes each finished row into all of them over NVLink while its other CTA
  groups keep computing (``gi_sssp_batch_peers``). No collective moves data; one barrier
  marks completion.
- ``sssp_batch_multi_gpu``: ``gi_sssp_batch`` then an NCCL all-gather of the rows (the
  baseline the fused path replaces; also the gloo-testable reference for the sharding).
"""
from __future__ import annotations

import numpy as np


def shard_bounds(k: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of k sources for `rank` (sizes differ by at most one)."""
    base, extra = divmod(k, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def padded_shard(srcs, rank: int, world: int):
    """Rank's sources padded (with its own first source, duplicates are allowed) to the
    common per-rank row count ceil(k/world) so that the gather has equal-sized parts.
    Returns (padded int32 array, number of real rows)."""
    srcs = np.asarray(srcs, dtype=np.int32)
    k = srcs.shape[0]
    per = -(-k // world) if k else 0
    lo, hi = shard_bounds(k, rank, world)
    mine = srcs[lo:hi]
    if per == 0:
        return np.zeros(0, np.int32), 0
    pad = np.full(per - mine.shape[0], mine[0] if mine.shape[0] else srcs[0], np.int32)
    return np.concatenate([mine, pad]), mine.shape[0]


def unpad_rows(gathered, k: int, world: int):
    """Drop the padding rows of a [world * per, n] gather -> [k, n] in source order."""
    per = -(-k // world) if k else 0
    rows = []
    for r in range(world):
        lo, hi = shard_bounds(k, r, world)
        rows.append(gathered[r * per: r * per + (hi - lo)])
    import torch
    if isinstance(gathered, torch.Tensor):
        return torch.cat(rows, 0)
    return np.concatenate(rows, 0)


def sssp_batch_multi_gpu(G, srcs, delta: int, compute=None, **opts):
    """All ranks call this with the same ``srcs``; returns the [k, n] int32 tensor of
    distances (uint32 bit patterns) on every rank.

    ``compute(local_srcs_int32_numpy) -> torch.Tensor [len, n] int32`` defaults to
    ``gi.sssp_batch`` on this rank's GPU (tests substitute a CPU stand-in under gloo)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    srcs = np.asarray(srcs, dtype=np.int32)
    k = srcs.shape[0]
    mine, nreal = padded_shard(srcs, rank, world)
    if compute is None:
        from . import gi

        def compute(s):
            out, _ = gi.sssp_batch(G, s, delta, **opts)
            return out
    local = compute(mine)
    if world == 1:
        return local[:k]
    backend = dist.get_backend()
    if backend == "nccl":
        gathered = torch.empty((local.shape[0] * world, local.shape[1]), dtype=local.dtype,
                               device=local.device)
        dist.all_gather_into_tensor(gathered, local.contiguous())
    else:
        parts = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(parts, local.contiguous())
        gathered = torch.cat(parts, 0)
    return unpad_rows(gathered, k, world)


def peer_row_addresses(bases, lo: int, n: int, itemsize: int = 4):
    """Device address of row `lo` in each rank's [k, n] matrix (base addresses `bases`)."""
    return [int(b) + lo * n * itemsize for b in bases]


def exchange_handles(out, rank: int, world: int, device: int, all_gather_object=None, ipc=None):
    """Map every rank's result matrix into this process. Returns (bases, opened) where
    bases[r] is the device address of rank r's matrix as seen from this rank and opened
    lists (address, offset) pairs to close after the final barrier."""
    if ipc is None:
        from . import gi as ipc
    if all_gather_object is None:
        import torch.distributed as dist
        all_gather_object = dist.all_gather_object
    mine = ipc.ipc_handle(out)
    allh = [None] * world
    all_gather_object(allh, mine)
    bases, opened = [], []
    for r in range(world):
        if r == rank:
            bases.append(int(out.data_ptr()))
        else:
            h, off = allh[r]
            addr = ipc.ipc_open(h, off, device)
            bases.append(addr)
            opened.append((addr, off))
    return bases, opened


def sssp_batch_fused_gather(G, srcs, delta: int, out=None, **opts):
    """All ranks call this with the same ``srcs``; returns the [k, n] int32 tensor of
    distances (uint32 bit patterns) on every rank, assembled by the kernels' own peer
    stores (``gi_sssp_batch_peers``)."""
    import torch
    import torch.distributed as dist
    from . import gi

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    srcs = np.asarray(srcs, dtype=np.int32)
    k = srcs.shape[0]
    n = G.n
    if out is None:
        out = torch.empty((k, n), dtype=torch.int32, device=f"cuda:{G.device}")
    if world == 1:
        bases, opened = [int(out.data_ptr())], []
    else:
        bases, opened = exchange_handles(out, rank, world, G.device)
    lo, hi = shard_bounds(k, rank, world)
    if hi > lo:
        gi.gi_sssp_batch_peers(G, srcs[lo:hi], delta, peer_row_addresses(bases, lo, n), rank,
                               gi.make_options(**opts) if opts else None)
    if world > 1:
        dist.barrier()  # every rank's kernel has completed: all rows are in every matrix
        for addr, off in opened:
            gi.ipc_close(addr, off, G.device)
    return out
