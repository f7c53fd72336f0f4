"""Multi-rank batch path (paper_1911_07260_b200/dist.py) on CPU with the gloo backend,
world_size 2: sharding, padding, all-gather and row order. The per-rank compute is the
oracle (a CPU stand-in for the GPU kernel), so the test checks the host logic only."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
import oracle
from paper_1911_07260_b200.dist import padded_shard, shard_bounds, unpad_rows


def test_shard_bounds_cover_exactly():
    for k in (0, 1, 5, 64, 65, 127):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                lo, hi = shard_bounds(k, r, world)
                assert 0 <= lo <= hi <= k
                seen.extend(range(lo, hi))
            assert seen == list(range(k))
            sizes = [shard_bounds(k, r, world)[1] - shard_bounds(k, r, world)[0] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def test_pad_unpad_roundtrip():
    srcs = np.arange(10, 17, dtype=np.int32)  # k = 7
    for world in (1, 2, 3, 4):
        per = -(-7 // world)
        parts = []
        for r in range(world):
            p, nreal = padded_shard(srcs, r, world)
            assert p.shape[0] == per
            parts.append(p)
        gathered = np.concatenate(parts)[:, None]
        assert unpad_rows(gathered, 7, world)[:, 0].tolist() == srcs.tolist()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1911_07260_b200.dist import sssp_batch_multi_gpu
    g = gen.grid(24, 24, 1, 100, 9, p_del=0.1)
    srcs = gen.sources(g.n, 7, 5)

    def compute(s):
        out, _, _ = oracle.dijkstra_many(g, s, threads=1)
        return torch.from_numpy(out.view(np.int32).copy())

    got = sssp_batch_multi_gpu(None, srcs, 10, compute=compute)
    q.put((rank, got.numpy().view(np.uint32).copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_batch_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = gen.grid(24, 24, 1, 100, 9, p_del=0.1)
    srcs = gen.sources(g.n, 7, 5)
    ref, _, _ = oracle.dijkstra_many(g, srcs)
    for r in (0, 1):
        assert np.array_equal(res[r], ref)


def test_peer_row_addresses():
    from paper_1911_07260_b200.dist import peer_row_addresses
    assert peer_row_addresses([1000, 5000], 0, 10) == [1000, 5000]
    assert peer_row_addresses([1 << 40, 7 << 40], 3, 1001) == [(1 << 40) + 3 * 1001 * 4, (7 << 40) + 3 * 1001 * 4]


class _FakeIpc:
    """Stands in for gi's IPC calls: a 'handle' names the rank; opening it returns a
    recognisable address so the exchange's bookkeeping can be checked without a GPU."""

    def __init__(self, rank):
        self.rank = rank

    def ipc_handle(self, out):
        return (b"rank%d" % self.rank).ljust(64, b"\0"), 256 * self.rank

    def ipc_open(self, h, off, device):
        r = int(h.rstrip(b"\0")[4:])
        return (r + 1) * 10**9 + off


class _FakeOut:
    def __init__(self, addr):
        self.addr = addr

    def data_ptr(self):
        return self.addr


def _worker_handles(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1911_07260_b200.dist import exchange_handles
    bases, opened = exchange_handles(_FakeOut(77 + rank), rank, world, 0, ipc=_FakeIpc(rank))
    q.put((rank, bases, opened))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_ipc_handle_exchange():
    """exchange_handles (the fused-gather setup of dist.sssp_batch_fused_gather): every rank
    ends with rank-ordered bases, its own matrix at its own index and the others opened."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_handles, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {r: (b, o) for r, b, o in (q.get(timeout=120) for _ in range(2))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == ([77, 2 * 10**9 + 256], [(2 * 10**9 + 256, 256)])
    assert res[1] == ([1 * 10**9 + 0, 78], [(10**9, 0)])
