"""The N>1 path on CPU: world_size 2 over gloo.  Each rank fills its shard
of a decision grid (a deterministic function of the flat index stands in for
the device sweep) and the all-gather must reproduce the single-rank grid
exactly, for shard counts that do and do not divide the grid."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_10187_b200.dist import ENTRY_INTS, gather_grid, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _entry(idx: torch.Tensor):
    # stand-in for the sweep: any pure function of the flat shape index
    cols = [idx * 7 + k * 1000003 for k in range(ENTRY_INTS)]
    return torch.stack(cols, 1).to(torch.int32)


def _worker(rank, world, port, n_entries, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local = torch.full((n_entries, ENTRY_INTS), -1, dtype=torch.int32)

        def fill(lo, hi):
            local[lo:hi] = _entry(torch.arange(lo, hi))

        gather_grid(local, n_entries, fill=fill)
        want = _entry(torch.arange(n_entries))
        q.put((rank, bool(torch.equal(local, want))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_entries", [32768, 32771, 5])
def test_gloo_sharded_grid_equals_single_rank(n_entries):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_entries, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


def test_shard_bounds_cover_exactly():
    for n in (1, 5, 32768, 393216, 393217):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                lo, hi, per = shard_bounds(n, world, r)
                assert hi - lo <= per
                seen.extend(range(lo, hi))
            assert seen == list(range(n))


# ---- build exchange protocol (dist.exchange_packed) on gloo -------------
def _blob(rank):
    # rank r sends 1000 * r + 37 bytes (rank 1 of 3 sends nothing), content
    # a function of (rank, position); counts carry the rank
    n = 0 if rank == 1 else 1000 * rank + 37
    return n, torch.arange(n, dtype=torch.int64).mul(31).add(rank * 7).remainder(251).to(torch.uint8)


def _xworker(rank, world, port, q):
    from paper_2604_10187_b200.dist import PACK_ALIGN, exchange_packed

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, data = _blob(rank)
        counts = [rank + 1, 2 * rank, 3 * rank, 40, 10] if n else [0, 0, 0, 40, 10]

        def pack(dst):
            assert dst.numel() >= n
            dst[:n] = data

        buf, stride, allc = exchange_packed(n, counts, pack, "cpu")
        ok = stride % PACK_ALIGN == 0 and buf.numel() == world * stride
        for r in range(world):
            nr, dr = _blob(r)
            ok = ok and stride >= nr and torch.equal(buf[r * stride: r * stride + nr], dr)
            want = [r + 1, 2 * r, 3 * r, 40, 10] if nr else [0, 0, 0, 40, 10]
            ok = ok and allc[r].tolist() == want
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_exchange_packed_blobs(world):
    """Variable-size blobs (one rank empty) land at rank * stride on every
    rank, with every rank's counts -- the layout wt_build_merge consumes."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_xworker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(world)}
