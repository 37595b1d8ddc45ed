"""The fused sharded sweep through real CUDA IPC: two processes on the same
GPU (gloo for the handle exchange and barriers) each map the other's grid
storage with wt_ipc_open and sweep their slice into both grids from the
kernel epilogue (wt_sweep_to).  Both grids must equal a full single-process
sweep bit for bit, and gathers must agree after finalize."""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here), here]
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2604_10187_b200 import capi, synthetic as S
        from paper_2604_10187_b200.dist import fused_sharded_sweep

        cfg = S.config_space(False)
        eng = capi.Engine(S.synthetic_tables(cfg), S.registry_arrays(cfg), n_sm=148)
        pairs = S.LLAMA3_8B
        g = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 5000)
        g.entries_tensor().fill_(-3)
        torch.cuda.synchronize()
        fused_sharded_sweep(g)
        ref = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 5000)
        ref.sweep()
        torch.cuda.synchronize()
        ok = bool(torch.equal(g.entries_tensor(), ref.entries_tensor()))
        q.put((rank, ok))
        dist.barrier()
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)[:500]))
    finally:
        dist.destroy_process_group()


def test_fused_sharded_sweep_over_ipc_two_processes():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    assert res == {0: True, 1: True}, res
