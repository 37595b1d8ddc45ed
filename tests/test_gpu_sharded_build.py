"""The device-resident multi-GPU build (dist.sharded_build): each rank fits
its contiguous registry slice from records in its HBM, packs the tables
(wt_build_pack), one all-gather moves the blobs, every rank merges them
(wt_build_merge) and resolves its engine image on the device.

On one GPU: the shards' packed blobs laid out exactly as the all-gather
leaves them, merged, must equal the single build of the whole registry bit
for bit (every array) and give the same decision grid.  Two processes on the
same GPU drive dist.sharded_build end to end (gloo moves the blobs through
the host; the pack / merge kernels and the layout are the real ones)."""
import os
import socket

import numpy as np
import pytest

import wtutil as U

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def capi():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_10187_b200 import capi as c

    c.lib()
    return c


def dev_records(rec):
    cv = {"g": torch.int64, "l": torch.int64, "w": torch.int32, "macro": torch.int32, "micro": torch.int32,
          "lat": torch.float64}
    return {k: torch.as_tensor(np.ascontiguousarray(rec[k])).to(dtype=cv[k], device="cuda") for k in cv}


INT_KEYS = ("macro_id", "coeff_off", "coeff_w", "awave_off", "awave_w", "awave_aoff", "anchor_l", "anchor_micro",
            "anchor_partial", "ext_aoff", "ext_l", "ext_micro", "ext_flags", "diag_samples", "diag_flags")
F64_KEYS = ("coeff_theta", "theta_ext", "diag_r2", "diag_mape")


def same_tables(a, b):
    for k in INT_KEYS:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    for k in F64_KEYS:
        np.testing.assert_array_equal(U.bits(a[k]), U.bits(b[k]), err_msg=k)
    assert a["W"] == b["W"] and a["n_tables"] == b["n_tables"] and a["p"] == b["p"]


def merge_on_one_gpu(capi, rec, ids_all, world, W, p=10, drop_rank=None):
    """What sharded_build does across ranks, with the all-gather replaced by
    laying the blobs out at rank * stride in one buffer."""
    from paper_2604_10187_b200.dist import PACK_ALIGN, macro_shards, records_of

    parts, counts, sizes = [], [], []
    for r, ids in enumerate(macro_shards(ids_all, world)):
        mine = records_of(rec, ids)
        if r == drop_rank or not len(ids) or not len(mine["g"]):
            parts.append(None)
            counts.append([0, 0, 0, W, p])
            sizes.append(0)
            continue
        b = capi.Build(dev_records(mine), ids, W, p)
        c, n = b.pack_info()
        parts.append(b)
        counts.append(list(c))
        sizes.append(n)
    stride = max(PACK_ALIGN, -(-max(sizes) // PACK_ALIGN) * PACK_ALIGN)
    buf = torch.full((world * stride,), 0xA5, dtype=torch.uint8, device="cuda")  # poison the padding
    for r, b in enumerate(parts):
        if b is not None:
            b.pack(buf[r * stride:(r + 1) * stride])
    merged = capi.Build.merge(buf, stride, np.array(counts, np.int64))
    for b in parts:
        if b is not None:
            b.close()
    return merged


@pytest.mark.parametrize("world", [2, 3, 8])
def test_packed_merge_equals_full_build(capi, world):
    from paper_2604_10187_b200 import synthetic as S

    cfg = S.config_space(False)
    rec = S.synthetic_records(cfg, micros_per_macro=2)
    full = capi.Build(dev_records(rec), cfg["id"], 40, 10)
    merged = merge_on_one_gpu(capi, rec, cfg["id"], world, 40)
    same_tables(merged.result(), full.result())
    # the merged build feeds the device image like a local one
    reg = S.registry_arrays(cfg)
    e1 = capi.Engine.from_build(merged, reg, n_sm=148)
    e2 = capi.Engine.from_build(full, reg, n_sm=148)
    pairs = S.LLAMA3_8B
    g1 = capi.Grid(e1, [q[0] for q in pairs], [q[1] for q in pairs], 1, 8192)
    g2 = capi.Grid(e2, [q[0] for q in pairs], [q[1] for q in pairs], 1, 8192)
    g1.sweep()
    g2.sweep()
    torch.cuda.synchronize()
    assert torch.equal(g1.entries_tensor(), g2.entries_tensor())
    for x in (g1, g2, e1, e2, merged, full):
        x.close()


def test_packed_merge_config3_with_empty_rank(capi):
    """Config 3 (4,608 tables) over 8 ranks, one of which holds no records:
    its tables are simply absent, like a single build over the same records."""
    from paper_2604_10187_b200 import synthetic as S
    from paper_2604_10187_b200.dist import macro_shards

    cfg = S.config_space(True)
    rec = S.synthetic_records(cfg, micros_per_macro=1)
    drop = set(macro_shards(cfg["id"], 8)[5].tolist())
    keep = ~np.isin(rec["macro"], list(drop))
    rec_k = {k: v[keep] for k, v in rec.items()}
    full = capi.Build(dev_records(rec_k), cfg["id"], 40, 10)
    merged = merge_on_one_gpu(capi, rec_k, cfg["id"], 8, 40)
    a, b = merged.result(), full.result()
    same_tables(a, b)
    assert a["n_tables"] == len(cfg["id"]) - len(drop)


def test_merge_rejects_mismatched_parts(capi):
    from paper_2604_10187_b200 import synthetic as S

    cfg = S.config_space(False)
    rec = S.synthetic_records(cfg)
    b = capi.Build(dev_records(rec), cfg["id"], 40, 10)
    c, n = b.pack_info()
    buf = torch.empty(2 * n, dtype=torch.uint8, device="cuda")
    b.pack(buf[:n])
    b.pack(buf[n:])
    bad = np.array([c, c], np.int64)
    bad[1, 3] = 39  # another W
    with pytest.raises(RuntimeError, match="different W"):
        capi.Build.merge(buf, n, bad)
    with pytest.raises(RuntimeError, match="no macro"):
        capi.Build.merge(buf, n, np.zeros((2, 5), np.int64))
    small = np.array([c, c], np.int64)
    with pytest.raises(RuntimeError, match="stride"):
        capi.Build.merge(buf, n - 256, small)
    with pytest.raises(RuntimeError, match="smaller"):
        b.pack(buf[: n - 1])
    b.close()


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
        from paper_2604_10187_b200.dist import global_w, shard_records, sharded_build, sharded_sweep

        cfg = S.config_space(False)
        rec = S.synthetic_records(cfg, micros_per_macro=2)
        ids, mine = shard_records(rec, cfg["id"], world, rank)
        W = global_w(mine["w"])
        st = torch.cuda.Stream()
        merged = sharded_build(dev_records(mine), ids, W, 10, device=0, stream=st)
        reg = S.registry_arrays(cfg)
        eng = capi.Engine.from_build(merged, reg, n_sm=148, stream=st)
        pairs = S.LLAMA3_8B
        g = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 5000, stream=st)
        sharded_sweep(g, stream=st)
        st.synchronize()
        full = capi.Build(dev_records(rec), cfg["id"], 0, 10)
        same_tables(merged.result(), full.result())
        ef = capi.Engine.from_build(full, reg, n_sm=148)
        ref = capi.Grid(ef, [p[0] for p in pairs], [p[1] for p in pairs], 1, 5000)
        ref.sweep()
        torch.cuda.synchronize()
        ok = bool(torch.equal(g.entries_tensor(), ref.entries_tensor()))
        q.put((rank, ok))
        dist.barrier()
    except Exception as e:  # noqa: BLE001
        import traceback

        q.put((rank, traceback.format_exc()[-1500:]))
    finally:
        dist.destroy_process_group()


def test_sharded_build_two_processes():
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
