"""The sharded fit on CPU: world_size 2 over gloo.  A deterministic per-macro
stand-in for the GPU fit (same CSR table layout as capi.fit_build) must give,
sharded by macro and merged, exactly the single-rank table set -- including
ranks without records and W <= 0 (the global max record wave)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_10187_b200.dist import macro_shards, merge_tables, records_of, sharded_fit


def fake_fit(records, ids, W, p, device=0):
    """Per macro (registry order): one coeff entry per distinct wave, two
    anchors per wave, one ext anchor, one step entry -- values derived from
    the macro's own records only (as build_dual_table)."""
    tabs = [m for m in ids if np.any(records["macro"] == m)]
    nt = len(tabs)
    out = {k: [] for k in ("macro_id", "theta_ext", "ext_flags", "W_arr", "lin_theta", "lin_r2", "lin_mape",
                           "lin_degenerate", "coeff_w", "coeff_theta", "diag_r2", "diag_mape", "diag_samples",
                           "diag_flags", "awave_w", "anchor_l", "anchor_micro", "anchor_partial", "ext_l",
                           "ext_micro", "step_l", "step_t")}
    offs = {k: [0] for k in ("coeff_off", "awave_off", "ext_aoff", "step_off")}
    aoff = [0]
    for m in tabs:
        r = records["macro"] == m
        waves = np.unique(records["w"][r])
        s = float(records["lat"][r].sum())
        out["macro_id"].append(m)
        out["theta_ext"] += [s, W, p, m]
        out["ext_flags"].append(int(m) % 3)
        out["W_arr"].append(W)
        out["lin_theta"] += [m, s, 1.0, 2.0]
        out["lin_r2"].append(s / 7)
        out["lin_mape"].append(s / 11)
        out["lin_degenerate"].append(0)
        for w in waves:
            out["coeff_w"].append(w)
            out["coeff_theta"] += [m, w, s, 1.0]
            out["diag_r2"].append(w / 3)
            out["diag_mape"].append(w / 5)
            out["diag_samples"].append(int((records["w"][r] == w).sum()))
            out["diag_flags"].append(0)
            out["awave_w"].append(w)
            out["anchor_l"] += [16, 32]
            out["anchor_micro"] += [m * 4, m * 4 + 1]
            out["anchor_partial"] += [0, 1]
            aoff.append(aoff[-1] + 2)
        out["ext_l"].append(64)
        out["ext_micro"].append(m * 4 + 2)
        out["step_l"].append(16)
        out["step_t"].append(s)
        offs["coeff_off"].append(offs["coeff_off"][-1] + len(waves))
        offs["awave_off"].append(offs["awave_off"][-1] + len(waves))
        offs["ext_aoff"].append(offs["ext_aoff"][-1] + 1)
        offs["step_off"].append(offs["step_off"][-1] + 1)
    res = {"n_tables": nt, "W": W, "p": p, "device_ms": 0.0}
    for k, v in out.items():
        res[k] = np.asarray(v)
    for k, v in offs.items():
        res[k] = np.asarray(v, np.int32)
    res["awave_aoff"] = np.asarray(aoff, np.int32)
    return res


def synthetic_records(seed=0):
    rng = np.random.default_rng(seed)
    n = 4000
    macro = rng.choice(np.array([3, 5, 8, 13, 21, 34, 55]), n)  # registry has ids without records too
    return {"g": rng.integers(1, 5000, n), "l": rng.integers(1, 200, n), "w": rng.integers(1, 40, n).astype(np.int32),
            "macro": macro.astype(np.int32), "micro": rng.integers(0, 8, n).astype(np.int32),
            "lat": rng.random(n)}


REGISTRY = np.array([1, 3, 5, 8, 13, 21, 34, 55, 89], np.int32)


def _equal(a, b):
    assert a["n_tables"] == b["n_tables"]
    for k in a:
        if isinstance(a[k], np.ndarray):
            np.testing.assert_array_equal(a[k], b[k], err_msg=k)


def test_merge_of_shards_equals_full_fit():
    rec = synthetic_records()
    full = fake_fit(rec, REGISTRY, 40, 10)
    for world in (1, 2, 3, 4, 9):
        parts = [fake_fit(records_of(rec, ids), ids, 40, 10) for ids in macro_shards(REGISTRY, world)]
        _equal(merge_tables(parts), full)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, W, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rec = synthetic_records()
        got = sharded_fit(rec, REGISTRY, W=W, p=10, fit=fake_fit)
        want = fake_fit(rec, REGISTRY, W if W > 0 else int(rec["w"].max()), 10)
        try:
            _equal(got, want)
            q.put((rank, True))
        except AssertionError as e:
            q.put((rank, str(e)[:500]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("W", [40, 0])
def test_gloo_sharded_fit_equals_single_rank(W):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, W, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
