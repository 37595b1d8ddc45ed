"""GPU parity of the exact pruning (segmask: configs strictly beaten in every
(wave row, L bucket) cell are skipped by k_sweep2 / k_eval4) on adversarial
tables: exact duplicates (ties -> smaller macro id must win), 1-ulp and
1e-12 relative neighbours (inside the dominance margin: never pruned),
clearly dominated rows (pruned), and rows where the winner changes with L.
Every decision is compared bit for bit with the C oracle, through the grid
sweep + gather and through the list evaluation (tune_batch), and with
pruning disabled (WT_PRUNE=0, subprocess) as a second witness."""
import os
import subprocess
import sys

import numpy as np
import pytest

import pyoracle as po
import wtutil as U

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))


def adversarial_tables():
    return U.adversarial_tables()


def run(capi, cfg, t, M, N, K, pairs):
    from paper_2604_10187_b200 import synthetic as S

    eng = capi.Engine(t, S.registry_arrays(cfg), n_sm=148)
    grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 4096)
    grid.sweep()
    n = len(M)
    res = {}
    for mode in ("grid", "list"):
        out = [torch.empty(n, dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
        dm = [torch.as_tensor(x).cuda() for x in (M, N, K)]
        if mode == "grid":
            grid.gather(*dm, capi.Engine.decisions(*out))
        else:
            eng.tune_batch(*dm, capi.Engine.decisions(*out))
        torch.cuda.synchronize()
        res[mode] = [o.cpu().numpy() for o in out]
    return res


def queries(pairs, n=60000, seed=3):
    rng = np.random.default_rng(seed)
    P = np.array(pairs)[rng.integers(0, len(pairs), n)]
    M = rng.integers(1, 4097, n).astype(np.int32)
    N, K = P[:, 0].astype(np.int32), P[:, 1].astype(np.int32)
    off = rng.random(n) < 0.3
    N[off] = rng.integers(16, 40000, off.sum())
    K[off] = rng.integers(1, 1 << 20, off.sum())  # L from 1 to 16k: every L bucket
    return M, N, K


def test_pruning_is_exact_on_adversarial_tables():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_10187_b200 import capi, synthetic as S

    cfg, t = adversarial_tables()
    pairs = S.LLAMA3_8B
    M, N, K = queries(pairs)
    res = run(capi, cfg, t, M, N, K, pairs)
    tiles = {int(i): (int(a), int(b), int(c)) for i, a, b, c in zip(cfg["id"], cfg["t_m"], cfg["t_n"], cfg["t_k"])}
    want = po.Oracle().tune(po.FlatTables(U.pytables_from_arrays(t), tiles), 148, 1, M, N, K)
    ok = want["status"] == 0
    assert ok.all()
    for mode, (mac, mic, lat) in res.items():
        np.testing.assert_array_equal(mac, want["macro"], err_msg=mode)
        np.testing.assert_array_equal(mic, want["micro"], err_msg=mode)
        np.testing.assert_array_equal(U.bits(lat), U.bits(want["lat"]), err_msg=mode)
    # ties resolved to the smaller id somewhere (the duplicated rows win)
    ids = np.array(cfg["id"])
    assert np.isin(res["list"][0], ids).all()


def test_pruning_matches_unpruned_run():
    """Same decisions with WT_PRUNE=0 (every config evaluated) and with the
    every-M grid sweep (WT_SWEEP_DEDUP=0: k_sweep2 with pruning) instead of
    the representative sweep."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    script = (
        "import sys, numpy as np; sys.path[:0] = [%r, %r, %r];"
        "import torch; import test_gpu_prune as T; from paper_2604_10187_b200 import capi, synthetic as S;"
        "cfg, t = T.adversarial_tables(); M, N, K = T.queries(S.LLAMA3_8B);"
        "r = T.run(capi, cfg, t, M, N, K, S.LLAMA3_8B);"
        "np.savez(sys.argv[1], gm=r['grid'][0], gl=r['grid'][2], lm=r['list'][0], ll=r['list'][2])"
    ) % (os.path.dirname(HERE), os.path.join(os.path.dirname(HERE), "oracle"), HERE)
    outs = []
    for i, env in enumerate(({"WT_PRUNE": "1"}, {"WT_PRUNE": "0"}, {"WT_PRUNE": "1", "WT_SWEEP_DEDUP": "0"})):
        f = os.path.join("/tmp", f"wt_prune_{i}_{os.getpid()}.npz")
        r = subprocess.run([sys.executable, "-c", script, f], env={**os.environ, **env},
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        outs.append(np.load(f))
        os.unlink(f)
    for o in outs[1:]:
        for k in ("gm", "lm"):
            np.testing.assert_array_equal(outs[0][k], o[k])
        for k in ("gl", "ll"):
            np.testing.assert_array_equal(outs[0][k].view(np.int64), o[k].view(np.int64))


def test_many_tile_classes_list_and_grid():
    """More segments than the kernels stage headers for in shared memory
    (320 distinct tile classes): the global-header variants of k_eval4 /
    k_sweep2 against the oracle."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_10187_b200 import capi, synthetic as S

    base = S.config_space(False)
    n = 320
    cfg = {k: np.resize(np.asarray(v), n) for k, v in base.items()}
    cfg["id"] = np.arange(n, dtype=np.int32)
    cfg["t_m"] = np.where(np.arange(n) % 2 == 0, 64, 128).astype(np.int64)
    cfg["t_n"] = (16 + 8 * (np.arange(n) // 2)).astype(np.int64)   # 160 widths x 2 heights = 320 classes
    cfg["t_k"] = np.full(n, 64, np.int64)
    t = S.synthetic_tables(cfg)
    pairs = S.LLAMA3_8B
    M, N, K = queries(pairs, n=20000, seed=4)
    res = run(capi, cfg, t, M, N, K, pairs)
    tiles = {int(i): (int(a), int(b), int(c)) for i, a, b, c in zip(cfg["id"], cfg["t_m"], cfg["t_n"], cfg["t_k"])}
    want = po.Oracle().tune(po.FlatTables(U.pytables_from_arrays(t), tiles), 148, 1, M, N, K)
    for mode, (mac, mic, lat) in res.items():
        np.testing.assert_array_equal(mac, want["macro"], err_msg=mode)
        np.testing.assert_array_equal(U.bits(lat), U.bits(want["lat"]), err_msg=mode)


@pytest.mark.parametrize("seed", [1, 2])
def test_odd_tiles_random_registry(seed):
    """Non-power-of-two tiles (t_m 48/80/112, t_n 24/40/72/200, t_k 32/96):
    runs of the grid heads break inside 64-wide blocks (multi-run blocks),
    G and L cross wave / bucket boundaries at odd places; grid gather and
    list evaluation against the oracle, bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_10187_b200 import capi, synthetic as S

    rows = [(tm, tn, tk, st, 4, 1, 1) for tm in (48, 80, 112) for tn in (24, 40, 72, 200) for tk in (32, 96)
            for st in (2, 3)]
    a = np.array(rows, np.int64)
    cfg = dict(id=(np.arange(len(a)) * 3 + 5).astype(np.int32), t_m=a[:, 0], t_n=a[:, 1], t_k=a[:, 2],
               stages=a[:, 3], warps=a[:, 4], cluster=a[:, 5], swizzle=a[:, 6])
    t = S.synthetic_tables(cfg, seed=seed)
    rng = np.random.default_rng(seed)
    pairs = [(int(x), int(y)) for x, y in rng.integers(100, 20000, (5, 2))]
    eng = capi.Engine(t, S.registry_arrays(cfg), n_sm=148)
    grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 3000)
    grid.sweep()
    n = 30001
    P = np.array(pairs)[rng.integers(0, len(pairs), n)]
    M = rng.integers(1, 3400, n).astype(np.int32)
    N, K = P[:, 0].astype(np.int32), P[:, 1].astype(np.int32)
    off = rng.random(n) < 0.5
    N[off] = rng.integers(1, 50000, off.sum())
    K[off] = rng.integers(1, 1 << 18, off.sum())
    res = {}
    for mode in ("grid", "list"):
        o = [torch.empty(n, dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
        dm = [torch.as_tensor(x).cuda() for x in (M, N, K)]
        (grid.gather if mode == "grid" else eng.tune_batch)(*dm, capi.Engine.decisions(*o))
        torch.cuda.synchronize()
        res[mode] = [x.cpu().numpy() for x in o]
    tiles = {int(i): (int(x), int(y), int(z)) for i, x, y, z in zip(cfg["id"], cfg["t_m"], cfg["t_n"], cfg["t_k"])}
    want = po.Oracle().tune(po.FlatTables(U.pytables_from_arrays(t), tiles), 148, 1, M, N, K)
    assert (want["status"] == 0).all()
    for mode, (mac, mic, lat) in res.items():
        np.testing.assert_array_equal(mac, want["macro"], err_msg=mode)
        np.testing.assert_array_equal(mic, want["micro"], err_msg=mode)
        np.testing.assert_array_equal(U.bits(lat), U.bits(want["lat"]), err_msg=mode)
