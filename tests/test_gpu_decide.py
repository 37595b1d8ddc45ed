"""GPU parity: the sm_100a decision kernels (through the C-ABI) against the
reference compiled verbatim (oracle/_ref) and the C restatement (oracle/).

Bar: macro / micro / wave / regime / comparisons / g / l bit-exact, predicted
latency bit-exact (BASELINE.json allows 1e-5 relative; the kernels use the
reference's exact fp64 operation order, so we assert bitwise equality).
"""
import numpy as np
import pytest

import pyoracle as po
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


@pytest.fixture(scope="module")
def ref():
    return po.Reference()


@pytest.fixture(scope="module")
def orc():
    return po.Oracle()


def dev(a, dt=torch.int32):
    return torch.as_tensor(np.ascontiguousarray(a)).to(dtype=dt, device="cuda")


def tune_gpu(capi, eng, M, N, K, topk=0, grid=None):
    n = len(M)
    o = dict(macro=torch.empty(n, dtype=torch.int32, device="cuda"),
             micro=torch.empty(n, dtype=torch.int32, device="cuda"),
             lat=torch.empty(n, dtype=torch.float64, device="cuda"),
             g=torch.empty(n, dtype=torch.int64, device="cuda"),
             l=torch.empty(n, dtype=torch.int64, device="cuda"),
             wave=torch.empty(n, dtype=torch.int32, device="cuda"),
             flags=torch.empty(n, dtype=torch.int32, device="cuda"),
             comps=torch.empty(n, dtype=torch.int32, device="cuda"),
             tail=torch.empty(n, dtype=torch.float64, device="cuda"))
    if topk:
        o["tkm"] = torch.empty(n * topk, dtype=torch.int32, device="cuda")
        o["tkl"] = torch.empty(n * topk, dtype=torch.float64, device="cuda")
    d = capi.Engine.decisions(o["macro"], o["micro"], o["lat"], o["g"], o["l"], o["wave"], o["flags"], o["comps"],
                              o["tail"], topk, o.get("tkm"), o.get("tkl"))
    Md, Nd, Kd = dev(M), dev(N), dev(K)
    if grid is None:
        eng.tune_batch(Md, Nd, Kd, d)
    else:
        grid.gather(Md, Nd, Kd, d)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in o.items()}


def assert_same(gpu, want, status_key="status"):
    st = want[status_key]
    gst = (gpu["flags"].astype(np.uint32) >> 24).astype(np.int32)
    np.testing.assert_array_equal(gst, st)
    ok = st == 0
    for k_g, k_w in (("macro", "macro"), ("micro", "micro"), ("g", "g"), ("l", "l"), ("wave", "w"),
                     ("comps", "comps")):
        np.testing.assert_array_equal(gpu[k_g][ok], want[k_w][ok], err_msg=k_g)
    np.testing.assert_array_equal(U.bits(gpu["lat"][ok]), U.bits(want["lat"][ok]))
    ex = (gpu["flags"] & 1) != 0
    np.testing.assert_array_equal(ex[ok], want["extrap"][ok] != 0)


# ------------------------------------------------------------------ fixtures
@pytest.fixture(scope="module")
def landscape(ref, tmpdir_session):
    reg, rec, tab = U.reference_fixture(ref, tmpdir_session)
    fam, tabs = po.parse_tables_json(tab)
    tiles, order = po.parse_registry_json(reg)
    return dict(reg=reg, rec=rec, tab=tab, tabs=tabs, tiles=tiles, arrays=U.arrays_from_pytables(tabs),
                registry=U.registry_from_json(reg))


@pytest.fixture(scope="module")
def synth256():
    from paper_2604_10187_b200 import synthetic as S

    cfg = S.config_space(full=False)
    t = S.synthetic_tables(cfg)
    return cfg, t, S.registry_arrays(cfg)


# --------------------------------------------------------------------- tests
def test_tune_matches_reference_on_its_landscape(capi, ref, orc, landscape):
    """Reference acceptance landscape (6x8 configs, W=10, sigma=5): GPU tune vs
    the reference's own tune() on 50k random shapes (acceptance.cpp:246-259
    style draws) plus the boundary shapes of every wave."""
    L = landscape
    eng = capi.Engine(L["arrays"], L["registry"], n_sm=132)
    rng = np.random.default_rng(33)
    n = 50000
    M = rng.integers(1, 9000, n)
    N = rng.integers(1, 9000, n)
    K = rng.integers(1, 9000, n)
    # wave boundaries: g = w*132 and w*132+1 for 64x64 tiles
    wb = np.array([w * 132 + d for w in range(1, 14) for d in (0, 1)])
    M = np.concatenate([M, wb * 64, np.full(len(wb), 64)])
    N = np.concatenate([N, np.full(len(wb), 64), wb * 64])
    K = np.concatenate([K, np.full(2 * len(wb), 1024)])
    h = ref.open(L["tab"], L["reg"], 132)
    want = ref.tune(h, M, N, K, nthreads=8)
    got = tune_gpu(capi, eng, M, N, K)
    assert (want["status"] == 0).all()
    assert_same(got, want)
    assert (want["evals"] == eng.n_configs).all()
    # restatement agrees with the reference too (pinning)
    flat = po.FlatTables(L["tabs"], L["tiles"])
    w2 = orc.tune(flat, 132, 1, M, N, K)
    assert_same(got, w2)
    ref.close(h)


def test_grid_gather_matches_reference_on_its_landscape(capi, ref, landscape):
    """The reference's own landscape through the serving path: grid sweep,
    run index, hashed gather and the pruned off-grid evaluation (plain
    outputs) against the reference's tune() itself."""
    L = landscape
    eng = capi.Engine(L["arrays"], L["registry"], n_sm=132)
    rng = np.random.default_rng(44)
    pairs = [(int(x), int(y)) for x, y in rng.integers(1, 9000, (6, 2))]
    grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 6000)
    grid.sweep()
    n = 40003
    P = np.array(pairs)[rng.integers(0, len(pairs), n)]
    M = rng.integers(1, 6500, n).astype(np.int32)
    N, K = P[:, 0].astype(np.int32), P[:, 1].astype(np.int32)
    off = rng.random(n) < 0.2
    N[off] = rng.integers(1, 9000, off.sum())
    K[off] = rng.integers(1, 9000, off.sum())
    out = [torch.empty(n, dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
    grid.gather(dev(M), dev(N), dev(K), capi.Engine.decisions(*out))
    torch.cuda.synchronize()
    mac, mic, lat = (o.cpu().numpy() for o in out)
    h = ref.open(L["tab"], L["reg"], 132)
    want = ref.tune(h, M, N, K, nthreads=8)
    ref.close(h)
    assert (want["status"] == 0).all()
    np.testing.assert_array_equal(mac, want["macro"])
    np.testing.assert_array_equal(mic, want["micro"])
    np.testing.assert_array_equal(U.bits(lat), U.bits(want["lat"]))


def test_sweep_grid_config1_bitexact(capi, orc, synth256):
    """Config 1: 4 Llama-3-8B pairs x M=1..8192 x 256 configs, every entry vs
    the oracle tune()."""
    from paper_2604_10187_b200 import synthetic as S

    cfg, t, reg = synth256
    eng = capi.Engine(t, reg, n_sm=148)
    pairs = S.LLAMA3_8B
    grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 8192)
    grid.sweep()
    torch.cuda.synchronize()
    ent = grid.entries_tensor().cpu().numpy()
    lat = ent[:, 0:2].copy().view(np.float64)[:, 0]
    M = np.tile(np.arange(1, 8193), len(pairs))
    N = np.repeat([p[0] for p in pairs], 8192)
    K = np.repeat([p[1] for p in pairs], 8192)
    tiles = {int(i): (int(a), int(b), int(c)) for i, a, b, c in zip(cfg["id"], cfg["t_m"], cfg["t_n"], cfg["t_k"])}
    flat = po.FlatTables(U.pytables_from_arrays(t), tiles)
    want = orc.tune(flat, 148, 1, M, N, K)
    assert (want["status"] == 0).all()
    np.testing.assert_array_equal(ent[:, 2], want["macro"])
    np.testing.assert_array_equal(ent[:, 3], want["micro"])
    np.testing.assert_array_equal(ent[:, 4], want["w"])
    np.testing.assert_array_equal(ent[:, 6], want["comps"])
    np.testing.assert_array_equal(U.bits(lat), U.bits(want["lat"]))
    np.testing.assert_array_equal(ent[:, 5] & 1, want["extrap"])
    # tail fraction of the winner (extension): (g - (w-1)*S)/S
    tail = ent[:, 7].copy().view(np.float32)
    exp = ((want["g"] - (want["w"] - 1) * 148) / 148.0).astype(np.float32)
    np.testing.assert_array_equal(tail, exp)


def test_gather_matches_tune_with_offgrid(capi, orc, synth256):
    """Config 2 stream (decode/prefill mix + 1% off-grid): gather answers ==
    evaluate-mode answers == oracle."""
    from paper_2604_10187_b200 import synthetic as S

    cfg, t, reg = synth256
    eng = capi.Engine(t, reg, n_sm=148)
    pairs = S.LLAMA3_8B
    grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 8192)
    grid.sweep()
    M, N, K = S.query_stream(300000, pairs, seed=55, off_grid_frac=0.02)
    got = tune_gpu(capi, eng, M, N, K, grid=grid)
    direct = tune_gpu(capi, eng, M, N, K)
    for k in ("macro", "micro", "wave", "comps", "flags", "g", "l"):
        np.testing.assert_array_equal(got[k], direct[k], err_msg=k)
    np.testing.assert_array_equal(U.bits(got["lat"]), U.bits(direct["lat"]))
    tiles = {int(i): (int(a), int(b), int(c)) for i, a, b, c in zip(cfg["id"], cfg["t_m"], cfg["t_n"], cfg["t_k"])}
    flat = po.FlatTables(U.pytables_from_arrays(t), tiles)
    sub = np.random.default_rng(0).choice(len(M), 40000, replace=False)
    want = orc.tune(flat, 148, 1, M[sub], N[sub], K[sub])
    assert_same({k: v[sub] for k, v in got.items()}, want)


@pytest.mark.parametrize("n_extra,offset", [(0, 0), (700, 0), (700, 1), (2100, 0)])
def test_hashed_gather_plain_outputs(capi, orc, synth256, n_extra, offset):
    """The common call (macro / micro / latency only) goes through the hashed
    pair table (k_gather_h): many pairs (probe chains), invalid dims, N = K = 0
    (never matches an empty slot), M outside the grid, n % 4 != 0 and
    misaligned arrays (scalar kernel); answers == evaluate mode == oracle.
    2100 extra pairs exceed the hashed-table cap (binary-search kernel)."""
    from paper_2604_10187_b200 import synthetic as S

    cfg, t, reg = synth256
    eng = capi.Engine(t, reg, n_sm=148)
    rng = np.random.default_rng(11 + n_extra)
    pairs = list(S.LLAMA3_8B) + [(int(a), int(b)) for a, b in rng.integers(1, 40000, (n_extra, 2))]
    grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 3, 300)
    grid.sweep()
    n = 50001
    P = np.array(pairs)[rng.integers(0, len(pairs), n)]
    M = rng.integers(1, 320, n).astype(np.int32)
    N, K = P[:, 0].astype(np.int32), P[:, 1].astype(np.int32)
    off = rng.random(n) < 0.05
    N[off] = rng.integers(1, 40000, off.sum())
    K[off] = rng.integers(1, 40000, off.sum())
    M[:7] = [0, -3, 1, 2, 300, 301, 5]
    N[:7] = [4096, 4096, 0, 4096, 4096, 4096, -1]
    K[:7] = [4096, 4096, 0, 4096, 4096, 4096, 4096]
    direct = tune_gpu(capi, eng, M, N, K)
    buf = [torch.empty(n + offset, dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
    out = [b[offset:] for b in buf]
    ins = [dev(np.concatenate([np.zeros(offset, np.int32), x]))[offset:] for x in (M, N, K)]
    grid.gather(*ins, capi.Engine.decisions(*out))
    torch.cuda.synchronize()
    mac, mic, lat = (o.cpu().numpy() for o in out)
    ok = (direct["flags"].astype(np.uint32) >> 24) == 0
    np.testing.assert_array_equal(mac, direct["macro"])
    np.testing.assert_array_equal(mic, direct["micro"])
    np.testing.assert_array_equal(U.bits(lat[ok]), U.bits(direct["lat"][ok]))
    assert (~ok).sum() >= 3
    tiles = {int(i): (int(a), int(b), int(c)) for i, a, b, c in zip(cfg["id"], cfg["t_m"], cfg["t_n"], cfg["t_k"])}
    flat = po.FlatTables(U.pytables_from_arrays(t), tiles)
    sub = np.random.default_rng(1).choice(n, 5000, replace=False)
    want = orc.tune(flat, 148, 1, M[sub], N[sub], K[sub])
    good = want["status"] == 0
    np.testing.assert_array_equal(mac[sub][good], want["macro"][good])
    np.testing.assert_array_equal(U.bits(lat[sub][good]), U.bits(want["lat"][good]))


def test_run_index_follows_entries(capi, synth256):
    """The run-compressed heads the gather serves from shared memory are
    rebuilt by a full sweep, invalidated by a partial one and rebuilt by
    finalize() after entries are written directly."""
    from paper_2604_10187_b200 import synthetic as S

    cfg, t, reg = synth256
    eng = capi.Engine(t, reg, n_sm=148)
    pairs = S.LLAMA3_8B
    grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 4096)
    M, N, K = S.query_stream(20003, pairs, seed=3, off_grid_frac=0.0, m_max=4096)
    n = len(M)

    def gather():
        out = [torch.empty(n, dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
        grid.gather(dev(M), dev(N), dev(K), capi.Engine.decisions(*out))
        torch.cuda.synchronize()
        return [o.cpu().numpy() for o in out]

    grid.sweep()
    want = tune_gpu(capi, eng, M, N, K)
    for step in ("full", "partial", "written", "finalized"):
        if step == "partial":
            grid.sweep(0, 1000)
        elif step == "written":
            ent = grid.entries_tensor()
            saved = ent.clone()
            ent.zero_()
            grid.finalize()
            mac, mic, lat = gather()
            assert (mac == 0).all() and (mic == 0).all() and (lat == 0).all()
            ent.copy_(saved)
            continue
        elif step == "finalized":
            grid.finalize()
        mac, mic, lat = gather()
        np.testing.assert_array_equal(mac, want["macro"], err_msg=step)
        np.testing.assert_array_equal(mic, want["micro"], err_msg=step)
        np.testing.assert_array_equal(U.bits(lat), U.bits(want["lat"]), err_msg=step)


def test_topk_matches_oracle(capi, orc, synth256):
    from paper_2604_10187_b200 import synthetic as S

    cfg, t, reg = synth256
    eng = capi.Engine(t, reg, n_sm=148)
    rng = np.random.default_rng(5)
    n = 3000
    M = rng.integers(1, 8193, n)
    P = np.array(S.LLAMA3_8B)[rng.integers(0, 4, n)]
    N, K = P[:, 0], P[:, 1]
    k = 4
    got = tune_gpu(capi, eng, M, N, K, topk=k)
    grid = capi.Grid(eng, [p[0] for p in S.LLAMA3_8B], [p[1] for p in S.LLAMA3_8B], 1, 8192, topk=k)
    grid.sweep()
    got_g = tune_gpu(capi, eng, M, N, K, topk=k, grid=grid)
    tiles = {int(i): (int(a), int(b), int(c)) for i, a, b, c in zip(cfg["id"], cfg["t_m"], cfg["t_n"], cfg["t_k"])}
    flat = po.FlatTables(U.pytables_from_arrays(t), tiles)
    for i in range(0, n, 7):
        st, mac, lat = orc.topk(flat, 148, 1, int(M[i]), int(N[i]), int(K[i]), k)
        assert st == 0
        np.testing.assert_array_equal(got["tkm"][i * k:(i + 1) * k], mac)
        np.testing.assert_array_equal(U.bits(got["tkl"][i * k:(i + 1) * k]), U.bits(lat))
        np.testing.assert_array_equal(got_g["tkm"][i * k:(i + 1) * k], mac)
        assert got["macro"][i] == mac[0]


def _mutilate(t, rng):
    """Tables exercising every fallback rule: erased coefficient waves,
    erased / emptied anchor maps, per-table W, an empty coeff table, NaN and
    +inf coefficients, ties."""
    tabs = U.pytables_from_arrays(t)
    for i, tb in enumerate(tabs):
        r = i % 9
        if r == 1:
            for w in rng.choice(sorted(tb.coeffs), 5, replace=False):
                del tb.coeffs[int(w)]
        elif r == 2:
            for w in rng.choice(sorted(tb.anchors), 6, replace=False):
                del tb.anchors[int(w)]
        elif r == 3:
            tb.ext_anchors = {}
        elif r == 4:
            tb.W = int(rng.integers(3, 40))
        elif r == 5:
            w = int(rng.integers(1, 41))
            tb.coeffs[w] = (float("nan"),) * 4
        elif r == 6:
            tb.coeffs = {w: c for w, c in tb.coeffs.items() if w % 3 == 0}
            tb.anchors = {w: d for w, d in tb.anchors.items() if w % 4 == 0}
        elif r == 7:
            tb.theta_ext = (0.0, 0.0, 0.0, float("inf"))
        elif r == 8 and i < 40:
            tb.coeffs[7] = tabs[i - 1].coeffs.get(7, (0.0, 0.0, 0.0, 1.0))  # exact ties across ids
    return tabs


def test_fallback_rules_and_errors(capi, orc, ref, synth256, tmpdir_session):
    cfg, t, reg = synth256
    rng = np.random.default_rng(9)
    tabs = _mutilate(t, rng)
    arr = U.arrays_from_pytables(tabs)
    eng = capi.Engine(arr, reg, n_sm=148)
    assert eng.info.has_fallback_rows == 1
    n = 60000
    M = rng.integers(1, 70000, n)
    N = rng.integers(1, 70000, n)
    K = rng.integers(1, 20000, n)
    M[:50] = 0  # invalid dims -> invalid_argument
    K[50:60] = -3
    got = tune_gpu(capi, eng, M, N, K)
    tiles = {int(i): (int(a), int(b), int(c)) for i, a, b, c in zip(cfg["id"], cfg["t_m"], cfg["t_n"], cfg["t_k"])}
    want = orc.tune(po.FlatTables(tabs, tiles), 148, 1, M, N, K)
    assert_same(got, want)
    ok = want["status"] == 0
    np.testing.assert_array_equal(((got["flags"] >> 1) & 1)[ok], (want["n_missing"] > 0)[ok])
    np.testing.assert_array_equal(((got["flags"] >> 2) & 1)[ok], (want["anchor_fb"] >= 0)[ok])
    # the same artefact through the reference itself (JSON round trip)
    tab = str(tmpdir_session / "mutilated.json")
    regp = str(tmpdir_session / "reg256.json")
    U.write_tables_json(tabs, tab)
    U.write_registry_json(reg, regp)
    h = ref.open(tab, regp, 148)
    sub = slice(60, 20060)
    wr = ref.tune(h, M[sub], N[sub], K[sub], nthreads=8)
    assert_same({k: v[sub] for k, v in got.items()}, wr)
    ref.close(h)


def test_empty_coeff_table_is_runtime_error(capi, orc, synth256):
    cfg, t, reg = synth256
    tabs = U.pytables_from_arrays(t)
    tabs[3].coeffs = {}
    eng = capi.Engine(U.arrays_from_pytables(tabs), reg, n_sm=148)
    M = np.array([1, 100000, 8192]); N = np.array([4096, 4096, 4096]); K = np.array([4096, 4096, 4096])
    got = tune_gpu(capi, eng, M, N, K)
    tiles = {int(i): (int(a), int(b), int(c)) for i, a, b, c in zip(cfg["id"], cfg["t_m"], cfg["t_n"], cfg["t_k"])}
    want = orc.tune(po.FlatTables(tabs, tiles), 148, 1, M, N, K)
    assert_same(got, want)
    assert want["status"][0] == 2  # w <= W for table 3 -> runtime_error


def test_all_infinite_candidates_are_runtime_error(capi, orc, synth256):
    """Coefficients that overflow: for large shapes every config predicts
    +inf, and tune() -- best_latency starts at +inf, strict < -- finds no
    winner (the reference dereferences null; the restatement reports
    runtime_error).  Small shapes keep finite candidates.  Grid (sweep +
    gather) and list paths must agree with the restatement."""
    from paper_2604_10187_b200 import synthetic as S

    cfg, t, reg = synth256
    t2 = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in t.items()}
    t2["coeff_theta"][0::4] = 1e308
    t2["theta_ext"][0::4] = 1e308
    eng = capi.Engine(t2, reg, n_sm=148)
    pairs = S.LLAMA3_8B[:2]
    grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 600)
    grid.sweep()
    rng = np.random.default_rng(4)
    M = np.concatenate([rng.integers(1, 600, 3000), rng.integers(1, 40, 1000)]).astype(np.int32)
    N = np.concatenate([np.full(3000, pairs[0][0]), rng.integers(1, 70, 1000)]).astype(np.int32)
    K = np.concatenate([np.full(3000, pairs[0][1]), rng.integers(1, 70, 1000)]).astype(np.int32)
    tiles = {int(i): (int(a), int(b), int(c)) for i, a, b, c in zip(cfg["id"], cfg["t_m"], cfg["t_n"], cfg["t_k"])}
    want = orc.tune(po.FlatTables(U.pytables_from_arrays(t2), tiles), 148, 1, M, N, K)
    assert (want["status"] == 2).any() and (want["status"] == 0).any()
    assert_same(tune_gpu(capi, eng, M, N, K, grid=grid), want)
    assert_same(tune_gpu(capi, eng, M, N, K), want)


def test_attention_family(capi, orc):
    """FlashAttention registries: g = n_heads*ceil(s_q/t_q), l = ceil(s_kv/t_kv)
    (kernel_map.cpp:258-263) -- the oracle evaluates it as dense with t_n=1."""
    from paper_2604_10187_b200 import synthetic as S

    cfg = S.config_space(False)
    t = S.synthetic_tables(cfg)
    reg = dict(family=2, id=cfg["id"], t_m=cfg["t_m"], t_n=cfg["t_n"], t_k=cfg["t_k"])
    eng = capi.Engine(t, reg, n_sm=148)
    rng = np.random.default_rng(3)
    n = 20000
    sq, heads, skv = rng.integers(1, 32768, n), rng.integers(1, 129, n), rng.integers(1, 65536, n)
    got = tune_gpu(capi, eng, sq, heads, skv)
    tiles = {int(i): (int(a), 1, int(c)) for i, a, c in zip(cfg["id"], cfg["t_m"], cfg["t_k"])}
    want = orc.tune(po.FlatTables(U.pytables_from_arrays(t), tiles), 148, 1, sq, heads, skv)
    assert_same(got, want)


def test_predict_and_nearest_anchor(capi, ref, landscape):
    L = landscape
    eng = capi.Engine(L["arrays"], L["registry"], n_sm=132)
    h = ref.open(L["tab"], L["reg"], 132)
    rng = np.random.default_rng(2)
    n = 4000
    cfgi = rng.integers(0, eng.n_configs, n).astype(np.int32)
    g = rng.integers(1, 3000, n)
    l = rng.integers(1, 200, n)
    lat = torch.empty(n, dtype=torch.float64, device="cuda")
    wave = torch.empty(n, dtype=torch.int32, device="cuda")
    ex = torch.empty(n, dtype=torch.int32, device="cuda")
    st = torch.empty(n, dtype=torch.int32, device="cuda")
    eng.predict_batch(dev(cfgi), dev(g, torch.int64), dev(l, torch.int64), lat, wave, ex, None, st)
    torch.cuda.synchronize()
    # engine configs are in ascending macro_id order; the artefact order may differ
    order = np.argsort([t.macro_id for t in L["tabs"]], kind="stable")
    lat, wave, ex = lat.cpu().numpy(), wave.cpu().numpy(), ex.cpu().numpy()
    for i in range(n):
        s, v, e, w, _ = ref.predict(h, int(order[cfgi[i]]), int(g[i]), int(l[i]))
        assert s == 0
        assert U.bits(np.array([v]))[0] == U.bits(lat[i:i + 1])[0]
        assert (e, w) == (ex[i], wave[i])
    ref.close(h)
    anchors = np.array([16, 32, 48, 64, 80], np.int64)
    ls = np.arange(0, 120, dtype=np.int64)
    out = torch.empty(len(ls), dtype=torch.int64, device="cuda")
    comps = torch.empty(len(ls), dtype=torch.int32, device="cuda")
    import ctypes as C

    a_d, l_d = dev(anchors, torch.int64), dev(ls, torch.int64)  # keep alive across the launch
    capi.check(capi.lib().wt_nearest_anchor_batch(C.c_void_p(a_d.data_ptr()), 5,
                                                   C.c_void_p(l_d.data_ptr()), C.c_int64(len(ls)),
                                                   C.c_void_p(out.data_ptr()), C.c_void_p(comps.data_ptr()),
                                                   C.c_void_p(0)))
    torch.cuda.synchronize()
    for i, lv in enumerate(ls):
        r, c = ref.nearest_anchor(anchors, int(lv))
        assert (r, c) == (out[i].item(), comps[i].item())


def test_sharded_sweep_equals_full(capi, synth256):
    """Any split of the flattened shape index (the multi-GPU shard unit)
    fills identical entries."""
    from paper_2604_10187_b200 import synthetic as S

    cfg, t, reg = synth256
    eng = capi.Engine(t, reg, n_sm=148)
    pairs = S.LLAMA3_8B
    g1 = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 5000)
    g2 = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 5000)
    g1.sweep()
    cuts = [0, 777, 5000, 5001, 12345, g2.n_entries]
    for a, b in zip(cuts[:-1], cuts[1:]):
        g2.sweep(a, b)
    torch.cuda.synchronize()
    assert torch.equal(g1.entries_tensor(), g2.entries_tensor())


@pytest.mark.parametrize("m_lo,m_hi", [(1, 5000), (37, 4133), (129, 129 + 63)])
def test_partial_sweep_writes_only_its_range(capi, orc, synth256, m_lo, m_hi):
    """The representative sweep (one M per interval of constant ceil(M/t_m),
    copied over the interval) writes exactly [begin, end): entries outside a
    partial range keep their poison, entries inside equal the full sweep and
    the restatement, for M ranges that start off the t_m multiples."""
    from paper_2604_10187_b200 import synthetic as S

    cfg, t, reg = synth256
    eng = capi.Engine(t, reg, n_sm=148)
    pairs = S.LLAMA3_8B[:3]
    full = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], m_lo, m_hi)
    full.sweep()
    part = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], m_lo, m_hi)
    n = part.n_entries
    assert full.n_representatives * 4 <= n  # the sweep evaluates one M per interval
    rng = np.random.default_rng(m_lo)
    for _ in range(4):
        a, b = sorted(int(x) for x in rng.integers(0, n + 1, 2))
        ent = part.entries_tensor()
        ent.fill_(-7)
        torch.cuda.synchronize()
        part.sweep(a, b)
        torch.cuda.synchronize()
        got = part.entries_tensor()
        assert bool((got[:a] == -7).all()) and bool((got[b:] == -7).all())
        assert torch.equal(got[a:b], full.entries_tensor()[a:b])
    # every full-grid entry against the restatement
    M = np.tile(np.arange(m_lo, m_hi + 1, dtype=np.int32), len(pairs))
    N = np.repeat(np.array([p[0] for p in pairs], np.int32), m_hi - m_lo + 1)
    K = np.repeat(np.array([p[1] for p in pairs], np.int32), m_hi - m_lo + 1)
    tiles = {int(i): (int(x), int(y), int(z)) for i, x, y, z in zip(cfg["id"], cfg["t_m"], cfg["t_n"], cfg["t_k"])}
    want = orc.tune(po.FlatTables(U.pytables_from_arrays(t), tiles), 148, 1, M, N, K)
    e = full.entries_tensor().cpu().numpy()
    lat = e[:, :2].copy().view(np.float64).ravel()
    np.testing.assert_array_equal(e[:, 2], want["macro"])
    np.testing.assert_array_equal(e[:, 3], want["micro"])
    np.testing.assert_array_equal(lat.view(np.int64), want["lat"].view(np.int64))


@pytest.mark.parametrize("env", [
    {"WT_SWEEP_RPT": "2", "WT_EVAL_RPT": "2", "WT_SWEEP_DEDUP": "0"},
    {"WT_SWEEP_SMEM_KB": "24", "WT_EVAL_SMEM_KB": "64", "WT_SWEEP_DEDUP": "0"},
    {"WT_SWEEP_RPT": "2", "WT_SWEEP_SMEM_KB": "160", "WT_EVAL_RPT": "4", "WT_EVAL_SMEM_KB": "160",
     "WT_SWEEP_DEDUP": "0"},
    {"WT_GATHER_VARIANT": "1"},
    {"WT_EVAL_RPT": "2", "WT_GATHER_VARIANT": "2"},
    {"WT_GATHER_VARIANT": "3"},
    {"WT_GATHER_VARIANT": "4"},
    {"WT_GATHER_RUNS_KB": "0"},
    {"WT_GATHER_VARIANT": "5"},
    {"WT_EVAL_MODE": "2"},
    {"WT_EVAL_KEY_BITS": "8"},
    {"WT_EVAL_KEY_BITS": "24"},
    {"WT_PRUNE": "0"},
    {"WT_EVAL_KERNEL": "3"},
    {"WT_EVAL4_RPT": "4"},
    {"WT_EVAL4_RPT": "1"},
    {"WT_EVAL_KEY_MODE": "3"},
    {"WT_BATCH_SLICE": "4100"},
    {"WT_SWEEP_SMEM_KB": "96", "WT_SWEEP_DEDUP": "0"},
    {"WT_SWEEP_DEDUP": "0"},
    {"WT_SWEEP_DEDUP": "0", "WT_PRUNE": "0"},
    {"WT_SWEEP_W": "0"},
])
def test_launch_variants(capi, env):
    """Every launch shape the tuning knobs can select stays bit-exact."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, os.path.join(here, "variant_check.py")], env={**os.environ, **env},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_tune_one_matches_batch(capi, landscape, synth256):
    """wt_tune_one (one warp, pinned mailbox) returns exactly the batch
    kernel's answer, field for field, including per-query error statuses and
    the reference landscape's fallback rows."""
    from paper_2604_10187_b200 import synthetic as S

    cfg, t, reg = synth256
    engines = [capi.Engine(t, reg, n_sm=148), capi.Engine(landscape["arrays"], landscape["registry"], n_sm=132)]
    rng = np.random.default_rng(11)
    M = np.concatenate([rng.integers(1, 70000, 400), [0, -3, 1, 2**31 - 1, 5]]).astype(np.int32)
    N = np.concatenate([rng.integers(1, 70000, 400), [5, 5, 0, 2**31 - 1, 2**31 - 1]]).astype(np.int32)
    K = np.concatenate([rng.integers(1, 70000, 400), [5, 5, 5, 7, 2**31 - 1]]).astype(np.int32)
    for eng in engines:
        want = tune_gpu(capi, eng, M, N, K)
        for i in range(len(M)):
            o = eng.tune_one(int(M[i]), int(N[i]), int(K[i]))
            assert o.flags == np.uint32(want["flags"][i]), i
            got = (o.macro_id, o.micro_id, o.wave, o.comparisons, o.g, o.l)
            exp = tuple(int(want[k][i]) for k in ("macro", "micro", "wave", "comps", "g", "l"))
            assert got == exp, (i, got, exp)
            assert U.bits(np.array([o.latency_us]))[0] == U.bits(want["lat"][i:i + 1])[0]
    assert engines[0].tune_one(4096, 4096, 4096).macro_id >= 0


def test_resident_server_matches_batch(capi, landscape, synth256):
    """wt_engine_set_resident: the polling CTA answers exactly as the batch
    kernel, restarts after its idle exit, and stops on request (so a device
    synchronisation afterwards returns at once)."""
    import time

    cfg, t, reg = synth256
    for eng in (capi.Engine(t, reg, n_sm=148), capi.Engine(landscape["arrays"], landscape["registry"], n_sm=132)):
        rng = np.random.default_rng(5)
        M = np.concatenate([rng.integers(1, 70000, 300), [0, 2**31 - 1]]).astype(np.int32)
        N = np.concatenate([rng.integers(1, 70000, 300), [7, 2**31 - 1]]).astype(np.int32)
        K = np.concatenate([rng.integers(1, 70000, 300), [7, 9]]).astype(np.int32)
        want = tune_gpu(capi, eng, M, N, K)
        eng.set_resident(2000)  # 2 ms idle exit: the sleeps below force restarts
        for i in range(len(M)):
            if i % 50 == 49:
                time.sleep(0.01)
            o = eng.tune_one(int(M[i]), int(N[i]), int(K[i]))
            assert o.flags == np.uint32(want["flags"][i]), i
            got = (o.macro_id, o.micro_id, o.wave, o.comparisons, o.g, o.l)
            assert got == tuple(int(want[k][i]) for k in ("macro", "micro", "wave", "comps", "g", "l")), i
            assert U.bits(np.array([o.latency_us]))[0] == U.bits(want["lat"][i:i + 1])[0]
        eng.set_resident(0)
        t0 = time.perf_counter()
        torch.cuda.synchronize()
        assert time.perf_counter() - t0 < 0.5


@pytest.mark.parametrize("chunk", [1000, 4096, 1 << 22])
def test_decide_host_pipeline_matches_device(capi, synth256, chunk):
    """wt_decide_host_sync (pinned host buffers, chunked H2D / gather / D2H
    over several streams with per-slot scratch) == the device-resident call,
    including a ragged last chunk and off-grid queries."""
    from paper_2604_10187_b200 import synthetic as S

    cfg, t, reg = synth256
    eng = capi.Engine(t, reg, n_sm=148)
    pairs = S.LLAMA3_8B
    grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 8192)
    grid.sweep()
    M, N, K = S.query_stream(30011, pairs, seed=9, off_grid_frac=0.05)
    n = len(M)
    out = [torch.empty(n, dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
    grid.gather(dev(M), dev(N), dev(K), capi.Engine.decisions(*out))
    torch.cuda.synchronize()
    Mp, Np, Kp = (torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in (M, N, K))
    mac = torch.empty(n, dtype=torch.int32).pin_memory()
    mic = torch.empty(n, dtype=torch.int32).pin_memory()
    lat = torch.empty(n, dtype=torch.float64).pin_memory()
    grid.decide_host(Mp, Np, Kp, mac, mic, lat, chunk=chunk)
    assert torch.equal(mac, out[0].cpu()) and torch.equal(mic, out[1].cpu())
    assert torch.equal(lat.view(torch.int64), out[2].cpu().view(torch.int64))


def test_sweep_to_fills_every_destination(capi, synth256):
    """The fused sweep's multi-destination epilogue (wt_sweep_to), driven in
    one process: rank slices swept into two local grids (standing in for
    peer-mapped storages) give, in both, exactly the single full sweep --
    with and without config splits (k_sweep_merge)."""
    from paper_2604_10187_b200 import synthetic as S
    from paper_2604_10187_b200.dist import shard_bounds

    cfg, t, reg = synth256
    eng = capi.Engine(t, reg, n_sm=148)
    pairs = S.LLAMA3_8B
    full = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 3001)
    full.sweep()
    for world in (2, 3):
        grids = [capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 3001) for _ in range(world)]
        for g in grids:
            g.entries_tensor().fill_(-7)
        ptrs = [g.entries_ptr for g in grids]
        for r, g in enumerate(grids):
            lo, hi, _ = shard_bounds(g.n_entries, world, r)
            g.sweep_to(ptrs[r:] + ptrs[:r], lo, hi)
        torch.cuda.synchronize()
        for g in grids:
            g.finalize()
            assert torch.equal(g.entries_tensor(), full.entries_tensor())
        # the finalized run index serves gathers
        M, N, K = S.query_stream(5000, pairs, seed=4, off_grid_frac=0.0, m_max=3001)
        outs = []
        for g in (grids[0], full):
            o = [torch.empty(len(M), dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
            g.gather(dev(M), dev(N), dev(K), capi.Engine.decisions(*o))
            torch.cuda.synchronize()
            outs.append([x.cpu() for x in o])
        for a, b in zip(*outs):
            assert torch.equal(a.view(torch.int64) if a.dtype == torch.float64 else a,
                               b.view(torch.int64) if b.dtype == torch.float64 else b)
