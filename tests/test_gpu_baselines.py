"""Ablation baselines on the GPU (reference
tuner.cpp:168-250) against the reference compiled verbatim (oracle/_ref) and
the restated fit (oracle/).

Bar: step t_wave bitwise (plain sequential sums, reproduced in order);
linear theta bitwise vs the restatement's fit_bucket on the same selected
samples and within 1e-9 of the reference's Eigen-shim fit; baseline_predict
and baseline_tune decisions bitwise when both sides hold the same predictor.
"""
import numpy as np
import pytest

import pyoracle as po
import wtutil as U

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def wt():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_10187_b200 import _core

    return _core


@pytest.fixture(scope="module")
def capi():
    from paper_2604_10187_b200 import capi as c

    c.lib()
    return c


@pytest.fixture(scope="module")
def ref():
    return po.Reference()


@pytest.fixture(scope="module")
def land(ref, tmpdir_session):
    reg, rec, tab = U.reference_fixture(ref, tmpdir_session)
    return dict(reg=reg, rec=rec, tab=tab, bp=po.ref_fit_baselines(ref, rec))


def _step_dict(bp):
    return {(int(m), int(l)): float(t) for m, l, t in zip(bp["step_macro"], bp["step_l"], bp["step_t"])}


def _core_bp(wt, kind, bp):
    """The reference's fitted predictor as a _core.BaselinePredictor."""
    p = wt.BaselinePredictor()
    if kind == 0:
        p.kind = "step"
        s = wt.StepPredictor()
        s.t_wave = _step_dict(bp)
        p.step = s
    else:
        p.kind = "linear"
        g = wt.GlobalLinearPredictor()
        th = bp["lin_theta"].reshape(-1, 4)
        g.theta = {int(m): wt.BilinearCoeffs(*map(float, th[i])) for i, m in enumerate(bp["lin_macro"])}
        p.linear = g
    return p


def test_fit_step_baseline_bitwise(wt, land):
    got = wt.fit_step_baseline(wt.read_records(land["rec"])).step.t_wave
    want = _step_dict(land["bp"])
    assert sorted(got) == sorted(want)
    for k, v in want.items():
        assert U.bits(np.array([got[k]]))[0] == U.bits(np.array([v]))[0], k


def test_fit_linear_baseline(wt, land):
    got = wt.fit_linear_baseline(wt.read_records(land["rec"])).linear.theta
    bp = land["bp"]
    # restatement: selected samples of every (macro, w, l) group in map order,
    # concatenated per macro, through the restated fit_bucket
    orc = po.Oracle()
    r = po.read_records_csv(land["rec"])
    order = np.lexsort((r["l"], r["w"], r["macro"]))
    keys = np.stack([r["macro"][order], r["w"][order], r["l"][order]], 1)
    cut = np.flatnonzero(np.any(np.diff(keys, axis=0) != 0, axis=1)) + 1
    per_macro = {}
    for grp in np.split(order, cut):
        st, _, _, gs, ts = orc.select_shared_micro(r["g"][grp], r["micro"][grp], r["lat"][grp])
        assert st == 0
        m, l = int(r["macro"][grp[0]]), int(r["l"][grp[0]])
        acc = per_macro.setdefault(m, ([], [], []))
        acc[0].extend(gs.astype(np.float64))
        acc[1].extend([float(l)] * len(gs))
        acc[2].extend(ts)
    th_ref = bp["lin_theta"].reshape(-1, 4)
    for i, m in enumerate(bp["lin_macro"]):
        c = got[int(m)]
        gc = np.array([c.alpha, c.beta, c.gamma, c.delta])
        st, co, _, _, _ = orc.fit_bucket(*per_macro[int(m)])
        assert st == 0
        np.testing.assert_array_equal(U.bits(gc), U.bits(co))
        np.testing.assert_allclose(gc, th_ref[i], rtol=1e-9, atol=1e-12)


def test_reference_unit_cases(wt):
    """tests/test_tuner.cpp:131-175, statement for statement."""
    bp = wt.BaselinePredictor()
    bp.kind = "step"
    s = wt.StepPredictor()
    s.t_wave = {(0, 16): 50.0}
    bp.step = s
    assert wt.baseline_predict(bp, 0, 10, 16, wt.HardwareSpec(4, 1, "")) == 150.0
    bp = wt.BaselinePredictor()
    bp.kind = "linear"
    g = wt.GlobalLinearPredictor()
    g.theta = {0: wt.BilinearCoeffs(0.01, 0.5, 0.2, 10.0)}
    bp.linear = g
    assert wt.baseline_predict(bp, 0, 100, 50, wt.HardwareSpec(4, 1, "")) == pytest.approx(120.0)
    recs = [wt.ProfileRecord(w * 100, 16, w, 0, 0, 50.0 * w) for w in range(1, 6)]
    assert wt.fit_step_baseline(recs).step.t_wave[(0, 16)] == pytest.approx(50.0)
    recs = [wt.ProfileRecord(g, l, w, 0, 0, 0.01 * g * l + 0.5 * g + 0.2 * l + 10)
            for w in range(1, 6) for l in (8, 16) for g in (w * 100 - 60, w * 100 - 20)]
    lb = wt.fit_linear_baseline(recs)
    assert lb.linear.theta[0].alpha == pytest.approx(0.01, rel=1e-9)
    assert wt.baseline_predict(lb, 0, 100, 50, wt.HardwareSpec(132, 1, "")) == pytest.approx(120.0, rel=1e-9)
    # errors: unknown macro -> out_of_range (IndexError), g < 1 -> invalid_argument (ValueError)
    with pytest.raises(IndexError, match="no linear baseline for macro 3"):
        wt.baseline_predict(lb, 3, 100, 50, wt.HardwareSpec(132, 1, ""))
    sb = wt.fit_step_baseline(recs)
    with pytest.raises(ValueError, match="grid size must be >= 1"):
        wt.baseline_predict(sb, 0, 0, 8, wt.HardwareSpec(132, 1, ""))
    assert wt.fit_step_baseline([]).step.t_wave == {}


@pytest.mark.parametrize("kind", [0, 1])
def test_baseline_predict_matches_reference(wt, ref, land, kind):
    bp = land["bp"]
    p = _core_bp(wt, kind, bp)
    rng = np.random.default_rng(kind)
    macros = np.unique(bp["step_macro"] if kind == 0 else bp["lin_macro"])
    for _ in range(300):
        m = int(rng.choice(np.append(macros, 99)))
        g, l = int(rng.integers(-2, 20000)), int(rng.integers(1, 200))
        st, want = po.ref_baseline_predict(ref, kind, bp, 132, 1, m, g, l)
        if st:
            with pytest.raises((IndexError, ValueError)):
                wt.baseline_predict(p, m, g, l, wt.HardwareSpec(132, 1, ""))
            continue
        got = wt.baseline_predict(p, m, g, l, wt.HardwareSpec(132, 1, ""))
        assert U.bits(np.array([got]))[0] == U.bits(np.array([want]))[0], (m, g, l)


@pytest.mark.parametrize("kind", [0, 1])
def test_baseline_tune_batch_matches_reference(wt, capi, ref, land, kind):
    """wt_baseline_tune_batch on 30k shapes vs the reference's baseline_tune()
    with the same predictor: macro, micro, latency (bits), wave, regime,
    comparisons, status."""
    bp = land["bp"]
    arrays = U.arrays_from_pytables(po.parse_tables_json(land["tab"])[1])
    eng = capi.Engine(arrays, U.registry_from_json(land["reg"]), n_sm=132)
    if kind == 0:
        b = capi.Baseline(eng, 0, bp["step_macro"], bp["step_l"], bp["step_t"])
    else:
        b = capi.Baseline(eng, 1, bp["lin_macro"], np.zeros(len(bp["lin_macro"]), np.int64), bp["lin_theta"])
    rng = np.random.default_rng(40 + kind)
    n = 30000
    M, N, K = (rng.integers(1, 9000, n) for _ in range(3))
    M[:3] = [0, 5, 1]
    dev = lambda a, dt=torch.int32: torch.as_tensor(np.ascontiguousarray(a)).to(dtype=dt, device="cuda")  # noqa
    o = dict(macro=torch.empty(n, dtype=torch.int32, device="cuda"), micro=torch.empty(n, dtype=torch.int32,
                                                                                          device="cuda"),
             lat=torch.empty(n, dtype=torch.float64, device="cuda"), wave=torch.empty(n, dtype=torch.int32,
                                                                                     device="cuda"),
             flags=torch.empty(n, dtype=torch.int32, device="cuda"), comps=torch.empty(n, dtype=torch.int32,
                                                                                      device="cuda"))
    d = capi.Engine.decisions(o["macro"], o["micro"], o["lat"], wave=o["wave"], flags=o["flags"], comps=o["comps"])
    b.tune_batch(dev(M), dev(N), dev(K), d)
    torch.cuda.synchronize()
    got = {k: v.cpu().numpy() for k, v in o.items()}
    h = ref.open(land["tab"], land["reg"], 132)
    want = po.ref_baseline_tune(ref, h, kind, bp, M, N, K)
    ref.close(h)
    st = (got["flags"].astype(np.uint32) >> 24).astype(np.int32)
    np.testing.assert_array_equal(st, want["status"])
    ok = want["status"] == 0
    assert ok.sum() > n - 10
    for k_g, k_w in (("macro", "macro"), ("micro", "micro"), ("wave", "w"), ("comps", "comps")):
        np.testing.assert_array_equal(got[k_g][ok], want[k_w][ok], err_msg=k_g)
    np.testing.assert_array_equal(U.bits(got["lat"][ok]), U.bits(want["lat"][ok]))
    np.testing.assert_array_equal((got["flags"][ok] & 1) != 0, want["extrap"][ok] != 0)
    # the C++ drop-in (single query) agrees with the batch
    p = _core_bp(wt, kind, bp)
    art, reg = wt.load_tables(land["tab"]), wt.ConfigRegistry.load(land["reg"])
    for i in range(3, 40):
        t = wt.baseline_tune(wt.DenseGemm(int(M[i]), int(N[i]), int(K[i])), p, art, reg, wt.HardwareSpec(132))
        assert (t.macro_id, t.micro_id, t.regime.w) == (got["macro"][i], got["micro"][i], got["wave"][i])
        assert t.stats.model_evals == len(art.tables)
    # a table without a baseline entry: out_of_range like the reference
    if kind == 1:
        q = wt.BaselinePredictor()
        q.kind = "linear"
        gl = wt.GlobalLinearPredictor()
        gl.theta = {0: wt.BilinearCoeffs(1.0, 1.0, 1.0, 1.0)}
        q.linear = gl
        with pytest.raises(IndexError, match="no linear baseline for macro 1"):
            wt.baseline_tune(wt.DenseGemm(100, 100, 100), q, art, reg, wt.HardwareSpec(132))
