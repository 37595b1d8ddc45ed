"""The Python drop-in (`_core`, reference bindings.cpp names) end to end on the
GPU: the reference's own smoke test (tests/python/test_smoke.py) re-expressed,
plus tune() / predict_latency() / build_tables() against the reference
compiled verbatim, including Tuned.flags text."""
import math

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
def ref():
    return po.Reference()


@pytest.fixture
def registry(wt):
    r = wt.ConfigRegistry()
    r.family = "dense_gemm"
    r.macros = [wt.MacroConfig(0, wt.GemmTiles(64, 64, 64)), wt.MacroConfig(1, wt.GemmTiles(128, 128, 64))]
    r.micros = [wt.MicroConfig(0, 2, 4), wt.MicroConfig(1, 3, 4)]
    for ma in (0, 1):
        for mi in (0, 1):
            r.add_feasible(ma, mi)
    r.validate()
    return r


def test_smoke_pipeline(wt, registry, ref, tmp_path):
    """test_smoke.py:test_full_pipeline with reference-simulated records."""
    hw = wt.HardwareSpec(132)
    regp, recp = str(tmp_path / "reg.json"), str(tmp_path / "rec.csv")
    registry.save(regp)
    # records from the reference's simulator for the same registry shape
    ref.fixture(132, 2, 2, 4, 4, 1.5, [8, 16, 32], 0.0, 9, str(tmp_path / "r2.json"), recp)
    records = wt.read_records(recp)
    reg2 = wt.ConfigRegistry.load(str(tmp_path / "r2.json"))
    tables = wt.build_tables(records, reg2, hw, W=4)
    assert len(tables.tables) == 2
    path = str(tmp_path / "tables.json")
    wt.save_tables(tables, path)
    loaded = wt.load_tables(path)
    assert [t.macro_id for t in loaded.tables] == [0, 1]
    decision = wt.tune(wt.DenseGemm(2000, 2000, 2048), loaded, reg2, hw)
    assert decision.macro_id in (0, 1)
    assert decision.stats.model_evals == 2
    again = wt.tune(wt.DenseGemm(2000, 2000, 2048), loaded, reg2, hw)
    assert (again.macro_id, again.micro_id) == (decision.macro_id, decision.micro_id)
    latency, regime = wt.predict_latency(loaded.tables[0], 200, 16, hw)
    assert latency > 0 and not regime.extrapolated
    # the reference's own build on the same records gives the same artefact
    ref.build(recp, str(tmp_path / "r2.json"), "", 132, 4, 10, str(tmp_path / "ref_tables.json"))
    assert open(tmp_path / "ref_tables.json", "rb").read() == open(path, "rb").read().replace(b"", b"")


def test_build_tables_byte_identical_to_reference(wt, ref, tmpdir_session, tmp_path):
    """build_dual_table on the GPU, saved by the drop-in, equals the reference's
    tables.json byte for byte (coefficients, diagnostics, flags, anchors)."""
    for shape in ((6, 8, 10, 5.0, 7), (3, 4, 6, 3.0, 42)):
        nm, nu, W, sigma, seed = shape
        reg, rec, tab = U.reference_fixture(ref, tmpdir_session, n_macros=nm, n_micros=nu, W=W, sigma=sigma,
                                            seed=seed)
        r = wt.ConfigRegistry.load(reg)
        art = wt.build_tables(wt.read_records(rec), r, wt.HardwareSpec(132, 1, "sim"), W=W, p=10)
        out = str(tmp_path / f"t{seed}.json")
        wt.save_tables(art, out)
        assert open(tab, "rb").read() == open(out, "rb").read()


def test_tune_and_flags_match_reference(wt, ref, tmpdir_session, tmp_path):
    reg, rec, tab = U.reference_fixture(ref, tmpdir_session)
    fam, tabs = po.parse_tables_json(tab)
    for i, t in enumerate(tabs):  # force every fallback rule
        if i % 2 == 0:
            for w in list(t.coeffs)[1::3]:
                del t.coeffs[w]
        if i % 3 == 1:
            t.anchors = {w: d for w, d in t.anchors.items() if w % 4 == 0}
            t.ext_anchors = {}
    mut = str(tmp_path / "mut.json")
    U.write_tables_json(tabs, mut)
    art = wt.load_tables(mut)
    r = wt.ConfigRegistry.load(reg)
    hw = wt.HardwareSpec(132)
    h = ref.open(mut, reg, 132)
    rng = np.random.default_rng(1)
    n_flags = 0
    for _ in range(300):
        M, N, K = (int(x) for x in rng.integers(1, 9000, 3))
        got = wt.tune(wt.DenseGemm(M, N, K), art, r, hw)
        want = ref.tune(h, [M], [N], [K])
        st, flags = ref.tune_flags(h, M, N, K)
        assert want["status"][0] == 0 and st == 0
        assert (got.macro_id, got.micro_id, got.g, got.l) == (want["macro"][0], want["micro"][0], want["g"][0],
                                                               want["l"][0])
        assert U.bits(np.array([got.predicted_latency_us]))[0] == U.bits(want["lat"])[0]
        assert (got.regime.extrapolated, got.regime.w) == (bool(want["extrap"][0]), want["w"][0])
        assert got.stats.anchor_comparisons == want["comps"][0] and got.stats.model_evals == len(tabs)
        assert list(got.flags) == flags
        n_flags += len(flags) > 0
    assert n_flags > 10
    ref.close(h)


def test_errors_match_reference(wt, registry):
    hw = wt.HardwareSpec(132)
    t = wt.DualTable()
    t.macro_id = 0
    t.W = 4
    t.coeff_table = {1: wt.BilinearCoeffs(0.01, 0.5, 0.2, 10.0)}
    t.anchor_table = {1: {16: 0}}
    t.ext_anchors = {16: 0}
    art = wt.TableArtifact()
    art.tables = [t]
    with pytest.raises(ValueError, match="dense_gemm dims must be >= 1"):
        wt.tune(wt.DenseGemm(0, 1, 1), art, registry, hw)
    t2 = wt.DualTable()
    t2.macro_id = 0
    t2.W = 4
    t2.anchor_table = {1: {16: 0}}
    art.tables = [t2]
    with pytest.raises(RuntimeError, match="dual table for macro 0 has no coefficient entries"):
        wt.tune(wt.DenseGemm(64, 64, 64), art, registry, hw)
    with pytest.raises(ValueError, match="empty anchor list"):
        wt.nearest_anchor([], 1)
    ref = po.Reference()
    for anchors, l in (([16, 32, 64], 40), ([32, 64], 48), ([32, 64], 5), ([32, 64], 500), ([7], 1000)):
        assert wt.nearest_anchor(anchors, l) == ref.nearest_anchor(anchors, l)
    lat, regime = wt.predict_latency(t, 100, 50, wt.HardwareSpec(4096))
    assert abs(lat - 120.0) < 1e-9


def test_fit_and_select_dropin(wt):
    s = [wt.FitSample(g, l, 0.01 * g * l + 0.5 * g + 0.2 * l + 10.0) for g in (3.0, 10.0, 47.0, 101.0)
         for l in (2.0, 17.0)]
    f = wt.fit_bucket(s)
    assert not f.degenerate and abs(f.coeffs.alpha - 0.01) < 1e-11 and abs(f.r2 - 1) < 1e-12
    rec = lambda g, m, t: wt.ProfileRecord(g, 4, 1, 0, m, t)  # noqa: E731
    sel = wt.select_shared_micro([rec(10, 0, 110), rec(20, 0, 90), rec(10, 1, 95), rec(20, 1, 85)])
    assert sel.micro_id == 1 and len(sel.samples) == 2 and not sel.partial_coverage
    sel = wt.select_shared_micro([rec(10, 0, 10), rec(20, 1, 500), rec(30, 1, 500)])
    assert sel.micro_id == 1 and sel.partial_coverage
    recs = [wt.ProfileRecord(g, l, w, 0, 0, 0.02 * g * l + 0.3 * g + 1.0 * l + 5.0)
            for w in range(1, 13) for l in (4, 8) for g in (w * 100 - 50, w * 100 - 10)]
    e = wt.fit_extrapolation(recs, 12, 10)
    assert not e.flags and abs(e.theta_ext.alpha - 0.02) < 1e-9 * 0.02 + 1e-12


def test_engine_batch_host(wt, ref, tmpdir_session):
    reg, rec, tab = U.reference_fixture(ref, tmpdir_session)
    eng = wt.Engine(wt.load_tables(tab), wt.ConfigRegistry.load(reg), wt.HardwareSpec(132))
    rng = np.random.default_rng(7)
    M, N, K = (rng.integers(1, 9000, 20000).astype(np.int32) for _ in range(3))
    ma, mi, lat = eng.tune_batch(M, N, K)
    h = ref.open(tab, reg, 132)
    want = ref.tune(h, M, N, K, nthreads=8)
    np.testing.assert_array_equal(ma, want["macro"])
    np.testing.assert_array_equal(mi, want["micro"])
    np.testing.assert_array_equal(U.bits(lat), U.bits(want["lat"]))
    ref.close(h)
    t = eng.tune(wt.DenseGemm(int(M[0]), int(N[0]), int(K[0])))
    assert t.macro_id == ma[0]


def test_reference_smoke_suite_verbatim_semantics(wt, registry, tmp_path):
    """tests/python/test_smoke.py of the reference, statement for statement,
    against this module (simulator + profile + fit + tune all on the GPU)."""
    import math

    g = wt.SyntheticKernelGround()
    g.set_entry(0, 0, wt.GroundEntry(20.0, 2.0))
    g.set_entry(0, 1, wt.GroundEntry(22.0, 1.8))
    g.set_entry(1, 0, wt.GroundEntry(70.0, 5.0))
    g.set_entry(1, 1, wt.GroundEntry(77.0, 4.5))
    hw = wt.HardwareSpec(132)
    # test_mapping_and_waves
    macro = wt.MacroConfig(0, wt.GemmTiles(128, 256, 64))
    gg, l = wt.map_workload(wt.DenseGemm(4096, 4096, 4096), macro)
    assert (gg, l) == (32 * 16, 64) and wt.wave_count(gg, hw) == math.ceil(512 / 132)
    # test_simulate_step_law
    assert wt.simulate(hw, 132, 1, 50.0) == 50.0
    assert wt.simulate(hw, 133, 1, 50.0) == 100.0
    noisy = wt.simulate(hw, 264, 1, 50.0, sigma=10.0, seed=3)
    assert noisy == wt.simulate(hw, 264, 1, 50.0, sigma=10.0, seed=3)
    # test_full_pipeline
    plan = wt.build_plan(hw, "dense_gemm", W=4, I=4, tau=1.5, loop_anchors=[8, 16, 32])
    assert 0 < len(plan.grid_points) <= 16
    records = wt.run_profile_sim(plan, registry, g, sigma=0.0, seed=9)
    assert len(records) == len(plan.grid_points) * 3 * 4
    tables = wt.build_tables(records, registry, hw, W=4)
    assert len(tables.tables) == 2
    path = str(tmp_path / "tables.json")
    wt.save_tables(tables, path)
    loaded = wt.load_tables(path)
    assert [t.macro_id for t in loaded.tables] == [0, 1]
    decision = wt.tune(wt.DenseGemm(2000, 2000, 2048), loaded, registry, hw)
    assert decision.macro_id in (0, 1) and decision.stats.model_evals == 2
    latency, regime = wt.predict_latency(loaded.tables[0], 200, 16, hw)
    assert latency > 0 and not regime.extrapolated
    # test_records_csv_roundtrip
    plan2 = wt.build_plan(hw, "dense_gemm", W=2, I=2, tau=1.5, loop_anchors=[8])
    recs = wt.run_profile_sim(plan2, registry, g, sigma=2.0, seed=1)
    p2 = str(tmp_path / "records.csv")
    wt.write_records(recs, p2)
    assert [r.latency_us for r in wt.read_records(p2)] == [r.latency_us for r in recs]
    # exhaustive oracle on the GPU simulator
    best = wt.oracle_best(hw, 3, wt.DenseGemm(2000, 2000, 2048), registry, g, sigma=0.0, reps=1)
    assert (best.macro_id, best.micro_id) in {(0, 0), (0, 1), (1, 0), (1, 1)}
