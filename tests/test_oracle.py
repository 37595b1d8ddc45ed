"""Pin the oracle (plain-C restatement, oracle/wt_oracle.c) before trusting it:
(1) the golden vectors of the reference's own tests (proj/tests/*.cpp,
test_smoke.py), transcribed; (2) the reference compiled verbatim
(oracle/_ref/libwtref.so) on random inputs, bit for bit."""
import math
import os
import subprocess

import numpy as np
import pytest

import pyoracle as po
import wtutil as U
from conftest import ROOT, have_reference_build

needs_ref = pytest.mark.skipif(not have_reference_build(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def orc():
    return po.Oracle()


@pytest.fixture(scope="module")
def ref():
    if not have_reference_build():
        pytest.skip("oracle/_ref not built")
    return po.Reference()


def one_table(coeffs, W, theta_ext=(0, 0, 0, 0), anchors=None, ext=None, macro=0, tiles=(64, 64, 64)):
    t = po.PyTable(macro, W, 10, "sim", dict(coeffs), tuple(theta_ext), anchors or {1: {16: 0}}, ext or {16: 0})
    return po.FlatTables([t], {macro: tiles})


# ------------------------------------------------------------ golden vectors
def test_mapping_golden(orc):
    lib = orc.lib
    import ctypes as C

    g, l = C.c_int64(), C.c_int64()
    assert lib.wto_map_dense(C.c_int64(128), C.c_int64(64), C.c_int64(4096), C.c_int64(128), C.c_int64(64),
                             C.c_int64(64), C.byref(g), C.byref(l)) == 0
    assert (g.value, l.value) == (1, 64)  # test_kernel_map.cpp:11-16
    lib.wto_map_dense(C.c_int64(4096), C.c_int64(4096), C.c_int64(4096), C.c_int64(128), C.c_int64(256),
                      C.c_int64(64), C.byref(g), C.byref(l))
    assert (g.value, l.value) == (512, 64)  # test_smoke.py:36-45
    # attention (16 heads, s_q 512, s_kv 2048) under (64, 64): dense with t_n=1
    lib.wto_map_dense(C.c_int64(512), C.c_int64(16), C.c_int64(2048), C.c_int64(64), C.c_int64(1),
                      C.c_int64(64), C.byref(g), C.byref(l))
    assert (g.value, l.value) == (128, 32)  # test_kernel_map.cpp:41-46
    assert lib.wto_map_dense(C.c_int64(0), C.c_int64(1), C.c_int64(1), C.c_int64(1), C.c_int64(1), C.c_int64(1),
                             C.byref(g), C.byref(l)) == 1
    w = C.c_int32()
    for gg, sm, bps, want in ((10, 4, 1, 3), (132, 132, 1, 1), (133, 132, 1, 2), (264, 132, 2, 1)):
        assert lib.wto_wave_count(C.c_int64(gg), sm, bps, C.byref(w)) == 0
        assert w.value == want  # test_kernel_map.cpp:54-59
    prev = 0
    for gg in range(1, 301):  # non-decreasing (test_kernel_map.cpp:61-68)
        lib.wto_wave_count(C.c_int64(gg), 7, 1, C.byref(w))
        assert w.value >= prev
        prev = w.value


def test_predict_golden(orc):
    # test_model.cpp:88-92
    ft = one_table({1: (0.01, 0.5, 0.2, 10.0)}, W=1000)
    st, lat, ex, w, used = orc.predict(ft, 0, 100, 50, 4096, 1)
    assert st == 0 and abs(lat - 120.0) < 1e-9 and not ex
    ft = one_table({1: (0.0, 0.0, 0.0, 7.5)}, W=1000)
    assert orc.predict(ft, 0, 12345, 678, 1 << 20, 1)[1] == 7.5


def test_regime_and_missing_wave_golden(orc):
    # test_tuner.cpp:60-80 shape: W=4 on 132 SMs; erase wave 2
    co = {w: (0.001 * w, 0.1, 0.2 * w, 5.0 * w) for w in (1, 2, 3, 4)}
    ft = one_table(co, W=4, theta_ext=(1, 1, 1, 1))
    st, lat, ex, w, used = orc.predict(ft, 0, 4 * 132, 16, 132, 1)
    assert (st, ex, w, used) == (0, 0, 4, -1)
    st, lat, ex, w, used = orc.predict(ft, 0, 4 * 132 + 1, 16, 132, 1)
    assert (st, ex) == (0, 1)
    del co[2]
    ft = one_table(co, W=4)
    st, lat, ex, w, used = orc.predict(ft, 0, 200, 16, 132, 1)
    assert (st, ex, w, used) == (0, 0, 2, 1)  # "missing_wave_2_used_1"
    assert lat == 0.001 * 200 * 16 + 0.1 * 200 + 0.2 * 16 + 5.0
    assert orc.predict(one_table({}, W=4), 0, 10, 1, 132, 1)[0] == 2  # empty -> runtime_error


def test_nearest_anchor_golden(orc):
    # test_tuner.cpp:34-58
    st, r, c = orc.nearest_anchor([16, 32, 64], 40)
    assert r == 32 and c <= math.ceil(math.log2(3)) + 1
    assert orc.nearest_anchor([32, 64], 48)[1] == 32
    assert orc.nearest_anchor([32, 64], 5)[1] == 32
    assert orc.nearest_anchor([32, 64], 500)[1] == 64
    assert orc.nearest_anchor([7], 1000)[1] == 7
    assert orc.nearest_anchor([], 1)[0] == 1
    anchors = [a * 10 for a in range(1, 34)]
    for l in (1, 55, 166, 329, 400):
        st, got, c = orc.nearest_anchor(anchors, l)
        assert c <= math.ceil(math.log2(33)) + 1
        best = min(anchors, key=lambda a: abs(l - a))
        assert abs(l - got) == abs(l - best)


def bilinear_samples(a, b, c, d):
    g, l, t = [], [], []
    for gg in (3.0, 10.0, 47.0, 101.0):
        for ll in (2.0, 17.0):
            g.append(gg); l.append(ll); t.append(a * gg * ll + b * gg + c * ll + d)
    return g, l, t


def test_fit_bucket_golden(orc):
    # test_model.cpp:23-61
    g, l, t = bilinear_samples(0.01, 0.5, 0.2, 10.0)
    st, co, r2, mape, dg = orc.fit_bucket(g, l, t)
    assert st == 0 and not dg
    for got, want in zip(co, (0.01, 0.5, 0.2, 10.0)):
        assert abs(got - want) <= 1e-9 * (1 + abs(want))
    assert abs(r2 - 1.0) <= 1e-12 * 2
    held = co[0] * 250 * 33 + co[1] * 250 + co[2] * 33 + co[3]
    assert abs(held - (0.01 * 250 * 33 + 0.5 * 250 + 0.2 * 33 + 10)) < 1e-9 * 200

    def ssr(c):
        return sum((tt - (c[0] * gg * ll + c[1] * gg + c[2] * ll + c[3])) ** 2 for gg, ll, tt in zip(g, l, t))

    base = ssr(co)
    for which in range(4):
        for sign in (-1, 1):
            c = list(co)
            step = 1e-6 * abs(c[which]) if c[which] else 1e-6
            c[which] += sign * step
            assert ssr(c) >= base
    # constant data (test_model.cpp:64-72)
    g = [x for x in (5.0, 9.0, 20.0, 31.0) for _ in (3.0, 11.0)]
    l = [y for _ in (5.0, 9.0, 20.0, 31.0) for y in (3.0, 11.0)]
    st, co, r2, mape, dg = orc.fit_bucket(g, l, [42.0] * 8)
    assert abs(co[0] * 100 * 50 + co[1] * 100 + co[2] * 50 + co[3] - 42.0) < 1e-9 * 43
    # single l -> reduced fit exact at the samples (:73-80)
    g = [5.0, 9.0, 20.0, 31.0, 44.0]
    st, co, r2, mape, dg = orc.fit_bucket(g, [8.0] * 5, [3 * x + 7 for x in g])
    assert dg
    for x in g:
        assert abs(co[0] * x * 8 + co[1] * x + co[2] * 8 + co[3] - (3 * x + 7)) < 1e-9 * (3 * x + 7)
    assert orc.fit_bucket([3.0, 5.0], [2.0, 2.0], [10.0, 14.0])[4] == 1  # n < 4 flagged
    # acceptance A5 recovery (acceptance.cpp:313-323)
    gs, ls, ts = [], [], []
    for gg in (3.0, 10.0, 47.0, 101.0, 250.0):
        for ll in (2.0, 17.0, 33.0):
            gs.append(gg); ls.append(ll); ts.append(0.013 * gg * ll + 0.47 * gg + 0.21 * ll + 9.5)
    co = orc.fit_bucket(gs, ls, ts)[1]
    for got, want in zip(co, (0.013, 0.47, 0.21, 9.5)):
        assert abs(got / want - 1.0) < 1e-9


def test_select_shared_micro_golden(orc):
    # test_model.cpp:94-119
    st, m, part, g, t = orc.select_shared_micro([10, 20, 10, 20], [0, 0, 1, 1], [110, 90, 95, 85])
    assert (m, part, len(g)) == (1, 0, 2)
    assert orc.select_shared_micro([10], [3], [50])[1] == 3
    assert orc.select_shared_micro([10, 10], [2, 5], [100, 100])[1] == 2
    st, m, part, g, t = orc.select_shared_micro([10, 20, 30], [0, 1, 1], [10, 500, 500])
    assert (m, part) == (1, 1)


@needs_ref
def test_reference_unit_and_acceptance_suites_pass():
    """The reference's own doctest suite + A1,A5,A7,A9 run against the oracle
    build (Eigen shim) -- this pins the shim's QR to the reference goldens."""
    unit = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_unit")], capture_output=True, text=True)
    assert unit.returncode == 0, unit.stdout[-2000:] + unit.stderr[-2000:]
    acc = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_acceptance"), "A1", "A5", "A7", "A9"],
                         capture_output=True, text=True)
    assert acc.returncode == 0 and acc.stdout.count("PASS") == 4, acc.stdout


# ------------------------------------------------- restatement vs reference
@needs_ref
def test_tune_restatement_matches_reference(orc, ref, tmpdir_session):
    reg, rec, tab = U.reference_fixture(ref, tmpdir_session)
    fam, tabs = po.parse_tables_json(tab)
    tiles, order = po.parse_registry_json(reg)
    flat = po.FlatTables(tabs, tiles)
    rng = np.random.default_rng(21)
    n = 30000
    M, N, K = rng.integers(1, 9000, n), rng.integers(1, 9000, n), rng.integers(1, 9000, n)
    h = ref.open(tab, reg, 132)
    r = ref.tune(h, M, N, K, nthreads=4)
    o = orc.tune(flat, 132, 1, M, N, K)
    for k in ("macro", "micro", "g", "l", "w", "extrap", "comps", "status"):
        np.testing.assert_array_equal(r[k], o[k], err_msg=k)
    np.testing.assert_array_equal(U.bits(r["lat"]), U.bits(o["lat"]))
    np.testing.assert_array_equal(r["flag_count"], o["n_missing"] + (o["anchor_fb"] >= 0))
    ref.close(h)


@needs_ref
def test_fallbacks_restatement_matches_reference(orc, ref, tmpdir_session):
    """Mutilated artefact (missing waves, empty maps, NaN/inf, per-table W):
    restatement == reference, including error statuses and flag counts."""
    reg, rec, tab = U.reference_fixture(ref, tmpdir_session)
    fam, tabs = po.parse_tables_json(tab)
    rng = np.random.default_rng(4)
    for i, t in enumerate(tabs):
        if i % 3 == 0:
            for w in list(t.coeffs)[1::2]:
                del t.coeffs[w]
        if i % 3 == 1:
            t.anchors = {w: d for w, d in t.anchors.items() if w % 3 == 0}
            t.ext_anchors = {}
        if i == 2:
            t.coeffs[3] = (float("nan"),) * 4
        if i == 4:
            t.W = 6
    path = str(tmpdir_session / "mut_ref.json")
    U.write_tables_json(tabs, path)
    tiles, order = po.parse_registry_json(reg)
    flat = po.FlatTables(tabs, tiles)
    n = 20000
    M, N, K = rng.integers(-2, 9000, n), rng.integers(1, 9000, n), rng.integers(1, 20000, n)
    h = ref.open(path, reg, 132)
    r = ref.tune(h, M, N, K, nthreads=4)
    o = orc.tune(flat, 132, 1, M, N, K)
    np.testing.assert_array_equal(r["status"], o["status"])
    ok = r["status"] == 0
    for k in ("macro", "micro", "w", "extrap", "comps"):
        np.testing.assert_array_equal(r[k][ok], o[k][ok], err_msg=k)
    np.testing.assert_array_equal(U.bits(r["lat"][ok]), U.bits(o["lat"][ok]))
    np.testing.assert_array_equal(r["flag_count"][ok], (o["n_missing"] + (o["anchor_fb"] >= 0))[ok])
    ref.close(h)


@needs_ref
def test_fit_restatement_matches_reference(orc, ref):
    rng = np.random.default_rng(8)
    for trial in range(300):
        n = int(rng.integers(1, 25))
        g = rng.integers(1, 6000, n).astype(float)
        l = rng.choice([8.0, 16.0, 32.0, 48.0, 64.0], n)
        if trial % 7 == 0:
            l[:] = 16.0
        t = 0.01 * g * l + 0.3 * g + rng.random() * l + 5 + rng.normal(0, 3, n)
        a = ref.fit_bucket(g, l, t)
        b = orc.fit_bucket(g, l, t)
        assert a[0] == b[0] == 0
        np.testing.assert_array_equal(U.bits(a[1]), U.bits(b[1]))
        assert U.bits(np.array([a[2], a[3]])).tolist() == U.bits(np.array([b[2], b[3]])).tolist()
        assert a[4] == b[4]


@needs_ref
def test_select_restatement_matches_reference(orc, ref):
    rng = np.random.default_rng(12)
    for trial in range(500):
        n = int(rng.integers(1, 30))
        g = rng.integers(1, 6, n)
        m = rng.integers(0, 4, n)
        t = rng.integers(1, 5, n).astype(float) * 10  # many ties and duplicates
        a = ref.select_shared_micro(g, m, t)
        b = orc.select_shared_micro(g, m, t)
        assert a[:3] == b[:3]
        np.testing.assert_array_equal(a[3], b[3])
        np.testing.assert_array_equal(U.bits(a[4]), U.bits(b[4]))


@needs_ref
def test_build_restatement_matches_reference(orc, ref, tmpdir_session):
    for seed, (nm, nu, W) in ((7, (6, 8, 10)), (3, (3, 4, 6))):
        reg, rec, tab = U.reference_fixture(ref, tmpdir_session, n_macros=nm, n_micros=nu, W=W, seed=seed)
        fam, tabs = po.parse_tables_json(tab)
        tiles, order = po.parse_registry_json(reg)
        records = po.read_records_csv(rec)
        st, b = orc.build(records, order, W, 10)
        assert st == 0 and b["n_tables"] == len(tabs)
        for i, t in enumerate(tabs):
            assert b["macro_id"][i] == t.macro_id
            lo, hi = b["coeff_off"][i], b["coeff_off"][i + 1]
            ws = list(b["coeff_w"][lo:hi])
            assert ws == sorted(t.coeffs)
            th = b["coeff_theta"][4 * lo:4 * hi]
            np.testing.assert_array_equal(U.bits(th), U.bits(np.array([t.coeffs[w] for w in ws]).reshape(-1)))
            np.testing.assert_array_equal(U.bits(b["theta_ext"][4 * i:4 * i + 4]), U.bits(np.array(t.theta_ext)))
            for j, w in enumerate(ws):
                r2, mape, ns, flags = t.diagnostics[w]
                assert (b["diag_r2"][lo + j], b["diag_mape"][lo + j], b["diag_samples"][lo + j]) == (r2, mape, ns)
            for j in range(b["awave_off"][i], b["awave_off"][i + 1]):
                w = int(b["awave_w"][j])
                got = {int(b["anchor_l"][q]): int(b["anchor_micro"][q])
                       for q in range(b["awave_aoff"][j], b["awave_aoff"][j + 1])}
                assert got == t.anchors[w]
            ext = {int(b["ext_l"][q]): int(b["ext_micro"][q]) for q in range(b["ext_aoff"][i], b["ext_aoff"][i + 1])}
            assert ext == t.ext_anchors
