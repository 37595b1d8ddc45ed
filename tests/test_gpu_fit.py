"""GPU parity for K2 (batched least-squares + dual-table build) against the
oracle restatement and the reference's own build_dual_table (oracle/_ref).

Bar: coefficients, theta_ext, R^2 and MAPE bit-identical to the restatement
(same operation order); anchors / micro ids / flags / sample counts exact;
the reference build compared through its JSON artefact."""
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
def orc():
    return po.Oracle()


@pytest.fixture(scope="module")
def ref():
    return po.Reference()


def test_fit_bucket_batch_bitexact(capi, orc):
    rng = np.random.default_rng(4)
    gs, ls, ts, off = [], [], [], [0]
    for b in range(600):
        n = int(rng.integers(1, 70))
        g = rng.integers(1, 6000, n).astype(float)
        l = rng.choice([8.0, 16.0, 32.0, 48.0, 64.0, 80.0], n)
        kind = b % 6
        if kind == 0:
            l[:] = 32.0  # single l -> reduced fit
        t = 0.013 * g * l + 0.47 * g + 0.21 * l + 9.5
        if kind == 1:
            t = np.full(n, 42.0)
        elif kind == 2:
            t = t * (1 + rng.normal(0, 0.02, n))
        elif kind == 3:
            g[:] = g[0]
        gs.append(g); ls.append(l); ts.append(t); off.append(off[-1] + n)
    g, l, t = np.concatenate(gs), np.concatenate(ls), np.concatenate(ts)
    co, r2, mape, dg = capi.fit_bucket_batch(g, l, t, off)
    for b in range(len(off) - 1):
        s = slice(off[b], off[b + 1])
        st, c2, r22, m2, d2 = orc.fit_bucket(g[s], l[s], t[s])
        assert st == 0
        np.testing.assert_array_equal(U.bits(co[b]), U.bits(c2), err_msg=f"bucket {b}")
        assert U.bits(np.array([r2[b], mape[b]])).tolist() == U.bits(np.array([r22, m2])).tolist()
        assert dg[b] == d2


def compare_build(gpu, want, tabs_ref=None):
    assert gpu["n_tables"] == want["n_tables"]
    nt = gpu["n_tables"]
    for k in ("macro_id", "ext_flags"):
        np.testing.assert_array_equal(gpu[k], want[k][:nt], err_msg=k)
    for k in ("coeff_off", "awave_off", "ext_aoff"):
        np.testing.assert_array_equal(gpu[k], want[k][:nt + 1], err_msg=k)
    nc, naw = gpu["coeff_off"][-1], gpu["awave_off"][-1]
    nan, nex = gpu["awave_aoff"][-1], gpu["ext_aoff"][-1]
    for k, m in (("coeff_w", nc), ("diag_samples", nc), ("diag_flags", nc), ("awave_w", naw),
                 ("anchor_l", nan), ("anchor_micro", nan), ("anchor_partial", nan), ("ext_l", nex),
                 ("ext_micro", nex)):
        np.testing.assert_array_equal(gpu[k], want[k][:m], err_msg=k)
    np.testing.assert_array_equal(gpu["awave_aoff"], want["awave_aoff"][:naw + 1])
    for k, m in (("coeff_theta", 4 * nc), ("diag_r2", nc), ("diag_mape", nc), ("theta_ext", 4 * nt)):
        np.testing.assert_array_equal(U.bits(gpu[k]), U.bits(want[k][:m]), err_msg=k)


@pytest.mark.parametrize("shape", [(6, 8, 10, 5.0, 7), (3, 4, 6, 3.0, 42), (2, 3, 3, 0.0, 1)])
def test_build_matches_reference_fixture(capi, orc, ref, tmpdir_session, shape):
    nm, nu, W, sigma, seed = shape
    reg, rec, tab = U.reference_fixture(ref, tmpdir_session, n_macros=nm, n_micros=nu, W=W, sigma=sigma, seed=seed)
    tiles, order = po.parse_registry_json(reg)
    records = po.read_records_csv(rec)
    gpu = capi.fit_build(records, order, W, 10)
    st, want = orc.build(records, order, W, 10)
    assert st == 0
    compare_build(gpu, want)
    # and the reference's own artefact (through JSON)
    fam, tabs = po.parse_tables_json(tab)
    assert [t.macro_id for t in tabs] == list(gpu["macro_id"])
    for i, t in enumerate(tabs):
        lo, hi = gpu["coeff_off"][i], gpu["coeff_off"][i + 1]
        got = {int(w): tuple(gpu["coeff_theta"][4 * j:4 * j + 4]) for j, w in zip(range(lo, hi), gpu["coeff_w"][lo:hi])}
        assert set(got) == set(t.coeffs)
        for w in got:
            assert U.bits(np.array(got[w])).tolist() == U.bits(np.array(t.coeffs[w])).tolist()
        assert U.bits(gpu["theta_ext"][4 * i:4 * i + 4]).tolist() == U.bits(np.array(t.theta_ext)).tolist()


def test_build_edge_records(capi, orc):
    """Duplicated (micro, g) rows (last write wins), partial micro coverage,
    unknown macro ids, sparse buckets, single-wave macros, W=0 (max wave)."""
    rng = np.random.default_rng(17)
    rows = []
    for macro in range(7):
        waves = [1] if macro == 3 else list(range(1, 1 + int(rng.integers(2, 13))))
        for w in waves:
            for l in (8, 16, 32):
                for gi in range(int(rng.integers(1, 5))):
                    g = (w - 1) * 100 + 10 + 20 * gi
                    for micro in range(3):
                        if macro == 5 and micro == 1 and gi == 0:
                            continue  # partial coverage
                        t = (5 + micro + 0.3 * macro) * w * (1 + l / 50) * (1 + 0.01 * rng.random())
                        rows.append((g, l, w, macro, micro, t))
                        if rng.random() < 0.1:
                            rows.append((g, l, w, macro, micro, t * 1.5))  # duplicate, last wins
    rows.append((10, 8, 1, 99, 0, 5.0))  # macro not in registry: ignored
    r = np.array(rows, dtype=object)
    rec = dict(g=r[:, 0].astype(np.int64), l=r[:, 1].astype(np.int64), w=r[:, 2].astype(np.int32),
               macro=r[:, 3].astype(np.int32), micro=r[:, 4].astype(np.int32), lat=r[:, 5].astype(np.float64))
    order = [6, 0, 5, 1, 2, 3, 4]
    for W in (0, 5, 12):
        gpu = capi.fit_build(rec, order, W, 4)
        st, want = orc.build(rec, order, W, 4)
        assert st == 0
        compare_build(gpu, want)


@pytest.mark.parametrize("const", ["l", "g", "w", "macro", "all_valid", "one_micro"])
def test_build_constant_fields(capi, orc, const):
    """Sort-key fields that are constant over the records pack to zero bits
    and drop out of the radix sort; the group / select / sample kernels then
    decode the remaining fields from the sorted keys (one packing pass).
    Every such case against the restatement."""
    rng = np.random.default_rng(23)
    rows = []
    for macro in range(1 if const == "macro" else 5):
        for w in ([3] if const == "w" else range(1, 6)):
            for l in ([16] if const == "l" else (8, 16, 32)):
                for gi in range(1 if const == "g" else 3):
                    g = 250 if const == "g" else (w - 1) * 100 + 10 + 20 * gi
                    for micro in range(1 if const == "one_micro" else 2):
                        t = (5 + micro + 0.3 * macro) * w * (1 + l / 50) * (1 + 0.01 * rng.random())
                        rows.append((g, l, w, macro, 10 * macro + micro, t))
    if const != "all_valid":
        rows.append((10, 8, 1, 99, 0, 5.0))  # a record of an unknown macro (not every record valid)
    r = np.array(rows, dtype=object)
    rec = dict(g=r[:, 0].astype(np.int64), l=r[:, 1].astype(np.int64), w=r[:, 2].astype(np.int32),
               macro=r[:, 3].astype(np.int32), micro=r[:, 4].astype(np.int32), lat=r[:, 5].astype(np.float64))
    order = list(range(5))
    for W in (0, 4):
        gpu = capi.fit_build(rec, order, W, 4)
        st, want = orc.build(rec, order, W, 4)
        assert st == 0
        compare_build(gpu, want)


def test_build_config4_scale_subset_parity(capi, orc):
    """Config 4 (4608 configs x 131 plan points x 5 anchors ~ 3.0M records):
    the full GPU build, checked bit for bit against the oracle on a 48-macro
    subset (tables depend only on their own macro's records)."""
    from paper_2604_10187_b200 import synthetic as S

    cfg = S.config_space(full=True)
    rec = S.synthetic_records(cfg, micros_per_macro=1)
    ids = cfg["id"]
    gpu = capi.fit_build(rec, ids, 40, 10)
    assert gpu["n_tables"] == len(ids)
    sub_ids = ids[::96]
    mask = np.isin(rec["macro"], sub_ids)
    sub = {k: v[mask] for k, v in rec.items()}
    st, want = orc.build(sub, sub_ids, 40, 10)
    assert st == 0
    pos = {int(m): i for i, m in enumerate(gpu["macro_id"])}
    for j, m in enumerate(want["macro_id"][:want["n_tables"]]):
        i = pos[int(m)]
        a0, a1 = gpu["coeff_off"][i], gpu["coeff_off"][i + 1]
        b0, b1 = want["coeff_off"][j], want["coeff_off"][j + 1]
        np.testing.assert_array_equal(gpu["coeff_w"][a0:a1], want["coeff_w"][b0:b1])
        np.testing.assert_array_equal(U.bits(gpu["coeff_theta"][4 * a0:4 * a1]), U.bits(want["coeff_theta"][4 * b0:4 * b1]))
        np.testing.assert_array_equal(U.bits(gpu["diag_r2"][a0:a1]), U.bits(want["diag_r2"][b0:b1]))
        np.testing.assert_array_equal(U.bits(gpu["theta_ext"][4 * i:4 * i + 4]), U.bits(want["theta_ext"][4 * j:4 * j + 4]))
    # predicted-vs-sampled error on the synthetic profile is reported, and sane
    assert np.median(gpu["diag_mape"]) < 0.05


@pytest.mark.parametrize("world", [2, 3, 8])
def test_macro_sharded_fit_equals_full_build(capi, world):
    """dist.sharded_fit's decomposition on one GPU: fit_build over each
    rank's contiguous registry slice, merged in rank order, is bit-identical
    to the single build (every array, every offset)."""
    from paper_2604_10187_b200 import synthetic as S
    from paper_2604_10187_b200.dist import macro_shards, merge_tables, records_of

    cfg = S.config_space(False)
    rec = S.synthetic_records(cfg, micros_per_macro=2)
    full = capi.fit_build(rec, cfg["id"], 40, 10)
    parts = [capi.fit_build(records_of(rec, ids), ids, 40, 10) for ids in macro_shards(cfg["id"], world)]
    got = merge_tables(parts)
    assert got["n_tables"] == full["n_tables"]
    for k, v in got.items():
        if isinstance(v, np.ndarray):
            if v.dtype == np.float64:
                np.testing.assert_array_equal(v.view(np.int64), full[k].view(np.int64), err_msg=k)
            else:
                np.testing.assert_array_equal(v, full[k], err_msg=k)


def test_memmap_artifacts_feed_fit_and_engine(capi, tmp_path):
    """Binary SoA images (artifact.py) loaded as memmap views go straight
    into wt_fit_build / wt_engine_create: same tables, same decisions."""
    import torch

    from paper_2604_10187_b200 import artifact as A, synthetic as S

    cfg = S.config_space(False)
    rec = {k: np.asarray(v, A.RECORD_FIELDS[k]) for k, v in S.synthetic_records(cfg).items()}
    A.save_records_bin(str(tmp_path / "r.wtr"), rec)
    rm = A.load_records_bin(str(tmp_path / "r.wtr"))
    f1 = capi.fit_build(rec, cfg["id"], 40, 10)
    f2 = capi.fit_build(rm, cfg["id"], 40, 10)
    for k in A.TABLE_FIELDS:
        if k in f1:
            np.testing.assert_array_equal(np.asarray(f1[k]), np.asarray(f2[k]), err_msg=k)
    t = {k: f1[k] for k in A.TABLE_FIELDS if k in f1}
    t["W"] = f1["W_arr"]
    A.save_tables_bin(str(tmp_path / "t.wtt"), t)
    tm = A.load_tables_bin(str(tmp_path / "t.wtt"))
    reg = S.registry_arrays(cfg)
    M, N, K = S.query_stream(5000, S.LLAMA3_8B, seed=2, off_grid_frac=0.5)
    outs = []
    for tab in (t, tm):
        eng = capi.Engine(tab, reg, n_sm=148)
        o = [torch.empty(len(M), dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
        eng.tune_batch(*(torch.from_numpy(x).cuda() for x in (M, N, K)), capi.Engine.decisions(*o))
        torch.cuda.synchronize()
        outs.append([x.cpu().numpy() for x in o])
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a.view(np.int64) if a.dtype == np.float64 else a,
                                      b.view(np.int64) if b.dtype == np.float64 else b)
