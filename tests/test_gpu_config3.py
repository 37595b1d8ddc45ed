"""GPU parity at BASELINE.json config 3 -- the build-time configuration the
bench times: 4,608 decomposed tile configs (every full config its own
macro_id) fitted on the GPU from the wave-structured synthetic
records, then the decision grid over the 6 Llama-3-70B / Qwen2-72B (N, K)
pairs x M = 1..65536 (393,216 shapes) swept with exact pruning.

Oracles:
  * the C restatement (oracle/wt_oracle.c, itself pinned bit-for-bit to the
    reference in tests/test_oracle.py): EVERY grid entry;
  * the reference compiled verbatim (oracle/_ref, tune() = tuner.cpp:159-166)
    on a stratified sample: wave boundaries of every tile class, random M per
    pair, the first and last M, and an off-grid slice;
  * a second GPU witness: the same grid swept with pruning disabled.
Bar: macro / micro / wave / comparisons bit-exact, latency bitwise."""
import os

import numpy as np
import pytest

import pyoracle as po
import wtutil as U

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

PAIRS = None
M_HI = 65536
SLOTS = 148


@pytest.fixture(scope="module")
def capi():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_10187_b200 import capi as c

    c.lib()
    return c


@pytest.fixture(scope="module")
def c3(capi):
    from paper_2604_10187_b200 import synthetic as S

    cfg = S.config_space(full=True)
    rec = S.synthetic_records(cfg, micros_per_macro=1)
    fit = capi.fit_build(rec, cfg["id"], 40, 10)
    t3 = {k: fit[k] for k in ("macro_id", "theta_ext", "coeff_off", "coeff_w", "coeff_theta", "awave_off",
                               "awave_w", "awave_aoff", "anchor_l", "anchor_micro", "ext_aoff", "ext_l",
                               "ext_micro")}
    t3["W"] = fit["W_arr"]
    eng = capi.Engine(t3, S.registry_arrays(cfg), n_sm=SLOTS)
    pairs = S.unique_pairs(S.LLAMA3_70B, S.QWEN2_72B)
    grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, M_HI)
    grid.sweep()
    torch.cuda.synchronize()
    flat = po.FlatTables(U.pytables_from_arrays(t3), U.tiles_of(cfg))
    yield dict(cfg=cfg, rec=rec, fit=fit, t3=t3, eng=eng, grid=grid, pairs=pairs, flat=flat)
    grid.close()
    eng.close()


def grid_queries(pairs):
    M = np.tile(np.arange(1, M_HI + 1, dtype=np.int64), len(pairs))
    N = np.repeat(np.array([p[0] for p in pairs], np.int64), M_HI)
    K = np.repeat(np.array([p[1] for p in pairs], np.int64), M_HI)
    return M, N, K


def read_entries(grid):
    e = grid.entries_tensor().cpu().numpy().copy()
    grid.finalize()  # taking the raw storage invalidated the run index
    torch.cuda.synchronize()
    return dict(lat=e[:, :2].copy().view(np.float64)[:, 0], macro=e[:, 2], micro=e[:, 3], wave=e[:, 4],
                flags=e[:, 5].view(np.uint32), comps=e[:, 6])


def wave_boundaries(cfg, pairs):
    """Flat grid indices of every M where some tile class's wave count
    changes (w <= R), plus M and M+1 around it, plus the first and last M."""
    cls = sorted({(int(a), int(b)) for a, b in zip(cfg["t_m"], cfg["t_n"])})
    idx = set()
    for pi, (N, _K) in enumerate(pairs):
        for tm, tn in cls:
            nt = -(-N // tn)
            for w in range(1, 42):
                mt = (w * SLOTS) // nt  # largest mt with mt * nt <= w * S
                for M in (mt * tm, mt * tm + 1, mt * tm - tm + 1):
                    if 1 <= M <= M_HI:
                        idx.add(pi * M_HI + M - 1)
        idx.add(pi * M_HI)
        idx.add(pi * M_HI + M_HI - 1)
    return np.array(sorted(idx), np.int64)


def test_config3_fit_matches_restatement(c3):
    """The GPU-fitted tables the sweep uses == the restatement's build of the
    same records (coefficients bitwise; anchors and micro ids exact)."""
    st, b = po.Oracle().build(c3["rec"], c3["cfg"]["id"], 40, 10)
    assert st == 0
    f = c3["fit"]
    nt = b["n_tables"]
    assert f["n_tables"] == nt == len(c3["cfg"]["id"])
    ncoef = int(b["coeff_off"][nt])
    for k in ("coeff_off", "awave_off", "ext_aoff"):
        np.testing.assert_array_equal(f[k], b[k][: nt + 1], err_msg=k)
    for k, n in (("coeff_w", ncoef), ("awave_w", int(b["awave_off"][nt])),
                 ("anchor_l", int(b["awave_aoff"][int(b["awave_off"][nt])])),
                 ("anchor_micro", int(b["awave_aoff"][int(b["awave_off"][nt])])),
                 ("ext_l", int(b["ext_aoff"][nt])), ("ext_micro", int(b["ext_aoff"][nt]))):
        np.testing.assert_array_equal(f[k], b[k][:n], err_msg=k)
    np.testing.assert_array_equal(U.bits(f["coeff_theta"]), U.bits(b["coeff_theta"][: 4 * ncoef]))
    np.testing.assert_array_equal(U.bits(f["theta_ext"]), U.bits(b["theta_ext"][: 4 * nt]))


def test_config3_every_grid_entry_matches_restatement(c3):
    """All 393,216 entries of the swept config-3 grid == the restatement's
    tune() (4,608 configs each)."""
    ent = read_entries(c3["grid"])
    M, N, K = grid_queries(c3["pairs"])
    want = U.oracle_tune_mt(po.Oracle(), c3["flat"], SLOTS, 1, M, N, K)
    assert (want["status"] == 0).all()
    np.testing.assert_array_equal(ent["macro"], want["macro"])
    np.testing.assert_array_equal(ent["micro"], want["micro"])
    np.testing.assert_array_equal(ent["wave"], want["w"])
    np.testing.assert_array_equal(ent["comps"], want["comps"])
    np.testing.assert_array_equal(U.bits(ent["lat"]), U.bits(want["lat"]))
    np.testing.assert_array_equal((ent["flags"] & 1) != 0, want["extrap"] != 0)


def test_config3_unpruned_witness(c3, capi):
    """Second witness: the same grid swept with every config evaluated."""
    ent = read_entries(c3["grid"])
    eng, pairs = c3["eng"], c3["pairs"]
    g2 = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, M_HI)
    eng.set_prune(False)
    try:
        g2.sweep()
        torch.cuda.synchronize()
    finally:
        eng.set_prune(True)
    e2 = read_entries(g2)
    g2.close()
    for k in ("macro", "micro", "wave", "flags", "comps"):
        np.testing.assert_array_equal(ent[k], e2[k], err_msg=k)
    np.testing.assert_array_equal(U.bits(ent["lat"]), U.bits(e2["lat"]))


def _ref_handle(c3, tmp):
    ref = po.Reference()
    tp, rp = os.path.join(str(tmp), "t3.json"), os.path.join(str(tmp), "r3.json")
    U.write_tables_json(U.pytables_from_arrays(c3["t3"]), tp)
    from paper_2604_10187_b200 import synthetic as S

    U.write_registry_json(S.registry_arrays(c3["cfg"]), rp)
    return ref, ref.open(tp, rp, SLOTS)


def test_config3_grid_and_gather_match_reference(c3, tmpdir_session):
    """Stratified sample against the reference's own tune(): wave boundaries
    of every tile class, random M per pair, first / last M -- read from the
    grid entries AND answered through the hashed gather (run index)."""
    ref, h = _ref_handle(c3, tmpdir_session)
    rng = np.random.default_rng(3)
    bnd = wave_boundaries(c3["cfg"], c3["pairs"])
    npair = len(c3["pairs"])
    rnd = (rng.integers(0, npair, 300) * M_HI + rng.integers(0, M_HI, 300)).astype(np.int64)
    firstlast = np.array([p * M_HI for p in range(npair)] + [p * M_HI + M_HI - 1 for p in range(npair)], np.int64)
    idx = np.unique(np.concatenate([rng.choice(bnd, min(len(bnd), 900), replace=False), rnd, firstlast]))
    M, N, K = (a[idx] for a in grid_queries(c3["pairs"]))
    thr = max(1, min(32, len(os.sched_getaffinity(0))))
    want = ref.tune(h, M, N, K, nthreads=thr)
    ref.close(h)
    assert (want["status"] == 0).all()
    assert (want["evals"] == len(c3["cfg"]["id"])).all()
    ent = read_entries(c3["grid"])
    for kg, kw in (("macro", "macro"), ("micro", "micro"), ("wave", "w"), ("comps", "comps")):
        np.testing.assert_array_equal(ent[kg][idx], want[kw], err_msg=kg)
    np.testing.assert_array_equal(U.bits(ent["lat"][idx]), U.bits(want["lat"]))
    # the same queries through the serving path (hashed gather, plain outputs)
    n = len(idx)
    out = [torch.empty(n, dtype=dt, device="cuda") for dt in (torch.int32, torch.int32, torch.float64)]
    dv = lambda a: torch.as_tensor(a.astype(np.int32)).cuda()
    c3["grid"].gather(dv(M), dv(N), dv(K), c3["eng"].decisions(*out))
    torch.cuda.synchronize()
    mac, mic, lat = (o.cpu().numpy() for o in out)
    np.testing.assert_array_equal(mac, want["macro"])
    np.testing.assert_array_equal(mic, want["micro"])
    np.testing.assert_array_equal(U.bits(lat), U.bits(want["lat"]))


def test_config3_offgrid_tune_batch(c3, capi, tmpdir_session):
    """Off-grid slice on the same engine: random (M, N, K) evaluated in full
    (pruned list evaluation) vs the restatement (20k) and the reference (300)."""
    rng = np.random.default_rng(8)
    n = 20000
    M = rng.integers(1, 65537, n).astype(np.int64)
    N = rng.integers(256, 65537, n).astype(np.int64)
    K = rng.integers(256, 32769, n).astype(np.int64)
    out = [torch.empty(n, dtype=dt, device="cuda") for dt in (torch.int32, torch.int32, torch.float64)]
    flags = torch.empty(n, dtype=torch.int32, device="cuda")
    dv = lambda a: torch.as_tensor(a.astype(np.int32)).cuda()
    d = c3["eng"].decisions(*out, flags=flags)
    c3["eng"].tune_batch(dv(M), dv(N), dv(K), d)
    # and the same stream through the grid (every query is off-grid there)
    out2 = [torch.empty(n, dtype=dt, device="cuda") for dt in (torch.int32, torch.int32, torch.float64)]
    c3["grid"].gather(dv(M), dv(N), dv(K), c3["eng"].decisions(*out2))
    torch.cuda.synchronize()
    mac, mic, lat = (o.cpu().numpy() for o in out)
    for a, b in zip(out, out2):
        assert torch.equal(a, b)
    assert ((flags.cpu().numpy().astype(np.uint32) >> 24) == 0).all()
    want = U.oracle_tune_mt(po.Oracle(), c3["flat"], SLOTS, 1, M, N, K)
    np.testing.assert_array_equal(mac, want["macro"])
    np.testing.assert_array_equal(mic, want["micro"])
    np.testing.assert_array_equal(U.bits(lat), U.bits(want["lat"]))
    ref, h = _ref_handle(c3, tmpdir_session)
    s = slice(0, 300)
    w2 = ref.tune(h, M[s], N[s], K[s], nthreads=max(1, min(32, len(os.sched_getaffinity(0)))))
    ref.close(h)
    np.testing.assert_array_equal(mac[s], w2["macro"])
    np.testing.assert_array_equal(mic[s], w2["micro"])
    np.testing.assert_array_equal(U.bits(lat[s]), U.bits(w2["lat"]))
