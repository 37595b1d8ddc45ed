"""The device-resident build path: records already in HBM -> K2 fit
(wt_fit_build_device, tables stay on the device) -> engine image built on
the device from them (wt_engine_create_from_build) -> decision grid.

Checked against the host-API path (wt_fit_build -> host CSR ->
wt_engine_create), itself pinned to the restatement / reference elsewhere:
tables bit-identical, grid entries bit-identical."""
import time

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


def same_tables(a, b):
    for k in ("macro_id", "coeff_off", "coeff_w", "awave_off", "awave_w", "awave_aoff", "anchor_l", "anchor_micro",
              "anchor_partial", "ext_aoff", "ext_l", "ext_micro", "ext_flags", "diag_samples", "diag_flags"):
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    for k in ("coeff_theta", "theta_ext", "diag_r2", "diag_mape"):
        np.testing.assert_array_equal(U.bits(a[k]), U.bits(b[k]), err_msg=k)
    assert a["W"] == b["W"] and a["n_tables"] == b["n_tables"]


def entries(grid):
    e = grid.entries_tensor().cpu().numpy().copy()
    grid.finalize()
    return e


@pytest.mark.parametrize("variant", ["config3", "holes"])
def test_device_build_matches_host_build(capi, variant):
    from paper_2604_10187_b200 import synthetic as S

    cfg = S.config_space(full=True)
    rec = S.synthetic_records(cfg, micros_per_macro=1 if variant == "config3" else 2)
    reg = S.registry_arrays(cfg)
    W = 40
    if variant == "holes":
        # macros without records (omitted tables), records of unknown macros
        # (ignored), a sparse wave, W from the data (W = 0)
        rng = np.random.default_rng(1)
        keep = ~np.isin(rec["macro"], rng.choice(len(cfg["id"]), 300, replace=False))
        keep &= ~((rec["w"] == 7) & (rng.random(len(keep)) < 0.7))
        rec = {k: v[keep] for k, v in rec.items()}
        rec["macro"] = rec["macro"].copy()
        rec["macro"][:50] = 99999
        W = 0
    host = capi.fit_build(rec, cfg["id"], W, 10)
    b = capi.Build(dev_records(rec), cfg["id"], W, 10)
    got = b.result()
    same_tables(got, host)
    # engine from the device tables == engine from the host tables
    e_dev = capi.Engine.from_build(b, reg, n_sm=148)
    e_host = capi.Engine(capi.engine_tables(host), reg, n_sm=148)
    assert e_dev.n_configs == e_host.n_configs == host["n_tables"]
    pairs = S.unique_pairs(S.LLAMA3_70B, S.QWEN2_72B)
    m_hi = 65536 if variant == "config3" else 8192
    gd = capi.Grid(e_dev, [p[0] for p in pairs], [p[1] for p in pairs], 1, m_hi)
    gh = capi.Grid(e_host, [p[0] for p in pairs], [p[1] for p in pairs], 1, m_hi)
    gd.sweep()
    gh.sweep()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(entries(gd), entries(gh))
    # off-grid list evaluation reads the anchor pool (ext slices uncompacted)
    M, N, K = S.query_stream(50000, pairs, seed=4, off_grid_frac=0.5, m_max=m_hi)
    outs = []
    for eng in (e_dev, e_host):
        o = [torch.empty(len(M), dtype=dt, device="cuda") for dt in (torch.int32, torch.int32, torch.float64)]
        eng.tune_batch(*(torch.as_tensor(x).cuda() for x in (M, N, K)), eng.decisions(*o))
        outs.append(o)
    torch.cuda.synchronize()
    for a, c in zip(*outs):
        assert torch.equal(a, c)
    for x in (gd, gh, e_dev, e_host, b):
        x.close()


def test_device_build_pipeline_time(capi):
    """Records in HBM -> grid resident (fit + engine + sweep + run index) on
    one stream: host wall clock of the whole chain, printed for the log."""
    from paper_2604_10187_b200 import synthetic as S

    cfg = S.config_space(full=True)
    reg = S.registry_arrays(cfg)
    recd = dev_records(S.synthetic_records(cfg))
    pairs = S.unique_pairs(S.LLAMA3_70B, S.QWEN2_72B)
    st = torch.cuda.current_stream()
    times = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        b = capi.Build(recd, cfg["id"], 40, 10, stream=st)
        e = capi.Engine.from_build(b, reg, n_sm=148, stream=st)
        g = capi.Grid(e, [p[0] for p in pairs], [p[1] for p in pairs], 1, 65536)
        g.sweep(stream=st)
        torch.cuda.synchronize()
        times.append((time.perf_counter() - t0) * 1e3)
        for x in (g, e, b):
            x.close()
    print(f"records->grid wall ms: {['%.2f' % t for t in times]}")
    assert min(times) < 1000
