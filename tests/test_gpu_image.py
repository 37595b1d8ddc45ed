"""The device image builder (wt_image_dev.cu) against the host-only plan
(wt_prune_plan, the same wt_rows.h functions on the CPU): pruning masks bit
for bit on the config-1 tables, the adversarial near-tie tables, tables with
missing waves / empty maps, and the GPU-fitted config-3 tables; plus the
engine-creation time from host tables (all image work on the device)."""
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


def masks_equal(capi, tables, reg):
    plan = capi.prune_plan(tables, reg, 148)
    eng = capi.Engine(tables, reg, n_sm=148)
    dev = eng.prune_masks(len(plan["seg_pos"]))
    eng.close()
    np.testing.assert_array_equal(dev, plan["masks"])
    return plan


def test_device_masks_match_host_plan_config1(capi):
    from paper_2604_10187_b200 import synthetic as S

    cfg = S.config_space(full=False)
    plan = masks_equal(capi, S.synthetic_tables(cfg), S.registry_arrays(cfg))
    kept = np.unpackbits(plan["masks"].view(np.uint8)).sum()
    assert 0 < kept < plan["masks"].size * 32


def test_device_masks_match_host_plan_adversarial(capi):
    cfg, t = U.adversarial_tables()
    masks_equal(capi, t, U.registry_arrays_of(cfg))


def test_device_masks_match_host_plan_holes(capi):
    """Missing coefficient waves, empty anchor maps, one empty table: the
    fallback rows (and the unprunable empty table) resolve identically."""
    from paper_2604_10187_b200 import synthetic as S

    cfg = S.config_space(full=False)
    t = S.synthetic_tables(cfg)
    tabs = U.pytables_from_arrays(t)
    rng = np.random.default_rng(2)
    for tb in tabs[::7]:
        for w in rng.choice(list(tb.coeffs), 5, replace=False):
            del tb.coeffs[int(w)]
    for tb in tabs[3::11]:
        for w in rng.choice(list(tb.anchors), 6, replace=False):
            tb.anchors[int(w)] = {}
    tabs[5].coeffs = {}
    masks_equal(capi, U.arrays_from_pytables(tabs), S.registry_arrays(cfg))


def test_device_masks_match_host_plan_config3(capi):
    from paper_2604_10187_b200 import synthetic as S

    cfg = S.config_space(full=True)
    fit = capi.fit_build(S.synthetic_records(cfg), cfg["id"], 40, 10)
    t3 = {k: fit[k] for k in ("macro_id", "theta_ext", "coeff_off", "coeff_w", "coeff_theta", "awave_off",
                               "awave_w", "awave_aoff", "anchor_l", "anchor_micro", "ext_aoff", "ext_l",
                               "ext_micro")}
    t3["W"] = fit["W_arr"]
    reg = S.registry_arrays(cfg)
    masks_equal(capi, t3, reg)
    capi.Engine(t3, reg, n_sm=148).close()  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng = capi.Engine(t3, reg, n_sm=148)
    ms = (time.perf_counter() - t0) * 1e3
    eng.close()
    print(f"config-3 engine creation from host tables: {ms:.2f} ms")
    assert ms < 200
