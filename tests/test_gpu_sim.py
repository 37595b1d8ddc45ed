"""GPU wave simulator (synthetic-profile generator) against
the reference's simulate() / SimulatorBackend compiled verbatim.

sigma = 0: makespans and profile records bit-identical (pure binary64 adds).
sigma > 0: Box-Muller goes through libm log/cos, whose last-ulp rounding
differs between glibc and CUDA, so the bar is 1e-12 relative."""
import json

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


def test_step_law_bitexact(capi):
    # acceptance A1 / test_wave_sim.cpp:13-42: zero variance -> 50 * ceil(g / 132)
    g = np.arange(1, 661)
    out = capi.simulate_batch(g, 50.0, 0.0, 0.5, 0.0, 0, 132)
    want = 50.0 * np.ceil(g / 132)
    np.testing.assert_array_equal(out, want)
    out4 = capi.simulate_batch([10], 50.0, 0.0, 0.5, 0.0, 42, 4)
    assert out4[0] == 150.0


def test_simulate_matches_reference(capi, ref):
    rng = np.random.default_rng(3)
    n = 400
    g = rng.integers(1, 3000, n)
    sig = rng.choice([0.0, 5.0, 20.0, 50.0], n)
    seed = rng.integers(0, 2**62, n).astype(np.uint64)
    mu = 50.0
    got = capi.simulate_batch(g, mu, sig, 0.01 * mu, 0.0, seed, 132)
    want = np.array([po.ref_simulate(ref, 132, int(g[i]), 1, mu, float(sig[i]), int(seed[i])) for i in range(n)])
    zero = sig == 0
    np.testing.assert_array_equal(got[zero], want[zero])
    rel = np.abs(got - want) / want
    assert rel.max() <= 1e-12, rel.max()
    assert (got == want).mean() > 0.5  # most draws are bit-identical even with noise


@pytest.mark.parametrize("sigma", [0.0, 5.0])
def test_profile_matches_reference_simulator_backend(capi, ref, tmp_path, sigma):
    """run_profile with SimulatorBackend (the acceptance landscape, 6x8 configs,
    W=10, anchors 8..64, seed 7) on the GPU vs the reference's records."""
    n_sm, nm, nu, W = 132, 6, 8, 10
    anchors = [8, 16, 32, 48, 64]
    reg, rec, tab = U.reference_fixture(ref, tmp_path, n_sm=n_sm, n_macros=nm, n_micros=nu, W=W, sigma=sigma,
                                        seed=7)
    gp = str(tmp_path / "ground.json")
    po.ref_ground(ref, nm, nu, gp)
    plan = str(tmp_path / "plan.json")
    ref.build_plan(n_sm, 1, W, 4, 1.5, anchors, plan)
    pts = [p["g"] for p in json.load(open(plan))["grid_points"]]
    ground = {(e["macro_id"], e["micro_id"]): e for e in json.load(open(gp))["entries"]}
    pairs = sorted(ground)  # feasible pairs in (macro, micro) order == run_profile order
    lat, st, ms = capi.profile_sim(pts, anchors, [p[0] for p in pairs], [p[1] for p in pairs],
                                   [ground[p]["base"] for p in pairs], [ground[p]["per_iter"] for p in pairs],
                                   [ground[p]["dispatch_gap"] for p in pairs], sigma, 7, n_sm)
    assert (st == 0).all()
    want = po.read_records_csv(rec)
    assert len(want["lat"]) == len(lat)
    g_rec = np.repeat(pts, len(anchors) * len(pairs))
    np.testing.assert_array_equal(want["g"], g_rec)
    if sigma == 0.0:
        np.testing.assert_array_equal(U.bits(lat), U.bits(want["lat"]))
    else:
        rel = np.abs(lat - want["lat"]) / want["lat"]
        assert rel.max() <= 1e-12, rel.max()
