"""The validation GEMM family (lib/libwtgemm.so) on the
GPU: every instantiation x swizzle against a torch fp32 reference of the same
product, ragged shapes, the measurement entry points, and the
profile -> fit -> tune loop through the reference's MeasurementBackend
interface (B200GemmBackend)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def gm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_10187_b200 import gemm

    gemm.lib()
    return gemm


@pytest.fixture(scope="module")
def wt():
    from paper_2604_10187_b200 import _core

    return _core


def _check(out, a, b):
    """bf16 output of an fp32-accumulated product: within two bf16 ulps of
    the fp32 reference plus a K-scaled absolute term for summation order."""
    ref = a.float() @ b.float().T
    err = (out.float() - ref).abs()
    tol = ref.abs() * (2.0 ** -7) + 1e-3 * math.sqrt(a.shape[1])
    bad = (err > tol).sum().item()
    assert bad == 0, f"{bad} elements out of tolerance; max err {err.max().item():.4g}"


# (24, 1024, 2048) and (40, 2056, 1024): decode-sized M -> the swap-AB tiles
# split K (fp32 partials reduced in slice order by the last slice)
@pytest.mark.parametrize("shape", [(512, 1024, 512), (333, 264, 200), (1, 8, 64), (1000, 4104, 1096),
                                   (24, 1024, 2048), (40, 2056, 1024)])
def test_family_numerics(gm, shape):
    M, N, K = shape
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    for cfg in range(len(gm.family())):
        for swz in gm.SWIZZLES:
            out = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
            gm.matmul(a, b, cfg, swz, out=out)
            torch.cuda.synchronize()
            _check(out, a, b)


@pytest.mark.parametrize("M", [768, 24])
def test_family_bitwise_deterministic(gm, M):
    """Same instantiation, same operands -> the same bits; swizzle only
    reorders tiles, so it cannot change any output element either (M = 24:
    split-K, whose slices are summed in slice order whichever finishes last)."""
    a = torch.randn(M, 1024, device="cuda").bfloat16()
    b = torch.randn(1536, 1024, device="cuda").bfloat16()
    for cfg in range(len(gm.family())):
        base = gm.matmul(a, b, cfg, 1)
        for swz in gm.SWIZZLES[1:]:
            assert torch.equal(gm.matmul(a, b, cfg, swz), base)
        assert torch.equal(gm.matmul(a, b, cfg, 1), base)


def test_measurement_entry_points(gm):
    fam = gm.family()
    a = torch.randn(1024, 2048, device="cuda").bfloat16()
    b = torch.randn(2048, 2048, device="cuda").bfloat16()
    t = gm.time_us(a, b, 1, 1, warmup=2, reps=5)
    flops = 2 * 1024 * 2048 * 2048
    assert 0 < t and flops / (t * 1e-6) < 2.5e15  # below the dense bf16 peak
    n = len(fam)
    cfg = np.arange(n)
    lat = gm.measure_batch(cfg, np.full(n, 2), np.full(n, 2048), np.full(n, 4096), np.full(n, 1024), 2, 5, 7)
    assert (lat > 0).all()
    # K not a multiple of 8 breaks TMA's 16-byte stride rule: reported as -1
    lat = gm.measure_batch([0, 1], [1, 1], [256, 256], [256, 256], [100, 1024], 1, 2, 7)
    assert lat[0] == -1 and lat[1] > 0
    with pytest.raises(gm.WtError):
        gm.matmul(torch.zeros(8, 100, device="cuda").bfloat16(), torch.zeros(8, 100, device="cuda").bfloat16(), 0)


def test_backend_profile_fit_tune(wt):
    """run_profile(plan, gemm_registry(), B200GemmBackend) -> build_tables ->
    tune(): the reference's whole pipeline on real tcgen05 kernels."""
    hw = wt.HardwareSpec(torch.cuda.get_device_properties(0).multi_processor_count, 1, "b200")
    reg = wt.gemm_registry()
    backend = wt.B200GemmBackend(warmup=1, measured=3, seed=5)
    plan = wt.build_plan(hw, "dense_gemm", W=3, I=2, tau=1.5, loop_anchors=[8, 32])
    records = backend.profile(plan, reg)
    assert len(records) == len(plan.grid_points) * 2 * len(reg.feasible)
    assert all(r.latency_us > 0 for r in records)
    # more K-loop iterations cost more (same grid point, same config)
    by = {(r.g, r.l, r.macro_id, r.micro_id): r.latency_us for r in records}
    longer = [by[(g, 32, a, b)] > by[(g, 8, a, b)] for (g, l, a, b) in by if l == 8]
    assert np.mean(longer) > 0.9
    art = wt.build_tables(records, reg, hw, W=3)
    assert len(art.tables) == len(reg.macros)
    d = wt.tune(wt.DenseGemm(2048, 4096, 2048), art, reg, hw)
    assert (d.macro_id, d.micro_id) in set(reg.feasible)
    assert d.predicted_latency_us > 0
    direct = backend.measure(wt.DenseGemm(2048, 4096, 2048), reg.macro(d.macro_id), reg.micro(d.micro_id))
    assert direct > 0
