"""GPU parity for 64-bit query dims (wt_tune_batch_i64 / wt_gather_batch_i64)
against the reference's own tune() -- whose DenseGemm carries i64 m, n, k
(kernel_map.hpp:25-27) -- and concurrent C-ABI calls from several host
threads (the reentrancy promised in wavetune_c.h)."""
import threading

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
def landscape(ref, tmpdir_session):
    reg, rec, tab = U.reference_fixture(ref, tmpdir_session)
    fam, tabs = po.parse_tables_json(tab)
    tiles, order = po.parse_registry_json(reg)
    return dict(reg=reg, tab=tab, tabs=tabs, tiles=tiles, arrays=U.arrays_from_pytables(tabs),
                registry=U.registry_from_json(reg))


def outputs(capi, n):
    o = dict(macro=torch.empty(n, dtype=torch.int32, device="cuda"),
             micro=torch.empty(n, dtype=torch.int32, device="cuda"),
             lat=torch.empty(n, dtype=torch.float64, device="cuda"),
             g=torch.empty(n, dtype=torch.int64, device="cuda"),
             l=torch.empty(n, dtype=torch.int64, device="cuda"),
             wave=torch.empty(n, dtype=torch.int32, device="cuda"),
             flags=torch.empty(n, dtype=torch.int32, device="cuda"),
             comps=torch.empty(n, dtype=torch.int32, device="cuda"))
    d = capi.Engine.decisions(o["macro"], o["micro"], o["lat"], o["g"], o["l"], o["wave"], o["flags"], o["comps"])
    return o, d


def wide_queries(rng, n, tiles, n_sm):
    """Mix of int32 queries and queries with one or more dims >= 2^31, kept
    where the reference's int wave count stays exact (< 2^31 waves for the
    smallest tile); a few beyond that, which must come back UNSUPPORTED."""
    tm = min(t[0] for t in tiles.values())
    tn = min(t[1] for t in tiles.values())
    M = rng.integers(1, 9000, n).astype(np.int64)
    N = rng.integers(1, 9000, n).astype(np.int64)
    K = rng.integers(1, 9000, n).astype(np.int64)
    kind = rng.integers(0, 5, n)
    big = lambda k: rng.integers(2 ** 31, 2 ** 31 + 2 ** 36, k)
    M[kind == 1] = big((kind == 1).sum())
    K[kind == 2] = big((kind == 2).sum())
    N[kind == 3] = big((kind == 3).sum())
    sel = kind == 4
    M[sel], N[sel] = big(sel.sum()), big(sel.sum())  # far beyond 2^31 waves
    # exact boundaries: 2^31 - 1 (int32 path) and 2^31 (wide path)
    M = np.concatenate([M, [2 ** 31 - 1, 2 ** 31, 2 ** 31 + 1, 64]])
    N = np.concatenate([N, [64, 64, 128, 2 ** 31]])
    K = np.concatenate([K, [2 ** 31, 2 ** 31 - 1, 4096, 2 ** 33]])
    gmax = [(-(-int(m) // tm)) * (-(-int(x) // tn)) for m, x in zip(M, N)]
    unsupported = np.array([(-(-g // n_sm)) >= 2 ** 31 for g in gmax])
    return M, N, K, unsupported


def check_vs_reference(got, want, unsupported):
    st = (got["flags"].astype(np.uint32) >> 24).astype(np.int32)
    assert (st[unsupported] == 5).all(), "WT_UNSUPPORTED expected beyond 2^31 waves"  # WT_UNSUPPORTED
    ok = ~unsupported
    assert (want["status"][ok] == 0).all()
    np.testing.assert_array_equal(st[ok], 0)
    for k_g, k_w in (("macro", "macro"), ("micro", "micro"), ("g", "g"), ("l", "l"), ("wave", "w"),
                     ("comps", "comps")):
        np.testing.assert_array_equal(got[k_g][ok], want[k_w][ok], err_msg=k_g)
    np.testing.assert_array_equal(U.bits(got["lat"][ok]), U.bits(want["lat"][ok]))


def test_tune_batch_i64_matches_reference(capi, ref, landscape):
    L = landscape
    eng = capi.Engine(L["arrays"], L["registry"], n_sm=132)
    rng = np.random.default_rng(71)
    M, N, K, unsup = wide_queries(rng, 20000, L["tiles"], 132)
    assert (M >= 2 ** 31).sum() > 1000 and (K >= 2 ** 31).sum() > 1000 and unsup.sum() > 100
    o, d = outputs(capi, len(M))
    dv = lambda a: torch.as_tensor(a, dtype=torch.int64, device="cuda")
    eng.tune_batch_i64(dv(M), dv(N), dv(K), d)
    torch.cuda.synchronize()
    got = {k: v.cpu().numpy() for k, v in o.items()}
    h = ref.open(L["tab"], L["reg"], 132)
    ok = ~unsup
    want = {k: np.zeros(len(M), v.dtype) for k, v in ref.tune(h, M[:1], N[:1], K[:1]).items()}
    part = ref.tune(h, M[ok], N[ok], K[ok], nthreads=8)
    for k in want:
        want[k][ok] = part[k]
    ref.close(h)
    check_vs_reference(got, want, unsup)
    # the int32 entry point on the narrow subset gives the same answers
    narrow = ok & (M < 2 ** 31) & (N < 2 ** 31) & (K < 2 ** 31)
    o2, d2 = outputs(capi, int(narrow.sum()))
    d32 = lambda a: torch.as_tensor(a[narrow].astype(np.int32), device="cuda")
    eng.tune_batch(d32(M), d32(N), d32(K), d2)
    torch.cuda.synchronize()
    for k in ("macro", "micro", "g", "l", "wave", "flags"):
        np.testing.assert_array_equal(o2[k].cpu().numpy(), got[k][narrow], err_msg=k)
    np.testing.assert_array_equal(U.bits(o2["lat"].cpu().numpy()), U.bits(got["lat"][narrow]))


def test_gather_batch_i64_matches_reference(capi, ref, landscape):
    L = landscape
    eng = capi.Engine(L["arrays"], L["registry"], n_sm=132)
    pairs = [(4096, 4096), (6144, 4096)]
    grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 4096)
    grid.sweep()
    rng = np.random.default_rng(72)
    M, N, K, unsup = wide_queries(rng, 12000, L["tiles"], 132)
    on = rng.random(len(M)) < 0.5  # half on the grid (int32 dims)
    P = np.array(pairs)[rng.integers(0, 2, len(M))]
    M[on], N[on], K[on] = rng.integers(1, 4097, on.sum()), P[on, 0], P[on, 1]
    unsup[on] = False
    o, d = outputs(capi, len(M))
    dv = lambda a: torch.as_tensor(a, dtype=torch.int64, device="cuda")
    grid.gather_i64(dv(M), dv(N), dv(K), d)
    torch.cuda.synchronize()
    got = {k: v.cpu().numpy() for k, v in o.items()}
    h = ref.open(L["tab"], L["reg"], 132)
    ok = ~unsup
    want = {k: np.zeros(len(M), v.dtype) for k, v in ref.tune(h, M[:1], N[:1], K[:1]).items()}
    part = ref.tune(h, M[ok], N[ok], K[ok], nthreads=8)
    for k in want:
        want[k][ok] = part[k]
    ref.close(h)
    check_vs_reference(got, want, unsup)


def test_concurrent_host_threads(capi, landscape):
    """Eight host threads issue batched tune / gather calls on their own
    streams at once (ctypes releases the GIL): every thread's answers equal
    the single-threaded ones."""
    L = landscape
    eng = capi.Engine(L["arrays"], L["registry"], n_sm=132)
    grid = capi.Grid(eng, [4096], [4096], 1, 4096)
    grid.sweep()
    torch.cuda.synchronize()
    rng = np.random.default_rng(73)
    n = 30000
    M = rng.integers(1, 5000, n).astype(np.int32)
    N = np.where(rng.random(n) < 0.5, 4096, rng.integers(1, 9000, n)).astype(np.int32)
    K = np.where(N == 4096, 4096, rng.integers(1, 9000, n)).astype(np.int32)
    Md, Nd, Kd = (torch.as_tensor(x, device="cuda") for x in (M, N, K))

    def run(kind, stream):
        o, d = outputs(capi, n)
        with torch.cuda.stream(stream):
            for _ in range(5):
                if kind == 0:
                    eng.tune_batch(Md, Nd, Kd, d, stream=stream)
                else:
                    grid.gather(Md, Nd, Kd, d, stream=stream)
        stream.synchronize()
        return {k: v.cpu().numpy() for k, v in o.items()}

    base = [run(k, torch.cuda.Stream()) for k in (0, 1)]
    results, errors = {}, []

    def worker(i):
        try:
            results[i] = run(i % 2, torch.cuda.Stream())
        except Exception as ex:  # pragma: no cover - reported below
            errors.append(repr(ex))

    th = [threading.Thread(target=worker, args=(i,)) for i in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for i in range(8):
        for k in ("macro", "micro", "flags"):
            np.testing.assert_array_equal(results[i][k], base[i % 2][k], err_msg=f"thread {i} {k}")
        np.testing.assert_array_equal(U.bits(results[i]["lat"]), U.bits(base[i % 2]["lat"]))
