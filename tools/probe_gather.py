"""Timing probe for the config-2 step components (diagnostic, not a bench line)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_10187_b200 import capi, synthetic as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
cfg = S.config_space(False)
t = S.synthetic_tables(cfg)
eng = capi.Engine(t, S.registry_arrays(cfg), n_sm=148)
pairs = S.LLAMA3_8B
grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 8192)
grid.sweep()
Mh, Nh, Kh = S.query_stream(n, pairs, seed=21)
P = np.array(pairs)
on = ((Nh[:, None] == P[None, :, 0]) & (Kh[:, None] == P[None, :, 1])).any(1)


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def mk(M, N, K):
    Md, Nd, Kd = (torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (M, N, K))
    m = len(M)
    o = [torch.empty(m, dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
    return Md, Nd, Kd, capi.Engine.decisions(*o), o


full = mk(Mh, Nh, Kh)
ong = mk(Mh[on], Nh[on], Kh[on])
off = mk(Mh[~on], Nh[~on], Kh[~on])
print("n", n, "on", int(on.sum()), "off", int((~on).sum()))
print("gather full  ms", timeit(lambda: grid.gather(*full[:4])))
print("gather on    ms", timeit(lambda: grid.gather(*ong[:4])))
print("gather off   ms", timeit(lambda: grid.gather(*off[:4])))
print("tune   off   ms", timeit(lambda: eng.tune_batch(*off[:4])))
m1 = min(1000000, int(on.sum()))
print("tune   on1M  ms", timeit(lambda: eng.tune_batch(ong[0][:m1], ong[1][:m1], ong[2][:m1], ong[3])))
