"""CUDA-event timings of the main paths under the current WT_* launch knobs
(diagnostic for A/B runs; not a bench line)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_10187_b200 import capi, synthetic as S  # noqa: E402


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


res = {"env": {k: v for k, v in os.environ.items() if k.startswith("WT_")}}
cfg3 = S.config_space(True)
e3 = capi.Engine(S.synthetic_tables(cfg3), S.registry_arrays(cfg3), n_sm=148)
p3 = S.unique_pairs(S.LLAMA3_70B, S.QWEN2_72B)
g3 = capi.Grid(e3, [p[0] for p in p3], [p[1] for p in p3], 1, 65536)
res["sweep3_ms"] = timeit(lambda: g3.sweep(), 3)
cfg = S.config_space(False)
eng = capi.Engine(S.synthetic_tables(cfg), S.registry_arrays(cfg), n_sm=148)
pairs = S.LLAMA3_8B
grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 8192)
res["sweep1_ms"] = timeit(lambda: grid.sweep())
for name, n, frac in (("eval_1M_ms", 1_000_000, 1.0), ("gather_100M_ms", 100_000_000, 0.01),
                      ("gather_ongrid_100M_ms", 100_000_000, 0.0)):
    M, N, K = (torch.from_numpy(x).cuda() for x in S.query_stream(n, pairs, seed=21, off_grid_frac=frac))
    o = [torch.empty(n, dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
    d = capi.Engine.decisions(*o)
    if frac == 1.0:
        res[name] = timeit(lambda: eng.tune_batch(M, N, K, d))
    else:
        res[name] = timeit(lambda: grid.gather(M, N, K, d))
    del M, N, K, o
print(json.dumps(res))
