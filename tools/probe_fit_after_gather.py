"""Fit device time standalone vs after large gather batches (pool interaction)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_10187_b200 import capi, synthetic as S  # noqa: E402

cfg3 = S.config_space(full=True)
rec4 = S.synthetic_records(cfg3, micros_per_macro=1)
for i in range(2):
    print("fit standalone", capi.fit_build(rec4, cfg3["id"], 40, 10)["device_ms"], flush=True)
cfg = S.config_space(False)
eng = capi.Engine(S.synthetic_tables(cfg), S.registry_arrays(cfg), n_sm=148)
pairs = S.LLAMA3_8B
grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 8192)
grid.sweep()
n = 100_000_000
M, N, K = (torch.from_numpy(x).cuda() for x in S.query_stream(n, pairs, seed=21))
o = [torch.empty(n, dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
for _ in range(3):
    grid.gather(M, N, K, capi.Engine.decisions(*o))
torch.cuda.synchronize()
for i in range(3):
    print("fit after gather", capi.fit_build(rec4, cfg3["id"], 40, 10)["device_ms"], flush=True)
