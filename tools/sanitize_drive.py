"""Small end-to-end drive of every decision kernel for compute-sanitizer
(memcheck / racecheck / synccheck): grid sweep + run index, hashed gather
with off-grid queries (keys, scan, scatter, k_eval4), tune_batch, the
single-query kernel, a small fit.  Sizes are tiny: the sanitizer is ~100x."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_10187_b200 import capi, synthetic as S  # noqa: E402

cfg = S.config_space(False)
t = S.synthetic_tables(cfg)
eng = capi.Engine(t, S.registry_arrays(cfg), n_sm=148)
pairs = S.LLAMA3_8B
grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 3, 700)
grid.sweep()
M, N, K = S.query_stream(6001, pairs, seed=5, off_grid_frac=0.2, m_max=800)
o = [torch.empty(len(M), dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
grid.gather(*(torch.from_numpy(x).cuda() for x in (M, N, K)), capi.Engine.decisions(*o))
o2 = [torch.empty(len(M), dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
eng.tune_batch(*(torch.from_numpy(x).cuda() for x in (M, N, K)), capi.Engine.decisions(*o2))
torch.cuda.synchronize()
assert torch.equal(o[0], o2[0]) and torch.equal(o[2].view(torch.int64), o2[2].view(torch.int64))
d = eng.tune_one(3000, 6144, 4096)
rec = S.synthetic_records(cfg)
keep = np.isin(rec["macro"], cfg["id"][:16])
small = {k: v[keep] for k, v in rec.items()}
fit = capi.fit_build(small, cfg["id"][:16], 40, 10)
print("sanitize drive ok", int(d.macro_id), fit["n_tables"])
