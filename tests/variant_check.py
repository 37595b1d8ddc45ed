"""Subprocess helper for test_gpu_decide.test_launch_variants: runs the list
and grid kernels under the launch shape selected by WT_* env vars and checks
them against the oracle.  Exit code 0 = bit-exact."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:0] = [os.path.dirname(HERE), os.path.join(os.path.dirname(HERE), "oracle"), HERE]

import numpy as np  # noqa: E402
import torch  # noqa: E402

import pyoracle as po  # noqa: E402
import wtutil as U  # noqa: E402
from paper_2604_10187_b200 import capi, synthetic as S  # noqa: E402

cfg = S.config_space(False)
t = S.synthetic_tables(cfg)
eng = capi.Engine(t, S.registry_arrays(cfg), n_sm=148)
pairs = S.LLAMA3_8B
grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 3000)
grid.sweep()
M, N, K = S.query_stream(40000, pairs, seed=8, off_grid_frac=0.3, m_max=3500)
n = len(M)
out = [torch.empty(n, dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
grid.gather(*(torch.from_numpy(x).cuda() for x in (M, N, K)), capi.Engine.decisions(*out))
torch.cuda.synchronize()
mac, mic, lat = (o.cpu().numpy() for o in out)
tiles = {int(i): (int(a), int(b), int(c)) for i, a, b, c in zip(cfg["id"], cfg["t_m"], cfg["t_n"], cfg["t_k"])}
want = po.Oracle().tune(po.FlatTables(U.pytables_from_arrays(t), tiles), 148, 1, M, N, K)
ok = (np.array_equal(mac, want["macro"]) and np.array_equal(mic, want["micro"])
      and np.array_equal(lat.view(np.int64), want["lat"].view(np.int64)))
print("variant", {k: v for k, v in os.environ.items() if k.startswith("WT_")}, "ok" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
