"""Drives one kernel family for an ncu capture (diagnostic; not a bench line).
usage: python tools/prof_kernels.py {sweep3|eval|gather|step|fit|build} [n]
(build = the bench's records-in-HBM -> grid chain at config 3/4, 3 times)
(step = the bench step: gather of the config-2 stream with 1% off-grid)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_10187_b200 import capi, synthetic as S  # noqa: E402

mode = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
if mode == "fit":
    cfg = S.config_space(True)
    rec = S.synthetic_records(cfg, micros_per_macro=1)
    for _ in range(2):
        r = capi.fit_build(rec, cfg["id"], 40, 10)
    print("fit device ms", r["device_ms"])
elif mode == "build":
    cfg = S.config_space(True)
    rec = S.synthetic_records(cfg, micros_per_macro=1)
    cv = {"g": torch.int64, "l": torch.int64, "w": torch.int32, "macro": torch.int32, "micro": torch.int32,
          "lat": torch.float64}
    recd = {k: torch.as_tensor(np.ascontiguousarray(rec[k])).to(dtype=cv[k], device="cuda") for k in cv}
    reg = S.registry_arrays(cfg)
    p3 = S.unique_pairs(S.LLAMA3_70B, S.QWEN2_72B)
    for _ in range(3):
        b = capi.Build(recd, cfg["id"], 40, 10)
        e = capi.Engine.from_build(b, reg, n_sm=148)
        g = capi.Grid(e, [p[0] for p in p3], [p[1] for p in p3], 1, 65536)
        g.sweep()
        torch.cuda.synchronize()
        for x in (g, e, b):
            x.close()
elif mode == "sweep3":
    cfg = S.config_space(True)
    eng = capi.Engine(S.synthetic_tables(cfg), S.registry_arrays(cfg), n_sm=148)
    p3 = S.unique_pairs(S.LLAMA3_70B, S.QWEN2_72B)
    g = capi.Grid(eng, [p[0] for p in p3], [p[1] for p in p3], 1, 65536)
    for _ in range(3):
        g.sweep()
    torch.cuda.synchronize()
else:
    cfg = S.config_space(False)
    eng = capi.Engine(S.synthetic_tables(cfg), S.registry_arrays(cfg), n_sm=148)
    pairs = S.LLAMA3_8B
    grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 8192)
    grid.sweep()
    frac = {"eval": 1.0, "step": 0.01}.get(mode, 0.0)
    M, N, K = (torch.from_numpy(x).cuda() for x in S.query_stream(n, pairs, seed=3, off_grid_frac=frac))
    o = [torch.empty(n, dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
    d = capi.Engine.decisions(*o)
    for _ in range(3):
        if mode == "eval":
            eng.tune_batch(M, N, K, d)
        else:
            grid.gather(M, N, K, d)
    torch.cuda.synchronize()
print("done", mode, n)
