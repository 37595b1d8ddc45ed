"""How the config-2 step depends on the tables' structure: the synthetic
tables' per-(config, wave) rows scaled by i.i.d. factors 1 + s*U[-1, 1]
(s = 0 / 0.05 / 0.2 / 0.5) break the near-monotone dominance of the
synthetic ground truth.  Per level: pruning survival (physical / logical
(query, config) evaluations of the off-grid list), step and off-grid times,
and a 20k-query parity check against the restatement.  Diagnostic."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_10187_b200 import capi, synthetic as S  # noqa: E402
import pyoracle as po  # noqa: E402
import wtutil as U  # noqa: E402

n = 100_000_000
cfg = S.config_space(False)
pairs = S.LLAMA3_8B
Mh, Nh, Kh = S.query_stream(n, pairs, seed=21)
Md, Nd, Kd = (torch.from_numpy(x).cuda() for x in (Mh, Nh, Kh))
out = [torch.empty(n, dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
dec = capi.Engine.decisions(*out)
P = np.array(pairs)
off = ~((Nh[:, None] == P[None, :, 0]) & (Kh[:, None] == P[None, :, 1])).any(1)
n_off = int(off.sum())
tiles = {int(i): (int(a), int(b), int(c)) for i, a, b, c in zip(cfg["id"], cfg["t_m"], cfg["t_n"], cfg["t_k"])}
st = torch.cuda.current_stream()
for s in (0.0, 0.05, 0.2, 0.5):
    t = S.synthetic_tables(cfg)
    th = t["coeff_theta"].reshape(-1, 4)
    f = 1.0 + s * (2.0 * np.random.default_rng(3).random(th.shape[0]) - 1.0)
    t["coeff_theta"] = (th * f[:, None]).reshape(-1)
    eng = capi.Engine(t, S.registry_arrays(cfg), n_sm=148)
    grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 8192)
    grid.sweep()
    step = lambda: grid.gather(Md, Nd, Kd, dec, stream=st)  # noqa: E731
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(10):
        step()
    b.record(st)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    capi.set_kernel_timing(True)
    step()
    g_ms, e_ms = capi.kernel_time_ms(0), capi.kernel_time_ms(1)
    capi.set_kernel_timing(False)
    ctr = torch.zeros(1, dtype=torch.int64, device="cuda")
    eng.count_evals(ctr)
    step()
    torch.cuda.synchronize()
    eng.count_evals(None)
    phys = int(ctr.item())
    # parity on a sample (on- and off-grid queries) against the restatement
    idx = np.concatenate([np.flatnonzero(off)[:10000], np.flatnonzero(~off)[:10000]])
    want = po.Oracle().tune(po.FlatTables(U.pytables_from_arrays(t), tiles), 148, 1, Mh[idx], Nh[idx], Kh[idx])
    ii = torch.from_numpy(idx).cuda()
    ok = (np.array_equal(out[0][ii].cpu().numpy(), want["macro"]) and np.array_equal(out[1][ii].cpu().numpy(), want["micro"])
          and np.array_equal(out[2][ii].cpu().numpy().view(np.int64), want["lat"].view(np.int64)))
    print(json.dumps({"row_scale_noise": s, "ms_per_step": round(ms, 4), "gather_ms": round(g_ms, 4),
                      "offgrid_ms": round(e_ms, 4), "offgrid_queries": n_off,
                      "survival": round(phys / (n_off * eng.n_configs), 4), "parity_20k": ok}), flush=True)
    grid.close()
    eng.close()
