"""Minimal GPU smoke of the list evaluation (tune_batch on 1e2 / 5e3 / 1e5 off-grid
queries) -- run under `timeout` before larger suites after touching wt_eval3.cu."""
import sys, time
sys.path[:0]=['/root/repo','/root/repo/oracle','/root/repo/tests']
import numpy as np, torch
from paper_2604_10187_b200 import capi, synthetic as S
cfg=S.config_space(False); t=S.synthetic_tables(cfg)
eng=capi.Engine(t,S.registry_arrays(cfg),n_sm=148)
for n in (100, 5000, 100000):
    M,N,K=S.query_stream(n,S.LLAMA3_8B,seed=1,off_grid_frac=1.0)
    o=[torch.empty(n,dtype=d,device='cuda') for d in (torch.int32,torch.int32,torch.float64)]
    t0=time.time()
    eng.tune_batch(*(torch.from_numpy(x).cuda() for x in (M,N,K)), capi.Engine.decisions(*o))
    torch.cuda.synchronize()
    print(n, "ok", time.time()-t0, flush=True)
