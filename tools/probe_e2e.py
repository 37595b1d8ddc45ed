"""e2e (host buffers, H2D + decide + D2H) throughput vs pipeline chunk size."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_10187_b200 import capi, synthetic as S  # noqa: E402

cfg = S.config_space(False)
eng = capi.Engine(S.synthetic_tables(cfg), S.registry_arrays(cfg), n_sm=148)
pairs = S.LLAMA3_8B
grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 8192)
grid.sweep()
n = 100_000_000
Mh, Nh, Kh = S.query_stream(n, pairs, seed=21)
Mp, Np, Kp = (torch.from_numpy(x).pin_memory() for x in (Mh, Nh, Kh))
mac = torch.empty(n, dtype=torch.int32).pin_memory()
mic = torch.empty(n, dtype=torch.int32).pin_memory()
lat = torch.empty(n, dtype=torch.float64).pin_memory()
for sh in [int(x) for x in sys.argv[1:]] or [19, 20, 21, 22]:
    ch = 1 << sh
    grid.decide_host(Mp, Np, Kp, mac, mic, lat, chunk=ch)
    t0 = time.perf_counter()
    for _ in range(3):
        grid.decide_host(Mp, Np, Kp, mac, mic, lat, chunk=ch)
    dt = (time.perf_counter() - t0) / 3
    print(f"chunk 2^{sh}: {dt * 1e3:.2f} ms/step, {n / dt:.3e} q/s", flush=True)
