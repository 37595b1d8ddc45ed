"""Device vs host timeline of the unsynced records-in-HBM -> grid chain
(config 3/4): CUDA events between the API calls on the build stream and the
host clock when each call returned.  Diagnostic (where the device idles)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_10187_b200 import capi, synthetic as S  # noqa: E402

cfg = S.config_space(True)
rec = S.synthetic_records(cfg, micros_per_macro=1)
cv = {"g": torch.int64, "l": torch.int64, "w": torch.int32, "macro": torch.int32, "micro": torch.int32,
      "lat": torch.float64}
recd = {k: torch.as_tensor(np.ascontiguousarray(rec[k])).to(dtype=cv[k], device="cuda") for k in cv}
reg = S.registry_arrays(cfg)
p3 = S.unique_pairs(S.LLAMA3_70B, S.QWEN2_72B)
st = torch.cuda.current_stream()
for rep in range(5):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    torch.cuda.synchronize()
    h = [time.perf_counter()]
    ev[0].record(st)
    b = capi.Build(recd, cfg["id"], 40, 10, stream=st)
    ev[1].record(st)
    h.append(time.perf_counter())
    e = capi.Engine.from_build(b, reg, n_sm=148, stream=st)
    ev[2].record(st)
    h.append(time.perf_counter())
    g = capi.Grid(e, [p[0] for p in p3], [p[1] for p in p3], 1, 65536, stream=st)
    ev[3].record(st)
    h.append(time.perf_counter())
    g.sweep(stream=st)
    ev[4].record(st)
    h.append(time.perf_counter())
    torch.cuda.synchronize()
    h.append(time.perf_counter())
    dev = [ev[0].elapsed_time(x) for x in ev]
    host = [(x - h[0]) * 1e3 for x in h]
    print(f"rep {rep}: device marks (ms from start) fit {dev[1]:.3f} engine {dev[2]:.3f} grid {dev[3]:.3f} "
          f"sweep {dev[4]:.3f} | host returns fit {host[1]:.3f} engine {host[2]:.3f} grid {host[3]:.3f} "
          f"sweep {host[4]:.3f} synced {host[5]:.3f}", flush=True)
    for x in (g, e, b):
        x.close()
