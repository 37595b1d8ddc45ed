"""Host wall time of each stage of the records-in-HBM -> grid chain
(config 3/4), synchronised after every stage, min over repetitions."""
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
st = {}
for rep in range(6):
    torch.cuda.synchronize()
    t = time.perf_counter()
    b = capi.Build(recd, cfg["id"], 40, 10)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    e = capi.Engine.from_build(b, reg, n_sm=148)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    g = capi.Grid(e, [p[0] for p in p3], [p[1] for p in p3], 1, 65536,
                  stream=torch.cuda.current_stream() if os.environ.get("GRID_ASYNC") else None)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    g.sweep()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    for k, v in (("fit", t1 - t), ("engine", t2 - t1), ("grid_create", t3 - t2), ("sweep", t4 - t3)):
        st.setdefault(k, []).append(v * 1e3)
    for x in (g, e, b):
        x.close()
print({k: round(min(v), 3) for k, v in st.items()})
