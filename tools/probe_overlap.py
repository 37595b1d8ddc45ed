"""Config-2 step time under the gather / off-grid-evaluation overlap settings
(WT_GATHER_OVERLAP chunks, WT_OVERLAP_GATHER_CTAS per SM; read once per
process).  Prints ms/step and a digest of the decisions (must not change)."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_10187_b200 import capi, synthetic as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
cfg = S.config_space(False)
t = S.synthetic_tables(cfg)
eng = capi.Engine(t, S.registry_arrays(cfg), n_sm=148)
pairs = S.LLAMA3_8B
grid = capi.Grid(eng, [p[0] for p in pairs], [p[1] for p in pairs], 1, 8192)
grid.sweep()
Mh, Nh, Kh = S.query_stream(n, pairs, seed=21)
Md, Nd, Kd = (torch.from_numpy(x).cuda() for x in (Mh, Nh, Kh))
o = [torch.full((n,), -7, dtype=d, device="cuda") for d in (torch.int32, torch.int32, torch.float64)]
dec = capi.Engine.decisions(*o)
st = torch.cuda.current_stream()
step = lambda: grid.gather(Md, Nd, Kd, dec, stream=st)  # noqa: E731
for _ in range(3):
    step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = []
for _ in range(3):
    a.record(st)
    for _ in range(10):
        step()
    b.record(st)
    torch.cuda.synchronize()
    res.append(a.elapsed_time(b) / 10)
capi.set_kernel_timing(True)
step()
g_ms, e_ms = capi.kernel_time_ms(0), capi.kernel_time_ms(1)
capi.set_kernel_timing(False)
h = hashlib.sha1()
for x in o:
    h.update(x.cpu().numpy().tobytes())
print(json.dumps({"overlap": os.environ.get("WT_GATHER_OVERLAP", "default"),
                  "ctas": os.environ.get("WT_OVERLAP_GATHER_CTAS", "default"),
                  "ms": [round(r, 4) for r in res], "gather_span_ms": round(g_ms, 4),
                  "eval_tail_ms": round(e_ms, 4), "digest": h.hexdigest()[:16]}), flush=True)
