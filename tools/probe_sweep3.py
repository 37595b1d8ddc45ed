"""Config-3 sweep device time (393,216 shapes x 4,608 configs), for launch-shape A/B via WT_SWEEP_* env."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_10187_b200 import capi, synthetic as S  # noqa: E402

cfg = S.config_space(True)
eng = capi.Engine(S.synthetic_tables(cfg), S.registry_arrays(cfg), n_sm=148)
p3 = S.unique_pairs(S.LLAMA3_70B, S.QWEN2_72B)
g = capi.Grid(eng, [p[0] for p in p3], [p[1] for p in p3], 1, 65536)
for _ in range(2):
    g.sweep()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    g.sweep()
e1.record()
torch.cuda.synchronize()
print({k: v for k, v in os.environ.items() if k.startswith("WT_SWEEP")}, "ms", e0.elapsed_time(e1) / 5)
