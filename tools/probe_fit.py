"""Config-4 fit timing (device_ms from the C-ABI + host wall), repeated."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_10187_b200 import capi, synthetic as S  # noqa: E402

cfg3 = S.config_space(full=True)
rec4 = S.synthetic_records(cfg3, micros_per_macro=1)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    t0 = time.perf_counter()
    fit = capi.fit_build(rec4, cfg3["id"], 40, 10, device=0)
    print(f"fit_build #{i}: device_ms {fit['device_ms']:.2f}, wall {1e3 * (time.perf_counter() - t0):.1f} ms",
          flush=True)
