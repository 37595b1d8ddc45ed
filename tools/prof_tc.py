"""Launch one tcgen05 family config on one shape a few times (ncu target).
usage: python tools/prof_tc.py CFG M N K [SWIZZLE] [REPS]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch  # noqa: E402

from paper_2604_10187_b200 import gemm  # noqa: E402

cfg, M, N, K = (int(x) for x in sys.argv[1:5])
swz = int(sys.argv[5]) if len(sys.argv) > 5 else 1
reps = int(sys.argv[6]) if len(sys.argv) > 6 else 3
a = torch.randn(M, K, device="cuda").bfloat16()
b = torch.randn(N, K, device="cuda").bfloat16()
for _ in range(reps):
    c = gemm.matmul(a, b, cfg, swz)
torch.cuda.synchronize()
print("us", gemm.time_us(a, b, cfg, swz, warmup=2, reps=10))
