import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2604_10187_b200 import gemm
M, N, K = 128, 4096, 4096
cfg = int(sys.argv[1])
a = torch.randn(M, K, device="cuda").bfloat16(); b = torch.randn(N, K, device="cuda").bfloat16()
for _ in range(5): gemm.matmul(a, b, cfg, 2)
torch.cuda.synchronize()
