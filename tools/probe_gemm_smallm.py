import sys, os, torch
sys.path.insert(0, '/root/repo')
from paper_2604_10187_b200 import gemm
fam = gemm.family()
for (M,N,K) in [(128,4096,4096),(128,6144,4096),(128,4096,14336),(128,28672,4096),(512,4096,4096),(512,6144,4096)]:
    a = torch.randn(M, K, device="cuda").bfloat16(); b = torch.randn(N, K, device="cuda").bfloat16()
    ref = a.float() @ b.float().T
    res=[]
    worst=0
    for c in range(len(fam)):
        out = gemm.matmul(a, b, c, 2)
        err = ((out.float()-ref).abs() - ref.abs()*2**-7).max().item()
        worst=max(worst,err)
        us = min(gemm.time_us(a, b, c, 2, warmup=3, reps=20) for _ in range(3))
        res.append((c, fam[c], round(us,1)))
    print(M,N,K, sorted(res, key=lambda r: r[2])[:4], 'worst excess err', round(worst,3), flush=True)
