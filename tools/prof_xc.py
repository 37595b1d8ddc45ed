"""Launch one CUTLASS cross-check config (tools/bin/libwtgemm_cutlass.so) a few
times (ncu target).  usage: python tools/prof_xc.py CFG M N K [SWIZZLE]"""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
L = C.CDLL(os.path.join(ROOT, "tools", "bin", "libwtgemm_cutlass.so"))
cfg, M, N, K = (int(x) for x in sys.argv[1:5])
swz = int(sys.argv[5]) if len(sys.argv) > 5 else 1
a = torch.randn(M, K, device="cuda").bfloat16()
b = torch.randn(N, K, device="cuda").bfloat16()
c = torch.empty(M, N, device="cuda").bfloat16()
for _ in range(3):
    rc = L.wt_gemm_run(cfg, swz, M, N, K, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                       C.c_void_p(c.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0, rc
torch.cuda.synchronize()
ref = a.float() @ b.float().T
print("maxerr", (c.float() - ref).abs().max().item())
us = C.c_double()
L.wt_gemm_time.argtypes = [C.c_int] * 5 + [C.c_void_p] * 3 + [C.c_int, C.c_int, C.POINTER(C.c_double)]
L.wt_gemm_time(cfg, swz, M, N, K, a.data_ptr(), b.data_ptr(), c.data_ptr(), 2, 10, C.byref(us))
print("us", us.value)
