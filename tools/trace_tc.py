import os,sys
sys.path.insert(0,'.')
import torch
from paper_2604_10187_b200 import gemm
cfg,M,N,K=(int(x) for x in sys.argv[1:5])
a=torch.randn(M,K,device='cuda').bfloat16(); b=torch.randn(N,K,device='cuda').bfloat16()
gemm.matmul(a,b,cfg,2); torch.cuda.synchronize()
gemm.matmul(a,b,cfg,2); torch.cuda.synchronize()
