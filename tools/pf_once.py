import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_04991_b200 import ops, _native as N
dev = torch.device("cuda:0")
M, n_out, k = 4096, 3072, 768
a = torch.randn(M, k, device=dev).half(); w = (torch.randn(n_out, k, device=dev) * 0.02).half()
out = torch.zeros(M, n_out, device=dev)
for _ in range(3):
    ops.gemm(a, w, k, N.EPI_F32, out=out, force_swap=0)
torch.cuda.synchronize(); print("ok")
