"""Launch the C2 lm_head GEMM (swap-AB, argmax epilogue) a few times, for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_04991_b200 import ops, _native as N
dev = torch.device("cuda:0")
B, H, V = int(os.environ.get("B", 32)), 768, 40000
w = (torch.randn(V, H, device=dev) * 0.02).half()
a = torch.randn(B, H, device=dev).half()
keys = torch.zeros(B, dtype=torch.int64, device=dev)
for _ in range(int(os.environ.get("REPS", 5))):
    ops.gemm(a, w, H, N.EPI_LOGITS, keys=keys)
torch.cuda.synchronize()
print("ok")
