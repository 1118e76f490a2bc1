"""One prefill-attention launch at the C2 shape (B=32, 12 heads, T=128, D=64) for ncu:
    ncu -k regex:attn_prefill python tools/pf_attn_once.py [T] [B]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2407_04991_b200 import ops  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 128
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
NH, D, cap = 12, 64, T + 64
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
q = (torch.randn(B * T, NH * D, device=dev, generator=g) * 0.5).half()
kc = (torch.randn(B, NH, cap, D, device=dev, generator=g) * 0.5).half()
vc = torch.randn(B, NH, cap, D, device=dev, generator=g).half()
start = torch.zeros(B, dtype=torch.int32, device=dev)
qb = torch.zeros(1, dtype=torch.int32, device=dev)
out = torch.empty(B * T, NH * D, dtype=torch.half, device=dev)
for _ in range(3):
    ops.attention(q, None, kc, vc, start, qb, 1.0 / math.sqrt(D), out, batch=B, heads=NH, head_dim=D, cap=cap,
                  seq_len=T)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    ops.attention(q, None, kc, vc, start, qb, 1.0 / math.sqrt(D), out, batch=B, heads=NH, head_dim=D, cap=cap,
                  seq_len=T)
e1.record()
e1.synchronize()
print(f"attention T={T} B={B}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per launch")
