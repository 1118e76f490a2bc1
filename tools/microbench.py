"""Per-operator timing of the C2 decode step shapes (CUDA events, warm clocks)."""
import os, sys, statistics, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_04991_b200 import ops, _native as N

dev = torch.device("cuda:0")
B, H, F, V, NH, D, cap, ctx = int(os.environ.get("B", 32)), 768, 3072, 40000, 12, 64, 192, 160
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
scr = ops.Scratch(dev, 64 << 20)

def t(fn, n=20, cold=True):
    ts = []
    for i in range(n + 3):
        if cold: flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1) * 1e3)
    return statistics.median(ts)

def loop(fn, n=50):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n

x = torch.randn(B, 832, device=dev).half(); x[:, H:] = 0
h = torch.zeros_like(x)
g = torch.ones(H, device=dev); bb = torch.zeros(H, device=dev)
f = torch.zeros(B, F, device=dev, dtype=torch.half)
res = {}
res["layernorm"] = (t(lambda: ops.layernorm(x, H, g, bb, h)), loop(lambda: ops.layernorm(x, H, g, bb, h)))
for name, n_out, k, epi in [("qkv", 3 * H, H, N.EPI_BIAS), ("wo", H, H, N.EPI_BIAS_RESID),
                            ("w1", F, H, N.EPI_BIAS_GELU), ("w2", H, F, N.EPI_BIAS_RESID),
                            ("lm_head", V, H, N.EPI_LOGITS)]:
    kp = ops.pad64(k)
    w = (torch.randn(n_out, kp, device=dev) * 0.02).half()
    a = torch.randn(B, kp, device=dev).half()
    out = torch.zeros(B, max(n_out, 64), device=dev, dtype=torch.half)
    bias = torch.zeros(n_out, device=dev)
    keys = torch.zeros(B, dtype=torch.int64, device=dev)
    for splits in ([0, 1] if name != "lm_head" else [0]):
        if epi == N.EPI_LOGITS:
            fn = lambda: ops.gemm(a, w, k, epi, keys=keys, scratch=scr, splits=splits)
        elif epi == N.EPI_BIAS_RESID:
            fn = lambda: ops.gemm(a, w, k, epi, out=out, resid=out, bias=bias, scratch=scr, splits=splits)
        else:
            fn = lambda: ops.gemm(a, w, k, epi, out=out, bias=bias, scratch=scr, splits=splits)
        cold = t(fn); warm = loop(fn)
        nbytes = n_out * kp * 2
        res[f"{name} splits={splits or 'auto'}"] = (cold, warm, nbytes / cold / 1e3)
q = torch.randn(B, 832, device=dev).half()
kc = torch.randn(B, NH, cap, D, device=dev).half(); vc = torch.randn_like(kc)
start = torch.zeros(B, dtype=torch.int32, device=dev); qb = torch.tensor([ctx - 1], dtype=torch.int32, device=dev)
ao = torch.zeros_like(q)
fn = lambda: ops.attention(q, None, kc, vc, start, qb, 0.125, ao, batch=B, heads=NH, head_dim=D, cap=cap, seq_len=1)
cold = t(fn); res["attn_decode"] = (cold, loop(fn), B * NH * ctx * D * 4 / cold / 1e3)
for k, v in res.items():
    print(f"{k:28s} cold {v[0]:8.2f} us  back-to-back {v[1]:8.2f} us" + (f"  cold GB/s {v[2]:8.1f}" if len(v) > 2 else ""))
