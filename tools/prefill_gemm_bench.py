"""Graph-timed prefill (non-swap) GEMM shapes at M tokens: TFLOP/s per epilogue."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_04991_b200 import ops, _native as N
dev = torch.device("cuda:0")
M = int(os.environ.get("M", 4096)); H, F = 768, 3072

def graph_time(fn, reps=10):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps): fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); g.replay(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    return statistics.median(ts)

a = torch.randn(M, 3072, device=dev).half()
for name, n_out, k, epi in [("qkv", 3 * H, H, N.EPI_BIAS), ("wo", H, H, N.EPI_BIAS_RESID),
                            ("w1", F, H, N.EPI_BIAS_GELU), ("w2", H, F, N.EPI_BIAS_RESID),
                            ("f32", F, H, N.EPI_F32)]:
    w = (torch.randn(n_out, k, device=dev) * 0.02).half()
    out = torch.zeros(M, n_out, device=dev, dtype=torch.float32 if epi == N.EPI_F32 else torch.half)
    bias = torch.zeros(n_out, device=dev)
    act = a[:, :k]
    if epi == N.EPI_BIAS_RESID:
        fn = lambda: ops.gemm(act, w, k, epi, out=out, resid=out, bias=bias, force_swap=0)
    else:
        fn = lambda: ops.gemm(act, w, k, epi, out=out, bias=bias, force_swap=0)
    t = graph_time(fn)
    print(f"{name:4s} {M}x{n_out}x{k}: {t:8.1f} us  {2*M*n_out*k/t/1e6:7.1f} TFLOP/s", flush=True)
