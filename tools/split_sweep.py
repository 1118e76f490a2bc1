"""Graph-timed sweep of split-K counts for the decode GEMM shapes at batch B."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_04991_b200 import ops, _native as N
dev = torch.device("cuda:0")
B = int(os.environ.get("B", 128)); H, F = 768, 3072

def graph_time(fn, reps):
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

for name, n_out, k, epi in [("qkv", 3 * H, H, N.EPI_BIAS), ("wo", H, H, N.EPI_BIAS_RESID),
                            ("w1", F, H, N.EPI_BIAS_GELU), ("w2", H, F, N.EPI_BIAS_RESID)]:
    kb = k // 64
    ws = [(torch.randn(n_out, k, device=dev) * 0.02).half() for _ in range(12)]
    a = torch.randn(B, k, device=dev).half()
    out = torch.zeros(B, n_out, device=dev, dtype=torch.half)
    bias = torch.zeros(n_out, device=dev)
    res = []
    for sp in [d for d in range(1, 17) if kb % d == 0]:
        it = [0]
        def fn():
            w = ws[it[0] % 12]; it[0] += 1
            if epi == N.EPI_BIAS_RESID: ops.gemm(a, w, k, epi, out=out, resid=out, bias=bias, splits=sp)
            else: ops.gemm(a, w, k, epi, out=out, bias=bias, splits=sp)
        res.append((sp, graph_time(fn, 48)))
    print(name, " ".join(f"s{sp}:{t:.1f}" for sp, t in res), flush=True)
