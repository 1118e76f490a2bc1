"""Per-kernel device time: capture N launches of one op into a CUDA graph and
time the replay (removes host/ctypes overhead from the measurement)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2407_04991_b200 import ops, _native as N

dev = torch.device("cuda:0"); torch.cuda.set_device(0)
B = int(os.environ.get("B", 32)); H, F, V, NH, D, cap, ctx = 768, 3072, 40000, 12, 64, 192, 160
REPS = 50

def graph_time(fn, reps=REPS):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        fn(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps): fn()
    torch.cuda.synchronize()
    g.replay(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); g.replay(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    return statistics.median(ts)

x = torch.randn(B, 832, device=dev).half(); h = torch.zeros_like(x)
g_ = torch.ones(H, device=dev); b_ = torch.zeros(H, device=dev)
print(f"layernorm 32x768        {graph_time(lambda: ops.layernorm(x, H, g_, b_, h)):8.2f} us")
for name, n_out, k, epi in [("qkv", 3 * H, H, N.EPI_BIAS), ("wo", H, H, N.EPI_BIAS_RESID),
                            ("w1", F, H, N.EPI_BIAS_GELU), ("w2", H, F, N.EPI_BIAS_RESID),
                            ("lm_head", V, H, N.EPI_LOGITS)]:
    kp = ops.pad64(k)
    # rotate through 8 weight copies so the weights do not stay L2-resident
    ws = [(torch.randn(n_out, kp, device=dev) * 0.02).half() for _ in range(4 if name == "lm_head" else 12)]
    a = torch.randn(B, kp, device=dev).half()
    out = torch.zeros(B, max(n_out, 64), device=dev, dtype=torch.half)
    bias = torch.zeros(n_out, device=dev)
    keys = torch.zeros(B, dtype=torch.int64, device=dev)
    it = [0]
    def fn():
        w = ws[it[0] % len(ws)]; it[0] += 1
        if epi == N.EPI_LOGITS: ops.gemm(a, w, k, epi, keys=keys)
        elif epi == N.EPI_BIAS_RESID: ops.gemm(a, w, k, epi, out=out, resid=out, bias=bias)
        else: ops.gemm(a, w, k, epi, out=out, bias=bias)
    t = graph_time(fn, reps=len(ws) * 4)
    print(f"{name:8s} {n_out}x{k}  {t:8.2f} us  {n_out * kp * 2 / t / 1e3:8.1f} GB/s")
q = torch.randn(B, 832, device=dev).half()
kcs = [torch.randn(B, NH, cap, D, device=dev).half() for _ in range(6)]
start = torch.zeros(B, dtype=torch.int32, device=dev); qb = torch.tensor([ctx - 1], dtype=torch.int32, device=dev)
ao = torch.zeros_like(q); it = [0]
def fa():
    kc = kcs[it[0] % 6]; it[0] += 1
    ops.attention(q, None, kc, kc, start, qb, 0.125, ao, batch=B, heads=NH, head_dim=D, cap=cap, seq_len=1)
t = graph_time(fa, reps=24)
print(f"attn_decode ctx {ctx}    {t:8.2f} us  {B * NH * ctx * D * 4 / t / 1e3:8.1f} GB/s")
ids = torch.zeros(B, dtype=torch.int32, device=dev); tok = torch.randn(V, H, device=dev).half(); pe = torch.randn(512, H, device=dev).half()
print(f"embed_ln 32              {graph_time(lambda: ops.embed_ln(ids, ids, tok, pe, H, x, h, g_, b_)):8.2f} us")
