"""Megakernel vs multi-kernel decode: token agreement and step time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_04991_b200 as P
from paper_2407_04991_b200 import model as PM, _native as N
from paper_2407_04991_b200.pruning import prune_position_embedding
from oracle import tinfer_oracle as O

which = os.environ.get("CFG", "small")
if which == "small":
    cfg = P.ModelConfig(512, 128, 2, 2, 64, 512, 128, P.DType.F16, 1, 2); B, SRC, NEW = 4, 8, 8
    m = P.init_random(cfg, 11)
else:
    cfg = P.ModelConfig(40000, 768, 12, 12, 64, 3072, 1024, P.DType.F16, 1, 2); B, SRC, NEW = int(os.environ.get("B", 32)), 128, 64
    m = prune_position_embedding(P.init_random(cfg, 42), 512)
prompts = O.synthetic_prompts(m.config.vocab_size, B, SRC)
prompts[0] = prompts[0][: SRC // 2]  # ragged: left padding
import bench
res = {}
for mk in ("0", "1"):
    os.environ["TF_MEGAKERNEL"] = mk
    os.environ["TF_MEGAKERNEL"] = mk
    out = P.batched_greedy_decode(m, prompts, NEW)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        out = P.batched_greedy_decode(m, prompts, NEW)
    torch.cuda.synchronize()
    res[mk] = (out, (time.perf_counter() - t0) / 3)
    print(f"TF_MEGAKERNEL={mk}: {res[mk][1]*1e3:.2f} ms per generate", flush=True)
a, b = res["0"][0], res["1"][0]
same = sum(x == y for x, y in zip(a, b))
first_div = [next((i for i, (u, v) in enumerate(zip(x, y)) if u != v), None) for x, y in zip(a, b)]
print(f"rows identical: {same}/{len(a)}; first divergence per row: {first_div}")
