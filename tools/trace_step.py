"""CUPTI trace of graph-replayed C2 decode steps: per-kernel device durations and
inter-kernel gaps (torch.profiler collects every kernel in the process)."""
import os, sys, json, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_04991_b200 as P
from paper_2407_04991_b200 import model as PM, _native as N
from paper_2407_04991_b200.pruning import prune_position_embedding
from oracle import tinfer_oracle as O

B = int(os.environ.get("B", 32)); SRC, NEW = 128, 64
cfg = P.ModelConfig(40000, 768, 12, 12, 64, 3072, 1024, P.DType.F16, 1, 2)
m = prune_position_embedding(P.init_random(cfg, 42), 512)
dm = m.device_model()
prompts = O.synthetic_prompts(40000, B, SRC)
ids, pos, pads, _ = PM._left_pad(m.config, prompts)
s = dm.session(B, SRC + NEW, SRC, NEW)
use_graph = int(os.environ.get("GRAPH", 1))
for _ in range(3):
    s.load_inputs(ids, pos, pads); s.forward(SRC, N.FWD_ARGMAX); s.decode(NEW - 1, use_graph=bool(use_graph))
torch.cuda.synchronize()
s.load_inputs(ids, pos, pads); s.forward(SRC, N.FWD_ARGMAX); s.decode(20, use_graph=bool(use_graph))
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s.decode(4, use_graph=bool(use_graph))
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
evs.sort(key=lambda e: e.time_range.start)
# one step = the last 87 kernels
per = collections.OrderedDict()
rows = []
prev_end = None
for e in evs:
    st, en = e.time_range.start, e.time_range.end
    gap = (st - prev_end) if prev_end is not None else 0
    prev_end = en
    rows.append((e.name[:60], en - st, gap))
n = len(rows)
print("kernels traced", n)
step = rows[-(n // 4):]
tot = sum(r[1] for r in step); gaps = sum(r[2] for r in step)
print(f"one step: {len(step)} kernels, busy {tot:.1f} us, gaps {gaps:.1f} us, span {tot+gaps:.1f} us")
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for name, d, g in step:
    a = agg[name]; a[0] += 1; a[1] += d; a[2] += g
for k, (c, d, g) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"n={c:3d} busy {d:8.1f} us ({d/c:6.2f}/launch) gaps-before {g:7.1f} us  {k}")
# critical-path attribution: end_i - end_{i-1}
ends = []
for e in evs:
    ends.append((e.name[:60], e.time_range.start, e.time_range.end))
ends = ends[-(n // 4):]
inc = collections.defaultdict(lambda: [0, 0.0])
for i in range(1, len(ends)):
    a = inc[ends[i][0]]; a[0] += 1; a[1] += ends[i][2] - ends[i - 1][2]
print("critical-path increments (end_i - end_{i-1}):")
for k, (c, d) in sorted(inc.items(), key=lambda kv: -kv[1][1]):
    print(f"  n={c:3d} {d:8.1f} us ({d/c:6.2f}/launch)  {k}")
