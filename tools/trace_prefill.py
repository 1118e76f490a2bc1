"""CUPTI trace of one C2 prefill forward (B=32, T=128): per-kernel device time."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_04991_b200 as P
from paper_2407_04991_b200 import model as PM, _native as N
from paper_2407_04991_b200.pruning import prune_position_embedding
from oracle import tinfer_oracle as O
B = int(os.environ.get("B", 32)); SRC = int(os.environ.get("SRC", 128))
cfg = P.ModelConfig(40000, 768, 12, 12, 64, 3072, 1024, P.DType.F16, 1, 2)
m = prune_position_embedding(P.init_random(cfg, 42), 512)
dm = m.device_model()
prompts = O.synthetic_prompts(40000, B, SRC)
ids, pos, pads, _ = PM._left_pad(m.config, prompts)
cap, mt = PM._session_shape(m.config, SRC, 64)
s = dm.session(B, cap, mt, 64)
for _ in range(3):
    s.load_inputs(ids, pos, pads); s.forward(SRC, N.FWD_ARGMAX)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
s.load_inputs(ids, pos, pads)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    s.forward(SRC, N.FWD_ARGMAX)
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
span = evs[-1].time_range.end - evs[0].time_range.start
agg = collections.defaultdict(lambda: [0, 0.0])
for e in evs:
    a = agg[e.name[:70]]; a[0] += 1; a[1] += e.time_range.end - e.time_range.start
print(f"prefill span {span:.1f} us, {len(evs)} kernels")
for k, (n, d) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  n={n:3d} {d:9.1f} us ({d/n:8.2f}/launch)  {k}")

inc = collections.defaultdict(lambda: [0, 0.0])
for i in range(1, len(evs)):
    a = inc[evs[i].name[:70]]; a[0] += 1; a[1] += evs[i].time_range.end - evs[i - 1].time_range.end
print("critical-path increments:")
for k, (n, d) in sorted(inc.items(), key=lambda kv: -kv[1][1]):
    print(f"  n={n:3d} {d:9.1f} us ({d/n:8.2f}/launch)  {k}")
