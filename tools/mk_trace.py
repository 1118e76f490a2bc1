"""Timeline of one megakernel decode step from per-task globaltimer stamps."""
import ctypes as C, os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2407_04991_b200 as P
from paper_2407_04991_b200 import model as PM, _native as N
from paper_2407_04991_b200.pruning import prune_position_embedding
from oracle import tinfer_oracle as O

B = int(os.environ.get("B", 32))
cfg = P.ModelConfig(40000, 768, 12, 12, 64, 3072, 1024, P.DType.F16, 1, 2)
m = prune_position_embedding(P.init_random(cfg, 42), 512)
prompts = O.synthetic_prompts(40000, B, 128)
P.batched_greedy_decode(m, prompts, 64)
dm = m.device_model()
sess = next(iter(dm._sessions.values()))
ni, na = C.c_int(), C.c_int()
N.check(N.lib().tf_debug_mk_trace(sess.handle, None, C.byref(ni), C.byref(na), None), "trace")
plan = np.zeros((ni.value + na.value, 4), np.int32)
trace = torch.zeros((ni.value + na.value) * 8, dtype=torch.int64, device="cuda")
N.check(N.lib().tf_debug_mk_trace(sess.handle, C.c_void_p(trace.data_ptr()), C.byref(ni), C.byref(na),
                                  plan.ctypes.data_as(C.c_void_p)), "trace")
P.batched_greedy_decode(m, prompts, 64)
torch.cuda.synchronize()
t = trace.cpu().numpy().reshape(-1, 8).astype(np.float64)
N.check(N.lib().tf_debug_mk_trace(sess.handle, None, None, None, None), "trace")
t0 = t[t > 0].min()
t = np.where(t > 0, (t - t0) / 1e3, np.nan)  # us
GN = ["QKV", "WO", "W1", "W2", "LM"]; AN = ["ATT", "R2", "R1", "EMB"]
rows = collections.OrderedDict()
for i in range(ni.value + na.value):
    ty, l = plan[i, 0], plan[i, 1]
    name = GN[ty] if i < ni.value else AN[ty]
    if name in ("LM", "EMB"):
        l = -1 if name == "EMB" else 99
    key = (l, name)
    rows.setdefault(key, []).append(t[i])
order = {"EMB": 0, "QKV": 1, "ATT": 2, "WO": 3, "R2": 4, "W1": 5, "W2": 6, "R1": 7, "LM": 8}
print(f"{'layer':>5} {'phase':>5} {'n':>4} {'start_min':>9} {'ready_max':>9} {'end_max':>9} {'dur_med':>8}")
for (l, name), v in sorted(rows.items(), key=lambda kv: (kv[0][0], order[kv[0][1]])):
    v = np.array(v)
    ready = np.nanmax(v[:, 1]) if not np.all(np.isnan(v[:, 1])) else np.nan
    print(f"{l:>5} {name:>5} {len(v):>4} {np.nanmin(v[:,0]):9.1f} {ready:9.1f} {np.nanmax(v[:,2]):9.1f} {np.nanmedian(v[:,2]-v[:,0]):8.2f}")

# sub-phase breakdown for one layer (median over tasks), relative to task stamp 0
L = int(os.environ.get("LAYER", 6))
def sub(name, cols):
    v = np.array(rows[(L, name)])
    out = []
    for a, b in cols:
        d = v[:, b] - v[:, a]
        out.append(f"{a}->{b}: {np.nanmedian(d):6.2f} (max {np.nanmax(d):6.2f})")
    print(f"layer {L} {name}: " + "  ".join(out))
sub("ATT", [(0, 1), (1, 3), (3, 4), (4, 5), (5, 6), (6, 7)])
sub("R1", [(0, 1), (1, 2)])
sub("R2", [(0, 1), (1, 2)])
for g in ("QKV", "WO", "W1", "W2"):
    sub(g, [(0, 1), (1, 5), (5, 2)])
