"""One C2 prefill forward (B=32, T=128) through a session, after two warm-up
forwards; for `ncu -k regex:gemm_pf2 ...` captures of the prefill GEMMs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2407_04991_b200 import _native as N  # noqa: E402
from paper_2407_04991_b200 import model as PM  # noqa: E402

w = bench.WORKLOADS["c2"]
m = bench.build_model(w)
prompts = bench.make_prompts(m.config.vocab_size, w, 0)
ids, pos, pads, _ = PM._left_pad(m.config, prompts)
cap, mt = PM._session_shape(m.config, ids.shape[1], w["new"])
s = m.device_model().session(len(prompts), cap, mt, w["new"])
for _ in range(3):
    s.load_inputs(ids, pos, pads)
    s.forward(ids.shape[1], N.FWD_ARGMAX)
torch.cuda.synchronize()
print("ok")
