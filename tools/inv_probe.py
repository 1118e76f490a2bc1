"""Probe: last-position logits of a prompt run alone (B=1) vs inside a batch,
compared bitwise (prefill swap-AB split-K for <= 256 tokens vs full-K tiles above)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2407_04991_b200 as P  # noqa: E402
from paper_2407_04991_b200 import _native as N  # noqa: E402
from paper_2407_04991_b200 import model as PM  # noqa: E402
from oracle import tinfer_oracle as O  # noqa: E402

cfg = P.ModelConfig(2048, 768, 2, 12, 64, 1024, 512, P.DType.F16, 1, 2)
m = P.init_random(cfg, 5)
dm = m.device_model()


def last_logits(prompts):
    ids, pos, pads, _ = PM._left_pad(cfg, prompts)
    cap, mt = PM._session_shape(cfg, ids.shape[1], 8)
    s = dm.session(len(prompts), cap, mt, 8, logits="last")
    s.load_inputs(ids, pos, pads)
    s.forward(ids.shape[1], N.FWD_LOGITS_LAST)
    torch.cuda.synchronize()
    return s.logits[:len(prompts)].float().cpu().numpy()


ps = O.synthetic_prompts(2048, 160, 40, seed=3)
for B in (2, 4, 8, 16, 128, 160):
    a = last_logits(ps[:1])[0]
    b = last_logits(ps[:B])[0]
    print(f"B={B} tokens={B * 40}: bitwise {np.array_equal(a, b)} max-abs {np.abs(a - b).max():.3e}")
