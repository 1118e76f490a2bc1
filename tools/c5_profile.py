"""Where the C5 sweep's time goes: for every length-bucketed group (one worker,
in plan order) the prefill forward, the graph-replayed decode and the host
remainder of one batched_greedy_decode-equivalent call, timed with CUDA events.
Usage: python tools/c5_profile.py [max_groups]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_04991_b200 as P  # noqa: E402
from paper_2407_04991_b200 import _native as N  # noqa: E402
from paper_2407_04991_b200 import model as M  # noqa: E402
from paper_2407_04991_b200 import pipeline as PL  # noqa: E402


def main():
    w = bench.WORKLOADS["c5"]
    model = bench.build_model(w)
    reqs = bench.make_prompts(model.config.vocab_size, w, 0)
    plan = PL.plan_batches([len(r) for r in reqs], w["batch"], 16)
    ng = int(sys.argv[1]) if len(sys.argv) > 1 else len(plan.groups)
    dm = model.device_model()
    rows = []
    for gi in range(min(ng, len(plan.groups))):
        prompts = [reqs[i] for i in plan.groups[gi]]
        P.batched_greedy_decode(model, prompts, w["new"])  # session + graphs for this shape
        ids, pos, pads, lens = M._left_pad(model.config, prompts)
        B, L = ids.shape
        cap, mt = M._session_shape(model.config, L, w["new"])
        s = dm.session(B, cap, mt, w["new"])
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.load_inputs(ids, pos, pads)
        e[0].record()
        s.forward(L, N.FWD_ARGMAX)
        e[1].record()
        s.decode(w["new"] - 1)
        e[2].record()
        s.fetch_tokens(w["new"])
        wall = (time.perf_counter() - t0) * 1e3
        pre, dec = e[0].elapsed_time(e[1]), e[1].elapsed_time(e[2])
        rows.append((B, L, pre, dec, wall))
    a = np.array(rows)
    print(f"groups {len(rows)}: prefill {a[:, 2].sum():.1f} ms, decode {a[:, 3].sum():.1f} ms, "
          f"wall {a[:, 4].sum():.1f} ms (host remainder {a[:, 4].sum() - a[:, 2].sum() - a[:, 3].sum():.1f} ms)")
    for B, L, pre, dec, wall in rows[:: max(1, len(rows) // 12)]:
        print(f"  B={int(B):3d} L={int(L):3d}: prefill {pre:6.2f} ms  decode {dec:6.2f} ms ({dec / 63 * 1e3:6.1f} us/step)  "
              f"wall {wall:6.2f} ms")


if __name__ == "__main__":
    main()
