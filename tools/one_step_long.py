"""One eager decode step at C5's longest bucket (pruned Ernie-base, batch 128,
src 512) inside an NVTX range "step", for ncu; optional arg: src length.
    ncu --nvtx --nvtx-include "step/" -k regex:attn_decode ... python tools/one_step_long.py 512"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2407_04991_b200 import _native as N  # noqa: E402


def main():
    src = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    w = dict(bench.WORKLOADS["c5"], src=src, requests=None)
    model = bench.build_model(w)
    run = bench.Runner(model, bench.make_prompts(model.config.vocab_size, w, 0), w)
    run.stage()
    run.sess.forward(run.ids.shape[1], N.FWD_ARGMAX)
    run.sess.decode(4, use_graph=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run.sess.decode(8, use_graph=True)
    e1.record()
    e1.synchronize()
    print(f"graph-replayed decode step at src {src}: {e0.elapsed_time(e1) / 8 * 1e3:.1f} us")
    torch.cuda.nvtx.range_push("step")
    run.sess.decode(1, use_graph=False)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()


if __name__ == "__main__":
    main()
