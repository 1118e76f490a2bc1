"""One graph-equivalent decode step of a workload inside an NVTX range "step",
for ncu (--nvtx --nvtx-include "step/"): prefill, a few warm decode steps, then
one eager decode step (the same kernels and PDL chaining the graph replays).
Usage: python tools/one_step.py [workload]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2407_04991_b200 import _native as N  # noqa: E402


def main():
    w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    model = bench.build_model(w)
    run = bench.Runner(model, bench.make_prompts(model.config.vocab_size, w, 0), w)
    run.stage()
    if run.beam:  # beam: prefill + select, warm steps, then one (T=1 forward + select) step
        import ctypes as C
        br, s = run.beam, run.sess
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        s.forward(br.L, N.FWD_LOGITS_LAST)
        N.check(N.lib().tf_beam_select(s.handle, C.byref(br.desc), st), "tf_beam_select")
        N.check(N.lib().tf_beam_decode(s.handle, C.byref(br.desc), 4, 0, st), "tf_beam_decode")
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("step")
        N.check(N.lib().tf_beam_decode(s.handle, C.byref(br.desc), 1, 0, st), "tf_beam_decode")
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        print("ok")
        return
    run.sess.forward(run.ids.shape[1], N.FWD_ARGMAX)
    run.sess.decode(4, use_graph=False)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("step")
    run.sess.decode(1, use_graph=False)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print("ok")


if __name__ == "__main__":
    main()
