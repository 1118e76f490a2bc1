"""Helper for test_gpu_beam_attention.py (run in a fresh process: the attention
switches are read once per process). Runs the device beam search on a D=64
model and saves the final beam scores and token/parent histories."""

import sys

import numpy as np
import torch

import paper_2407_04991_b200 as P
from paper_2407_04991_b200.beam import BeamRun
from oracle import tinfer_oracle as O


def main():
    out, K, new = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    lens = [int(x) for x in sys.argv[4].split(",")]
    cfg = P.ModelConfig(8192, 256, 2, 4, 64, 1024, 512, P.DType.F16, 1, 2)
    m = P.init_random(cfg, 42)
    prompts = O.synthetic_prompts(8192, len(lens), max(lens), seed=5)
    prompts = [p[:n] for p, n in zip(prompts, lens)]
    run = BeamRun(m, prompts, new, K)
    with torch.cuda.device(run.dm.device):
        run.stage_inputs()
        run.run_device(use_graph=True)
        torch.cuda.synchronize()
        s = run.s
        np.savez(out, scores=s.scores.cpu().numpy(), tok=s.tok_hist.cpu().numpy(), par=s.par_hist.cpu().numpy(),
                 seqs=np.array([len(x) for x in run.finish()[0]]))


if __name__ == "__main__":
    main()
