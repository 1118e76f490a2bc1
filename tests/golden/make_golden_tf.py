"""Teacher-forced golden vectors at the BENCHMARKED configs, from the UNMODIFIED
reference (run in the build container; ~10 min on 8 cores).

    python tests/golden/make_golden_tf.py [c2] [c3] [taps]

For C2 (Ernie-base-sized, 512 positions, batch 32, src 128, 64 new) and C3
(vocab pruned 40k -> 10k, 256 positions, batch 128, src 128, 64 new) the
reference's own ``batched_greedy_decode`` (model.py:613-667) runs free on the
F16 model with the bench's synthetic prompts (``bench.make_prompts``, rank 0);
a hook on ``_forward_tokens`` (model.py:440-504) records every step's logits.
Stored per (step, row): the reference tokens, the top-5 ids / values of the
logits (ties to the lower id, model.py:594) and the top-1 margin. The GPU test
(tests/test_gpu_parity_tf.py) feeds the reference tokens back step by step
(teacher forcing), so every step of every row is compared, not only the prefix
before a first low-margin divergence.

``taps``: the 2L+1 hidden-state taps (the input of every
layer_norm_f32 call, model.py:460, 484, 497) at the last position of two C2
prompts, for the reference's F16 and F32 paths.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from oracle import ref_loader  # noqa: E402

T = ref_loader.load()
M, TS, PR = T.model, T.tensor, T.pruning

import bench  # noqa: E402  (prompt construction + Zipf counts, same as the bench)
from make_golden import master_config, run_batched_with_logits, save, taps_of  # noqa: E402


def top5(step_logits):
    """top-5 ids (descending value, ties to the lower id) and values."""
    order = np.argsort(-step_logits, axis=-1, kind="stable")[..., :5]
    vals = np.take_along_axis(step_logits, order, axis=-1)
    s = np.sort(step_logits, axis=-1)
    margin = (s[..., -1] - s[..., -2]).astype(np.float32)
    return order.astype(np.int32), vals.astype(np.float16), margin


def c2_model():
    master = M.init_random(master_config(), seed=bench.SEED)
    return master, PR.prune_position_embedding(master, 512)


def run(tag, model, prompts, new):
    ts = time.time()
    seqs, steps = run_batched_with_logits(model, prompts, new)
    ids, vals, margin = top5(steps)
    save(f"{tag}_tf.npz", prompts=np.array(prompts, np.int32), tokens=np.array(seqs, np.int32),
         top5_ids=ids, top5_vals=vals, margin=margin, seconds=np.array(time.time() - ts))


def main(which):
    T.kernels.warmup()
    master, c2 = c2_model()
    if "c2" in which:
        w = bench.WORKLOADS["c2"]
        run("c2", c2, bench.make_prompts(40000, w, 0), w["new"])
    if "taps" in which:
        w = bench.WORKLOADS["c2"]
        prompts = bench.make_prompts(40000, w, 0)[:2]
        out = {"prompts": np.array(prompts, np.int32)}
        for tag, m in (("f16", c2), ("f32", M.cast_model(c2, TS.DType.F32))):
            taps = []
            for p in prompts:
                t, _ = taps_of(m, p)  # taps [2L+1, T, H] of row 0 -> last position
                taps.append(t[:, -1])
            out[f"taps_{tag}"] = np.stack(taps).astype(np.float32)
        save("c2_taps.npz", **out)
    if "c3" in which:
        w = bench.WORKLOADS["c3"]
        vmap = PR.build_pruned_vocab(bench.zipf_keep_ids(), 10000, specials=[0, 1, 2])
        c3 = PR.prune_position_embedding(PR.prune_token_embedding(master, vmap), w["positions"])
        run("c3", c3, bench.make_prompts(10000, w, 0), w["new"])


if __name__ == "__main__":
    main(set(sys.argv[1:]) or {"c2", "c3", "taps"})
