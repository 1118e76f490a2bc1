"""Generate golden vectors from the UNMODIFIED reference (run in the build container).

    python tests/golden/make_golden.py

Imports ``/root/reference/pkg/src/tinfer`` through ``oracle/ref_loader.py`` and
writes small ``.npz`` fixtures next to this file. They pin both the oracle
(``oracle/tinfer_oracle.py``, checked in ``tests/test_oracle_golden.py``) and the
GPU path (``tests/test_gpu_*.py``) to the reference's own outputs on identical
random-init weights and synthetic prompts. ``/root/reference`` does not exist on
the GPU box, so only these committed fixtures travel.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref_loader  # noqa: E402
from oracle import tinfer_oracle as O  # noqa: E402

T = ref_loader.load()
M, TS, PR, PL = T.model, T.tensor, T.pruning, T.pipeline
F32, F16 = TS.DType.F32, TS.DType.F16


def cfg(**kw):
    return M.ModelConfig(**kw)


def tiny_config(dtype=F32):
    return cfg(vocab_size=8, hidden_size=4, num_layers=1, num_heads=1, head_dim=4,
               ffn_size=8, max_position=32, dtype=dtype, eos_token=1, pad_token=2)


def small_config(dtype=F32, **over):
    base = dict(vocab_size=64, hidden_size=32, num_layers=2, num_heads=2, head_dim=16,
                ffn_size=64, max_position=64, dtype=dtype, eos_token=1, pad_token=2)
    base.update(over)
    return cfg(**base)


def c1_config(dtype=F32):
    return cfg(vocab_size=8192, hidden_size=256, num_layers=2, num_heads=4, head_dim=64,
               ffn_size=1024, max_position=512, dtype=dtype, eos_token=1, pad_token=2)


def master_config(dtype=F16):
    return cfg(vocab_size=40000, hidden_size=768, num_layers=12, num_heads=12, head_dim=64,
               ffn_size=3072, max_position=1024, dtype=dtype, eos_token=1, pad_token=2)


def digest(model):
    h = hashlib.sha256()
    for _, t in model.named_tensors():
        h.update(t.array.tobytes())
    return h.hexdigest()


def prompts_for(V, B, S, seed=42):
    s = T.rng.SplitMix64(T.rng.derive_seed(seed, "prompts"))
    ids = s.randint(B * S, V - 3) + 3
    return [list(map(int, r)) for r in ids.reshape(B, S)]


def run_batched_with_logits(model, prompts, max_new):
    """batched_greedy_decode with a hook on _forward_tokens that records the
    per-step logits ([B, V], f32 values) the reference argmaxes."""
    rec = []
    orig = M._forward_tokens

    def hook(*a, **k):
        out = orig(*a, **k)
        rec.append(np.asarray(out, np.float32).copy())
        return out

    M._forward_tokens = hook
    try:
        seqs = M.batched_greedy_decode(model, prompts, max_new)
    finally:
        M._forward_tokens = orig
    return seqs, np.stack(rec)


def margins(step_logits):
    """top-1 minus top-2 per (step, row)."""
    s = np.sort(step_logits, axis=-1)
    return (s[..., -1] - s[..., -2]).astype(np.float32)


def taps_of(model, ids):
    taps = []
    ln = M.layer_norm_f32
    M.layer_norm_f32 = lambda x, g, b, eps: (taps.append(x.copy()), ln(x, g, b, eps))[1]
    try:
        logits = M.forward_full(model, ids).array
    finally:
        M.layer_norm_f32 = ln
    return np.stack([t[0] for t in taps]).astype(np.float32), logits


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def main():
    T.kernels.warmup()
    t0 = time.time()

    # --- tiny + small configs (reference conftest.py:15-40) -----------------
    tiny = M.init_random(tiny_config(), seed=7)
    save("tiny.npz",
         digest=np.array(digest(tiny)),
         ff_ids=np.array([3, 5, 7, 2, 6, 4]),
         ff_logits=M.forward_full(tiny, [3, 5, 7, 2, 6, 4]).array,
         greedy=np.array(M.greedy_decode(tiny, [3, 4], 10)))

    small = M.init_random(small_config(), seed=7)
    small16 = M.cast_model(small, F16)
    bprompts = [[5, 9, 11], [7, 3, 3, 3, 20, 21], [50], [12, 13, 14, 15]]
    bat = M.batched_greedy_decode(small, bprompts, 8)
    bat16 = M.batched_greedy_decode(small16, bprompts, 8)
    taps, tap_logits = taps_of(small, [10, 20, 30, 40, 50, 60])
    taps16, tap_logits16 = taps_of(small16, [10, 20, 30, 40, 50, 60])
    save("small.npz",
         digest=np.array(digest(small)),
         digest16=np.array(digest(small16)),
         greedy=np.array(M.greedy_decode(small, [5, 9, 11, 20], 12)),
         greedy16=np.array(M.greedy_decode(small16, [5, 9, 11, 20], 12)),
         ff_ids=np.array([10, 20, 30, 40, 50, 60]),
         ff_logits=tap_logits, ff_logits16=tap_logits16,
         taps=taps, taps16=taps16,
         batched=np.array([s + [-1] * (20 - len(s)) for s in bat]),
         batched16=np.array([s + [-1] * (20 - len(s)) for s in bat16]),
         embed_ids=np.array([3, 1, 4, 1, 5]),
         embed=M.embed(small, [3, 1, 4, 1, 5], start_position=2).array)

    # --- C1: the reference's tiny Ernie-style config (BASELINE configs[0]) ---
    out = {}
    for tag, dt in (("f32", F32), ("f16", F16)):
        m = M.init_random(c1_config(dt), seed=42)
        prompts = prompts_for(8192, 4, 64)
        M.batched_greedy_decode(m, prompts[:1], 2)  # warm specialisations
        ts = time.time()
        seqs, steps = run_batched_with_logits(m, prompts, 32)
        dt_s = time.time() - ts
        out[f"digest_{tag}"] = np.array(digest(m))
        out[f"tokens_{tag}"] = np.array(seqs)
        out[f"prefill_logits_{tag}"] = steps[0]
        out[f"argmax_{tag}"] = steps.argmax(-1)
        out[f"margin_{tag}"] = margins(steps)
        out[f"seconds_{tag}"] = np.array(dt_s)
        if tag == "f32":
            out["prompts"] = np.array(prompts)
    save("c1.npz", **out)

    # --- master Ernie-base (P=1024) trimmed to 512 positions (C2 model), short run
    master = M.init_random(master_config(), seed=42)
    c2 = PR.prune_position_embedding(master, 512)
    prompts = prompts_for(40000, 2, 128)
    ts = time.time()
    seqs, steps = run_batched_with_logits(c2, prompts, 6)
    c2_secs = time.time() - ts
    save("c2_short.npz",
         digest_master=np.array(digest(master)),
         prompts=np.array(prompts), tokens=np.array(seqs),
         prefill_logits=steps[0].astype(np.float16),
         argmax=steps.argmax(-1), margin=margins(steps),
         seconds=np.array(c2_secs))

    # --- pruning (pruning.py) + batching (pipeline.py) known answers ---------
    zs = O.Stream(O.derive_seed(42, "zipf"))
    rank = np.argsort(zs.u64(40000), kind="stable")
    counts = np.empty(40000, np.int64)
    counts[rank] = 10 ** 9 // (np.arange(40000) + 1)
    vmap = PR.build_pruned_vocab(counts, 10000, specials=[0, 1, 2])
    thr = PR.build_pruned_vocab_by_threshold(counts[:200], 10 ** 6, specials=[1])
    # pruned C1 generation (kept set covers prompt + original output: exact in F32)
    m1 = M.init_random(c1_config(), seed=42)
    p1 = prompts_for(8192, 1, 16)[0]
    orig = M.greedy_decode(m1, p1, 12)
    kept = tuple(sorted(set(orig) | {0, 1, 2} | set(range(3, 600))))
    pm = PR.prune_token_embedding(m1, PR.PrunedVocabMap(kept_old_ids=kept, threshold=len(kept)))
    pm = PR.prune_position_embedding(pm, 128)
    got = M.greedy_decode(pm, [kept.index(t) for t in p1], 12)
    rs = O.Stream(O.derive_seed(7, "lengths"))
    lens = (rs.randint(300, 481) + 32).tolist()
    plan = PL.plan_batches(lens, 32, 16)
    save("pruning.npz",
         zipf_counts=counts, kept_c3=np.array(vmap.kept_old_ids),
         kept_threshold=np.array(thr.kept_old_ids),
         c1_prompt=np.array(p1), c1_orig=np.array(orig), c1_kept=np.array(kept),
         c1_pruned_tokens=np.array(got),
         plan_lengths=np.array(lens),
         plan_groups=np.array([i for g in plan.groups for i in g]),
         plan_sizes=np.array([len(g) for g in plan.groups]),
         plan_pads=np.array(plan.group_pad))
    print(f"golden generation done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
