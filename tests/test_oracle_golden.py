"""Pins the CPU oracle (oracle/tinfer_oracle.py) to golden vectors produced by
the unmodified reference (tests/golden/make_golden.py). CPU only."""

import numpy as np

from conftest import golden
from oracle import tinfer_oracle as O


def small(f16=False):
    return O.Config(64, 32, 2, 2, 16, 64, 64, f16)


def test_tiny_forward_and_greedy():
    g = golden("tiny.npz")
    c = O.Config(8, 4, 1, 1, 4, 8, 32, False)
    w = O.init_weights(c, 7)
    assert O.weights_digest(w, c) == str(g["digest"])
    got = O.forward_full(w, c, list(g["ff_ids"]))
    assert np.max(np.abs(got - g["ff_logits"])) <= 1e-5
    assert O.greedy_decode(w, c, [3, 4], 10) == g["greedy"].tolist()


def test_small_known_answer_and_digests():
    g = golden("small.npz")
    c = small()
    w = O.init_weights(c, 7)
    assert O.weights_digest(w, c) == str(g["digest"])
    # survey-derived known answer
    assert O.greedy_decode(w, c, [5, 9, 11, 20], 12) == \
        [5, 9, 11, 20, 46, 11, 4, 46, 9, 46, 9, 46, 11, 58, 46, 9]
    w16 = O.cast_weights(w, True)
    assert O.weights_digest(w16, small(True)) == str(g["digest16"])
    assert O.greedy_decode(w16, small(True), [5, 9, 11, 20], 12) == g["greedy16"].tolist()


def test_small_logits_and_taps():
    g = golden("small.npz")
    for f16, lk, tk in ((False, "ff_logits", "taps"), (True, "ff_logits16", "taps16")):
        c = small(f16)
        w = O.cast_weights(O.init_weights(small(), 7), f16)
        taps = []
        cache = O.Cache.new(c, 1, 6)
        ids = np.asarray(g["ff_ids"]).reshape(1, -1)
        logits = O.forward_tokens(w, c, ids, np.arange(6).reshape(1, -1), cache,
                                  np.zeros(1, np.int64), all_logits=True, taps=taps)[0]
        tol = 1e-5 if not f16 else 2e-3
        assert np.max(np.abs(logits - g[lk])) <= tol
        assert len(taps) == 2 * c.num_layers + 1
        assert np.array_equal(taps[0][0], g[tk][0])  # embed sum is bit-exact
        assert np.max(np.abs(np.stack([t[0] for t in taps]) - g[tk])) <= tol


def test_small_batched_and_embed():
    g = golden("small.npz")
    c = small()
    w = O.init_weights(c, 7)
    bp = [[5, 9, 11], [7, 3, 3, 3, 20, 21], [50], [12, 13, 14, 15]]
    got = O.batched_greedy_decode(w, c, bp, 8)
    assert [s + [-1] * (20 - len(s)) for s in got] == g["batched"].tolist()
    w16 = O.cast_weights(w, True)
    got16 = O.batched_greedy_decode(w16, small(True), bp, 8)
    assert [s + [-1] * (20 - len(s)) for s in got16] == g["batched16"].tolist()
    assert np.array_equal(O.embed(w, c, list(g["embed_ids"]), 2), g["embed"])


def test_c1_tokens_and_prefill_logits():
    g = golden("c1.npz")
    prompts = O.synthetic_prompts(8192, 4, 64)
    assert prompts == g["prompts"].tolist()
    for tag, f16, tol in (("f32", False, 1e-5), ("f16", True, 4e-3)):
        c = O.config_c1(f16)
        w = O.init_weights(c, 42)
        assert O.weights_digest(w, c) == str(g["digest_" + tag])
        rec = []
        seqs = O.batched_greedy_decode(w, c, prompts, 32, step_logits=rec)
        assert seqs == g["tokens_" + tag].tolist()
        assert np.max(np.abs(rec[0] - g["prefill_logits_" + tag])) <= tol


def test_c2_short_master_digest_and_tokens():
    g = golden("c2_short.npz")
    c = O.config_master()
    w = O.init_weights(c, 42)
    assert O.weights_digest(w, c) == str(g["digest_master"])
    w2, c2 = O.prune_weights(w, c, tuple(range(c.vocab_size)), new_max_position=512)
    prompts = g["prompts"].tolist()
    assert prompts == O.synthetic_prompts(40000, 2, 128)
    rec = []
    seqs = O.batched_greedy_decode(w2, c2, prompts, 6, step_logits=rec)
    assert np.max(np.abs(rec[0] - g["prefill_logits"].astype(np.float32))) <= 8e-3
    # tokens equal wherever the reference's top-1 margin clears the tolerance
    ref = g["tokens"]
    for b in range(2):
        for s in range(6):
            if g["margin"][s, b] > 4e-2:
                assert seqs[b][128 + s] == ref[b][128 + s]


def test_pruning_and_batching_known_answers():
    g = golden("pruning.npz")
    assert O.build_pruned_vocab(g["zipf_counts"], 10000, [0, 1, 2]) == tuple(g["kept_c3"])
    c = O.config_c1(False)
    w = O.init_weights(c, 42)
    kept = tuple(int(i) for i in g["c1_kept"])
    w2, c2 = O.prune_weights(w, c, kept, new_max_position=128)
    prompt = [kept.index(t) for t in g["c1_prompt"]]
    assert O.greedy_decode(w2, c2, prompt, 12) == g["c1_pruned_tokens"].tolist()
    assert [kept[t] for t in g["c1_pruned_tokens"]] == g["c1_orig"].tolist()
    groups, pads = O.plan_batches(g["plan_lengths"].tolist(), 32, 16)
    assert [i for gr in groups for i in gr] == g["plan_groups"].tolist()
    assert [len(gr) for gr in groups] == g["plan_sizes"].tolist()
    assert pads == g["plan_pads"].tolist()
