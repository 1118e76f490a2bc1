"""GPU parity at the benchmark shapes the small tests do not reach: batch 128
(bn = 128 swap-AB tiles, split-KV attention), pruned vocabulary, long and ragged
prompts (multi-tile prefill attention), and the device-side prompt remap."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2407_04991_b200 as P  # noqa: E402
from paper_2407_04991_b200 import pruning as PR  # noqa: E402
from oracle import tinfer_oracle as O  # noqa: E402

MARGIN = 4e-2


def check_margin_gated(got, ref, rec, prompts):
    for b, (g, r) in enumerate(zip(got, ref)):
        n = len(prompts[b])
        assert g[:n] == r[:n]
        for s in range(len(r) - n):
            if g[n + s] != r[n + s]:
                top = np.sort(rec[s][b])[-2:]
                assert top[1] - top[0] < MARGIN, (b, s, g[n + s], r[n + s])
                break


def small_ernie(v=2048, p=1024):
    return (v, 256, 2, 4, 64, 1024, p)


@pytest.fixture(scope="module")
def pair():
    args = small_ernie()
    m = P.init_random(P.ModelConfig(*args, P.DType.F16, 1, 2), 5)
    w = O.init_weights(O.Config(*args, True, 1, 2), 5)
    return m, w, O.Config(*args, True, 1, 2)


def test_batch_128_matches_oracle(cuda_device, pair):
    m, w, oc = pair
    prompts = O.synthetic_prompts(oc.vocab_size, 128, 24, seed=9)
    got = P.batched_greedy_decode(m, prompts, 6)
    rec = []
    ref = O.batched_greedy_decode(w, oc, prompts, 6, step_logits=rec)
    check_margin_gated(got, ref, rec, prompts)


def test_long_ragged_prompts_match_oracle(cuda_device, pair):
    m, w, oc = pair
    s = O.Stream(O.derive_seed(3, "ragged"))
    lens = (s.randint(6, 400) + 130).tolist()
    ids = (s.randint(sum(lens), oc.vocab_size - 3) + 3).tolist()
    prompts, k = [], 0
    for n in lens:
        prompts.append(ids[k:k + n])
        k += n
    got = P.batched_greedy_decode(m, prompts, 5)
    rec = []
    ref = O.batched_greedy_decode(w, oc, prompts, 5, step_logits=rec)
    check_margin_gated(got, ref, rec, prompts)
    # batched == single, bitwise, at multi-tile prompt lengths
    assert got[2] == P.greedy_decode(m, prompts[2], 5)


def test_pruned_model_and_device_remap(cuda_device, pair):
    m, w, oc = pair
    counts = np.arange(oc.vocab_size)[::-1].copy()
    vmap = PR.build_pruned_vocab(counts, 700, specials=[0, 1, 2])
    pm = PR.prune_token_embedding(m, vmap)
    kept = vmap.kept_old_ids
    prompts_old = [[kept[(7 * i + 3 * j) % len(kept)] for j in range(20)] for i in range(8)]
    prompts_new = [vmap.remap(p) for p in prompts_old]
    a = P.batched_greedy_decode(pm, prompts_new, 6)
    b = P.batched_greedy_decode(pm, prompts_old, 6, prompt_vocab_map=vmap)
    assert [x[20:] for x in a] == [x[20:] for x in b]
    # pruned-vocab logits == unpruned logits restricted to the kept ids (bitwise)
    full = P.forward_full(m, prompts_old[0]).array[-1]
    pr = P.forward_full(pm, prompts_new[0]).array[-1]
    assert np.array_equal(full[list(kept)], pr)


def test_ragged_batch_tiles_match_oracle(cuda_device, pair):
    """Batch 100: two 64-row decode tiles, the second partial (rows past the
    batch masked in every epilogue), with ragged prompts."""
    m, w, oc = pair
    s = O.Stream(O.derive_seed(4, "tiles"))
    lens = (s.randint(100, 40) + 8).tolist()
    ids = (s.randint(sum(lens), oc.vocab_size - 3) + 3).tolist()
    prompts, k = [], 0
    for n in lens:
        prompts.append(ids[k:k + n])
        k += n
    got = P.batched_greedy_decode(m, prompts, 5)
    rec = []
    ref = O.batched_greedy_decode(w, oc, prompts, 5, step_logits=rec)
    check_margin_gated(got, ref, rec, prompts)


def test_generation_up_to_max_position(cuda_device, pair):
    """prompt + max_new_tokens == max_position: the last generated token sits in
    the last position / cache slot."""
    m, w, oc = pair
    P_max = oc.max_position
    s = O.Stream(O.derive_seed(5, "maxpos"))
    prompts = [(s.randint(P_max - 4, oc.vocab_size - 3) + 3).tolist(), [7, 8, 9]]
    got = P.batched_greedy_decode(m, prompts, 4)
    rec = []
    ref = O.batched_greedy_decode(w, oc, prompts, 4, step_logits=rec)
    check_margin_gated(got, ref, rec, prompts)
    with pytest.raises(P.PositionError):
        P.batched_greedy_decode(m, prompts, 5)
