"""Token-type embeddings (north star (1): word / position / type gather-sum).

The reference embeds token + position only (model.py:453-455), so this is an
extension with parity UNPINNED by reference code: the embedding is checked
bit-exactly against numpy q16(tok[id] + pos[p] + type[t]) (the reference's
gather-sum rule with one more f32 term), and generation against the oracle
restatement extended the same way (oracle/tinfer_oracle.py forward_tokens
``types``)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2407_04991_b200 as P  # noqa: E402
from oracle import tinfer_oracle as O  # noqa: E402

ARGS = (512, 128, 2, 2, 64, 512, 128)


def typed_model():
    m = P.init_random(P.ModelConfig(*ARGS, P.DType.F16, 1, 2), 11)
    return P.init_type_embedding(m, 3, 11)


def test_type_embedding_bit_exact(cuda_device):
    m = typed_model()
    ids, types = [5, 9, 11, 20, 7], [0, 0, 1, 2, 1]
    got = P.embed(m, ids, start_position=3, type_ids=types).array
    want = (m.token_embedding.array[ids].astype(np.float32) + m.position_embedding.array[3:8].astype(np.float32)
            + m.type_embedding.array[types].astype(np.float32))
    assert np.array_equal(got, np.clip(want, -65504, 65504).astype(np.float16))
    with pytest.raises(P.VocabError):
        P.embed(m, ids, type_ids=[0, 0, 3, 0, 0])
    with pytest.raises(P.ParameterError):
        P.embed(P.init_random(P.ModelConfig(*ARGS, P.DType.F16, 1, 2), 11), ids, type_ids=[0] * 5)


def test_typed_generation_matches_oracle(cuda_device):
    m = typed_model()
    oc = O.Config(*ARGS, True, 1, 2)
    w = O.init_weights(oc, 11)
    w["type_embedding"] = m.type_embedding.array.astype(np.float32)
    prompts = [[5, 9, 11, 20, 7], [3, 4], [100, 200, 300, 17]]
    types = [[0, 0, 0, 1, 1], [2, 0], [0, 1, 0, 1]]
    got = P.batched_greedy_decode(m, prompts, 8, type_ids=types, gen_type_id=1)
    rec = []
    want = O.batched_greedy_decode(w, oc, prompts, 8, step_logits=rec, type_ids=types, gen_type=1)
    for b, (g, r) in enumerate(zip(got, want)):
        n = len(prompts[b])
        assert g[:n] == r[:n]
        for s in range(len(r) - n):
            if g[n + s] != r[n + s]:
                top = np.sort(rec[s][b])[-2:]
                assert top[1] - top[0] < 4e-2, (b, s)
                break
    # types change the result (the table is really used), and the typed
    # forward_full logits match the oracle within the north-star tolerance
    assert got != P.batched_greedy_decode(m, prompts, 8)
    lg = P.forward_full(m, prompts[0], type_ids=types[0]).array.astype(np.float32)
    ref = O.forward_tokens(w, oc, np.asarray([prompts[0]]), np.arange(5)[None], O.Cache.new(oc, 1, 5),
                           np.zeros(1, np.int64), all_logits=True, types=np.asarray([types[0]]))[0]
    assert np.max(np.abs(lg - ref)) <= 2e-2
