"""Host-side API behaviour that needs no GPU: configs, init determinism, TINF IO,
pruning selection, argument validation (errors raised before any launch)."""

import json

import numpy as np
import pytest

import paper_2407_04991_b200 as P
from paper_2407_04991_b200 import pruning as PR
from conftest import golden


def small(**kw):
    base = dict(vocab_size=64, hidden_size=32, num_layers=2, num_heads=2, head_dim=16,
                ffn_size=64, max_position=64, dtype=P.DType.F32, eos_token=1, pad_token=2)
    base.update(kw)
    return P.ModelConfig(**base)


@pytest.fixture(scope="module")
def small_model():
    return P.init_random(small(), 7)


def test_config_validation_and_json():
    with pytest.raises(P.ConfigError):
        small(hidden_size=65)
    with pytest.raises(P.ConfigError):
        small(vocab_size=2)
    cfg = P.reference_config()
    assert P.ModelConfig.from_json(cfg.to_json()) == cfg
    doc = json.loads(cfg.to_json())
    assert set(doc) == {"vocab_size", "hidden_size", "num_layers", "num_heads", "head_dim",
                        "ffn_size", "max_position", "dtype", "eos_token", "pad_token"}
    doc["surprise"] = 1
    with pytest.raises(P.FormatError):
        P.ModelConfig.from_json(json.dumps(doc))


def test_init_random_bit_identical_to_reference(small_model):
    import hashlib
    h = hashlib.sha256()
    for _, t in small_model.named_tensors():
        h.update(t.array.tobytes())
    assert h.hexdigest() == str(golden("small.npz")["digest"])
    m16 = P.cast_model(small_model, P.DType.F16)
    h = hashlib.sha256()
    for _, t in m16.named_tensors():
        h.update(t.array.tobytes())
    assert h.hexdigest() == str(golden("small.npz")["digest16"])


def test_save_load_roundtrip(small_model, tmp_path):
    p = tmp_path / "m.tinf"
    P.save_model(small_model, p)
    again = P.load_model(p)
    assert again.config == small_model.config
    for (n0, t0), (n1, t1) in zip(small_model.named_tensors(), again.named_tensors()):
        assert n0 == n1 and np.array_equal(t0.array, t1.array)
    P.write_tinf(str(p), [("zzz", small_model.lm_head)])
    with pytest.raises(P.FormatError):
        P.load_model(p)


def test_validation_precedes_device(small_model):
    # every check fires on the host, before any CUDA call (works without a GPU)
    with pytest.raises(P.VocabError):
        P.embed(small_model, [64])
    with pytest.raises(P.PositionError):
        P.embed(small_model, [0, 0], start_position=63)
    with pytest.raises(P.ParameterError):
        P.greedy_decode(small_model, [], 4)
    with pytest.raises(P.PositionError):
        P.greedy_decode(small_model, [1] * 10, 64)
    with pytest.raises(P.ParameterError):
        P.greedy_decode(small_model, [1], -1)
    assert P.greedy_decode(small_model, [4, 2], 0) == [4, 2]
    assert P.batched_greedy_decode(small_model, [], 4) == []
    with pytest.raises(P.ParameterError):
        P.KVCache(small_model.config, capacity=0)
    with pytest.raises(P.ParameterError):
        P.decode_step(small_model, 3, P.KVCache(small_model.config, batch=2))
    with pytest.raises(P.PositionError):
        P.forward_full(small_model, [3] * 65)


def test_pruning_known_answers(small_model):
    m = PR.build_pruned_vocab([5, 1, 9], keep_count=2)
    assert m.kept_old_ids == (0, 2) and m.old_to_new == {0: 0, 2: 1}
    assert PR.build_pruned_vocab([3, 3], keep_count=1).kept_old_ids == (0,)
    assert set(PR.build_pruned_vocab([9, 0, 0, 8, 7], 3, specials=[1, 2]).kept_old_ids) == {0, 1, 2}
    with pytest.raises(P.ParameterError):
        PR.build_pruned_vocab([1, 2], keep_count=3)
    assert PR.build_pruned_vocab_by_threshold([5, 0, 9, 2], 2, specials=[1]).kept_old_ids == (0, 1, 2, 3)
    g = golden("pruning.npz")
    assert PR.build_pruned_vocab(g["zipf_counts"], 10000, [0, 1, 2]).kept_old_ids == tuple(g["kept_c3"])
    assert PR.build_pruned_vocab_by_threshold(g["zipf_counts"][:200], 10 ** 6, [1]).kept_old_ids == \
        tuple(g["kept_threshold"])
    vm = PR.build_pruned_vocab(np.arange(64)[::-1], keep_count=8, specials=[1, 2])
    pm = PR.prune_token_embedding(small_model, vm)
    assert pm.config.vocab_size == 8
    for new, old in vm.new_to_old.items():
        assert np.array_equal(pm.token_embedding.array[new], small_model.token_embedding.array[old])
        assert np.array_equal(pm.lm_head.array[:, new], small_model.lm_head.array[:, old])
    assert pm.layers[0].wq.array is small_model.layers[0].wq.array
    with pytest.raises(P.DimensionError):
        PR.prune_token_embedding(small_model, PR.PrunedVocabMap((0, 3, 4), 3))
    tr = PR.prune_position_embedding(small_model, 8)
    assert tr.position_embedding.array.tobytes() == small_model.position_embedding.array[:8].tobytes()
    assert PR.prune_position_embedding(small_model, 64) is small_model
    table = vm.remap_table(64)
    assert table[vm.kept_old_ids[3]] == 3 and (table >= -1).all()
    assert (table[[i for i in range(64) if i not in vm.kept_old_ids]] == -1).all()


def test_vocab_map_tsv(tmp_path):
    vm = PR.build_pruned_vocab([4, 0, 8, 1, 9], keep_count=3, specials=[1])
    p = tmp_path / "map.tsv"
    PR.write_vocab_map(p, vm)
    assert PR.read_vocab_map(p).kept_old_ids == vm.kept_old_ids
    p.write_text("3\t0\n7\t2\n", encoding="utf-8")
    with pytest.raises(P.FormatError):
        PR.read_vocab_map(p)


def test_beam_backtrack_vectorised_matches_per_request_walk():
    """beam._backtrack follows every request's parents at once; the result equals
    the per-request walk (first max score -> lowest beam index; cut after the
    first eos) on random histories."""
    from paper_2407_04991_b200.beam import _backtrack

    class C:
        eos_token = 1

    def walk(prompts, scores, th, ph, K):
        out = []
        for r, p in enumerate(prompts):
            k = int(np.argmax(scores[r * K:(r + 1) * K]))
            rev = []
            for t in range(th.shape[0] - 1, -1, -1):
                rev.append(int(th[t, r * K + k]))
                k = int(ph[t, r * K + k])
            gen = []
            for tok in reversed(rev):
                gen.append(tok)
                if tok == C.eos_token:
                    break
            out.append(list(p) + gen)
        return out

    g = np.random.default_rng(0)
    for R, K, T in [(5, 4, 9), (64, 4, 128), (3, 1, 5), (7, 8, 1)]:
        scores = g.standard_normal(R * K).astype(np.float32)
        scores[:K] = 0.5  # tie inside request 0
        th = g.integers(0, 6, (T, R * K)).astype(np.int32)
        ph = g.integers(0, K, (T, R * K)).astype(np.int32)
        prompts = [[9] * int(x) for x in g.integers(1, 4, R)]
        assert _backtrack(C, prompts, scores, th, ph, K) == walk(prompts, scores, th, ph, K)
