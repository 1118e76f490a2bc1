"""Text layer on CPU: tokenizer (test_tokenizer.py restated),
the reference's synthetic vocabulary / corpus generators pinned to golden
vectors produced by the unmodified reference (tests/golden/make_golden_text.py),
text-level run_pipeline == run_sequential with a CPU stand-in for the device
generation, the JSON-lines IO, the CLI's host-side commands, and — when the
reference tree is mounted (build container only) — the reference's own
test_tokenizer.py run against the ``tinfer`` name bound to this package."""

import json
import os
import subprocess
import sys
import threading
import time

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2407_04991_b200 as P
from paper_2407_04991_b200 import cli, ladder
from paper_2407_04991_b200 import pipeline as PL
from paper_2407_04991_b200.errors import ConfigError, FormatError, ParameterError, TinferError, VocabError
from paper_2407_04991_b200.tokenizer import UNK_RENDER, Vocab, build, read_vocab, write_vocab

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "text.json"), encoding="utf-8"))
BASE = Vocab(("<unk>", "<eos>", "<pad>", "a", "b", "ab"), 0, 1, 2)


def brute_encode(vocab, text):
    ids, i = [], 0
    index = {t: k for k, t in enumerate(vocab.tokens)}
    while i < len(text):
        for j in range(len(text), i, -1):
            if text[i:j] in index:
                ids.append(index[text[i:j]])
                i = j
                break
        else:
            ids.append(vocab.unk)
            i += 1
    return ids


class TestTokenizer:
    def test_vocab_invariants(self):
        for bad in (dict(tokens=("<unk>", "<eos>", "<pad>", "")),
                    dict(tokens=("<unk>", "<eos>", "<pad>", "x", "x")),
                    dict(tokens=("<unk>", "<eos>", "<pad>"), eos=0),
                    dict(tokens=("<unk>", "<eos>", "<pad>"), pad=7)):
            kw = dict(unk=0, eos=1, pad=2)
            kw.update(bad)
            with pytest.raises(VocabError):
                Vocab(**kw)
        assert BASE.special_ids == {0, 1, 2} and len(BASE) == 6

    def test_encode_rules(self):
        tok = build(BASE)
        assert tok.encode("ab") == [5]
        assert tok.encode("") == []
        assert tok.encode("azb") == [3, 0, 4]
        assert build(Vocab(("<unk>", "<eos>", "<pad>", "a ", "b"), 0, 1, 2)).encode("a b") == [3, 4]
        assert build(Vocab(("<unk>", "<eos>", "<pad>", "日", "日本"), 0, 1, 2)).encode("日本日x") == [4, 3, 0]

    def test_decode_rules(self):
        tok = build(BASE)
        assert tok.decode([]) == "" and tok.decode([0]) == UNK_RENDER
        assert tok.decode(tok.encode("abab")) == "abab"
        with pytest.raises(VocabError):
            tok.decode([6])

    @given(st.lists(st.text(alphabet="abc", min_size=1, max_size=4), min_size=1, max_size=30, unique=True),
           st.text(alphabet="abcd", max_size=40))
    @settings(max_examples=200, deadline=None)
    def test_matches_brute_force(self, extra, text):
        toks = ["<unk>", "<eos>", "<pad>"] + [t for t in extra if t not in ("<unk>", "<eos>", "<pad>")]
        v = Vocab(tuple(toks), 0, 1, 2)
        got = build(v).encode(text)
        assert got == brute_encode(v, text) and len(got) <= len(text)

    def test_tsv_roundtrip_and_errors(self, tmp_path):
        v = Vocab(("<unk>", "<eos>", "<pad>", "a", "b c", "日本"), 0, 1, 2, (0, 0, 0, 12, 5, 99))
        write_vocab(tmp_path / "1.tsv", v)
        again = read_vocab(tmp_path / "1.tsv")
        assert again == v
        write_vocab(tmp_path / "2.tsv", again)
        assert (tmp_path / "1.tsv").read_bytes() == (tmp_path / "2.tsv").read_bytes()
        (tmp_path / "h.tsv").write_text("<unk>\t0\n", encoding="utf-8")
        with pytest.raises(FormatError):
            read_vocab(tmp_path / "h.tsv")
        with pytest.raises(FormatError):
            write_vocab(tmp_path / "t.tsv", Vocab(("<unk>", "<eos>", "<pad>", "a\tb"), 0, 1, 2))
        (tmp_path / "f.tsv").write_text("#unk=0\n#eos=1\n#pad=2\na\tnope\n", encoding="utf-8")
        with pytest.raises(FormatError):
            read_vocab(tmp_path / "f.tsv")


class TestGeneratorsGolden:
    """Byte-identical to the reference's generators (same SplitMix64 streams)."""

    def test_vocab(self):
        assert list(ladder.gen_vocab(128, seed=9).tokens) == GOLD["vocab_128_9"]
        assert list(ladder.gen_vocab(4096, seed=42).tokens[:64]) == GOLD["vocab_4096_42_head"]

    def test_dataset_and_lengths(self):
        v = ladder.gen_vocab(128, seed=9)
        assert ladder.gen_dataset(40, seed=4, mean=12, max_len=30, vocab=v) == GOLD["dataset_40_4_12_30"]
        assert ladder.sample_lengths(2000, P.SplitMix64(123), mean=60, max_len=100) == GOLD["lengths_2000_123"]

    def test_keep_count(self):
        v = ladder.gen_vocab(256, seed=3)
        texts = ladder.gen_dataset(40, seed=5, mean=20, max_len=60, vocab=v)
        counts = P.scan_frequencies(texts, build(v))
        assert ladder.choose_keep_count(counts, 0.99, sorted(v.special_ids)) == GOLD["keep_count_256_3"]

    def test_concatenations_reencode(self):
        v = ladder.gen_vocab(64, seed=2)
        ids = [5, 9, 3, 60, 5]
        assert build(v).encode("".join(v.tokens[i] for i in ids)) == ids

    def test_format_stability(self, tmp_path):
        """Acceptance 10 (test_acceptance.py:245-265): TINF, vocab TSV, JSONL round trips."""
        m = P.init_random(P.ModelConfig(64, 16, 1, 2, 8, 32, 24, P.DType.F32, 1, 2), 7)
        P.write_tinf(str(tmp_path / "w1.tinf"), m.named_tensors())
        P.write_tinf(str(tmp_path / "w2.tinf"), P.read_tinf(str(tmp_path / "w1.tinf")))
        assert (tmp_path / "w1.tinf").read_bytes() == (tmp_path / "w2.tinf").read_bytes()
        v = ladder.gen_vocab(128, seed=9)
        texts = ladder.gen_dataset(40, seed=4, mean=12, max_len=30, vocab=v)
        ladder.write_dataset_jsonl(tmp_path / "d1.jsonl", texts)
        ladder.write_dataset_jsonl(tmp_path / "d2.jsonl", PL.read_jsonl_texts(tmp_path / "d1.jsonl"))
        assert (tmp_path / "d1.jsonl").read_bytes() == (tmp_path / "d2.jsonl").read_bytes()


# ------------------------------------------------------------------ pipeline
def _model(vocab_size=256):
    return P.init_random(P.ModelConfig(vocab_size, 16, 1, 2, 8, 32, 128, P.DType.F16, 1, 2), 3)


def fake_generate(model, prompts, settings):
    """Deterministic, batch-independent CPU stand-in for the device generation."""
    V, eos = model.config.vocab_size, model.config.eos_token
    out = []
    for p in prompts:
        seq = list(p)
        for _ in range(settings.max_new_tokens):
            nxt = (sum(seq[-3:]) * 31 + len(seq)) % V
            seq.append(nxt)
            if nxt == eos:
                break
        out.append(seq)
    return out


@pytest.fixture
def cpu_gen(monkeypatch):
    monkeypatch.setattr(PL, "_generate", fake_generate)
    monkeypatch.setattr(PL, "_devices", lambda s: [None] * (1 if s.devices is None else len(s.devices)))


class TestTextPipeline:
    def setup_method(self):
        self.vocab = ladder.gen_vocab(256, seed=3)
        self.tok = build(self.vocab)
        self.texts = ladder.gen_dataset(37, seed=5, mean=14, max_len=40, vocab=self.vocab)
        self.model = _model()

    @pytest.mark.parametrize("cap,devices", [(1, None), (2, None), (8, ("a", "b", "c"))])
    def test_matches_sequential_in_order(self, cpu_gen, cap, devices):
        s = PL.PipelineSettings(queue_capacity=cap, max_batch_size=4, bucket_width=3, max_new_tokens=5,
                                devices=devices)
        seq, st = PL.run_sequential(self.texts, self.model, self.tok, s)
        pipe, pst = PL.run_pipeline(self.texts, self.model, self.tok, s, watchdog_seconds=60)
        assert [w.output_text for w in pipe] == [w.output_text for w in seq]
        assert [w.sample_index for w in pipe] == list(range(len(self.texts)))
        assert pst.stages["preprocess"].items == len(self.texts) == pst.stages["inference"].items
        assert all("inference" in w.timestamps for w in pipe)

    def test_empty_and_single(self, cpu_gen):
        s = PL.PipelineSettings(max_new_tokens=3)
        assert PL.run_pipeline([], self.model, self.tok, s)[0] == []
        one, _ = PL.run_pipeline(self.texts[:1], self.model, self.tok, s)
        assert one[0].output_text == PL.run_sequential(self.texts[:1], self.model, self.tok, s)[0][0].output_text

    def test_incompatible_tokenizer(self, cpu_gen):
        with pytest.raises(ConfigError):
            PL.run_pipeline(self.texts, _model(128), self.tok, PL.PipelineSettings())
        with pytest.raises(ParameterError):
            PL.run_pipeline(self.texts, self.model, self.tok, PL.PipelineSettings(queue_capacity=0))

    def test_stage_failure_raises_without_deadlock(self, cpu_gen):
        def hook(item):
            if item.sample_index == 5:
                raise ValueError("poisoned")
        s = PL.PipelineSettings(queue_capacity=1, max_batch_size=2, preprocess_hook=hook)
        t0 = time.time()
        with pytest.raises(TinferError) as e:
            PL.run_pipeline(self.texts, self.model, self.tok, s, watchdog_seconds=30)
        assert isinstance(e.value.__cause__, ValueError) and time.time() - t0 < 20
        assert threading.active_count() < 20

    def test_overlap_with_slow_preprocess(self, cpu_gen):
        s = PL.PipelineSettings(max_batch_size=2, preprocess_hook=lambda w: time.sleep(0.002))
        _, st = PL.run_pipeline(self.texts, self.model, self.tok, s)
        assert st.wall_seconds > 0 and st.stages["preprocess"].busy_seconds > 0

    def test_results_jsonl(self, cpu_gen, tmp_path):
        items, _ = PL.run_sequential(self.texts[:5], self.model, self.tok, PL.PipelineSettings(max_new_tokens=2))
        PL.write_results_jsonl(tmp_path / "r.jsonl", items)
        rows = [json.loads(x) for x in (tmp_path / "r.jsonl").read_text(encoding="utf-8").splitlines()]
        assert [sorted(r) for r in rows] == [["content", "sample_index", "summary"]] * 5
        (tmp_path / "bad.jsonl").write_text('{"x": 1}\n', encoding="utf-8")
        with pytest.raises(FormatError):
            PL.read_jsonl_texts(tmp_path / "bad.jsonl")


# ------------------------------------------------------------------ CLI (host commands)
class TestCliHost:
    def test_usage_errors_exit_1(self, capsys):
        with pytest.raises(SystemExit) as e:
            cli.main([])
        assert e.value.code == 1
        assert cli.main(["prune", "--model", "/nonexistent.tinf", "--vocab", "v", "--corpus", "c",
                         "--out-model", "o", "--out-vocab", "ov"]) == 1

    def test_gen_init_prune(self, tmp_path):
        d = str(tmp_path)
        assert cli.main(["gen-vocab", "--size", "256", "--seed", "3", "--out", f"{d}/v.tsv"]) == 0
        assert cli.main(["gen-data", "--vocab", f"{d}/v.tsv", "--n", "30", "--mean", "12", "--max", "30",
                         "--out", f"{d}/d.jsonl"]) == 0
        cfg = P.ModelConfig(256, 16, 1, 2, 8, 32, 128, P.DType.F32, 1, 2)
        (tmp_path / "c.json").write_text(cfg.to_json(), encoding="utf-8")
        assert cli.main(["init-model", "--config", f"{d}/c.json", "--out", f"{d}/m.tinf"]) == 0
        assert cli.main(["prune", "--model", f"{d}/m.tinf", "--vocab", f"{d}/v.tsv", "--corpus", f"{d}/d.jsonl",
                         "--keep-count", "64", "--max-position", "80", "--out-model", f"{d}/p.tinf",
                         "--out-vocab", f"{d}/pv.tsv", "--out-map", f"{d}/map.tsv"]) == 0
        pm = P.load_model(f"{d}/p.tinf")
        pv = read_vocab(f"{d}/pv.tsv")
        assert pm.config.vocab_size == len(pv) == 64 and pm.config.max_position == 80
        from paper_2407_04991_b200.pruning import read_vocab_map
        vmap = read_vocab_map(f"{d}/map.tsv")
        m = P.load_model(f"{d}/m.tinf")
        kept = np.asarray(vmap.kept_old_ids)
        assert np.array_equal(pm.token_embedding.array, m.token_embedding.array[kept])
        assert np.array_equal(pm.lm_head.array, m.lm_head.array[:, kept])


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/tests"), reason="reference tree not mounted")
def test_reference_tokenizer_suite_through_tinfer_name(tmp_path):
    """The reference's own tests/test_tokenizer.py, unmodified, with ``tinfer``
    resolving to pkg/src/tinfer (this package)."""
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "pkg", "src"), ROOT]))
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", str(tmp_path),
                          "/root/reference/pkg/tests/test_tokenizer.py"], env=env, cwd=str(tmp_path),
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
