"""Text layer, ablation ladder and CLI on the GPU.

* run_pipeline (tokenizer thread -> length-bucketed dynamic batches -> one
  inference worker per device -> detokenizer) equals run_sequential on the
  native path, with one and with two inference workers (two on cuda:0 here;
  the box has one GPU) — reference pipeline.py:178-394 equivalence.
* run_ablation times all four stages on the GPU only after its gates passed;
  every injected fault raises CorrectnessError and no report is produced
  (reference bench.py:376-467, test_bench.py:128-177).
* the CLI's bench exits 2 on an injected fault without printing speed figures,
  and `run` writes one JSON line per sample (acceptance 9, test_cli.py:86-133).
"""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2407_04991_b200 as P  # noqa: E402
from paper_2407_04991_b200 import cli, ladder  # noqa: E402
from paper_2407_04991_b200 import pipeline as PL  # noqa: E402
from paper_2407_04991_b200.errors import CorrectnessError  # noqa: E402
from paper_2407_04991_b200.tokenizer import build  # noqa: E402


def small_cfg(vocab=256, positions=128, dtype=P.DType.F32):
    return P.ModelConfig(vocab, 64, 2, 2, 32, 128, positions, dtype, 1, 2)


@pytest.fixture(scope="module")
def setup():
    model = P.init_random(small_cfg(), seed=11)
    vocab = ladder.gen_vocab(256, seed=3)
    texts = ladder.gen_dataset(40, seed=5, mean=20, max_len=60, vocab=vocab)
    return model, vocab, texts


def quick(**kw):
    base = dict(max_new_tokens=6, max_batch_size=4, repeats=2, warmup_samples=4, oracle_samples=2)
    base.update(kw)
    return ladder.BenchOptions(**base)


@pytest.mark.parametrize("devices", [None, ("cuda:0", "cuda:0")])
def test_pipeline_equals_sequential_on_device(cuda_device, setup, devices):
    model, vocab, texts = setup
    m16 = P.cast_model(model, P.DType.F16)
    tok = build(vocab)
    s = PL.PipelineSettings(queue_capacity=2, max_batch_size=8, bucket_width=4, max_new_tokens=8, devices=devices)
    seq, _ = PL.run_sequential(texts, m16, tok, s)
    pipe, st = PL.run_pipeline(texts, m16, tok, s, watchdog_seconds=300)
    assert [w.output_text for w in pipe] == [w.output_text for w in seq]
    assert [w.generated_ids for w in pipe] == [w.generated_ids for w in seq]
    assert st.stages["inference"].items == len(texts)
    # every sample's generation equals its stand-alone decode (batch invariance)
    for w in seq[:6]:
        alone = P.greedy_decode(m16, w.token_ids, 8)
        assert alone[len(w.token_ids):] == w.generated_ids


def test_full_ladder_reports(cuda_device, setup):
    model, vocab, texts = setup
    reports = ladder.run_ablation(model, vocab, texts, ladder.LADDER, quick())
    assert [r.stage_name for r in reports] == list(ladder.LADDER)
    assert reports[0].speedup_vs_baseline == 1.0
    for r in reports:
        assert r.wall_seconds > 0 and r.samples_per_sec > 0 and r.tokens_per_sec > 0
        assert r.config_fingerprint == reports[0].config_fingerprint
    sps = {r.stage_name: r.samples_per_sec for r in reports}
    assert sps["fast_transformer"] > sps["baseline"]  # KV cache beats recompute on the device too
    again = ladder.reports_from_json(ladder.emit_report(reports, "json"))
    assert [r.stage_name for r in again] == list(ladder.LADDER)


@pytest.mark.parametrize("fault", ["cache", "fusion", "pruning", "pipeline"])
def test_injected_faults_abort(cuda_device, setup, fault):
    model, vocab, texts = setup
    with pytest.raises(CorrectnessError):
        ladder.run_ablation(model, vocab, texts, ladder.LADDER, quick(inject_fault=fault))


def test_pruned_stage_restricted_logits_exact(cuda_device, setup):
    """Row/column selection is exact on the device: the pruned model's logits over
    kept ids equal the original's bitwise (reference test_pruning.py:217-226)."""
    model, vocab, texts = setup
    m16 = P.cast_model(model, P.DType.F16)
    pruned, ptok, vmap, _ = ladder.build_pruned_stage(m16, vocab, texts, quick())
    kept = np.asarray(vmap.kept_old_ids)
    ids = [i for i in build(vocab).encode(texts[0]) if i in vmap.old_to_new][:40]
    want = P.forward_full(m16, ids).array[:, kept]
    got = P.forward_full(pruned, vmap.remap(ids)).array
    assert np.array_equal(want, got)


def test_cli_bench_and_run(cuda_device, tmp_path, capsys):
    d = str(tmp_path)
    P.save_model(P.init_random(small_cfg(positions=128), seed=11), f"{d}/m.tinf")
    assert cli.main(["gen-vocab", "--size", "256", "--seed", "3", "--out", f"{d}/v.tsv"]) == 0
    assert cli.main(["gen-data", "--vocab", f"{d}/v.tsv", "--n", "16", "--mean", "12", "--max", "40",
                     "--out", f"{d}/d.jsonl"]) == 0
    capsys.readouterr()
    rc = cli.main(["bench", "--model", f"{d}/m.tinf", "--vocab", f"{d}/v.tsv", "--data", f"{d}/d.jsonl",
                   "--max-new", "4", "--repeats", "1", "--inject-fault", "cache"])
    out = capsys.readouterr().out
    assert rc == 2 and "samples/s" not in out and "speedup" not in out
    rc = cli.main(["bench", "--model", f"{d}/m.tinf", "--vocab", f"{d}/v.tsv", "--data", f"{d}/d.jsonl",
                   "--max-new", "4", "--repeats", "1", "--format", "json", "--out", f"{d}/r.json"])
    assert rc == 0
    doc = json.loads((tmp_path / "r.json").read_text())
    assert [r["stage_name"] for r in doc["reports"]] == list(ladder.LADDER)
    for stage in ("baseline", "pipeline"):
        assert cli.main(["run", "--model", f"{d}/m.tinf", "--vocab", f"{d}/v.tsv", "--data", f"{d}/d.jsonl",
                         "--stage", stage, "--max-new", "4", "--out", f"{d}/{stage}.jsonl"]) == 0
        rows = [json.loads(x) for x in (tmp_path / f"{stage}.jsonl").read_text().splitlines()]
        assert [r["sample_index"] for r in rows] == list(range(16))
