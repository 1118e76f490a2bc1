"""The per-GPU worker path of the data layer on real CUDA workers: run_sharded
spawns two worker processes on cuda:0 (each builds its own replica and runs the
native generation), and the gathered outputs equal the in-process sequential
run on the same plan (reference pipeline.py:178-209 equivalence)."""

import pytest

pytestmark = pytest.mark.gpu

import paper_2407_04991_b200 as P  # noqa: E402
from paper_2407_04991_b200 import pipeline as PL  # noqa: E402
from oracle import tinfer_oracle as O  # noqa: E402


def test_run_sharded_cuda_workers_match_sequential(cuda_device):
    args = (2048, 256, 2, 4, 64, 1024, 512)
    cfg = P.ModelConfig(*args, P.DType.F16, 1, 2)
    spec = PL.ModelSpec(config_json=cfg.to_json(), seed=5)
    s = O.Stream(O.derive_seed(3, "lengths"))
    lens = (s.randint(40, 90) + 8).tolist()
    reqs = O.synthetic_prompts(2048, 1, sum(lens))[0]
    reqs = [reqs[sum(lens[:i]):sum(lens[:i + 1])] for i in range(len(lens))]
    settings = PL.PipelineSettings(max_batch_size=16, bucket_width=8, max_new_tokens=12)
    got, stats = PL.run_sharded(reqs, spec, settings, devices=["cuda:0", "cuda:0"], timeout=600)
    seq, _ = PL.run_sequential_ids(reqs, spec.build(), settings)
    assert got == seq
    assert len(stats.per_worker_seconds) == 2 and all(t > 0 for t in stats.per_worker_seconds)
    assert stats.generated_tokens == sum(len(g) - len(r) for g, r in zip(got, reqs))
