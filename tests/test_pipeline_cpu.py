"""Data layer on CPU: the reference planner's known answers, LPT assignment,
the torchrun-mode sharding over a world_size-2 gloo group, and the
process-per-device runner (with a CPU stand-in generator; on the GPU box the
workers run batched_greedy_decode)."""

import os
import tempfile

import numpy as np
import pytest
import torch.multiprocessing as tmp

import paper_2407_04991_b200 as P
from paper_2407_04991_b200 import pipeline as PL
from conftest import golden
from oracle import tinfer_oracle as O

TINY = dict(vocab_size=48, hidden_size=16, num_layers=1, num_heads=2, head_dim=8, ffn_size=32,
            max_position=64, dtype=P.DType.F32, eos_token=1, pad_token=2)


def cpu_runner(model, prompts, settings):
    """Test stand-in for the GPU generator: the oracle on the worker's replica."""
    c = model.config
    oc = O.Config(c.vocab_size, c.hidden_size, c.num_layers, c.num_heads, c.head_dim, c.ffn_size,
                  c.max_position, c.dtype is P.DType.F16, c.eos_token, c.pad_token)
    w = {n: t.array.astype(np.float32) for n, t in model.named_tensors()}
    return O.batched_greedy_decode(w, oc, prompts, settings.max_new_tokens)


def requests(n=40, seed=3):
    s = O.Stream(O.derive_seed(seed, "req"))
    lens = (s.randint(n, 20) + 1).tolist()
    toks = (s.randint(sum(lens), 45) + 3).tolist()
    out, k = [], 0
    for L in lens:
        out.append(toks[k:k + L])
        k += L
    return out


def test_plan_batches_matches_reference_golden():
    g = golden("pruning.npz")
    plan = PL.plan_batches(g["plan_lengths"].tolist(), 32, 16)
    assert [i for gr in plan.groups for i in gr] == g["plan_groups"].tolist()
    assert [len(gr) for gr in plan.groups] == g["plan_sizes"].tolist()
    assert plan.group_pad == g["plan_pads"].tolist()
    assert PL.plan_batches([3, 5, 1, 7, 7, 2], 2, 1).groups == [[3, 4], [1], [0, 5], [2]]
    with pytest.raises(P.ParameterError):
        PL.plan_batches([1], 0, 1)


def test_assign_groups_covers_and_balances():
    lens = [int(x) for x in np.random.default_rng(0).integers(32, 513, 500)]
    plan = PL.plan_batches(lens, 32, 16)
    for w in (1, 2, 4, 8):
        a = PL.assign_groups(plan, w, 64)
        flat = sorted(g for part in a for g in part)
        assert flat == list(range(len(plan.groups)))
        loads = [sum(PL.group_cost(plan, g, 64) for g in part) for part in a]
        assert max(loads) - min(loads) <= max(PL.group_cost(plan, g, 64) for g in range(len(plan.groups)))
        assert a == PL.assign_groups(plan, w, 64)  # deterministic


def _gloo_rank(rank, world, port, out_path):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    model = P.init_random(P.ModelConfig(**TINY), 5)
    reqs = requests()
    settings = PL.PipelineSettings(max_batch_size=8, bucket_width=4, max_new_tokens=6)
    plan = PL.plan_batches([len(r) for r in reqs], settings.max_batch_size, settings.bucket_width)
    local = {}
    for gi in PL.rank_share(plan, world, rank, settings.max_new_tokens):
        g = plan.groups[gi]
        for i, s in zip(g, cpu_runner(model, [reqs[i] for i in g], settings)):
            local[i] = s
    t = PL.max_over_ranks(float(rank + 1))
    merged = PL.gather_outputs(local, len(reqs), world)
    if rank == 0:
        seq, _ = PL.run_sequential_ids(reqs, model, settings, runner=cpu_runner)
        with open(out_path, "w") as fh:
            fh.write(f"{int(merged == seq)} {t}")
    dist.barrier()
    dist.destroy_process_group()


def test_torchrun_mode_sharding_gloo_world2():
    port = 29500 + os.getpid() % 1000
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "r.txt")
        tmp.spawn(_gloo_rank, args=(2, port, out), nprocs=2, join=True)
        ok, t = open(out).read().split()
    assert ok == "1"  # gathered shards == sequential run, in request order
    assert float(t) == 2.0  # max over ranks


def test_run_sharded_two_workers_matches_sequential():
    cfg = P.ModelConfig(**TINY)
    spec = PL.ModelSpec(config_json=cfg.to_json(), seed=5)
    reqs = requests(30)
    settings = PL.PipelineSettings(max_batch_size=8, bucket_width=4, max_new_tokens=5)
    got, stats = PL.run_sharded(reqs, spec, settings, devices=["cpu", "cpu"], runner=cpu_runner,
                                timeout=300)
    seq, _ = PL.run_sequential_ids(reqs, spec.build(), settings, runner=cpu_runner)
    assert got == seq
    assert stats.generated_tokens == 30 * 5 - sum(  # eos may cut rows short
        5 - (len(s) - len(r)) for s, r in zip(seq, reqs))
    assert len(stats.per_worker_seconds) == 2


def _failing_runner(model, prompts, settings):
    raise RuntimeError("injected fault")


def test_run_sharded_worker_failure_names_device():
    cfg = P.ModelConfig(**TINY)
    spec = PL.ModelSpec(config_json=cfg.to_json(), seed=5)
    with pytest.raises(P.TinferError, match="cpu"):
        PL.run_sharded(requests(6), spec, PL.PipelineSettings(max_new_tokens=2), devices=["cpu"],
                       runner=_failing_runner, timeout=120)


def test_bench_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks
    (never silently one): the dry run rendezvouses over gloo and rank 0
    reports both ranks; a WORLD_SIZE that disagrees with --gpus is an error."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["ranks_joined"] == 2
    bad = dict(env, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"], cwd=root, env=bad,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode != 0
