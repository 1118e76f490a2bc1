"""Data layer (paper §3.3): length-bucketed batching and per-GPU worker processes.

Replaces the reference's 4-stage threaded pipeline (pipeline.py:265-394), whose
inference stage is one thread calling ``batched_greedy_decode`` per group
(pipeline.py:152-166), with:

* :func:`plan_batches` — the reference's planner verbatim in behaviour
  (pipeline.py:60-87): stable descending-length sort, a group closes at
  ``max_batch_size`` or when the gap to the group head exceeds ``bucket_width``.
* :func:`assign_groups` — deterministic longest-processing-time assignment of the
  groups to G devices by cost ~ batch x (padded prompt + new tokens).
* :func:`run_sharded` — one spawned worker process per GPU, each holding a full
  model replica (built locally from a :class:`ModelSpec`, so no weights cross
  process boundaries), pulling its groups and returning (sample_index, ids) to
  the host. No collective on the data path: requests are independent.
* :func:`run_sequential` — the same groups on one device in-process (the
  equivalence oracle for the sharded run, like reference pipeline.py:178-209).

Results come back in original request order regardless of grouping: padding is
masked out of attention, so each request's tokens do not depend on its batch
(batched == single, tested bitwise).

Text pre/post-processing (tokenizer) is out of scope; requests are
token-id lists.
"""

from __future__ import annotations

import os
import time
import traceback
from dataclasses import dataclass, field
from typing import Callable, Sequence

from .errors import ParameterError, TinferError


@dataclass
class BatchPlan:
    groups: list[list[int]]
    max_batch_size: int
    bucket_width: int
    group_pad: list[int]

    def __post_init__(self):
        if len(self.groups) != len(self.group_pad):
            raise ParameterError("groups and group_pad must align")
        for g in self.groups:
            if not g:
                raise ParameterError("empty batch group")
            if len(g) > self.max_batch_size:
                raise ParameterError("group exceeds max_batch_size")


def plan_batches(lengths: Sequence[int], max_batch_size: int, bucket_width: int) -> BatchPlan:
    """Length-sorted greedy grouping (reference pipeline.py:60-87)."""
    if max_batch_size < 1:
        raise ParameterError("max_batch_size must be >= 1")
    if bucket_width < 0:
        raise ParameterError("bucket_width must be >= 0")
    order = sorted(range(len(lengths)), key=lambda i: -lengths[i])  # stable
    groups: list[list[int]] = []
    pads: list[int] = []
    for idx in order:
        if groups and len(groups[-1]) < max_batch_size and pads[-1] - lengths[idx] <= bucket_width:
            groups[-1].append(idx)
        else:
            groups.append([idx])
            pads.append(lengths[idx])
    return BatchPlan(groups=groups, max_batch_size=max_batch_size, bucket_width=bucket_width,
                     group_pad=pads)


def padding_waste(plan: BatchPlan, lengths: Sequence[int]) -> int:
    return sum(plan.group_pad[gi] - lengths[i] for gi, g in enumerate(plan.groups) for i in g)


def group_cost(plan: BatchPlan, gi: int, max_new: int) -> int:
    return len(plan.groups[gi]) * (plan.group_pad[gi] + max_new)


def assign_groups(plan: BatchPlan, n_workers: int, max_new: int) -> list[list[int]]:
    """LPT: groups by descending cost, each to the least-loaded worker (ties to
    the lower worker id). Deterministic; every group assigned exactly once."""
    if n_workers < 1:
        raise ParameterError("n_workers must be >= 1")
    order = sorted(range(len(plan.groups)), key=lambda gi: (-group_cost(plan, gi, max_new), gi))
    load = [0] * n_workers
    out: list[list[int]] = [[] for _ in range(n_workers)]
    for gi in order:
        w = min(range(n_workers), key=lambda j: (load[j], j))
        out[w].append(gi)
        load[w] += group_cost(plan, gi, max_new)
    return out


@dataclass
class PipelineSettings:
    max_batch_size: int = 128
    bucket_width: int = 16
    max_new_tokens: int = 64
    beam_width: int = 1

    def validate(self) -> None:
        if self.max_batch_size < 1:
            raise ParameterError("max_batch_size must be >= 1")
        if self.bucket_width < 0:
            raise ParameterError("bucket_width must be >= 0")
        if self.max_new_tokens < 0:
            raise ParameterError("max_new_tokens must be >= 0")
        if not 1 <= self.beam_width <= 8:
            raise ParameterError("beam_width must be in [1, 8]")


@dataclass
class ModelSpec:
    """How a worker builds its replica: a TINF path, or config + seed with the
    optional pruning transforms (all deterministic, bit-identical per worker)."""
    config_json: str | None = None
    seed: int = 42
    tinf_path: str | None = None
    keep_count: int | None = None
    keep_ids: tuple[int, ...] | None = None
    max_position: int | None = None

    def build(self):
        from . import model as M
        from . import pruning as PR
        if self.tinf_path:
            m = M.load_model(self.tinf_path)
        else:
            m = M.init_random(M.ModelConfig.from_json(self.config_json), self.seed)
        if self.keep_ids is not None:
            m = PR.prune_token_embedding(m, PR.PrunedVocabMap(tuple(self.keep_ids), len(self.keep_ids)))
        if self.max_position is not None:
            m = PR.prune_position_embedding(m, self.max_position)
        return m


@dataclass
class RunStats:
    wall_seconds: float = 0.0
    per_worker_seconds: list[float] = field(default_factory=list)
    generated_tokens: int = 0
    latencies: list[float] = field(default_factory=list)  # per request: enqueue -> ids back


def _generate(model, prompts, settings: PipelineSettings):
    from .beam import beam_search_decode
    from .model import batched_greedy_decode
    if settings.beam_width > 1:
        return beam_search_decode(model, prompts, settings.max_new_tokens, settings.beam_width)
    return batched_greedy_decode(model, prompts, settings.max_new_tokens)


def run_sequential(requests: Sequence[Sequence[int]], model, settings: PipelineSettings,
                   runner: Callable | None = None):
    """All groups on the current device in plan order; returns (outputs, stats)."""
    settings.validate()
    run = runner or _generate
    t0 = time.perf_counter()
    plan = plan_batches([len(r) for r in requests], settings.max_batch_size, settings.bucket_width)
    out: list[list[int] | None] = [None] * len(requests)
    stats = RunStats()
    for g in plan.groups:
        seqs = run(model, [list(requests[i]) for i in g], settings)
        done = time.perf_counter()
        for i, s in zip(g, seqs):
            out[i] = s
            stats.generated_tokens += len(s) - len(requests[i])
            stats.latencies.append(done - t0)
    stats.wall_seconds = time.perf_counter() - t0
    return out, stats


def _worker_main(rank: int, device: str, spec: ModelSpec, settings: PipelineSettings,
                 task_q, result_q, runner):
    try:
        if device.startswith("cuda"):
            import torch
            torch.cuda.set_device(torch.device(device))
        model = spec.build()
        run = runner or _generate
        busy = 0.0
        while True:
            task = task_q.get()
            if task is None:
                break
            gi, idx, prompts = task
            t0 = time.perf_counter()
            seqs = run(model, prompts, settings)
            busy += time.perf_counter() - t0
            result_q.put(("ok", rank, gi, idx, seqs, time.perf_counter()))
        result_q.put(("done", rank, busy))
    except BaseException:  # report, never hang the host
        result_q.put(("error", rank, traceback.format_exc()))


def run_sharded(requests: Sequence[Sequence[int]], spec: ModelSpec, settings: PipelineSettings,
                devices: Sequence[str] | None = None, runner: Callable | None = None,
                timeout: float = 3600.0):
    """Generate for every request on G worker processes (one per device).

    Groups are pre-assigned by LPT (`assign_groups`) and queued per worker, so
    the assignment is deterministic; outputs are returned in request order. A
    worker failure raises TinferError naming the worker's device."""
    import multiprocessing as mp

    settings.validate()
    if devices is None:
        import torch
        devices = [f"cuda:{i}" for i in range(torch.cuda.device_count())]
    if not devices:
        raise TinferError("no devices for run_sharded")
    t0 = time.perf_counter()
    plan = plan_batches([len(r) for r in requests], settings.max_batch_size, settings.bucket_width)
    assign = assign_groups(plan, len(devices), settings.max_new_tokens)
    ctx = mp.get_context("spawn")
    result_q = ctx.Queue()
    queues, procs = [], []
    for rank, dev in enumerate(devices):
        q = ctx.Queue()
        for gi in assign[rank]:
            g = plan.groups[gi]
            q.put((gi, g, [list(requests[i]) for i in g]))
        q.put(None)
        p = ctx.Process(target=_worker_main, args=(rank, dev, spec, settings, q, result_q, runner),
                        daemon=True)
        p.start()
        queues.append(q)
        procs.append(p)
    out: list[list[int] | None] = [None] * len(requests)
    stats = RunStats(per_worker_seconds=[0.0] * len(devices))
    finished = 0
    deadline = time.time() + timeout
    try:
        while finished < len(devices):
            remaining = deadline - time.time()
            if remaining <= 0:
                raise TinferError("run_sharded timed out")
            try:
                msg = result_q.get(timeout=min(remaining, 5.0))
            except Exception:
                dead = [devices[i] for i, p in enumerate(procs) if not p.is_alive() and p.exitcode]
                if dead:
                    raise TinferError(f"worker on {dead[0]} died")
                continue
            if msg[0] == "ok":
                _, rank, gi, idx, seqs, when = msg
                for i, s in zip(idx, seqs):
                    out[i] = s
                    stats.generated_tokens += len(s) - len(requests[i])
                    stats.latencies.append(when - t0)
            elif msg[0] == "done":
                stats.per_worker_seconds[msg[1]] = msg[2]
                finished += 1
            else:
                raise TinferError(f"worker on {devices[msg[1]]} failed:\n{msg[2]}")
    finally:
        for p in procs:
            p.join(timeout=10.0)
            if p.is_alive():
                p.terminate()
    stats.wall_seconds = time.perf_counter() - t0
    return out, stats


# ---------------------------------------------------------------------------
# torchrun mode (bench.py): each rank takes its LPT share, rank 0 gathers
# ---------------------------------------------------------------------------
def rank_share(plan: BatchPlan, world: int, rank: int, max_new: int) -> list[int]:
    return assign_groups(plan, world, max_new)[rank]


def gather_outputs(local: dict[int, list[int]], n: int, world: int):
    """Gather {request index: ids} from every rank onto rank 0 (gloo or nccl
    process group). Returns the ordered list on rank 0, None elsewhere."""
    import torch.distributed as dist
    if world == 1:
        return [local[i] for i in range(n)]
    parts = [None] * world if dist.get_rank() == 0 else None
    dist.gather_object(local, parts, dst=0)
    if dist.get_rank() != 0:
        return None
    merged: dict[int, list[int]] = {}
    for p in parts:
        merged.update(p)
    return [merged[i] for i in range(n)]


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def worker_env() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))
