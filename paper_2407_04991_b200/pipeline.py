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
* :func:`run_sequential_ids` — the same groups on one device in-process (the
  equivalence oracle for the sharded run, like reference pipeline.py:178-209).

Results come back in original request order regardless of grouping: padding is
masked out of attention, so each request's tokens do not depend on its batch
(batched == single, tested bitwise).

Text level (reference API, pipeline.py:30-425): :class:`WorkItem`,
:func:`run_sequential` / :func:`run_pipeline` over strings with a
:class:`~.tokenizer.Tokenizer` — tokenise, length-bucketed dynamic batching,
GPU generation (one inference worker thread per device in ``settings.devices``;
the native calls release the GIL), detokenise — and the JSON-lines IO
(:func:`read_jsonl_texts`, :func:`write_results_jsonl`). Outputs of the two are
equal (group membership only changes padding, which is masked out).
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
    """Reference fields and defaults (pipeline.py:90-110) plus two extensions:
    ``beam_width`` (beam search, 1 = greedy) and ``devices`` (the CUDA devices
    that run inference: one inference worker per device; None = the current
    device)."""
    queue_capacity: int = 8
    max_batch_size: int = 8
    bucket_width: int = 16
    max_new_tokens: int = 32
    fused: bool = True
    use_cache: bool = True  # False: full-recompute decode (ladder baseline)
    preprocess_hook: Callable | None = None
    beam_width: int = 1
    devices: tuple | None = None

    def validate(self) -> None:
        if self.queue_capacity < 1:
            raise ParameterError("queue_capacity must be >= 1")
        if self.max_batch_size < 1:
            raise ParameterError("max_batch_size must be >= 1")
        if self.bucket_width < 0:
            raise ParameterError("bucket_width must be >= 0")
        if self.max_new_tokens < 0:
            raise ParameterError("max_new_tokens must be >= 0")
        if not 1 <= self.beam_width <= 8:
            raise ParameterError("beam_width must be in [1, 8]")
        if self.devices is not None and len(self.devices) == 0:
            raise ParameterError("devices must name at least one device")


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
    from .model import batched_greedy_decode, greedy_decode
    if settings.beam_width > 1:
        return beam_search_decode(model, prompts, settings.max_new_tokens, settings.beam_width)
    if not settings.use_cache:
        return [greedy_decode(model, p, settings.max_new_tokens, use_cache=False, fused=settings.fused)
                for p in prompts]
    return batched_greedy_decode(model, prompts, settings.max_new_tokens, fused=settings.fused)


def run_sequential_ids(requests: Sequence[Sequence[int]], model, settings: PipelineSettings,
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


# ---------------------------------------------------------------------------
# text level: the reference's pipeline API (pipeline.py:30-425) over GPU workers
# ---------------------------------------------------------------------------
@dataclass
class WorkItem:
    sample_index: int
    text: str
    token_ids: list[int] | None = None
    generated_ids: list[int] | None = None
    output_text: str | None = None
    timestamps: dict[str, tuple[float, float]] = field(default_factory=dict)


@dataclass
class StageTiming:
    busy_seconds: float = 0.0
    queue_wait_seconds: float = 0.0
    items: int = 0


@dataclass
class StageStats:
    stages: dict[str, StageTiming]
    wall_seconds: float


STAGE_NAMES = ("preprocess", "inference", "postprocess")


def _check_compatible(model, tokenizer) -> None:
    """Same contract as pipeline.py:123-131: the tokenizer's vocabulary is the
    model's (size and eos/pad ids)."""
    from .errors import ConfigError
    c = model.config
    if len(tokenizer.vocab) != c.vocab_size:
        raise ConfigError(f"tokenizer vocab size {len(tokenizer.vocab)} != model vocab size {c.vocab_size}")
    if tokenizer.vocab.eos != c.eos_token or tokenizer.vocab.pad != c.pad_token:
        raise ConfigError("tokenizer specials do not match the model config")


def _tokenize(item: WorkItem, tokenizer, settings: PipelineSettings) -> None:
    t0 = time.perf_counter()
    if settings.preprocess_hook is not None:
        settings.preprocess_hook(item)
    item.token_ids = tokenizer.encode(item.text)
    item.timestamps["preprocess"] = (t0, time.perf_counter())


def _generate_group(group: list[WorkItem], model, settings: PipelineSettings) -> None:
    t0 = time.perf_counter()
    seqs = _generate(model, [w.token_ids for w in group], settings)
    t1 = time.perf_counter()
    for w, seq in zip(group, seqs):
        w.generated_ids = list(seq[len(w.token_ids):])
        w.timestamps["inference"] = (t0, t1)


def _detokenize(item: WorkItem, tokenizer) -> None:
    t0 = time.perf_counter()
    gen = list(item.generated_ids)
    if gen and gen[-1] == tokenizer.vocab.eos:  # the eos that ended generation is not text
        gen = gen[:-1]
    item.output_text = tokenizer.decode(gen)
    item.timestamps["postprocess"] = (t0, time.perf_counter())


def _devices(settings: PipelineSettings) -> list:
    import torch
    if settings.devices is None:
        return [torch.device("cuda", torch.cuda.current_device())] if torch.cuda.is_available() else [None]
    return [torch.device(d) for d in settings.devices]


def run_sequential(items: Sequence[str], model, tokenizer, settings: PipelineSettings):
    """Tokenise everything, plan the groups, generate group by group on one
    device, detokenise (pipeline.py:178-209); the equivalence oracle of
    :func:`run_pipeline`. Returns (work items in input order, StageStats)."""
    settings.validate()
    _check_compatible(model, tokenizer)
    wall0 = time.perf_counter()
    work = [WorkItem(sample_index=i, text=t) for i, t in enumerate(items)]
    timing = {n: StageTiming() for n in STAGE_NAMES}
    dev = _devices(settings)[0]

    def timed(name, n, fn):
        t0 = time.perf_counter()
        fn()
        timing[name].busy_seconds = time.perf_counter() - t0
        timing[name].items = n

    def pre():
        for w in work:
            _tokenize(w, tokenizer, settings)

    def infer():
        plan = plan_batches([len(w.token_ids) for w in work], settings.max_batch_size, settings.bucket_width)
        with _on_device(dev):
            for g in plan.groups:
                _generate_group([work[i] for i in g], model, settings)

    timed("preprocess", len(work), pre)
    timed("inference", len(work), infer)
    timed("postprocess", len(work), lambda: [_detokenize(w, tokenizer) for w in work])
    return work, StageStats(stages=timing, wall_seconds=time.perf_counter() - wall0)


class _on_device:
    """CUDA current device for this host thread (None: leave as is)."""

    def __init__(self, dev):
        self.dev = dev

    def __enter__(self):
        if self.dev is not None and self.dev.type == "cuda":
            import torch
            torch.cuda.set_device(self.dev)

    def __exit__(self, *exc):
        return False


class _own_stream:
    """A private CUDA stream for this worker thread (workers sharing a GPU then
    overlap: each runs its own sessions and graphs on its own stream)."""

    def __init__(self, dev):
        self.dev, self.ctx = dev, None

    def __enter__(self):
        if self.dev is not None and self.dev.type == "cuda":
            import torch
            self.ctx = torch.cuda.stream(torch.cuda.Stream(self.dev))
            self.ctx.__enter__()

    def __exit__(self, *exc):
        if self.ctx is not None:
            self.ctx.__exit__(*exc)
        return False


class _Stop:
    """First failure wins; every loop polls it (and the optional deadline), so
    no stage can block forever on a queue."""

    def __init__(self, deadline: float | None):
        import threading
        self.event = threading.Event()
        self.lock = threading.Lock()
        self.error: BaseException | None = None
        self.stage: str | None = None
        self.deadline = deadline

    def fail(self, stage: str, exc: BaseException) -> None:
        with self.lock:
            if self.error is None:
                self.error, self.stage = exc, stage
        self.event.set()

    def stopped(self) -> bool:
        if not self.event.is_set() and self.deadline is not None and time.perf_counter() > self.deadline:
            self.fail("watchdog", TinferError("pipeline watchdog expired"))
        return self.event.is_set()


_END = object()


def _put(q, obj, stop: _Stop, tm: StageTiming | None) -> bool:
    import queue as _q
    t0 = time.perf_counter()
    while not stop.stopped():
        try:
            q.put(obj, timeout=0.05)
        except _q.Full:
            continue
        if tm is not None:
            tm.queue_wait_seconds += time.perf_counter() - t0
        return True
    return False


def _get(q, stop: _Stop, tm: StageTiming | None):
    import queue as _q
    t0 = time.perf_counter()
    while not stop.stopped():
        try:
            obj = q.get(timeout=0.05)
        except _q.Empty:
            continue
        if tm is not None:
            tm.queue_wait_seconds += time.perf_counter() - t0
        return obj
    return _END


def run_pipeline(items: Sequence[str], model, tokenizer, settings: PipelineSettings,
                 watchdog_seconds: float | None = None):
    """Concurrent stages over bounded queues (pipeline.py:265-394): a tokenizer
    thread with dynamic batching (per-length-bin groups flushed as soon as they
    hold ``max_batch_size`` items; leftovers planned with :func:`plan_batches`),
    one inference thread per CUDA device of ``settings.devices`` pulling groups
    from a shared queue (each device holds its own weight replica; the native
    generation releases the GIL), and a detokenizer thread. Results come back in
    input order and equal :func:`run_sequential`'s. Any stage failure stops
    every stage and is re-raised as ``TinferError`` (cause attached); an expired
    watchdog does the same."""
    import queue
    import threading

    settings.validate()
    _check_compatible(model, tokenizer)
    wall0 = time.perf_counter()
    n = len(items)
    devs = _devices(settings)
    q_tok = queue.Queue(settings.queue_capacity)
    q_grp = queue.Queue(settings.queue_capacity)
    q_det = queue.Queue(settings.queue_capacity)
    q_out = queue.Queue()
    stop = _Stop(None if watchdog_seconds is None else wall0 + watchdog_seconds)
    timing = {name: StageTiming() for name in STAGE_NAMES}
    tlock = threading.Lock()
    span = settings.bucket_width + 1

    def tokenizer_stage():
        tm, bins = timing["preprocess"], {}
        try:
            while True:
                w = _get(q_tok, stop, tm)
                if w is _END:
                    break
                t0 = time.perf_counter()
                _tokenize(w, tokenizer, settings)
                tm.busy_seconds += time.perf_counter() - t0
                tm.items += 1
                key = len(w.token_ids) // span
                b = bins.setdefault(key, [])
                b.append(w)
                if len(b) == settings.max_batch_size:
                    del bins[key]
                    if not _put(q_grp, b, stop, tm):
                        return
            rest = [w for b in bins.values() for w in b]
            if rest:
                plan = plan_batches([len(w.token_ids) for w in rest], settings.max_batch_size,
                                    settings.bucket_width)
                for g in plan.groups:
                    if not _put(q_grp, [rest[i] for i in g], stop, tm):
                        return
            for _ in devs:  # one end marker per inference worker
                _put(q_grp, _END, stop, None)
        except BaseException as exc:
            stop.fail("preprocess", exc)

    live = [len(devs)]

    def inference_stage(dev):
        tm = timing["inference"]
        try:
            with _on_device(dev), _own_stream(dev):
                while True:
                    g = _get(q_grp, stop, None)
                    if g is _END:
                        break
                    t0 = time.perf_counter()
                    _generate_group(g, model, settings)
                    with tlock:
                        tm.busy_seconds += time.perf_counter() - t0
                        tm.items += len(g)
                    if not _put(q_det, g, stop, None):
                        return
            with tlock:
                live[0] -= 1
                last = live[0] == 0
            if last:
                _put(q_det, _END, stop, None)
        except BaseException as exc:
            stop.fail("inference", exc)

    def detokenizer_stage():
        tm = timing["postprocess"]
        try:
            while True:
                g = _get(q_det, stop, tm)
                if g is _END:
                    break
                t0 = time.perf_counter()
                for w in g:
                    _detokenize(w, tokenizer)
                tm.busy_seconds += time.perf_counter() - t0
                tm.items += len(g)
                for w in g:
                    q_out.put(w)
        except BaseException as exc:
            stop.fail("postprocess", exc)

    threads = [threading.Thread(target=tokenizer_stage, name="preprocess", daemon=True),
               *[threading.Thread(target=inference_stage, args=(d,), name=f"inference{i}", daemon=True)
                 for i, d in enumerate(devs)],
               threading.Thread(target=detokenizer_stage, name="postprocess", daemon=True)]
    for t in threads:
        t.start()
    results: dict[int, WorkItem] = {}
    fed = 0
    try:
        while len(results) < n and not stop.stopped():
            if fed < n:
                if _put(q_tok, WorkItem(sample_index=fed, text=items[fed]), stop, None):
                    fed += 1
                    if fed == n:
                        _put(q_tok, _END, stop, None)
                continue
            w = _get(q_out, stop, None)
            if w is not _END:
                results[w.sample_index] = w
        if n == 0:
            _put(q_tok, _END, stop, None)
    finally:
        done = len(results) == n
        if not done and not stop.event.is_set():
            stop.fail("orchestrator", TinferError("pipeline ended early"))
        stop.event.set()  # release every worker still polling a queue
        for t in threads:
            t.join(timeout=10.0)
    if not done:
        raise TinferError(f"pipeline stage {stop.stage!r} failed") from stop.error
    ordered = [results[i] for i in range(n)]
    return ordered, StageStats(stages=timing, wall_seconds=time.perf_counter() - wall0)


def read_jsonl_texts(path) -> list[str]:
    """JSON lines, one object with a ``content`` string each (pipeline.py:402-416);
    blank lines skipped; ``FormatError`` names the bad line."""
    import json

    from .errors import FormatError
    texts = []
    with open(path, "r", encoding="utf-8") as fh:
        for ln, line in enumerate(fh):
            line = line.rstrip("\n")
            if not line:
                continue
            try:
                obj = json.loads(line)
            except json.JSONDecodeError as e:
                raise FormatError(f"line {ln}: bad JSON: {e}") from None
            if not isinstance(obj, dict) or "content" not in obj:
                raise FormatError(f"line {ln}: expected an object with 'content'")
            texts.append(obj["content"])
    return texts


def write_results_jsonl(path, items: Sequence[WorkItem]) -> None:
    """One ``{"content", "summary", "sample_index"}`` object per line, sorted
    keys, UTF-8 unescaped (pipeline.py:419-425)."""
    import json
    with open(path, "w", encoding="utf-8") as fh:
        for w in items:
            fh.write(json.dumps({"content": w.text, "summary": w.output_text, "sample_index": w.sample_index},
                                ensure_ascii=False, sort_keys=True) + "\n")
