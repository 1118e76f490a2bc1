"""Session workspace planning: lifetime-disjoint activation
buffers share storage.

The reference plans memory for its operator-graph IR (graphopt.py:265-346):
``analyze_lifetimes`` gives every intermediate tensor the interval (producer
index, last consumer index) (graphopt.py:265-282), ``plan_memory`` assigns
tensors to buffers first-fit in definition order — the lowest-index buffer that
is large enough and lifetime-disjoint wins, else a new buffer opens
(graphopt.py:302-330) — and ``check_plan`` rejects any same-buffer overlap or
undersized buffer with ``PlanError`` (graphopt.py:333-346). Intervals are closed
(graphopt.py:298-299: touching intervals overlap).

Here the "graph" is the fixed kernel sequence of one native forward
(csrc/tinfer_sm100.cu ``forward``: embed, then per layer QKV -> attention -> Wo
-> [LN2] -> FFN1 -> FFN2 -> [LN1 of the next layer], then [final LN] ->
lm_head -> collect), and the planned tensors are the session's named
activation buffers x, h, q, attn, ffn. One name is written by every layer, so
its lifetime is the SET of intervals between each write and the last read of
that value; two names may share a buffer when no interval of one overlaps an
interval of the other. For the forward this yields {ffn, q} and {h, attn}
sharing storage (q lives QKV -> attention, ffn FFN1 -> FFN2; h lives
LN -> consumer GEMM, attn attention -> Wo), x alone.

Safe under programmatic dependent launch: every kernel touches these buffers
only after ``griddepcontrol.wait`` (its early prologue reads weights or the
KV cache, never an activation buffer), and that wait orders it after the
complete predecessor chain. Sharing is used only when no buffer carries
padding columns (ld == logical width), so a buffer never exposes another
buffer's values to a GEMM's zero-weight K padding.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import PlanError

Interval = tuple[int, int]
Op = tuple[str, tuple[str, ...], tuple[str, ...]]  # (kernel, reads, writes)

ALIGN = 1024  # byte alignment of every buffer in the arena (TMA needs 16; one swizzle atom)


def forward_ops(n_layers: int) -> list[Op]:
    """The native forward's kernel sequence with the activation buffers each
    kernel reads and writes, covering both LayerNorm forms (stand-alone LN
    kernels in prefill, LN folded into the consuming GEMM in decode): a plan
    valid for this sequence is valid for either."""
    ops: list[Op] = [("embed", (), ("x", "h"))]
    for layer in range(n_layers):
        if layer > 0:
            ops.append((f"ln1.{layer}", ("x",), ("h",)))
        ops += [
            (f"qkv.{layer}", ("h", "x"), ("q",)),
            (f"attention.{layer}", ("q",), ("attn",)),
            (f"wo.{layer}", ("attn", "x"), ("x",)),
            (f"ln2.{layer}", ("x",), ("h",)),
            (f"ffn1.{layer}", ("h", "x"), ("ffn",)),
            (f"ffn2.{layer}", ("ffn", "x"), ("x",)),
        ]
    ops += [("final_ln", ("x",), ("h",)), ("lm_head", ("h", "x"), ()), ("collect", (), ())]
    return ops


def forward_kernels(n_layers: int, folded: bool) -> list[str]:
    """The kernels one native forward launches: a decode step (T = 1) folds
    every LayerNorm into the consuming GEMM (5 per layer), a prefill runs the
    stand-alone LayerNorm kernels (csrc/tinfer_sm100.cu forward)."""
    names = ["embed"]
    for layer in range(n_layers):
        if layer > 0 and not folded:
            names.append(f"ln1.{layer}")
        names += [f"qkv.{layer}", f"attention.{layer}", f"wo.{layer}"]
        if not folded:
            names.append(f"ln2.{layer}")
        names += [f"ffn1.{layer}", f"ffn2.{layer}"]
    if not folded:
        names.append("final_ln")
    return names + ["lm_head", "collect"]


def analyze_lifetimes(ops: list[Op], live_out: tuple[str, ...] = ()) -> dict[str, list[Interval]]:
    """Per buffer name, the (write index, last read index) interval of every
    value written to it, in order. A value never read spans its write only
    (graphopt.py:274-278); names in ``live_out`` are read after the sequence,
    so their last value extends to len(ops)."""
    out: dict[str, list[Interval]] = {}
    start: dict[str, int] = {}
    last: dict[str, int] = {}
    for i, (_, reads, writes) in enumerate(ops):
        for name in reads:
            if name not in start:
                raise PlanError(f"op {i} ({ops[i][0]}) reads {name!r} before any write")
            last[name] = i
        for name in writes:
            if name in start:
                out.setdefault(name, []).append((start[name], last[name]))
            start[name] = last[name] = i
    for name, s in start.items():
        out.setdefault(name, []).append((s, len(ops) if name in live_out else last[name]))
    return out


def _overlap(a: Interval, b: Interval) -> bool:
    return not (a[1] < b[0] or b[1] < a[0])


def _sets_overlap(a: list[Interval], b: list[Interval]) -> bool:
    return any(_overlap(x, y) for x in a for y in b)


@dataclass
class ArenaPlan:
    buffer_sizes: list[int]
    assignment: dict[str, int]  # name -> buffer index (offset 0 inside the buffer)
    tensor_bytes: dict[str, int]
    lifetimes: dict[str, list[Interval]]

    @property
    def buffer_count(self) -> int:
        return len(self.buffer_sizes)

    @property
    def peak_bytes(self) -> int:
        return sum(self.buffer_sizes)

    def offsets(self, align: int = ALIGN) -> list[int]:
        """Byte offset of each buffer in one contiguous arena."""
        offs, o = [], 0
        for size in self.buffer_sizes:
            offs.append(o)
            o += -(-size // align) * align
        return offs

    def arena_bytes(self, align: int = ALIGN) -> int:
        return sum(-(-s // align) * align for s in self.buffer_sizes)


def plan_memory(sizes: dict[str, int], lifetimes: dict[str, list[Interval]],
                order: str = "definition") -> ArenaPlan:
    """First-fit buffer assignment. ``order="definition"`` is the reference's
    rule exactly (names by first write; graphopt.py:305-330); ``"size"`` visits
    larger tensors first (ties by first write), which lets the small buffers
    fill the large ones' gaps — the order the sessions use."""
    names = sorted(lifetimes, key=lambda n: lifetimes[n][0][0])
    if order == "size":
        names = sorted(names, key=lambda n: (-sizes[n], lifetimes[n][0][0]))
    elif order != "definition":
        raise PlanError(f"unknown plan order {order!r}")
    buffer_sizes: list[int] = []
    members: list[list[str]] = []
    assignment: dict[str, int] = {}
    for name in names:
        for bi, size in enumerate(buffer_sizes):
            if size < sizes[name]:
                continue
            if any(_sets_overlap(lifetimes[name], lifetimes[m]) for m in members[bi]):
                continue
            assignment[name] = bi
            members[bi].append(name)
            break
        else:
            buffer_sizes.append(sizes[name])
            members.append([name])
            assignment[name] = len(buffer_sizes) - 1
    return ArenaPlan(buffer_sizes, assignment, {n: sizes[n] for n in names},
                     {n: list(lifetimes[n]) for n in names})


def check_plan(plan: ArenaPlan) -> None:
    """Raise PlanError on any same-buffer lifetime overlap or undersized buffer
    (graphopt.py:333-346)."""
    by_buffer: dict[int, list[str]] = {}
    for name, bi in plan.assignment.items():
        by_buffer.setdefault(bi, []).append(name)
        if plan.tensor_bytes[name] > plan.buffer_sizes[bi]:
            raise PlanError(f"tensor {name!r} does not fit its buffer")
    for bi, names in by_buffer.items():
        for i in range(len(names)):
            for j in range(i + 1, len(names)):
                a, b = names[i], names[j]
                if _sets_overlap(plan.lifetimes[a], plan.lifetimes[b]):
                    raise PlanError(f"tensors {a!r} and {b!r} share buffer {bi} with overlapping lifetimes")


def session_plan(rows: int, hidden: int, ffn: int, ldk_h: int, ldk_f: int, n_layers: int) -> ArenaPlan:
    """The arena plan of a session's activation buffers ([rows, ld] f16 each).
    Buffers with padding columns are planned apart (every name its own buffer)."""
    sizes = {"x": rows * ldk_h * 2, "h": rows * ldk_h * 2, "q": rows * ldk_h * 2,
             "attn": rows * ldk_h * 2, "ffn": rows * ldk_f * 2}
    lifetimes = analyze_lifetimes(forward_ops(n_layers))
    if ldk_h != hidden or ldk_f != ffn:
        # disjointness is not enough here: no sharing at all
        lifetimes = {n: [(0, 1 << 30)] for n in sizes}
    plan = plan_memory(sizes, lifetimes, order="size")
    check_plan(plan)
    return plan
