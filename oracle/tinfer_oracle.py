"""CPU oracle for the Ernie-style generation path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm (``/root/reference/pkg/src/tinfer``),
used as the checker by ``tests/``, ``__graft_entry__.smoke()`` and as the
``cpu_baseline`` / ``--impl reference`` leg of ``bench.py``. The product package
never imports this module; its CUDA path fails loudly when the extension is
missing instead of falling back here.

Pinned against the real reference: ``tests/golden/make_golden.py`` imports the
unmodified reference (via ``oracle/ref_loader.py``) in the build container and
writes golden vectors to ``tests/golden/*.npz``; ``tests/test_oracle_golden.py``
checks this module against them (weights bit-exact, tokens exact, logits within
1e-5 for F32 / f16-ulp for F16).

Every function cites the reference file:line it restates. Differences from the
reference are limited to GEMM/attention summation order (numpy BLAS instead of
numba's strictly sequential k-loop, kernels.py:48-109), which is why logits are
compared with a tolerance rather than bitwise.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

F16_MAX = 65504.0
WEIGHT_SCALE = 0.05  # model.py:37
LN_EPS = 1e-5  # model.py:460

# ---------------------------------------------------------------------------
# splitmix64 (rng.py:14-63)
# ---------------------------------------------------------------------------
_G = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * _C1
    z = (z ^ (z >> np.uint64(27))) * _C2
    return z ^ (z >> np.uint64(31))


class Stream:
    """rng.py:26-54 — output n (1-based) is mix(seed + n*GAMMA)."""

    def __init__(self, seed: int):
        self.seed = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        self.count = 0

    def u64(self, n):
        idx = np.arange(self.count + 1, self.count + n + 1, dtype=np.uint64)
        self.count += n
        with np.errstate(over="ignore"):
            return _mix(self.seed + idx * _G)

    def uniform(self, n, lo, hi):
        u = (self.u64(n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
        return lo + u * (hi - lo)

    def randint(self, n, bound):
        return (self.u64(n) % np.uint64(bound)).astype(np.int64)


def derive_seed(seed: int, label: str) -> int:
    """rng.py:57-63."""
    h = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        for ch in label.encode("utf-8"):
            h = _mix((h ^ np.uint64(ch)) * _G)
    return int(h)


# ---------------------------------------------------------------------------
# config + weights (model.py:40-224)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class Config:
    vocab_size: int
    hidden_size: int
    num_layers: int
    num_heads: int
    head_dim: int
    ffn_size: int
    max_position: int
    f16: bool
    eos_token: int = 1
    pad_token: int = 2


def tensor_shapes(c: Config):
    """Canonical order and shapes, model.py:190-207."""
    h, v, p, f = c.hidden_size, c.vocab_size, c.max_position, c.ffn_size
    out = [("token_embedding", (v, h)), ("position_embedding", (p, h))]
    for i in range(c.num_layers):
        pre = f"layers.{i}."
        out += [(pre + "attn_norm.gamma", (h,)), (pre + "attn_norm.beta", (h,)),
                (pre + "attn.wq", (h, h)), (pre + "attn.bq", (h,)),
                (pre + "attn.wk", (h, h)), (pre + "attn.bk", (h,)),
                (pre + "attn.wv", (h, h)), (pre + "attn.bv", (h,)),
                (pre + "attn.wo", (h, h)), (pre + "attn.bo", (h,)),
                (pre + "ffn_norm.gamma", (h,)), (pre + "ffn_norm.beta", (h,)),
                (pre + "ffn.w1", (h, f)), (pre + "ffn.b1", (f,)),
                (pre + "ffn.w2", (f, h)), (pre + "ffn.b2", (h,))]
    out += [("final_norm.gamma", (h,)), ("final_norm.beta", (h,)), ("lm_head", (h, v))]
    return out


def round_f16(x):
    """tensor.py:95-100: clip to +-65504, RNE to f16, returned as f32 values."""
    return np.clip(x, -F16_MAX, F16_MAX).astype(np.float16).astype(np.float32)


def quant(x, f16: bool):
    """model.py:400-404."""
    return round_f16(x) if f16 else x


def init_weights(c: Config, seed: int) -> dict:
    """model.py:210-224: one stream, canonical order, f64 uniform -> f32 (+1 for
    gammas) -> storage rounding. Returns f32 arrays (f16-representable if f16)."""
    s = Stream(seed)
    w = {}
    for name, shape in tensor_shapes(c):
        n = int(np.prod(shape))
        vals = s.uniform(n, -WEIGHT_SCALE, WEIGHT_SCALE).astype(np.float32)
        if name.endswith("norm.gamma"):
            vals = vals + np.float32(1.0)
        w[name] = quant(vals.reshape(shape), c.f16)
    return w


def cast_weights(w: dict, f16: bool) -> dict:
    """model.py:247-256 (values only)."""
    return {k: quant(v.astype(np.float32), f16) for k, v in w.items()}


def weights_digest(w: dict, c: Config) -> str:
    """sha256 over canonical-order storage bytes (pins init_random)."""
    import hashlib
    h = hashlib.sha256()
    dt = np.float16 if c.f16 else np.float32
    for name, _ in tensor_shapes(c):
        h.update(np.ascontiguousarray(w[name].astype(dt)).tobytes())
    return h.hexdigest()


# ---------------------------------------------------------------------------
# numerics (kernels.py, tensor.py:153-160)
# ---------------------------------------------------------------------------
def layer_norm(x, g, b):
    """tensor.py:153-160: two-pass f32 LN."""
    mean = x.mean(axis=-1, keepdims=True)
    c = x - mean
    var = (c * c).mean(axis=-1, keepdims=True)
    inv = np.float32(1.0) / np.sqrt(var + np.float32(LN_EPS))
    return c * inv * g + b


def gelu(x):
    """kernels.py:36-45, tanh approximation in f32."""
    x = x.astype(np.float32)
    inner = np.float32(0.7978845608028654) * (x + np.float32(0.044715) * (x * x * x))
    return np.float32(0.5) * x * (np.float32(1.0) + np.tanh(inner))


def attend(q, k, v, start, qbase, scale):
    """kernels.py:148-233: row t of batch b attends slots [start[b], qbase+t];
    empty window -> zeros. q [B,NH,Tq,D], k/v [B,NH,L,D]."""
    B, NH, Tq, D = q.shape
    L = k.shape[2]
    s = np.einsum("bhtd,bhld->bhtl", q, k).astype(np.float32) * np.float32(scale)
    slot = np.arange(L)[None, None, None, :]
    hi = (qbase + np.arange(Tq))[None, None, :, None]
    lo = np.asarray(start).reshape(B, 1, 1, 1)
    mask = (slot >= lo) & (slot <= hi)
    s = np.where(mask, s, -np.inf)
    m = s.max(axis=-1, keepdims=True)
    m = np.where(np.isfinite(m), m, 0.0).astype(np.float32)
    e = np.where(mask, np.exp(s - m), 0.0).astype(np.float32)
    z = e.sum(axis=-1, keepdims=True)
    inv = np.where(z > 0, np.float32(1.0) / np.where(z > 0, z, 1), 0).astype(np.float32)
    return np.einsum("bhtl,bhld->bhtd", e * inv, v).astype(np.float32)


# ---------------------------------------------------------------------------
# KV cache + forward core (model.py:293-504)
# ---------------------------------------------------------------------------
@dataclass
class Cache:
    """model.py:293-348, [L, B, NH, cap, D] f32 values (f16-rounded if f16)."""
    k: np.ndarray
    v: np.ndarray
    len: int = 0

    @classmethod
    def new(cls, c: Config, batch: int, capacity: int):
        shape = (c.num_layers, batch, c.num_heads, capacity, c.head_dim)
        return cls(np.zeros(shape, np.float32), np.zeros(shape, np.float32), 0)


def forward_tokens(w, c: Config, ids, pos, cache: Cache, start, all_logits=False,
                   taps=None, types=None):
    """model.py:440-504. ids/pos [B,T] int; returns logits [B,V] (last row) or
    [B,T,V]. ``taps`` (list) collects the 2L+1 residual-stream LN inputs
    (SURVEY appendix B). ``types`` [B,T] (extension, no reference code): adds
    w["type_embedding"][types] to the f32 gather-sum before the rounding."""
    f16 = c.f16
    B, T = ids.shape
    H, NH, D = c.hidden_size, c.num_heads, c.head_dim
    qbase = cache.len
    length = qbase + T
    if length > cache.k.shape[3]:
        raise OverflowError("cache capacity exceeded")
    scale = 1.0 / math.sqrt(D)
    x = w["token_embedding"][ids.reshape(-1)] + w["position_embedding"][pos.reshape(-1)]
    if types is not None:
        x = x + w["type_embedding"][np.asarray(types).reshape(-1)]
    x = quant(x, f16).reshape(B, T, H)
    for li in range(c.num_layers):
        p = f"layers.{li}."
        if taps is not None:
            taps.append(x.copy())
        h = quant(layer_norm(x, w[p + "attn_norm.gamma"], w[p + "attn_norm.beta"]), f16)
        h2 = h.reshape(B * T, H)
        q = quant(h2 @ w[p + "attn.wq"] + w[p + "attn.bq"], f16)
        k = quant(h2 @ w[p + "attn.wk"] + w[p + "attn.bk"], f16)
        v = quant(h2 @ w[p + "attn.wv"] + w[p + "attn.bv"], f16)
        qh = q.reshape(B, T, NH, D).transpose(0, 2, 1, 3)
        cache.k[li, :, :, qbase:length] = k.reshape(B, T, NH, D).transpose(0, 2, 1, 3)
        cache.v[li, :, :, qbase:length] = v.reshape(B, T, NH, D).transpose(0, 2, 1, 3)
        a = quant(attend(qh, cache.k[li, :, :, :length], cache.v[li, :, :, :length],
                         start, qbase, scale), f16)
        merged = a.transpose(0, 2, 1, 3).reshape(B * T, H)
        o = quant(merged @ w[p + "attn.wo"] + w[p + "attn.bo"], f16)
        x = quant(x + o.reshape(B, T, H), f16)
        if taps is not None:
            taps.append(x.copy())
        h = quant(layer_norm(x, w[p + "ffn_norm.gamma"], w[p + "ffn_norm.beta"]), f16)
        f = quant(gelu(h.reshape(B * T, H) @ w[p + "ffn.w1"] + w[p + "ffn.b1"]), f16)
        o = quant(f @ w[p + "ffn.w2"] + w[p + "ffn.b2"], f16)
        x = quant(x + o.reshape(B, T, H), f16)
    cache.len = length
    if taps is not None:
        taps.append(x.copy())
    h = quant(layer_norm(x, w["final_norm.gamma"], w["final_norm.beta"]), f16)
    if all_logits:
        return quant(h.reshape(B * T, H) @ w["lm_head"], f16).reshape(B, T, -1)
    return quant(h[:, -1, :] @ w["lm_head"], f16)


def embed(w, c: Config, ids, start_position=0):
    """model.py:521-534."""
    t = len(ids)
    x = w["token_embedding"][np.asarray(ids)] + w["position_embedding"][start_position:start_position + t]
    return quant(x, c.f16)


def forward_full(w, c: Config, ids):
    """model.py:537-551: all-position logits [T, V]."""
    t = len(ids)
    cache = Cache.new(c, 1, t)
    arr = np.asarray(ids, np.int64).reshape(1, t)
    pos = np.arange(t, dtype=np.int64).reshape(1, t)
    return forward_tokens(w, c, arr, pos, cache, np.zeros(1, np.int64), all_logits=True)[0]


def greedy_decode(w, c: Config, prompt, max_new):
    """model.py:571-606 (use_cache=True)."""
    seq = [int(t) for t in prompt]
    if max_new == 0:
        return seq
    n = len(seq)
    cache = Cache.new(c, 1, n + max_new)
    logits = forward_tokens(w, c, np.asarray(seq, np.int64).reshape(1, -1),
                            np.arange(n, dtype=np.int64).reshape(1, -1), cache,
                            np.zeros(1, np.int64))
    for _ in range(max_new):
        nxt = int(np.argmax(logits[0]))
        seq.append(nxt)
        if nxt == c.eos_token or len(seq) - n == max_new:
            break
        logits = forward_tokens(w, c, np.asarray([[nxt]], np.int64),
                                np.asarray([[cache.len]], np.int64), cache, np.zeros(1, np.int64))
    return seq


def left_pad(c: Config, prompts):
    """model.py:634-641: ids [B,L] padded with pad_token, positions 0..n-1 for
    real tokens and 0 for pads, pads[b] = L - n_b."""
    lens = [len(p) for p in prompts]
    B, L = len(prompts), max(lens)
    pads = np.asarray([L - n for n in lens], np.int64)
    ids = np.full((B, L), c.pad_token, np.int64)
    pos = np.zeros((B, L), np.int64)
    for i, p in enumerate(prompts):
        ids[i, pads[i]:] = p
        pos[i, pads[i]:] = np.arange(lens[i])
    return ids, pos, pads, lens


def batched_greedy_decode(w, c: Config, prompts, max_new, step_logits=None,
                          teacher=None, type_ids=None, gen_type=0):
    """model.py:613-667. ``step_logits`` (list) collects per-step [B,V] logits;
    ``teacher`` ([B, max_new] ids) forces the fed tokens (teacher forcing) while
    still recording the argmax as the output. ``type_ids`` (per-prompt lists) /
    ``gen_type`` (extension): token types of the prompts (pads: 0) and of every
    generated token."""
    if not prompts:
        return []
    ids, pos, pads, lens = left_pad(c, prompts)
    B, L = ids.shape
    cache = Cache.new(c, B, min(L + max_new, c.max_position))
    seqs = [list(map(int, p)) for p in prompts]
    if max_new == 0:
        return seqs
    types = None
    if type_ids is not None:
        types = np.zeros((B, L), np.int64)
        for i, tp in enumerate(type_ids):
            types[i, pads[i]:] = tp
    logits = forward_tokens(w, c, ids, pos, cache, pads, types=types)
    done = [False] * B
    for step in range(max_new):
        if step_logits is not None:
            step_logits.append(logits.copy())
        nxt = np.argmax(logits, axis=1)
        feed = np.empty((B, 1), np.int64)
        newpos = np.empty((B, 1), np.int64)
        for i in range(B):
            tok = int(nxt[i])
            if not done[i]:
                seqs[i].append(tok)
                if tok == c.eos_token or len(seqs[i]) - lens[i] == max_new:
                    done[i] = True
            feed[i, 0] = tok if teacher is None else int(teacher[i][step])
            newpos[i, 0] = cache.len - pads[i]
        if all(done) or step == max_new - 1:
            break
        logits = forward_tokens(w, c, feed, newpos, cache, pads,
                                types=None if type_ids is None else np.full((B, 1), gen_type, np.int64))
    return seqs


# ---------------------------------------------------------------------------
# beam search (NEW semantics, no reference code: parity unpinned — SURVEY §8c)
# ---------------------------------------------------------------------------
def log_softmax_f32(logits):
    """log-softmax over f16-rounded logits in f32 (SURVEY §8c beam oracle)."""
    x = logits.astype(np.float32)
    m = x.max(axis=-1, keepdims=True)
    z = np.exp(x - m).sum(axis=-1, keepdims=True, dtype=np.float32)
    return (x - m - np.log(z)).astype(np.float32)


def beam_search_decode(w, c: Config, prompts, max_new, beam):
    """Fixed-width beam search over the reference forward core.

    Semantics (documented in DESIGN.md §beam): every request keeps ``beam``
    hypotheses; at step 0 only beam 0 is live (the others start at -inf). Each
    step, candidate score = beam score + log_softmax(f16 logits) in f32; the top
    ``beam`` candidates over the flat (beam, token) index are kept, ties to the
    lowest flat index. A hypothesis that emitted eos is frozen: it proposes only
    itself (score unchanged, token eos) once. No length penalty. Returns the
    highest-scoring hypothesis per request (lowest beam index on ties), prompt
    included, truncated after its first eos.
    """
    if not prompts:
        return []
    R, K = len(prompts), beam
    flat = [p for p in prompts for _ in range(K)]
    ids, pos, pads, lens = left_pad(c, flat)
    B, L = ids.shape
    cache = Cache.new(c, B, min(L + max_new, c.max_position))
    logits = forward_tokens(w, c, ids, pos, cache, pads)
    V = logits.shape[1]
    score = np.full((R, K), -np.inf, np.float32)
    score[:, 0] = 0.0
    hist = np.zeros((R, K, 0), np.int64)
    finished = np.zeros((R, K), bool)
    for step in range(max_new):
        lp = log_softmax_f32(logits).reshape(R, K, V)
        cand = (score[:, :, None] + lp).astype(np.float32)
        # frozen hypotheses propose only themselves with eos
        for r in range(R):
            for b in range(K):
                if finished[r, b]:
                    cand[r, b, :] = -np.inf
                    cand[r, b, c.eos_token] = score[r, b]
        flatc = cand.reshape(R, K * V)
        order = np.argsort(-flatc, axis=1, kind="stable")[:, :K]
        parent = order // V
        tok = order % V
        new_score = np.take_along_axis(flatc, order, axis=1).astype(np.float32)
        hist = np.concatenate([np.take_along_axis(hist, parent[:, :, None], axis=1),
                               tok[:, :, None]], axis=2)
        finished = np.take_along_axis(finished, parent, axis=1) | (tok == c.eos_token)
        score = new_score
        if step == max_new - 1 or finished.all():
            break
        # reorder cache rows by parent beam (axis 1 of [L,B,NH,cap,D])
        src = (np.arange(R)[:, None] * K + parent).reshape(-1)
        cache.k[:] = cache.k[:, src]
        cache.v[:] = cache.v[:, src]
        feed = tok.reshape(B, 1)
        newpos = (cache.len - pads).reshape(B, 1)
        logits = forward_tokens(w, c, feed, newpos, cache, pads)
    out = []
    for r in range(R):
        best = int(np.argmax(score[r]))  # first max -> lowest beam index
        gen = []
        for t in hist[r, best]:
            gen.append(int(t))
            if int(t) == c.eos_token:
                break
        out.append(list(map(int, prompts[r])) + gen)
    return out


# ---------------------------------------------------------------------------
# pruning (pruning.py:66-142) and batching (pipeline.py:60-87)
# ---------------------------------------------------------------------------
def build_pruned_vocab(counts, keep_count, specials=()):
    """pruning.py:66-86: top keep_count by count (ties to lower id), specials
    forced in; returns sorted kept old ids."""
    counts = np.asarray(counts, np.int64)
    kept = set(int(s) for s in specials)
    order = np.lexsort((np.arange(len(counts)), -counts))
    for tid in order:
        if len(kept) >= keep_count:
            break
        kept.add(int(tid))
    return tuple(sorted(kept))


def prune_weights(w, c: Config, kept_old_ids, new_max_position=None):
    """pruning.py:104-142: token rows + lm_head columns selected, eos/pad
    remapped, position table truncated."""
    idx = np.asarray(kept_old_ids, np.int64)
    o2n = {o: n for n, o in enumerate(kept_old_ids)}
    w2 = dict(w)
    w2["token_embedding"] = w["token_embedding"][idx]
    w2["lm_head"] = np.ascontiguousarray(w["lm_head"][:, idx])
    c2 = replace(c, vocab_size=len(idx), eos_token=o2n[c.eos_token], pad_token=o2n[c.pad_token])
    if new_max_position is not None and new_max_position != c.max_position:
        w2["position_embedding"] = w["position_embedding"][:new_max_position].copy()
        c2 = replace(c2, max_position=new_max_position)
    return w2, c2


def plan_batches(lengths, max_batch_size, bucket_width):
    """pipeline.py:60-87: stable descending-length sort, greedy chunking."""
    order = sorted(range(len(lengths)), key=lambda i: -lengths[i])
    groups, pads, cur, head = [], [], [], 0
    for i in order:
        if cur and (len(cur) == max_batch_size or head - lengths[i] > bucket_width):
            groups.append(cur)
            pads.append(head)
            cur = []
        if not cur:
            head = lengths[i]
        cur.append(i)
    if cur:
        groups.append(cur)
        pads.append(head)
    return groups, pads


# ---------------------------------------------------------------------------
# benchmark config pins (SURVEY §8 "Config pins")
# ---------------------------------------------------------------------------
def config_c1(f16=False):
    return Config(8192, 256, 2, 4, 64, 1024, 512, f16, 1, 2)


def config_master(f16=True):
    return Config(40000, 768, 12, 12, 64, 3072, 1024, f16, 1, 2)


def synthetic_prompts(vocab_size, batch, src_len, seed=42, label="prompts"):
    """SplitMix64(derive_seed(seed, label)).randint(., V-3)+3."""
    s = Stream(derive_seed(seed, label))
    ids = s.randint(batch * src_len, vocab_size - 3) + 3
    return [list(map(int, r)) for r in ids.reshape(batch, src_len)]


def sequence_logprob(w, c: Config, prompt, gen):
    """Sum of log_softmax(f16 logits) of ``gen`` given ``prompt`` (beam score of a
    hypothesis, eos included), through the reference forward core."""
    seq = list(prompt) + list(gen)
    logits = forward_full(w, c, seq[:-1]) if gen else None
    total = np.float32(0.0)
    for t, tok in enumerate(gen):
        lp = log_softmax_f32(logits[len(prompt) - 1 + t][None, :])[0]
        total = np.float32(total + lp[tok])
    return float(total)
