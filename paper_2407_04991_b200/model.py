"""Model construction and generation API — drop-in for the reference ``tinfer.model``.

Same public names, signatures, argument checks and exceptions as the reference
(model.py:40-667); the compute runs on the B200 through the native runtime
(``device.py`` -> ``libtinfer_sm100.so``). Validation happens on the host before
any launch, exactly like the reference (model.py:507-583, 622-633).

Host-side objects (``ModelConfig``, ``Model``, ``init_random``, ``cast_model``,
TINF save/load) are restatements of the reference; ``init_random`` reproduces the
reference's weights bit-for-bit (same splitmix64 stream and canonical order).

Numerics on the device: f16 storage, f32 accumulation,
every activation quantised at the reference's points (model.py:455-504). An F32
``Model`` is rounded to f16 on upload; the values returned to the host carry the
model's dtype tag. Argmax ties break to the lowest token id (model.py:594).
"""

from __future__ import annotations

import itertools
import json
import math
from dataclasses import dataclass, fields
from pathlib import Path

import numpy as np

from .errors import (
    CapacityError,
    ConfigError,
    DimensionError,
    FormatError,
    ParameterError,
    PositionError,
    VocabError,
)
from .rng import SplitMix64, derive_seed
from .tensor import DType, Tensor, read_tinf, round_to, write_tinf

WEIGHT_SCALE = 0.05


# ---------------------------------------------------------------------------
# configuration (reference model.py:40-103)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class ModelConfig:
    vocab_size: int
    hidden_size: int
    num_layers: int
    num_heads: int
    head_dim: int
    ffn_size: int
    max_position: int
    dtype: DType
    eos_token: int
    pad_token: int

    def __post_init__(self):
        for name in ("vocab_size", "hidden_size", "num_layers", "num_heads", "head_dim",
                     "ffn_size", "max_position"):
            v = getattr(self, name)
            if not isinstance(v, int) or v < 1:
                raise ConfigError(f"{name} must be a positive integer, got {v!r}")
        if self.hidden_size != self.num_heads * self.head_dim:
            raise ConfigError(f"hidden_size ({self.hidden_size}) != num_heads*head_dim "
                              f"({self.num_heads}*{self.head_dim})")
        for name in ("eos_token", "pad_token"):
            v = getattr(self, name)
            if not isinstance(v, int) or v < 0:
                raise ConfigError(f"{name} must be a non-negative integer")
        if self.vocab_size <= max(self.eos_token, self.pad_token):
            raise ConfigError("vocab_size must exceed eos_token and pad_token")
        if not isinstance(self.dtype, DType):
            raise ConfigError("dtype must be a DType")

    def to_json(self) -> str:
        d = _config_dict(self)
        d["dtype"] = self.dtype.value
        return json.dumps(d, sort_keys=True)

    @classmethod
    def from_json(cls, text: str) -> "ModelConfig":
        try:
            d = json.loads(text)
        except json.JSONDecodeError as e:
            raise FormatError(f"bad config JSON: {e}") from None
        want = {f.name for f in fields(cls)}
        if not isinstance(d, dict) or set(d) != want:
            raise FormatError(f"config fields {sorted(d) if isinstance(d, dict) else d} "
                              f"!= expected {sorted(want)}")
        d["dtype"] = DType.from_name(d["dtype"])
        return cls(**d)


def reference_config(dtype: DType = DType.F32) -> ModelConfig:
    """The reference's desk-scale benchmark configuration (model.py:99-103)."""
    return ModelConfig(vocab_size=4096, hidden_size=128, num_layers=4, num_heads=4,
                       head_dim=32, ffn_size=512, max_position=512, dtype=dtype,
                       eos_token=1, pad_token=2)


def _config_dict(c: ModelConfig) -> dict:
    return {f.name: getattr(c, f.name) for f in fields(ModelConfig)}


# ---------------------------------------------------------------------------
# weights (reference model.py:106-256)
# ---------------------------------------------------------------------------
@dataclass
class LayerWeights:
    attn_norm_gamma: Tensor
    attn_norm_beta: Tensor
    wq: Tensor
    bq: Tensor
    wk: Tensor
    bk: Tensor
    wv: Tensor
    bv: Tensor
    wo: Tensor
    bo: Tensor
    ffn_norm_gamma: Tensor
    ffn_norm_beta: Tensor
    w1: Tensor
    b1: Tensor
    w2: Tensor
    b2: Tensor


_LAYER_FIELDS = (("attn_norm.gamma", "attn_norm_gamma"), ("attn_norm.beta", "attn_norm_beta"),
                 ("attn.wq", "wq"), ("attn.bq", "bq"), ("attn.wk", "wk"), ("attn.bk", "bk"),
                 ("attn.wv", "wv"), ("attn.bv", "bv"), ("attn.wo", "wo"), ("attn.bo", "bo"),
                 ("ffn_norm.gamma", "ffn_norm_gamma"), ("ffn_norm.beta", "ffn_norm_beta"),
                 ("ffn.w1", "w1"), ("ffn.b1", "b1"), ("ffn.w2", "w2"), ("ffn.b2", "b2"))


def _tensor_shapes(c: ModelConfig) -> list[tuple[str, tuple[int, ...]]]:
    """Canonical tensor order and shapes (reference model.py:190-207)."""
    h, f = c.hidden_size, c.ffn_size
    per_layer = {"attn_norm.gamma": (h,), "attn_norm.beta": (h,), "attn.wq": (h, h),
                 "attn.bq": (h,), "attn.wk": (h, h), "attn.bk": (h,), "attn.wv": (h, h),
                 "attn.bv": (h,), "attn.wo": (h, h), "attn.bo": (h,), "ffn_norm.gamma": (h,),
                 "ffn_norm.beta": (h,), "ffn.w1": (h, f), "ffn.b1": (f,), "ffn.w2": (f, h),
                 "ffn.b2": (h,)}
    out = [("token_embedding", (c.vocab_size, h)), ("position_embedding", (c.max_position, h))]
    for i in range(c.num_layers):
        out += [(f"layers.{i}.{n}", per_layer[n]) for n, _ in _LAYER_FIELDS]
    out += [("final_norm.gamma", (h,)), ("final_norm.beta", (h,)), ("lm_head", (h, c.vocab_size))]
    return out


class Model:
    """Weights plus config. Treated as immutable once built; tests that mutate a
    weight reset ``_f32 = None``, which also invalidates the device mirror."""

    def __init__(self, config: ModelConfig, token_embedding: Tensor,
                 position_embedding: Tensor, layers: list[LayerWeights],
                 final_norm_gamma: Tensor, final_norm_beta: Tensor, lm_head: Tensor):
        self.config = config
        self.token_embedding = token_embedding
        self.position_embedding = position_embedding
        self.layers = layers
        self.final_norm_gamma = final_norm_gamma
        self.final_norm_beta = final_norm_beta
        self.lm_head = lm_head
        self._f32: dict[str, np.ndarray] | None = None
        self._device = None  # (memo token, {device index: DeviceModel})
        # extension (north star: word/position/TYPE gather-sum): optional
        # [n_types, H] table, kept outside named_tensors / ModelConfig so the
        # reference's TINF layout and JSON field set are unchanged
        self.type_embedding: Tensor | None = None
        self._check_shapes()

    def _check_shapes(self):
        c = self.config
        expect = dict(_tensor_shapes(c))
        for name, t in self.named_tensors():
            if tuple(t.shape) != expect[name]:
                raise ConfigError(f"weight {name} has shape {list(t.shape)}, expected "
                                  f"{list(expect[name])}")
            if t.dtype is not c.dtype:
                raise ConfigError(f"weight {name} dtype != config dtype")

    def named_tensors(self) -> list[tuple[str, Tensor]]:
        out = [("token_embedding", self.token_embedding),
               ("position_embedding", self.position_embedding)]
        for i, lw in enumerate(self.layers):
            out += [(f"layers.{i}.{n}", getattr(lw, attr)) for n, attr in _LAYER_FIELDS]
        out += [("final_norm.gamma", self.final_norm_gamma),
                ("final_norm.beta", self.final_norm_beta), ("lm_head", self.lm_head)]
        return out

    def f32(self, name: str) -> np.ndarray:
        """f32 view of one weight, memoised per name (model.py:177-184)."""
        if self._f32 is None:
            self._f32 = {}
        if name not in self._f32:
            self._f32[name] = dict(self.named_tensors())[name].array.astype(np.float32, copy=False)
        return self._f32[name]

    def weight_bytes(self) -> dict[str, int]:
        return {name: t.nbytes for name, t in self.named_tensors()}

    # -------------------------------------------------------------- device mirror
    def device_model(self, device=None):
        """The packed device copy on ``device`` (default: current CUDA device),
        rebuilt whenever ``_f32`` was reset after a weight mutation."""
        import torch

        from .device import DeviceModel

        if not torch.cuda.is_available():
            from .errors import DeviceError
            raise DeviceError("CUDA device required: the generation path has no CPU fallback")
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if self._f32 is None:  # the memo token: tests reset it after mutating a weight
            self._f32 = {}
        if self._device is None or self._device[0] is not self._f32:
            self._device = (self._f32, {})
        mirrors = self._device[1]
        if dev.index not in mirrors:
            with torch.cuda.device(dev):
                mirrors[dev.index] = DeviceModel(self, dev)
        return mirrors[dev.index]


def set_type_embedding(model: Model, table) -> Model:
    """Attach (or clear, ``table=None``) a token-type embedding [n_types, H]
    (extension: the reference embeds token + position only, model.py:453-455).
    Rounded to the model dtype; invalidates the device mirror like a weight
    mutation."""
    if table is None:
        model.type_embedding = None
    else:
        arr = np.asarray(table.array if isinstance(table, Tensor) else table, dtype=np.float32)
        if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] != model.config.hidden_size:
            raise ParameterError(f"type embedding must be [n_types >= 1, {model.config.hidden_size}]")
        model.type_embedding = Tensor(round_to(arr, model.config.dtype), model.config.dtype)
    model._f32 = None
    return model


def init_type_embedding(model: Model, n_types: int, seed: int) -> Model:
    """Random type table with the init_random distribution (uniform [-0.05,
    0.05) from SplitMix64(derive_seed(seed, "type_embedding")))."""
    if n_types < 1:
        raise ParameterError("n_types must be >= 1")
    s = SplitMix64(derive_seed(seed, "type_embedding"))
    vals = s.uniform(n_types * model.config.hidden_size, -0.05, 0.05).astype(np.float32)
    return set_type_embedding(model, vals.reshape(n_types, model.config.hidden_size))


def _check_types(model: Model, type_ids, n: int) -> np.ndarray | None:
    if type_ids is None:
        return None
    if model.type_embedding is None:
        raise ParameterError("type_ids given but the model has no type embedding")
    t = np.asarray(list(map(int, type_ids)), np.int32)
    if t.size != n:
        raise ParameterError("type_ids must have one entry per token")
    nt = model.type_embedding.shape[0]
    if t.size and (t.min() < 0 or t.max() >= nt):
        raise VocabError(f"type id out of range [0, {nt})")
    return t


def init_random(config: ModelConfig, seed: int) -> Model:
    """Deterministic random weights, bit-identical to the reference
    (model.py:210-224): one splitmix64 stream over the canonical order, uniform
    in [-0.05, 0.05) as f64 -> f32, +1 on norm gammas, then storage rounding."""
    stream = SplitMix64(seed)
    arrays: dict[str, Tensor] = {}
    for name, shape in _tensor_shapes(config):
        count = int(np.prod(shape))
        vals = stream.uniform(count, -WEIGHT_SCALE, WEIGHT_SCALE).astype(np.float32)
        if name.endswith("norm.gamma"):
            vals = vals + np.float32(1.0)
        arrays[name] = Tensor(round_to(vals.reshape(shape), config.dtype), config.dtype)
    return _model_from_dict(config, arrays)


def _model_from_dict(config: ModelConfig, arrays: dict[str, Tensor]) -> Model:
    layers = [LayerWeights(**{attr: arrays[f"layers.{i}.{n}"] for n, attr in _LAYER_FIELDS})
              for i in range(config.num_layers)]
    return Model(config, arrays["token_embedding"], arrays["position_embedding"], layers,
                 arrays["final_norm.gamma"], arrays["final_norm.beta"], arrays["lm_head"])


def cast_model(model: Model, dtype: DType) -> Model:
    """Same weights re-rounded to another storage precision (model.py:247-256)."""
    if dtype is model.config.dtype:
        return model
    cfg = ModelConfig(**{**_config_dict(model.config), "dtype": dtype})
    arrays = {name: Tensor(round_to(t.array.astype(np.float32), dtype), dtype)
              for name, t in model.named_tensors()}
    return _model_from_dict(cfg, arrays)


def config_path_for(weights_path: str | Path) -> Path:
    p = Path(weights_path)
    return p.with_suffix(".json") if p.suffix == ".tinf" else Path(str(p) + ".json")


def save_model(model: Model, weights_path: str | Path) -> None:
    write_tinf(str(weights_path), model.named_tensors())
    config_path_for(weights_path).write_text(model.config.to_json() + "\n", encoding="utf-8")


def load_model(weights_path: str | Path, device=None) -> Model:
    """TINF v1 + JSON config (model.py:267-286).

    ``device`` (extension): load straight to that CUDA device — the file is
    memory-mapped (no host copy, no f32 materialisation), each tensor's bytes
    are uploaded as stored and packed by the device kernels
    (:class:`~.device.DeviceModel`), and the returned Model's host tensors are
    views of the mapping (read lazily if a host accessor touches them)."""
    from .tensor import map_tinf
    cfg = ModelConfig.from_json(config_path_for(weights_path).read_text(encoding="utf-8"))
    named = read_tinf(str(weights_path)) if device is None else map_tinf(str(weights_path))
    if [n for n, _ in named] != [n for n, _ in _tensor_shapes(cfg)]:
        raise FormatError("weight file tensors do not match the config layout")
    model = _model_from_dict(cfg, dict(named))
    if device is not None:
        model.device_model(device)
    return model


# ---------------------------------------------------------------------------
# counters (reference model.py:376-393)
# ---------------------------------------------------------------------------
@dataclass
class OpCounters:
    attn_macs: int = 0
    gemm_macs: int = 0
    launches: int = 0
    kernels: int = 0  # extension: sm_100a kernels actually launched


COUNTERS = OpCounters()


def reset_counters() -> None:
    COUNTERS.attn_macs = COUNTERS.gemm_macs = COUNTERS.launches = COUNTERS.kernels = 0


def snapshot_counters() -> OpCounters:
    return OpCounters(COUNTERS.attn_macs, COUNTERS.gemm_macs, COUNTERS.launches, COUNTERS.kernels)


def _ref_launches(c: ModelConfig, fused: bool) -> int:
    """Operator launches the reference's _forward_tokens issues (model.py:407-437):
    per layer the q/k/v/o and FFN GEMMs (bias [+ GELU] fused into one launch, or
    a GEMM + bias_add [+ gelu] launch each when unfused) and one attention; the
    lm_head GEMM has no bias."""
    return c.num_layers * (7 if fused else 14) + 1


def _count_forward(c: ModelConfig, B: int, T: int, qbase: int, start_sum: int, logit_rows: int,
                   kernels: int, fused: bool = True) -> None:
    """MAC and launch accounting identical to the reference's _gemm/_attend
    bookkeeping (model.py:407-437); ``kernels`` counts the native kernels."""
    H, F, M = c.hidden_size, c.ffn_size, B * T
    COUNTERS.gemm_macs += c.num_layers * M * (4 * H * H + 2 * H * F) + logit_rows * H * c.vocab_size
    series = (qbase + 1 + qbase + T) * T // 2
    valid = B * series - start_sum * T
    COUNTERS.attn_macs += c.num_layers * 2 * c.num_heads * c.head_dim * valid
    COUNTERS.launches += _ref_launches(c, fused)
    COUNTERS.kernels += kernels


def _count_decode_steps(c: ModelConfig, B: int, L: int, steps: int, start_sum: int, fused: bool = True) -> None:
    """``steps`` single-token forwards at cache lengths L, L+1, ... in closed
    form: the same totals as calling _count_forward once per step."""
    if steps <= 0:
        return
    H, F = c.hidden_size, c.ffn_size
    COUNTERS.gemm_macs += steps * (c.num_layers * B * (4 * H * H + 2 * H * F) + B * H * c.vocab_size)
    # step k (qbase = L + k - 1, T = 1) attends qbase + 1 slots per row, minus its pad
    slots = (L + 1 + L + steps) * steps // 2
    COUNTERS.attn_macs += c.num_layers * 2 * c.num_heads * c.head_dim * (B * slots - start_sum * steps)
    COUNTERS.launches += steps * _ref_launches(c, fused)


# ---------------------------------------------------------------------------
# KV cache (reference model.py:293-369), device-resident
# ---------------------------------------------------------------------------
class KVCache:
    """Append-only K/V store [L, B, NH, capacity, D] in f16 on the GPU.

    Slots [0, len) are written once by the QKV GEMM epilogue and never rewritten.
    The host accessors return the reference's single-sequence views."""

    def __init__(self, config: ModelConfig, batch: int = 1, capacity: int | None = None):
        if capacity is None:
            capacity = config.max_position
        if not 1 <= capacity <= config.max_position:
            raise ParameterError("cache capacity must be in [1, max_position]")
        self.config = config
        self.batch = batch
        self.capacity = capacity
        self.len = 0
        self._sess = None  # (DeviceModel, Session) bound on first use
        self._own = None  # (k, v) device storage written before a session is bound

    def _session(self, dm):
        if self._sess is None or self._sess[0] is not dm:
            from .device import Session
            kc, vc = self._own if self._own is not None else (None, None)
            if self._sess is not None:  # rebinding keeps the stored slots
                kc, vc = self._sess[1].k_cache, self._sess[1].v_cache
            s = Session(dm, self.batch, self.capacity, 1, 1, logits=True, k_cache=kc, v_cache=vc)
            s.len = self.len
            self._sess = (dm, s)
            self._own = None
        return self._sess[1]

    def _device_storage(self, create: bool = False):
        """(k, v) device tensors [L, B, NH, cap, D] f16: the bound session's, or
        storage of this cache alone (``write`` before any forward)."""
        if self._sess is not None:
            return self._sess[1].k_cache, self._sess[1].v_cache
        if self._own is None and create:
            import torch
            from .errors import DeviceError
            if not torch.cuda.is_available():
                raise DeviceError("CUDA device required: the KV cache lives in device memory")
            c = self.config
            shape = (c.num_layers, self.batch, c.num_heads, self.capacity, c.head_dim)
            self._own = (torch.zeros(shape, dtype=torch.float16, device="cuda"),
                         torch.zeros(shape, dtype=torch.float16, device="cuda"))
        return self._own if self._own is not None else (None, None)

    def write(self, layer: int, k: np.ndarray, v: np.ndarray) -> None:
        """Store f32 K/V rows [B, NH, T, D] at slots [len, len+T), rounded to f16
        (model.py:326-342: saturating RNE); ``commit`` advances len."""
        import torch
        k, v = np.asarray(k, np.float32), np.asarray(v, np.float32)
        c = self.config
        want = (self.batch, c.num_heads, k.shape[2] if k.ndim == 4 else -1, c.head_dim)
        if k.ndim != 4 or k.shape != want or v.shape != want:
            raise DimensionError(f"write expects K/V of shape {list(want)}")
        if not 0 <= layer < c.num_layers:
            raise ParameterError(f"layer {layer} out of range")
        lo, hi = self.len, self.len + k.shape[2]
        if hi > self.capacity:
            raise CapacityError(f"cache capacity {self.capacity} exceeded")
        kc, vc = self._device_storage(create=True)
        kc[layer, :, :, lo:hi] = torch.from_numpy(round_to(k, DType.F16)).to(kc.device)
        vc[layer, :, :, lo:hi] = torch.from_numpy(round_to(v, DType.F16)).to(vc.device)

    def commit(self, t: int) -> None:
        self.len += t

    def view(self, layer: int, length: int) -> tuple[np.ndarray, np.ndarray]:
        """f32 copies of slots [0, length) of one layer, [B, NH, length, D]
        (model.py:347-348; f16 -> f32 is exact)."""
        kc, vc = self._device_storage()
        c = self.config
        if kc is None:
            z = np.zeros((self.batch, c.num_heads, length, c.head_dim), np.float32)
            return z, z.copy()
        return (kc[layer, :, :, :length].float().cpu().numpy(), vc[layer, :, :, :length].float().cpu().numpy())

    def _accessor(self, which: str, layer: int) -> Tensor:
        c = self.config
        kc, vc = self._device_storage()
        t = kc if which == "k" else vc
        if t is None:
            sel = np.zeros((c.num_heads, self.capacity, c.head_dim), np.float16)
        else:
            sel = t[layer, 0].cpu().numpy()  # one layer of one sequence crosses the bus
        if c.dtype is DType.F32:
            return Tensor(sel.astype(np.float32), DType.F32)
        return Tensor(sel, DType.F16)

    def keys(self, layer: int) -> Tensor:
        return self._accessor("k", layer)

    def values(self, layer: int) -> Tensor:
        return self._accessor("v", layer)

    def fingerprint(self) -> bytes:
        """Filled-slot bytes in slot-major order (reference model.py:359-369);
        only the filled slots are copied to the host."""
        kc, vc = self._device_storage()
        if kc is None or self.len == 0:
            return b""
        ks = kc[:, :, :, :self.len].cpu().numpy()
        vs = vc[:, :, :, :self.len].cpu().numpy()
        if self.config.dtype is DType.F32:
            ks, vs = ks.astype(np.float32), vs.astype(np.float32)
        parts = []
        for slot in range(self.len):
            parts.append(ks[:, :, :, slot].tobytes())
            parts.append(vs[:, :, :, slot].tobytes())
        return b"".join(parts)


# ---------------------------------------------------------------------------
# validation helpers (reference model.py:507-514)
# ---------------------------------------------------------------------------
def _check_ids(config: ModelConfig, ids) -> list[int]:
    # int() per id as the reference does (model.py:507-514); one min/max range
    # check, and the first offending id reported by the scalar loop
    out = list(map(int, ids))
    if not out or (min(out) >= 0 and max(out) < config.vocab_size):
        return out
    for t in out:
        if not 0 <= t < config.vocab_size:
            raise VocabError(f"token id {t} out of range [0, {config.vocab_size})")
    return out


def _host_logits(arr_f16: np.ndarray, dtype: DType) -> Tensor:
    if dtype is DType.F32:
        return Tensor(arr_f16.astype(np.float32), DType.F32)
    return Tensor(np.ascontiguousarray(arr_f16), DType.F16)


# ---------------------------------------------------------------------------
# public single-sequence operations (reference model.py:521-606)
# ---------------------------------------------------------------------------
def embed(model: Model, token_ids, start_position: int = 0, type_ids=None) -> Tensor:
    """Token rows plus position rows [start, start+T) (plus type rows when
    ``type_ids`` is given; extension), rounded to the model dtype."""
    import torch

    from . import ops

    c = model.config
    ids = _check_ids(c, token_ids)
    t = len(ids)
    if t == 0:
        raise ParameterError("embed requires at least one token")
    if start_position < 0 or start_position + t > c.max_position:
        raise PositionError(f"positions [{start_position}, {start_position + t}) exceed "
                            f"max_position {c.max_position}")
    dm = model.device_model()
    with torch.cuda.device(dm.device):
        dev_ids = torch.tensor(ids, dtype=torch.int32, device=dm.device)
        dev_pos = torch.arange(start_position, start_position + t, dtype=torch.int32, device=dm.device)
        x = torch.empty((t, c.hidden_size), dtype=torch.float16, device=dm.device)
        types = _check_types(model, type_ids, t)
        dev_types = None if types is None else torch.from_numpy(types).to(dm.device)
        ops.embed_ln(dev_ids, dev_pos, dm.tok_emb, dm.pos_emb, c.hidden_size, x, type_ids=dev_types,
                     type_emb=dm.type_emb if types is not None else None)
        COUNTERS.kernels += 1
        arr = x.cpu().numpy()
    # the device stores f16 (F32 models are rounded on upload): an F16 model's
    # rows are bit-identical to the reference; an F32 model gets the f16 values
    return _host_logits(arr, c.dtype)


def forward_full(model: Model, token_ids, fused: bool = True, type_ids=None) -> Tensor:
    """Full-recompute causal forward; next-token logits for every position [T, V]."""
    import torch

    from . import _native as N

    c = model.config
    ids = _check_ids(c, token_ids)
    t = len(ids)
    if t == 0:
        raise ParameterError("forward_full requires at least one token")
    if t > c.max_position:
        raise PositionError(f"sequence length {t} exceeds max_position")
    dm = model.device_model()
    with dm.lock, torch.cuda.device(dm.device):
        s = dm.session(1, t, t, 1, logits=True)
        s.load_inputs(np.asarray(ids, np.int32), np.arange(t, dtype=np.int32), np.zeros(1, np.int32),
                      types=_check_types(model, type_ids, t))
        n = s.forward(t, N.FWD_LOGITS_ALL)
        out = s.logits[:t].cpu().numpy()
    _count_forward(c, 1, t, 0, 0, t, n, fused)
    return _host_logits(out, c.dtype)


def hidden_states(model: Model, token_ids) -> Tensor:
    """Extension (no reference counterpart; the parity tap of SURVEY appendix B):
    the residual stream at every LayerNorm input of one causal forward over
    ``token_ids``, shape [2L+1, T, H] in the model dtype. ``[0]`` is
    ``embed(token_ids)``; ``[2l+1]`` is layer l's ffn_norm input (after the
    attention residual, model.py:481-484); ``[2l+2]`` the next attn_norm input
    (after the FFN residual, model.py:493 -> 460), the last one the final_norm
    input (model.py:497)."""
    import torch

    from . import _native as N

    c = model.config
    ids = _check_ids(c, token_ids)
    t = len(ids)
    if t == 0:
        raise ParameterError("hidden_states requires at least one token")
    if t > c.max_position:
        raise PositionError(f"sequence length {t} exceeds max_position")
    dm = model.device_model()
    with dm.lock, torch.cuda.device(dm.device):
        s = dm.session(1, t, t, 1, logits=True)
        s.load_inputs(np.asarray(ids, np.int32), np.arange(t, dtype=np.int32), np.zeros(1, np.int32))
        taps = s.forward_taps(t, N.FWD_LOGITS_LAST).cpu().numpy()
    return _host_logits(taps, c.dtype)


def decode_step(model: Model, token_id: int, cache: KVCache, fused: bool = True) -> Tensor:
    """Incremental decode of one token into ``cache``; returns [1, V] logits."""
    import torch

    from . import _native as N

    c = model.config
    if cache.batch != 1:
        raise ParameterError("decode_step expects a single-sequence cache")
    if cache.len >= cache.capacity:
        raise CapacityError(f"cache is full (capacity {cache.capacity})")
    (tid,) = _check_ids(c, [token_id])
    dm = model.device_model()
    with dm.lock, torch.cuda.device(dm.device):
        s = cache._session(dm)
        s.load_inputs(np.asarray([tid], np.int32), np.asarray([cache.len], np.int32),
                      np.zeros(1, np.int32), length=cache.len)
        n = s.forward(1, N.FWD_LOGITS_LAST)
        out = s.logits[:1].cpu().numpy()
    _count_forward(c, 1, 1, cache.len, 0, 1, n, fused)
    cache.len += 1
    return _host_logits(out, c.dtype)


def greedy_decode(model: Model, prompt, max_new_tokens: int, use_cache: bool = True,
                  fused: bool = True, type_ids=None, gen_type_id: int = 0) -> list[int]:
    """Greedy generation; stops at eos_token or after max_new_tokens."""
    c = model.config
    ids = _check_ids(c, prompt)
    if len(ids) < 1:
        raise ParameterError("prompt must contain at least one token")
    if max_new_tokens < 0:
        raise ParameterError("max_new_tokens must be >= 0")
    if len(ids) + max_new_tokens > c.max_position:
        raise PositionError(f"prompt ({len(ids)}) + max_new_tokens ({max_new_tokens}) "
                            f"exceeds max_position {c.max_position}")
    if max_new_tokens == 0:
        return list(ids)
    if use_cache or type_ids is not None:
        return batched_greedy_decode(model, [ids], max_new_tokens, fused=fused,
                                     type_ids=None if type_ids is None else [type_ids],
                                     gen_type_id=gen_type_id)[0]
    seq = list(ids)
    for _ in range(max_new_tokens):
        logits = forward_full(model, seq, fused).array
        nxt = int(np.argmax(logits[-1]))
        seq.append(nxt)
        if nxt == c.eos_token:
            break
    return seq


# ---------------------------------------------------------------------------
# batched generation (reference model.py:613-667)
# ---------------------------------------------------------------------------
def _left_pad(c: ModelConfig, prompts):
    lens = [len(p) for p in prompts]
    B, L = len(prompts), max(lens)
    if min(lens) == L:  # equal lengths: no padding, one array conversion
        ids = np.asarray(prompts, dtype=np.int32).reshape(B, L)
        pos = np.broadcast_to(np.arange(L, dtype=np.int32), (B, L)).copy()
        return ids, pos, np.zeros(B, np.int32), lens
    pads = np.asarray([L - n for n in lens], np.int32)
    flat = np.fromiter(itertools.chain.from_iterable(prompts), np.int32, count=sum(lens))
    ids = np.full((B, L), c.pad_token, np.int32)
    # row i's tokens land in columns [pads[i], L): one scatter over the flat ids
    cols = np.arange(L, dtype=np.int32)
    live = cols[None, :] >= pads[:, None]
    ids[live] = flat
    pos = np.maximum(cols[None, :] - pads[:, None], 0).astype(np.int32)
    return ids, pos, pads, lens


def _session_shape(c: ModelConfig, L: int, max_new_tokens: int) -> tuple[int, int]:
    """(capacity, max_tokens) of the session serving prompts of padded length L:
    rounded up to multiples of 64 so groups of nearby lengths share one session
    (and its captured decode graph); capacity never exceeds max_position and
    always covers L + max_new_tokens (the reference sizes it exactly,
    model.py:643-644 — a larger cache changes nothing but memory)."""
    r64 = lambda n: (n + 63) // 64 * 64  # noqa: E731
    cap = min(r64(L + max_new_tokens), c.max_position)
    return max(cap, min(L + max_new_tokens, c.max_position)), r64(L)


def _equal_length_ids(c: ModelConfig, prompts, max_new_tokens: int) -> np.ndarray | None:
    """Fast path of _validate_prompts for a batch of equal-length integer prompts
    (one array conversion and vectorised range checks). None whenever any check
    would fail or the input is not such a batch: the caller then runs the
    per-id validation, which raises the reference's errors."""
    try:
        arr = np.asarray(prompts)
    except (ValueError, TypeError):
        return None
    if arr.ndim != 2 or arr.dtype.kind not in "iu" or arr.shape[1] < 1 or max_new_tokens < 0:
        return None
    if arr.shape[1] + max_new_tokens > c.max_position or arr.min() < 0 or arr.max() >= c.vocab_size:
        return None
    return arr


def _validate_prompts(c: ModelConfig, prompts, max_new_tokens: int) -> list[list[int]]:
    checked = []
    for p in prompts:
        ids = _check_ids(c, p)
        if len(ids) < 1:
            raise ParameterError("every prompt needs at least one token")
        if len(ids) + max_new_tokens > c.max_position:
            raise PositionError("prompt ({}) + max_new_tokens exceeds max_position".format(len(ids)))
        checked.append(ids)
    if max_new_tokens < 0:
        raise ParameterError("max_new_tokens must be >= 0")
    return checked


class GenerateStats:
    """Per-call evidence for the benchmark (bytes moved, kernels launched)."""

    def __init__(self):
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self.launches = 0


LAST_STATS = GenerateStats()


def batched_greedy_decode(model: Model, prompts: list[list[int]], max_new_tokens: int,
                          fused: bool = True, prompt_vocab_map=None, type_ids=None,
                          gen_type_id: int = 0) -> list[list[int]]:
    """KV-cached greedy generation for a group of prompts in lockstep.

    Prompts are left-padded; padded slots are masked out of attention. The whole
    generation runs on the device: prefill, then ``max_new_tokens - 1`` decode
    steps replayed from one CUDA graph, each feeding the previous step's
    in-kernel argmax; the host syncs once to read the tokens back. Sequences are
    cut after their first eos (done rows keep being fed, as in the reference,
    model.py:656-661, so the cut is exact).

    ``prompt_vocab_map`` (a ``pruning.PrunedVocabMap``; extension, not in the
    reference): the prompts are in the ORIGINAL vocabulary of a pruned model and
    are remapped on the device by the embedding kernel (ids outside the kept set
    become the model's unk id 0); returned prompts stay as given and
    generated ids are in the pruned vocabulary.

    ``type_ids`` / ``gen_type_id`` (extension; the model needs a type table,
    :func:`set_type_embedding`): one type id per prompt token, and the type of
    every generated token; the embedding adds the type row (word + position +
    type gather-sum)."""
    import torch

    from . import _native as N

    c = model.config
    if not prompts:
        return []
    table = arr = None
    if prompt_vocab_map is not None:
        table = prompt_vocab_map.remap_table()
        for p in prompts:  # original-vocabulary ids: only the sign/length checks apply
            if len(p) < 1 or any(int(t) < 0 for t in p):
                raise VocabError("prompt ids must be non-negative and non-empty")
            if len(p) + max_new_tokens > c.max_position:
                raise PositionError("prompt + max_new_tokens exceeds max_position")
        checked = [[int(t) for t in p] for p in prompts]
        seqs = [list(p) for p in checked]
    else:
        arr = _equal_length_ids(c, prompts, max_new_tokens)
        if arr is not None:  # every prompt valid, same length: no per-id Python work
            checked = seqs = arr.tolist()
        else:
            checked = _validate_prompts(c, prompts, max_new_tokens)
            seqs = [list(p) for p in checked]
    if max_new_tokens == 0:
        return seqs
    if arr is not None:
        B, L = arr.shape
        ids, pads, lens = arr.astype(np.int32), np.zeros(B, np.int32), [L] * B
        pos = np.broadcast_to(np.arange(L, dtype=np.int32), (B, L)).copy()
    else:
        ids, pos, pads, lens = _left_pad(c, checked)
    B, L = ids.shape
    types = None
    if type_ids is not None:
        if len(type_ids) != len(checked):
            raise ParameterError("type_ids must have one list per prompt")
        types = np.zeros((B, L), np.int32)  # pad slots: type 0 (masked out of attention)
        for i, (tp, p) in enumerate(zip(type_ids, checked)):
            types[i, pads[i]:] = _check_types(model, tp, len(p))
    if model.type_embedding is not None:
        _check_types(model, [gen_type_id], 1)
    cap, max_tokens = _session_shape(c, L, max_new_tokens)
    dm = model.device_model()
    stats = GenerateStats()
    # the session is this thread's own (DeviceModel.session), so concurrent
    # generate calls from several host threads (each on its own stream) overlap
    with torch.cuda.device(dm.device):
        s = dm.session(B, cap, max_tokens, max_new_tokens)
        s.set_remap(table)
        s.set_gen_type(gen_type_id)
        stats.h2d_bytes = s.load_inputs(ids, pos, pads, types=types)
        n_pre = s.forward(L, N.FWD_ARGMAX)
        n_dec = s.decode(max_new_tokens - 1)
        toks = s.fetch_tokens(max_new_tokens)
        stats.d2h_bytes = toks.nbytes
    stats.launches = n_pre + n_dec
    _count_forward(c, B, L, 0, int(pads.sum()), B, n_pre, fused)
    _count_decode_steps(c, B, L, max_new_tokens - 1, int(pads.sum()), fused)
    COUNTERS.kernels += n_dec
    global LAST_STATS
    LAST_STATS = stats
    # append up to and including each row's first eos (model.py:656-661)
    hit = toks == c.eos_token
    cut = np.where(hit.any(axis=1), hit.argmax(axis=1) + 1, toks.shape[1])
    for i in range(B):
        seqs[i].extend(toks[i, :cut[i]].tolist())
    return seqs
