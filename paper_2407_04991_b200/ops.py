"""Operator API over the C ABI (replaces the reference ``tinfer.kernels``).

Each function takes CUDA ``torch.Tensor`` operands (torch is only the device
allocator and stream provider here) and launches one hand-written sm_100a kernel
through ``libtinfer_sm100.so``:

* :func:`gemm` — tcgen05 GEMM with fused epilogues (kernels.gemm_f32 +
  bias_add + gelu, kernels.py:96-126).
* :func:`attention` — masked attention over the KV cache (kernels.attend_f32,
  kernels.py:216-233).
* :func:`layernorm` / :func:`embed_ln` — tensor.layer_norm_f32
  (tensor.py:153-160) and the embedding gather-sum (model.py:453-455).

Weights are K-major ``W^T [out, ld]`` f16 with K zero-padded to a multiple of
64 (see :func:`pack_kmajor`).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .errors import DimensionError


def pad64(k: int) -> int:
    return (k + 63) // 64 * 64


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def pack_kmajor(w_in_out: np.ndarray, device) -> torch.Tensor:
    """[in, out] (reference layout) -> f16 W^T [out, pad64(in)] on ``device``."""
    k, n = w_in_out.shape
    buf = np.zeros((n, pad64(k)), dtype=np.float16)
    buf[:, :k] = np.asarray(w_in_out, dtype=np.float32).T.astype(np.float16)
    return torch.from_numpy(buf).to(device)


class Scratch:
    """Split-K workspace + zeroed tile counters shared by sequential GEMMs."""

    def __init__(self, device, workspace_bytes: int = 64 << 20, n_counters: int = 1 << 16):
        self.ws = torch.empty(workspace_bytes // 4, dtype=torch.float32, device=device)
        self.counters = torch.zeros(n_counters, dtype=torch.int32, device=device)
        self.workspace_bytes = workspace_bytes
        self.n_counters = n_counters


def gemm(act: torch.Tensor, wt: torch.Tensor, k: int, epilogue: int, *, out=None, bias=None,
         resid=None, scratch: Scratch | None = None, force_swap: int = -1, splits: int = 0,
         keys=None, qkv=None, m_tok: int | None = None, n_feat: int | None = None, ln=None,
         stats=None):
    """out[m, n] = epilogue(act[m, :k] . wt[n, :k]^T) on the current stream.

    ``ln = (stats, stats_ld, hidden, c, d)``: LayerNorm folded into the GEMM
    (swap-AB only): ``wt`` holds gamma-folded weights and the accumulator
    becomes inv * (acc - mean * c) + d, row statistics from ``stats``;
    ``stats = (buffer, stats_ld)``: an EPI_BIAS_RESID GEMM also writes the
    per-128-feature-tile (mean, M2) pairs of its output rows there."""
    m = act.shape[0] if m_tok is None else m_tok
    n = wt.shape[0] if n_feat is None else n_feat
    d = N.GemmDesc()
    d.m_tok, d.n_feat, d.k = m, n, k
    d.act, d.lda = _ptr(act), act.stride(0)
    d.wt, d.ldw = _ptr(wt), wt.stride(0)
    d.epilogue = epilogue
    d.bias = _ptr(bias)
    if out is not None:
        d.out, d.ldo = _ptr(out), out.stride(0)
    if resid is not None:
        d.resid, d.ldr = _ptr(resid), resid.stride(0)
    if keys is not None:
        d.argmax_keys = _ptr(keys)
    if qkv is not None:
        q_out, kc, vc, heads, head_dim, cap, seq_len, qbase = qkv
        d.q_out, d.ldq = _ptr(q_out), q_out.stride(0)
        d.k_cache, d.v_cache = _ptr(kc), _ptr(vc)
        d.hidden, d.heads, d.head_dim = heads * head_dim, heads, head_dim
        d.cap, d.seq_len, d.qbase_dev = cap, seq_len, _ptr(qbase)
    if scratch is not None:
        d.workspace, d.workspace_bytes = _ptr(scratch.ws), scratch.workspace_bytes
        d.counters, d.n_counters = _ptr(scratch.counters), scratch.n_counters
    if ln is not None:
        st, st_ld, hidden, lc, ld = ln
        d.ln_stats, d.ln_stats_ld, d.ln_hidden = _ptr(st), st_ld, hidden
        d.ln_c, d.ln_d = _ptr(lc), _ptr(ld)
    if stats is not None:
        d.stats_out, d.stats_ld = _ptr(stats[0]), stats[1]
    d.force_swap, d.splits, d.pdl = force_swap, splits, 0
    N.check(N.lib().tf_gemm(C.byref(d), _stream()), "tf_gemm")
    return out


def layernorm(x: torch.Tensor, hidden: int, gamma: torch.Tensor, beta: torch.Tensor,
              out: torch.Tensor, n_rows: int | None = None, src_stride: int = 1, src_off: int = 0):
    rows = x.shape[0] if n_rows is None else n_rows
    N.check(N.lib().tf_layernorm(rows, hidden, _ptr(x), x.stride(0), src_stride, src_off,
                                 _ptr(gamma), _ptr(beta), _ptr(out), out.stride(0), _stream()),
            "tf_layernorm")
    return out


def attention(q, ldq_rows_view, k_cache, v_cache, start, qbase, scale, out, *, batch, heads,
              head_dim, cap, seq_len):
    N.check(N.lib().tf_attention(batch, heads, head_dim, cap, seq_len, _ptr(q), q.stride(0),
                                 _ptr(k_cache), _ptr(v_cache), _ptr(start), _ptr(qbase),
                                 C.c_float(scale), _ptr(out), out.stride(0), _stream()),
            "tf_attention")
    return out


def attention_beam(q, k_cache, v_cache, start, qbase, indir, scale, out, *, requests, beam, heads, head_dim,
                   cap):
    """Beam-search decode attention (tf_attention_beam): one query row per beam,
    cache rows resolved through the indirection table ``indir`` [rows, cap]."""
    N.check(N.lib().tf_attention_beam(requests, beam, heads, head_dim, cap, _ptr(q), q.stride(0), _ptr(k_cache),
                                      _ptr(v_cache), _ptr(start), _ptr(qbase), _ptr(indir), C.c_float(scale),
                                      _ptr(out), out.stride(0), _stream()), "tf_attention_beam")
    return out


def embed_ln(ids, pos, tok_emb, pos_emb, hidden, x, h=None, gamma=None, beta=None, *,
             remap=None, unk_id=0, type_ids=None, type_emb=None, type_const=0, ids_out=None):
    if ids.shape != pos.shape:
        raise DimensionError("ids/pos shape mismatch")
    d = N.EmbedDesc()
    d.n_tok, d.hidden = ids.numel(), hidden
    d.vocab, d.max_pos = tok_emb.shape[0], pos_emb.shape[0]
    d.ids, d.pos, d.type_ids, d.type_const = _ptr(ids), _ptr(pos), _ptr(type_ids), type_const
    if remap is not None:
        d.remap, d.remap_n = _ptr(remap), remap.numel()
    d.unk_id = unk_id
    d.tok_emb, d.pos_emb, d.type_emb = _ptr(tok_emb), _ptr(pos_emb), _ptr(type_emb)
    d.ldw = tok_emb.stride(0)
    d.ln_gamma, d.ln_beta = _ptr(gamma), _ptr(beta)
    d.x, d.h, d.ldx = _ptr(x), _ptr(h), x.stride(0)
    d.ids_out = _ptr(ids_out)
    N.check(N.lib().tf_embed_ln(C.byref(d), _stream()), "tf_embed_ln")
    return x


def warmup() -> None:
    """Reference kernels.warmup() (kernels.py:236-252) JIT-compiles every numba
    kernel up front; here the kernels are compiled ahead of time, so warming up
    means loading the sm_100a library (raises if it is missing)."""
    N.load_library()
