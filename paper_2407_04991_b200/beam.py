"""Beam search on the device (north star (3), BASELINE configs[3] "C4").

The reference has no beam search, so the semantics are this
package's, stated once in ``oracle/tinfer_oracle.py::beam_search_decode`` (the
CPU restatement built on the reference's forward core) and implemented here on
the GPU:

* every request keeps ``beam_width`` hypotheses (rows ``r*K + k``); at step 0 only
  beam 0 is live;
* candidate score = beam score + log_softmax(f16-rounded logits) in f32; the top
  ``K`` over the flat (beam, token) index survive, ties to the lower index;
* a hypothesis that emitted eos is frozen (proposes only itself with eos); no
  length penalty;
* the result per request is the best final hypothesis (lowest beam index on
  ties), prompt included, cut after its first eos.

Device flow (one host sync): replicated prefill of the K copies of each prompt
-> ``tf_beam_select`` -> ``max_new - 1`` x (T=1 forward + select) replayed from
one CUDA graph. The KV cache is never reordered: decode attention reads slots
through a per-row indirection table that the select kernel rewrites.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .model import COUNTERS, ModelConfig, Model, _count_forward, _left_pad, _validate_prompts


def _backtrack(c: ModelConfig, prompts, scores, tok_hist, par_hist, K: int):
    out = []
    steps = tok_hist.shape[0]
    for r, prompt in enumerate(prompts):
        row = scores[r * K:(r + 1) * K]
        k = int(np.argmax(row))  # first max -> lowest beam index
        rev = []
        for t in range(steps - 1, -1, -1):
            b = r * K + k
            rev.append(int(tok_hist[t, b]))
            k = int(par_hist[t, b])
        gen = []
        for tok in reversed(rev):
            gen.append(tok)
            if tok == c.eos_token:
                break
        out.append(list(prompt) + gen)
    return out


def beam_search_decode(model: Model, prompts: list[list[int]], max_new_tokens: int,
                       beam_width: int = 4, use_graph: bool = True) -> list[list[int]]:
    """Beam search for a group of prompts; returns one sequence per prompt."""
    import torch

    from .errors import ParameterError

    c = model.config
    if not prompts:
        return []
    if not 1 <= beam_width <= 8:
        raise ParameterError("beam_width must be in [1, 8]")
    checked = _validate_prompts(c, prompts, max_new_tokens)
    if max_new_tokens == 0:
        return [list(p) for p in checked]
    R, K = len(checked), beam_width
    flat = [p for p in checked for _ in range(K)]
    ids, pos, pads, _ = _left_pad(c, flat)
    B, L = ids.shape
    cap = min(L + max_new_tokens, c.max_position)
    dm = model.device_model()
    with dm.lock, torch.cuda.device(dm.device):
        s = dm.session(B, cap, L, max_new_tokens, logits="last", beam=K)
        s.load_inputs(ids, pos, pads)
        s.indir.copy_((torch.arange(B, device=dm.device, dtype=torch.int32) % K)[:, None].expand(B, cap))
        init = torch.full((B,), float("-inf"), dtype=torch.float32, device=dm.device)
        init[::K] = 0.0
        s.scores.copy_(init)
        s.finished.zero_()
        d = N.BeamDesc()
        d.requests, d.beam, d.max_new, d.prompt_len, d.eos = R, K, max_new_tokens, L, c.eos_token
        d.scores, d.finished, d.tokens = s.scores.data_ptr(), s.finished.data_ptr(), s.beam_tokens.data_ptr()
        d.tok_hist, d.par_hist = s.tok_hist.data_ptr(), s.par_hist.data_ptr()
        stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        n_pre = s.forward(L, N.FWD_LOGITS_LAST)
        N.check(N.lib().tf_beam_select(s.handle, C.byref(d), stream), "tf_beam_select")
        if max_new_tokens > 1:
            N.check(N.lib().tf_beam_decode(s.handle, C.byref(d), max_new_tokens - 1,
                                           1 if use_graph else 0, stream), "tf_beam_decode")
            s.len += max_new_tokens - 1
        per_step = N.lib().tf_session_launches_per_step(s.handle)
        scores = s.scores.cpu().numpy()
        tok_hist = s.tok_hist.cpu().numpy()
        par_hist = s.par_hist.cpu().numpy()
    _count_forward(c, B, L, 0, int(pads.sum()), B, n_pre + 1)
    for step in range(1, max_new_tokens):
        _count_forward(c, B, 1, L + step - 1, int(pads.sum()), B, per_step)
    return _backtrack(c, checked, scores, tok_hist, par_hist, K)
