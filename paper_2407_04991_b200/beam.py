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
from .model import ModelConfig, Model, _count_forward, _left_pad, _session_shape, _validate_prompts


def _backtrack(c: ModelConfig, prompts, scores, tok_hist, par_hist, K: int):
    """Best hypothesis per request (first max -> lowest beam index), followed back
    through the parent history for every request at once (one vectorised gather
    per step), cut after its first eos."""
    R, steps = len(prompts), tok_hist.shape[0]
    k = np.argmax(np.asarray(scores).reshape(R, K), axis=1)
    base = np.arange(R) * K
    toks = np.empty((R, steps), dtype=np.int64)
    for t in range(steps - 1, -1, -1):
        b = base + k
        toks[:, t] = tok_hist[t, b]
        k = par_hist[t, b]
    hit = toks == c.eos_token
    cut = np.where(hit.any(axis=1), hit.argmax(axis=1) + 1, steps)
    return [list(p) + toks[r, :cut[r]].tolist() for r, p in enumerate(prompts)]


class BeamRun:
    """Device state of one beam-search call (prepare -> run_device -> finish)."""

    def __init__(self, model: Model, prompts, max_new_tokens: int, beam_width: int, validated: bool = False):
        import torch

        from .errors import ParameterError

        c = model.config
        if not 1 <= beam_width <= 8:
            raise ParameterError("beam_width must be in [1, 8]")
        if beam_width > c.vocab_size:
            raise ParameterError("beam_width must not exceed vocab_size")
        self.model, self.c = model, c
        # validated: the caller already ran _validate_prompts on these prompts
        self.prompts = prompts if validated else _validate_prompts(c, prompts, max_new_tokens)
        self.new, self.K, self.R = max_new_tokens, beam_width, len(self.prompts)
        # each request's padded row repeated for its K beams
        ids, pos, pads, _ = _left_pad(c, self.prompts)
        self.ids, self.pos, self.pads = (np.repeat(a, self.K, axis=0) for a in (ids, pos, pads))
        self.B, self.L = self.ids.shape
        cap, max_tokens = _session_shape(c, self.L, max_new_tokens)
        self.dm = model.device_model()
        with torch.cuda.device(self.dm.device):
            self.s = self.dm.session(self.B, cap, max_tokens, max_new_tokens, logits="last", beam=self.K)
        d = N.BeamDesc()
        d.requests, d.beam, d.max_new, d.prompt_len, d.eos = self.R, self.K, max_new_tokens, self.L, c.eos_token
        s = self.s
        d.scores, d.finished, d.tokens = s.scores.data_ptr(), s.finished.data_ptr(), s.beam_tokens.data_ptr()
        d.tok_hist, d.par_hist = s.tok_hist.data_ptr(), s.par_hist.data_ptr()
        self.desc = d
        self.launches = 0

    def stage_inputs(self) -> int:
        """H2D of ids/positions/pads + device-side state init; returns H2D bytes."""
        import torch
        s, B, K = self.s, self.B, self.K
        nbytes = s.load_inputs(self.ids, self.pos, self.pads)
        s.indir.copy_((torch.arange(B, device=s.indir.device, dtype=torch.int32) % K)[:, None]
                      .expand(B, s.capacity))
        # prompt slots hold identical K/V in every beam row of a request: all
        # beams read them from beam 0's row (children inherit the entry), so the
        # shared prefix streams from DRAM once per request instead of once per beam
        s.indir[:, :self.L] = 0
        s.scores.fill_(float("-inf"))
        s.scores[::K] = 0.0
        s.finished.zero_()
        return nbytes

    def run_device(self, use_graph: bool = True) -> None:
        import torch
        s = self.s
        stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        n_pre = s.forward(self.L, N.FWD_LOGITS_LAST)
        N.check(N.lib().tf_beam_select(s.handle, C.byref(self.desc), stream), "tf_beam_select")
        per_step = 0
        if self.new > 1:
            N.check(N.lib().tf_beam_decode(s.handle, C.byref(self.desc), self.new - 1,
                                           1 if use_graph else 0, stream), "tf_beam_decode")
            s.len += self.new - 1
            per_step = N.lib().tf_session_launches_per_step(s.handle)
        self.launches = n_pre + 1 + (self.new - 1) * per_step
        _count_forward(self.c, self.B, self.L, 0, int(self.pads.sum()), self.B, n_pre + 1)
        for step in range(1, self.new):
            _count_forward(self.c, self.B, 1, self.L + step - 1, int(self.pads.sum()), self.B, per_step)

    def finish(self):
        """D2H of scores and histories, host backtrack; returns (seqs, D2H bytes)."""
        s = self.s
        scores = s.scores.cpu().numpy()
        tok_hist = s.tok_hist.cpu().numpy()
        par_hist = s.par_hist.cpu().numpy()
        nbytes = scores.nbytes + tok_hist.nbytes + par_hist.nbytes
        return _backtrack(self.c, self.prompts, scores, tok_hist, par_hist, self.K), nbytes


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
    if beam_width > c.vocab_size:
        raise ParameterError("beam_width must not exceed vocab_size")
    checked = _validate_prompts(c, prompts, max_new_tokens)
    if max_new_tokens == 0:
        return [list(p) for p in checked]
    dm = model.device_model()
    with dm.lock, torch.cuda.device(dm.device):  # the session is created and used under the lock
        run = BeamRun(model, checked, max_new_tokens, beam_width, validated=True)
        h2d = run.stage_inputs()
        run.run_device(use_graph)
        seqs, d2h = run.finish()
    from . import model as M
    st = M.GenerateStats()
    st.h2d_bytes, st.d2h_bytes, st.launches = h2d, d2h, run.launches
    M.LAST_STATS = st
    return seqs
