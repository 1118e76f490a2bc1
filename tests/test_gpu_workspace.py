"""Planned session arenas on the device (workspace.py).

Sessions carve x / h / q / attn / ffn out of one arena in which the
lifetime-disjoint buffers share storage ({ffn, q}, {h, attn}). Generation with
the planned arena must equal generation with every buffer separate BITWISE —
greedy (prefill + graph-replayed decode), beam search, and full-sequence
logits — which is the reference's "planned matches fresh bitwise" contract
(test_graphopt.py:392-402) applied to the native forward.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2407_04991_b200 as P  # noqa: E402
from paper_2407_04991_b200 import workspace as W  # noqa: E402


def _cfg():
    # no padding columns (hidden, ffn multiples of 64), so the plan shares
    return P.ModelConfig(512, 128, 2, 2, 64, 256, 128, P.DType.F16, 1, 2)


def _unshared(rows, hidden, ffn, ldk_h, ldk_f, n_layers):
    sizes = {"x": rows * ldk_h * 2, "h": rows * ldk_h * 2, "q": rows * ldk_h * 2,
             "attn": rows * ldk_h * 2, "ffn": rows * ldk_f * 2}
    return W.plan_memory(sizes, {n: [(0, 1 << 30)] for n in sizes})


def _run(model, prompts):
    greedy = P.batched_greedy_decode(model, prompts, 12)
    beam = P.beam_search_decode(model, prompts[:2], 8, beam_width=3)
    logits = P.forward_full(model, prompts[1]).array
    return greedy, beam, logits


def test_planned_arena_matches_separate_buffers(cuda_device, monkeypatch):
    model = P.init_random(_cfg(), seed=5)
    rng = np.random.default_rng(3)
    prompts = [rng.integers(3, 512, size=n).tolist() for n in (9, 17, 5, 30)]
    dm = model.device_model()
    s = dm.session(4, 64, 32, 12)
    assert s.plan.buffer_count == 3
    assert s.q.data_ptr() == s.ffn.data_ptr() and s.h.data_ptr() == s.attn.data_ptr()
    planned = _run(model, prompts)
    dm.close()
    model._f32 = None  # the memo token: a fresh device mirror, new sessions with the unshared plan
    monkeypatch.setattr(W, "session_plan", _unshared)
    dm2 = model.device_model()
    s2 = dm2.session(4, 64, 32, 12)
    assert s2.plan.buffer_count == 5
    fresh = _run(model, prompts)
    assert planned[0] == fresh[0]
    assert planned[1] == fresh[1]
    assert np.array_equal(planned[2], fresh[2])
