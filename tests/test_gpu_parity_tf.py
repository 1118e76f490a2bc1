"""Teacher-forced parity at the BENCHMARKED configs against the unmodified
reference (tests/golden/make_golden_tf.py; SURVEY §8c protocol).

C2 (Ernie-base-sized, 512 positions, batch 32, src 128, 64 new) and C3 (vocab
pruned 40k -> 10k, 256 positions, batch 128, src 128, 64 new) run on the GPU
through the native session with the reference's own generated tokens fed back
at every step (teacher forcing), so every (step, row) is compared -- not only
the prefix before a row's first low-margin divergence:

* logits: the GPU's f16 logits at the reference's top-5 ids are within
  LOGIT_TOL (max-abs 2e-2, the north-star tolerance) of the reference's;
* tokens: the GPU argmax equals the reference token wherever the reference's
  top-1 margin exceeds 2 x LOGIT_TOL (below that, f16 accumulation-order
  differences may legitimately flip it).

Hidden states: the 2L+1 LayerNorm inputs at the last
position of two C2 prompts, against the reference's F16 path (same quantisation
points) and F32 path.
"""

import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import bench  # noqa: E402  (the bench's model construction: same weights as the golden)
import paper_2407_04991_b200 as P  # noqa: E402
from paper_2407_04991_b200 import _native as N  # noqa: E402
from conftest import golden  # noqa: E402

LOGIT_TOL = 2e-2
MARGIN = 2 * LOGIT_TOL
# hidden states: max-abs error relative to the tap's own scale (max |x| of
# that tap), vs the reference F16 path and F32 path
TAP_TOL_F16 = 5e-3
TAP_TOL_F32 = 5e-3
REPORT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                      "parity_tf_report.json")

_models = {}


def model_for(wname):
    if wname not in _models:
        _models[wname] = bench.build_model(bench.WORKLOADS[wname])
    return _models[wname]


def _report(key, value):
    os.makedirs(os.path.dirname(REPORT), exist_ok=True)
    data = {}
    if os.path.exists(REPORT):
        with open(REPORT) as fh:
            data = json.load(fh)
    data[key] = value
    with open(REPORT, "w") as fh:
        json.dump(data, fh, indent=1)


def teacher_forced_check(model, g):
    """Run prefill + (new - 1) decode steps fed with the reference tokens;
    yield (step, logits [B, V] f32) for each of the `new` logit rows."""
    prompts, tokens = g["prompts"], g["tokens"]
    B, L = prompts.shape
    new = g["top5_ids"].shape[0]
    dm = model.device_model()
    pads = np.zeros(B, np.int32)
    with dm.lock, torch.cuda.device(dm.device):
        s = dm.session(B, L + new, L, 1, logits="last")
        s.load_inputs(prompts.astype(np.int32), np.broadcast_to(np.arange(L, dtype=np.int32), (B, L)).copy(), pads)
        s.forward(L, N.FWD_LOGITS_LAST)
        yield 0, s.logits[:B].float().cpu().numpy()
        for step in range(1, new):
            slot = L + step - 1
            ids = tokens[:, slot].astype(np.int32).reshape(B, 1)
            s.load_inputs(ids, np.full((B, 1), slot, np.int32), pads, length=slot)
            s.forward(1, N.FWD_LOGITS_LAST)
            yield step, s.logits[:B].float().cpu().numpy()


@pytest.mark.parametrize("wname", ["c2", "c3"])
def test_teacher_forced_logits_and_tokens(cuda_device, wname):
    g = golden(f"{wname}_tf.npz")
    model = model_for(wname)
    ids5, vals5, margin = g["top5_ids"], g["top5_vals"].astype(np.float32), g["margin"]
    worst, checked, gated, flips = 0.0, 0, 0, []
    for step, lg in teacher_forced_check(model, g):
        got5 = np.take_along_axis(lg, ids5[step].astype(np.int64), axis=1)
        worst = max(worst, float(np.max(np.abs(got5 - vals5[step]))))
        am = lg.argmax(axis=1)
        sure = margin[step] > MARGIN
        checked += int(sure.sum())
        gated += int((~sure).sum())
        bad = np.nonzero(sure & (am != ids5[step, :, 0]))[0]
        flips += [(step, int(b), int(am[b]), int(ids5[step, b, 0]), float(margin[step, b])) for b in bad]
    _report(f"{wname}_teacher_forced", {"max_abs_top5_logit_err": worst, "tokens_checked": checked,
                                        "low_margin_skipped": gated, "flips": flips[:20]})
    assert worst <= LOGIT_TOL, worst
    assert not flips, flips[:10]
    assert checked > 0.8 * (checked + gated)


def test_hidden_state_taps_c2(cuda_device):
    g = golden("c2_taps.npz")
    model = model_for("c2")
    L = model.config.num_layers
    errs = {"f16": [], "f32": []}
    for r, p in enumerate(g["prompts"]):
        taps = P.hidden_states(model, p.tolist()).array.astype(np.float32)
        assert taps.shape == (2 * L + 1, len(p), model.config.hidden_size)
        last = taps[:, -1]
        for tag in ("f16", "f32"):
            ref = g[f"taps_{tag}"][r]
            scale = np.maximum(1.0, np.abs(ref).max(axis=1))
            errs[tag].append((np.abs(last - ref).max(axis=1) / scale).tolist())
        # taps[0] is the embedding sum: bit-exact vs the reference F16 path
        assert np.array_equal(last[0], g["taps_f16"][r][0])
    _report("c2_taps", {k: [max(v) for v in zip(*e)] for k, e in errs.items()})
    assert max(max(e) for e in errs["f16"]) <= TAP_TOL_F16
    assert max(max(e) for e in errs["f32"]) <= TAP_TOL_F32
