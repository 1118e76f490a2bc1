"""The beam attention plan written by the cluster select (TF_BEAM_PLAN, default
on) must reproduce the attention CTAs' own derivation of it exactly: the same
units in the same order, so generation is bitwise identical with the plan and
without it, across beam widths 2..8, ragged prompts (left pads) and windows
crossing several 64-slot chunks. Each setting runs in a child process (the
switch is read once per process)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np
import paper_2407_04991_b200 as P
cfg = P.ModelConfig(512, 128, 2, 2, 64, 256, 512, P.DType.F16, 1, 2)
m = P.init_random(cfg, 17)
rng = np.random.default_rng(5)
out = {}
for K, lens, new in ((2, (3, 70, 130), 40), (3, (100, 9), 30), (5, (64, 65, 1), 24), (8, (150, 20), 20)):
    prompts = [rng.integers(3, 512, size=n).tolist() for n in lens]
    out[str(K)] = P.beam_search_decode(m, prompts, new, beam_width=K)
print(json.dumps(out))
"""


def _run(plan: str):
    env = dict(os.environ, TF_BEAM_PLAN=plan, PYTHONPATH=ROOT)
    res = subprocess.run([sys.executable, "-c", CHILD], env=env, cwd=ROOT, capture_output=True, text=True,
                         timeout=900)
    assert res.returncode == 0, res.stderr[-3000:]
    return json.loads(res.stdout.strip().splitlines()[-1])


def test_beam_plan_matches_in_kernel_derivation(cuda_device):
    with_plan, without = _run("1"), _run("0")
    assert with_plan.keys() == without.keys()
    for k in with_plan:
        assert with_plan[k] == without[k], k
