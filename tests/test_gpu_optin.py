"""The A/B switches of the decode path stay correct: each runs the smoke
generation in a fresh process (the switches are read once per process) and is
checked against the oracle with the same margin-gated protocol."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [
    {"TF_LN_FUSE": "0"},    # stand-alone LayerNorm kernels instead of the fused statistics path
    {"TF_L2PF": "0"},       # no next-layer L2 prefetch
])
def test_decode_switch_matches_oracle(cuda_device, env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.smoke()"], cwd=ROOT, env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "smoke ok" in r.stdout
