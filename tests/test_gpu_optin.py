"""The opt-in decode variants (measured slower than the default path, kept for
A/B measurements) stay correct: each runs the smoke generation
in a fresh process (the switches are read once per process) and is checked
against the oracle with the same margin-gated protocol."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [
    {"TF_DGEMM": "1"},      # whole-K narrow-tile decode GEMM, LN fused into the operand
    {"TF_LN_COOP": "1"},    # cluster-cooperative LN in the QKV / FFN1 split-K GEMMs
    {"TF_ROWLN": "1"},      # residual GEMMs as one whole-row cluster with the LayerNorm in the epilogue
    {"TF_L2PF": "0"},       # no next-layer L2 prefetch
    {"TF_LN_TAIL": "1"},    # LayerNorm of a row by the CTA that completes it in the residual GEMM
    {"TF_PF_PERSIST": "1"},  # persistent prefill GEMM with two TMEM accumulators
    {"TF_ATTN_WO": "1"},    # output projection inside the attention + head-sum/residual/LN row kernel
])
def test_optin_decode_variant_matches_oracle(cuda_device, env):
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", "import __graft_entry__ as g; g.smoke()"], cwd=ROOT, env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "smoke ok" in r.stdout
