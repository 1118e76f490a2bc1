"""Beam-grouped decode attention (attn_decode_beam_ring_kernel: one CTA per
(head, request), shared prompt chunks staged once for all beams) is bitwise the
per-row kernel (attn_decode_pf_kernel, TF_ATTN_BEAM=0): same per-chunk
arithmetic and merge order. Compared on the final beam scores and the
token/parent histories of whole beam searches, with ragged prompts (left pad,
partially shared chunks), beam widths 2/3/4/8 (8: the plane pool forces
several staging batches / ring turns; 2-5 take the two-CTAs-per-SM ring) and windows up to 8 chunks. The oracle comparison of
beam search itself is test_gpu_beam.py."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def dump(tmp_path, tag, env, K, new, lens):
    out = str(tmp_path / f"{tag}.npz")
    e = dict(os.environ)
    e.update(env)
    e["PYTHONPATH"] = ROOT + os.pathsep + e.get("PYTHONPATH", "")
    r = subprocess.run([sys.executable, "tests/_beam_dump.py", out, str(K), str(new), lens], cwd=ROOT, env=e,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return np.load(out)


@pytest.mark.parametrize("K,new,lens", [
    (4, 40, "300,130,257,64,1,90"),
    (3, 24, "200,17,129"),
    (8, 30, "420,60"),
    (2, 20, "64,63,65"),
])
def test_beam_kernel_bitwise_per_row_kernel(cuda_device, tmp_path, K, new, lens):
    b = dump(tmp_path, "rows", {"TF_ATTN_BEAM": "0"}, K, new, lens)
    a = dump(tmp_path, "beam", {"TF_ATTN_BEAM": "2"}, K, new, lens)
    for k in ("scores", "tok", "par", "seqs"):
        assert np.array_equal(a[k], b[k]), k
    assert np.isfinite(b["scores"]).any()
