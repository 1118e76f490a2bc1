"""The reference's OWN test files, unmodified, run on the GPU against the
``tinfer`` name bound to this package (pkg/src/tinfer) — the drop-in check.

The files come from the byte-identical copy ``oracle/make_ref.py`` stages under
``oracle/_ref`` (git-ignored; it travels to the GPU box with the snapshot). Each
file runs in a subprocess with ``PYTHONPATH=pkg/src:<repo>`` so ``import tinfer``
resolves to this package and every model call runs the sm_100a kernels.

Known, documented deviations (EXPECTED below): the reference's F32 model path
is exact f32 arithmetic on the CPU, and a few of its tests assert bitwise or
1e-5 agreement with that arithmetic (or with an f64 straight-line forward).
This path stores f16 and accumulates f32 on tensor cores for every model
(DESIGN.md §4): those checks hold here within the north-star tolerance (they
are restated with tolerances / margin gating in tests/test_gpu_model.py and
tests/test_gpu_parity_tf.py), not bitwise. Everything else must pass as written
(``graph-opt`` reports the fused forward's plan, cli.py / workspace.py).
"""

import json
import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import make_ref  # noqa: E402

FILES = ["test_tokenizer.py", "test_pipeline.py", "test_pruning.py", "test_model.py", "test_bench.py",
         "test_cli.py"]
# test id (file::class::name) -> why it cannot hold on an f16 tensor-core path / is out of scope
_F16 = ("F32 model on an f16-storage path: the reference asserts exact f32 arithmetic; this path rounds F32 "
        "weights/activations to f16 (restated with the north-star tolerance in tests/test_gpu_model.py)")
EXPECTED: dict[str, str] = {
    "test_model.py::TestEmbed::test_single_token_definition": _F16 + " — the embedding of an F32 model is the "
    "f16-rounded sum, bit-exact for F16 models (tests/test_gpu_model.py)",
    "test_model.py::TestForwardFull::test_matches_straightline_oracle_tiny": _F16 + " — max-abs 9e-5 vs the "
    "1e-5 bound on an f64 straight-line forward",
    "test_model.py::TestForwardFull::test_matches_straightline_oracle_multihead": _F16 + " — max-abs 3.2e-4 vs "
    "the 1e-5 bound",
}


def _run(path, tmp_path):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "pkg", "src"), ROOT]))
    xml = tmp_path / (os.path.basename(path) + ".xml")
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "--rootdir", str(tmp_path),
                          f"--junitxml={xml}", path], env=env, cwd=str(tmp_path), capture_output=True, text=True,
                         timeout=3000)
    out = {}
    if xml.exists():
        for case in ET.parse(xml).getroot().iter("testcase"):
            cls = case.get("classname", "").split(".")[-1]
            tid = f"{os.path.basename(path)}::{cls}::{case.get('name')}"
            bad = case.find("failure") if case.find("failure") is not None else case.find("error")
            skipped = case.find("skipped") is not None
            out[tid] = "skipped" if skipped else ("failed" if bad is not None else "passed")
            if bad is not None:
                out[tid + "#msg"] = (bad.get("message") or "")[:300]
    return res, out


@pytest.mark.parametrize("name", FILES)
def test_reference_suite(cuda_device, tmp_path, name):
    root = make_ref.ref_root()
    if root is None:
        pytest.skip("reference copy not staged (python oracle/make_ref.py in the build container)")
    res, outcomes = _run(os.path.join(root, "tests", name), tmp_path)
    assert outcomes, res.stdout[-3000:] + res.stderr[-3000:]
    report = os.path.join(ROOT, "gpurun_out", "reference_suite")
    os.makedirs(report, exist_ok=True)
    with open(os.path.join(report, name + ".json"), "w") as fh:
        json.dump(outcomes, fh, indent=1, sort_keys=True)
    failed = sorted(t for t, v in outcomes.items() if v == "failed" and t not in EXPECTED)
    assert not failed, "\n".join(f"{t}: {outcomes.get(t + '#msg', '')}" for t in failed)
