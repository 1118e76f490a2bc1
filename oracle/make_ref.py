"""Recipe: stage the UNMODIFIED reference package + its tests under oracle/_ref/
(TEST / BASELINE INFRASTRUCTURE ONLY; oracle/_ref/ is git-ignored, so no
reference source enters history, but it travels to the GPU box with the
snapshot like the built .so files).

    python oracle/make_ref.py          # run by __graft_entry__.build() when /root/reference exists

What uses it (never the product package):
* bench.py --impl reference / cpu_baseline: the reference's own numba CPU path
  (kernels.py:48-233 via model.batched_greedy_decode) timed on the box's cores;
* tests/test_gpu_reference_suite.py: the reference's own tests/*.py run on the
  GPU box against the ``tinfer`` name bound to this package (pkg/src/tinfer).

The files are copied byte for byte; a manifest with their sha256 is written
next to them so a stale or edited copy is detected.
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import sys

SRC = "/root/reference/pkg"
HERE = os.path.dirname(os.path.abspath(__file__))
DST = os.path.join(HERE, "_ref", "pkg")


def stage(src: str = SRC, dst: str = DST) -> str | None:
    if not os.path.isdir(src):
        return None
    manifest = {}
    for sub in ("src/tinfer", "tests"):
        os.makedirs(os.path.join(dst, sub), exist_ok=True)
        for name in sorted(os.listdir(os.path.join(src, sub))):
            if not name.endswith(".py"):
                continue
            a, b = os.path.join(src, sub, name), os.path.join(dst, sub, name)
            shutil.copyfile(a, b)
            with open(b, "rb") as fh:
                manifest[f"{sub}/{name}"] = hashlib.sha256(fh.read()).hexdigest()
    with open(os.path.join(dst, "MANIFEST.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
    return dst


def ref_root() -> str | None:
    """Where the reference package lives: the mount (build container) or the
    staged copy (GPU box)."""
    if os.path.isdir(os.path.join(SRC, "src", "tinfer")):
        return SRC
    if os.path.isdir(os.path.join(DST, "src", "tinfer")):
        return DST
    return None


if __name__ == "__main__":
    out = stage()
    print(out or "reference not mounted; nothing staged")
    sys.exit(0)
