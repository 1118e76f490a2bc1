"""Alias loader for the reference hot path (`tinfer_ref`) — TEST INFRASTRUCTURE ONLY.

Used by ``tests/golden/make_golden.py`` inside the build container to import the
UNMODIFIED reference modules from ``/root/reference/pkg/src/tinfer`` and generate
golden vectors, and by ``bench.py``'s reference arm / cpu_baseline on the GPU box
(from the byte-identical copy ``oracle/make_ref.py`` stages under ``oracle/_ref``)
to time the reference's own numba CPU path. Never imported by the product package.

Why a loader: the reference ``tinfer/__init__.py:41`` imports ``tinfer.tokenizer``,
which is missing from the mount, so ``import tinfer`` fails. The
hot-path modules (errors, rng, kernels, tensor, model) do not need it; pruning and
pipeline import it only for type names, so a stub module with those names suffices
(SURVEY §8c).
"""

from __future__ import annotations

import importlib.util
import os
import sys
import types

PKG = "tinfer_ref"


def _ref_src() -> str:
    """The reference package: the mount (build container) or the copy staged by
    oracle/make_ref.py under oracle/_ref (travels to the GPU box)."""
    from oracle import make_ref
    root = make_ref.ref_root()
    return os.path.join(root, "src", "tinfer") if root else "/root/reference/pkg/src/tinfer"


REF_SRC = _ref_src()


def load(with_pruning: bool = True):
    """Return the ``tinfer_ref`` package with errors/rng/kernels/tensor/model
    (and pruning/pipeline, via a tokenizer stub) loaded from the reference."""
    if PKG in sys.modules and hasattr(sys.modules[PKG], "model"):
        return sys.modules[PKG]
    if not os.path.isdir(REF_SRC):
        raise RuntimeError(f"reference sources not found at {REF_SRC}")
    # numba cache=True pickles the module name; a cache dir populated under
    # another name breaks alias loads (SURVEY §8c trap)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tinfer_ref_numba_cache")
    pkg = types.ModuleType(PKG)
    pkg.__path__ = [REF_SRC]
    sys.modules[PKG] = pkg
    names = ["errors", "rng", "kernels", "tensor", "model"]
    if with_pruning:
        stub = types.ModuleType(f"{PKG}.tokenizer")

        class Tokenizer:  # type-name stub only; never called by the selection code
            pass

        class Vocab:
            pass

        stub.Tokenizer = Tokenizer
        stub.Vocab = Vocab
        sys.modules[stub.__name__] = stub
        pkg.tokenizer = stub
        names += ["pruning", "pipeline"]
    for n in names:
        spec = importlib.util.spec_from_file_location(f"{PKG}.{n}", f"{REF_SRC}/{n}.py")
        m = importlib.util.module_from_spec(spec)
        sys.modules[spec.name] = m
        spec.loader.exec_module(m)
        setattr(pkg, n, m)
    return pkg
