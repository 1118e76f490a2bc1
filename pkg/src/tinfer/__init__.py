"""``tinfer`` — the reference package name (pkg/src/tinfer) bound to the B200 path.

A user of the reference keeps ``import tinfer`` / ``from tinfer.model import
...`` and gets the sm_100a implementation: each reference module name is an
alias of the module here that restates it (same objects, so ``isinstance`` and
``except`` clauses work across both names):

    tinfer.errors    -> paper_2407_04991_b200.errors     (errors.py)
    tinfer.rng       -> paper_2407_04991_b200.rng        (rng.py)
    tinfer.tensor    -> paper_2407_04991_b200.tensor     (tensor.py: DType, Tensor, TINF IO)
    tinfer.model     -> paper_2407_04991_b200.model      (model.py: the generation API)
    tinfer.kernels   -> paper_2407_04991_b200.ops        (kernels.py: operator API over the C ABI)
    tinfer.pruning   -> paper_2407_04991_b200.pruning    (pruning.py)
    tinfer.tokenizer -> paper_2407_04991_b200.tokenizer  (the tokenizer the reference imports)
    tinfer.pipeline  -> paper_2407_04991_b200.pipeline   (pipeline.py)
    tinfer.bench     -> paper_2407_04991_b200.ladder     (bench.py: the ablation ladder)
    tinfer.cli       -> paper_2407_04991_b200.cli        (cli.py)

Not provided: ``tinfer.graphopt`` (the operator-graph IR; outside the
generation hot path).
"""

from __future__ import annotations

import importlib
import os
import sys

_ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..", ".."))
if os.path.isdir(os.path.join(_ROOT, "paper_2407_04991_b200")) and _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

_IMPL = "paper_2407_04991_b200"
_ALIASES = {"errors": "errors", "rng": "rng", "tensor": "tensor", "model": "model", "kernels": "ops",
            "pruning": "pruning", "tokenizer": "tokenizer", "pipeline": "pipeline", "bench": "ladder",
            "cli": "cli"}

for _name, _target in _ALIASES.items():
    _mod = importlib.import_module(f"{_IMPL}.{_target}")
    sys.modules[f"{__name__}.{_name}"] = _mod
    globals()[_name] = _mod

from paper_2407_04991_b200 import *  # noqa: E402,F401,F403  (the reference's top-level re-exports)
from paper_2407_04991_b200 import __version__  # noqa: E402,F401
