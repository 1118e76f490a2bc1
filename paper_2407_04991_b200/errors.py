"""Error taxonomy of the generation path.

Names and meanings mirror the reference ``tinfer.errors`` (errors.py:9-62) so
callers can catch the same classes. The native library never throws: every
C-ABI entry point returns an ``int`` status, and :func:`raise_for_status` maps a
non-zero status onto the matching class here (include/tinfer_sm100.h lists the
codes).
"""

from __future__ import annotations


class TinferError(Exception):
    """Root of every error raised by this package."""


class DimensionError(TinferError):
    """Operand shapes disagree."""


class PrecisionError(TinferError):
    """Operand storage precisions disagree."""


class NumericError(TinferError):
    """A non-finite value where only finite values are allowed."""


class ConfigError(TinferError):
    """A model configuration breaks one of its invariants."""


class VocabError(TinferError):
    """A token id or vocabulary entry is invalid."""


class PositionError(TinferError):
    """A position lies outside the model's position table."""


class CapacityError(TinferError):
    """The KV cache has no free slot left."""


class ParameterError(TinferError):
    """An argument lies outside its documented range."""


class FormatError(TinferError):
    """A weight, vocabulary or dataset file is malformed."""


class CorrectnessError(TinferError):
    """An equivalence check failed; results must not be trusted or timed."""


class BindingError(TinferError):
    """Reference graph-optimizer error (graphopt); defined for ``except`` compatibility."""


class GraphError(TinferError):
    """Reference graph-optimizer error (graphopt); defined for ``except`` compatibility."""


class PlanError(TinferError):
    """Reference arena-planner error (graphopt); defined for ``except`` compatibility."""


class DeviceError(TinferError):
    """The CUDA extension is missing, or a kernel launch / CUDA call failed."""


# C-ABI status codes (include/tinfer_sm100.h, enum tf_status)
TF_OK = 0
TF_ERR_ARG = 1
TF_ERR_SHAPE = 2
TF_ERR_CUDA = 3
TF_ERR_UNSUPPORTED = 4
TF_ERR_CAPACITY = 5

_STATUS_CLASS = {
    TF_ERR_ARG: ParameterError,
    TF_ERR_SHAPE: DimensionError,
    TF_ERR_CUDA: DeviceError,
    TF_ERR_UNSUPPORTED: DeviceError,
    TF_ERR_CAPACITY: CapacityError,
}


def raise_for_status(status: int, what: str, detail: str = "") -> None:
    """Translate a C-ABI status into the matching exception (no-op on 0)."""
    if status == TF_OK:
        return
    cls = _STATUS_CLASS.get(status, DeviceError)
    msg = f"{what} failed with status {status}"
    if detail:
        msg += f": {detail}"
    raise cls(msg)
