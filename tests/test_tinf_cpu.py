"""TINF v1 header index and memory-mapped view (the host half of the
direct-to-device loader) agree with the reference-format reader, and reject
the same malformed files (tensor.py:179-232)."""

import numpy as np
import pytest

import paper_2407_04991_b200 as P
from paper_2407_04991_b200.errors import FormatError
from paper_2407_04991_b200.tensor import map_tinf, tinf_index


@pytest.mark.parametrize("dtype", [P.DType.F32, P.DType.F16])
def test_map_equals_read(tmp_path, dtype):
    m = P.init_random(P.ModelConfig(64, 16, 2, 2, 8, 32, 24, dtype, 1, 2), 3)
    path = str(tmp_path / "m.tinf")
    P.write_tinf(path, m.named_tensors())
    a, b = map_tinf(path), P.read_tinf(path)
    assert [n for n, _ in a] == [n for n, _ in b]
    for (_, x), (_, y) in zip(a, b):
        assert x.dtype is y.dtype and np.array_equal(x.array, y.array)
    idx = tinf_index(path)
    assert [e[2] for e in idx] == [t.shape for _, t in b]


def test_index_rejects_truncated_and_bad_magic(tmp_path):
    m = P.init_random(P.ModelConfig(64, 16, 1, 2, 8, 32, 24, P.DType.F16, 1, 2), 3)
    path = tmp_path / "m.tinf"
    P.write_tinf(str(path), m.named_tensors())
    data = path.read_bytes()
    (tmp_path / "t.tinf").write_bytes(data[:-3])
    with pytest.raises(FormatError):
        tinf_index(str(tmp_path / "t.tinf"))
    (tmp_path / "b.tinf").write_bytes(b"XXXX" + data[4:])
    with pytest.raises(FormatError):
        tinf_index(str(tmp_path / "b.tinf"))
