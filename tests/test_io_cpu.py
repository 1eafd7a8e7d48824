"""Host-side COO ingestion (coo.py:95-157 of the reference): text round trip, comments, 1-based
coordinates, min-max normalisation, and the reference's error messages (ParseError /
ValidationError naming the offending line), mirroring pkg/tests/test_tensor_store.py:20-79."""

import numpy as np
import pytest

from paper_2210_06014_b200.coo import SparseCooTensor, load_coo, split_dataset, write_coo
from paper_2210_06014_b200.errors import ConfigError, ParseError, ValidationError


def _write(tmp_path, text):
    p = tmp_path / "t.tns"
    p.write_text(text)
    return p


def test_round_trip(tmp_path):
    rng = np.random.default_rng(1)
    idx = np.unique(rng.integers(0, 7, size=(60, 3)), axis=0)
    vals = rng.normal(size=idx.shape[0])
    t = SparseCooTensor((7, 7, 7), idx, vals)
    p = tmp_path / "x.tns"
    write_coo(p, t)
    back = load_coo(p, 3, dims=(7, 7, 7))
    assert np.array_equal(back.idx, t.idx) and np.array_equal(back.vals, t.vals)
    assert back.dims == (7, 7, 7)


def test_comments_blank_lines_and_default_dims(tmp_path):
    p = _write(tmp_path, "# header\n\n1 1 1 2.5\n3 2 4 -1\n# tail\n")
    t = load_coo(p, 3)
    assert t.dims == (3, 2, 4)
    assert t.idx.tolist() == [[0, 0, 0], [2, 1, 3]]
    assert t.vals.tolist() == [2.5, -1.0]


@pytest.mark.parametrize("text,exc,msg", [
    ("1 1 1 5.0 # c\n", ParseError, "line 1: expected 4 fields, got 6"),   # inline '#'
    ("1 1 1 2\n1 2 3\n", ParseError, "line 2: expected 4 fields, got 3"),
    ("1 1 1 2\n1 x 1 2\n", ParseError, "line 2: bad coordinate"),
    ("1 1 1 2\n1 2 1 abc\n", ParseError, "line 2: bad value 'abc'"),
    ("1 1 1 2\n0 2 1 1\n", ValidationError, "line 2: coordinates are 1-based"),
    ("1 1 1 2\n2 2 2 1\n1 1 1 3\n", ValidationError, r"line 3: duplicate coordinate \(1, 1, 1\)"),
    ("# only comments\n", ValidationError, "no entries"),
])
def test_errors_name_the_line(tmp_path, text, exc, msg):
    with pytest.raises(exc, match=msg):
        load_coo(_write(tmp_path, text), 3)


def test_normalize(tmp_path):
    t = load_coo(_write(tmp_path, "1 1 1 10\n1 1 2 20\n1 1 3 30\n"), 3, normalize=(1, 5))
    assert t.vals.tolist() == [1.0, 3.0, 5.0]
    with pytest.raises(ConfigError):
        load_coo(_write(tmp_path, "1 1 1 2\n1 1 2 2\n"), 3, normalize=(1, 5))


def test_tensor_validation():
    with pytest.raises(ValidationError, match="order must be >= 3"):
        SparseCooTensor((3, 3), np.zeros((1, 2), int), [1.0])
    with pytest.raises(ValidationError, match="out of range"):
        SparseCooTensor((3, 3, 3), [[0, 0, 3]], [1.0])
    with pytest.raises(ValidationError, match=r"duplicate coordinate \(1, 2, 3\)"):
        SparseCooTensor((3, 3, 3), [[0, 1, 2], [1, 1, 1], [0, 1, 2]], [1.0, 2.0, 3.0])
    with pytest.raises(ValidationError, match="at least one entry"):
        SparseCooTensor((3, 3, 3), np.zeros((0, 3), int), [])


def test_split_partition_law():
    rng = np.random.default_rng(3)
    idx = np.unique(rng.integers(0, 20, size=(500, 3)), axis=0)
    t = SparseCooTensor((20, 20, 20), idx, rng.uniform(size=idx.shape[0]))
    s = split_dataset(t, 0.1, seed=4)
    assert s.test.nnz == int(round(t.nnz * 0.1)) and s.train.nnz + s.test.nnz == t.nnz
    both = np.concatenate([s.train.idx, s.test.idx])
    assert np.unique(both, axis=0).shape[0] == t.nnz
    s2 = split_dataset(t, 0.1, seed=4)
    assert np.array_equal(s.test.idx, s2.test.idx)
    with pytest.raises(ConfigError):
        split_dataset(t, 1.0, seed=0)


def test_nan_value_loads_like_the_reference(tmp_path):
    """float('nan') is a value the reference's scanner accepts (coo.py:118-121)."""
    t = load_coo(_write(tmp_path, "1 1 1 nan\n2 1 1 3\n"), 3)
    assert np.isnan(t.vals[0]) and t.vals[1] == 3.0


def test_comment_only_file_has_no_entries(tmp_path):
    with pytest.raises(ValidationError, match="no entries"):
        load_coo(_write(tmp_path, "# nothing\n\n"), 3)
