"""Host-side matrix file I/O (matcore.py:154-204): format, round trip and
the error cases the reference raises MatrixInputError for."""
import numpy as np
import pytest

from paper_2010_00465_b200 import MatrixInputError, read_matrix, write_matrix


def test_round_trip_is_exact(tmp_path, rng):
    a = rng.standard_normal((7, 5)) * 10.0 ** rng.uniform(-200, 200, (7, 5))
    p = tmp_path / "m.txt"
    write_matrix(str(p), a)
    b = read_matrix(str(p))
    assert b.dtype == np.float64 and b.shape == (7, 5)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    assert p.read_text().splitlines()[0] == "7 5"


def test_blank_lines_ignored(tmp_path):
    p = tmp_path / "m.txt"
    p.write_text("\n2 2\n\n1 2\n  \n3.5 -4e-3\n\n")
    assert np.array_equal(read_matrix(str(p)), [[1.0, 2.0], [3.5, -4e-3]])


@pytest.mark.parametrize("text,frag", [
    ("", "empty file"),
    ("2\n1 2\n", "header"),
    ("a b\n1\n", "non-integer"),
    ("0 2\n", "positive"),
    ("2 2\n1 2\n", "expected 2 data lines"),
    ("2 2\n1 2\n3\n", "line 3: expected 2 entries"),
    ("1 2\n1 x\n", "non-numeric"),
    ("1 1\nnan\n", "finite"),
    ("1 1\ninf\n", "finite"),
])
def test_malformed_files_raise(tmp_path, text, frag):
    p = tmp_path / "bad.txt"
    p.write_text(text)
    with pytest.raises(MatrixInputError) as ei:
        read_matrix(str(p))
    assert frag in str(ei.value)
    assert str(p) in str(ei.value)
