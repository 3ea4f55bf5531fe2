"""Matrix Market / permutation I/O (mmio.py): the reference's documented
semantics (mmio.py:1-9) — coordinate real/integer general/symmetric/
skew-symmetric, square only, explicit zeros kept, duplicates summed,
symmetric storage mirrored — and exact round trips."""

import io

import numpy as np
import pytest

import paper_1812_06160_b200 as jv
from paper_1812_06160_b200.errors import MatrixFormatError
from paper_1812_06160_b200 import workloads as W

G = """%%MatrixMarket matrix coordinate real general
% a comment
2 2 4
1 1 4.0
2 1 1.0

1 2 2.0
2 2 3.0
"""


def test_general():
    a = jv.parse_matrix_market(G)
    assert a.n == 2 and a.nnz == 4
    assert np.array_equal(a.to_dense(), [[4.0, 2.0], [1.0, 3.0]])
    assert np.array_equal(jv.parse_matrix_market(G.encode()).to_dense(), a.to_dense())


def test_symmetric_and_skew_and_integer():
    s = jv.parse_matrix_market("%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 2.0\n2 1 1.0\n")
    assert np.array_equal(s.to_dense(), [[2.0, 1.0], [1.0, 0.0]]) and s.nnz == 3
    k = jv.parse_matrix_market("%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 3.0\n")
    assert np.array_equal(k.to_dense(), [[0.0, -3.0], [3.0, 0.0]])
    i = jv.parse_matrix_market("%%MatrixMarket matrix coordinate integer general\n1 1 1\n1 1 7\n")
    assert i.to_dense()[0, 0] == 7.0


def test_explicit_zero_kept_and_duplicates_summed():
    a = jv.parse_matrix_market(
        "%%MatrixMarket matrix coordinate real general\n2 2 4\n1 1 0.0\n2 2 1.5\n2 2 2.5\n1 2 1\n")
    assert a.nnz == 3
    assert list(a.row_cols(0)) == [0, 1] and a.row_vals(0)[0] == 0.0
    assert list(a.row_vals(1)) == [4.0]


@pytest.mark.parametrize("text, msg", [
    ("%%MatrixMarket matrix array real general\n1 1\n1\n", "layout"),
    ("%%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n", "pattern"),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n", "field"),
    ("%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n", "symmetry"),
    ("%%MatrixMarket matrix coordinate real general\n2 3 0\n", "square"),
    ("%%MatrixMarket matrix coordinate real general\n", "size"),
    ("%%MatrixMarket matrix coordinate real general\n2 2\n", "size"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", "out of range"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n", "entry"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n", "entry"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", "declared"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 1.0\n", "more entries"),
    ("%%MatrixMarket tensor coordinate real general\n1 1 1\n1 1 1\n", "header"),
])
def test_errors(text, msg):
    with pytest.raises(MatrixFormatError, match=msg):
        jv.parse_matrix_market(text)


def test_round_trip_exact(tmp_path):
    a = W.random_diag_dominant(300, 7, seed=4)
    a.val[5] = 0.0                       # explicit zero survives
    a.val[7] = 1.0 / 3.0
    p = tmp_path / "a.mtx"
    jv.write_matrix_market_file(a, p)
    b = jv.read_matrix_market_file(p)
    assert np.array_equal(b.row_start, a.row_start) and np.array_equal(b.col, a.col)
    assert np.array_equal(b.val, a.val)
    buf = io.StringIO()
    jv.write_matrix_market(a, buf)
    assert np.array_equal(jv.parse_matrix_market(buf.getvalue()).val, a.val)


def test_permutation_files(tmp_path):
    perm = jv.Permutation(np.array([2, 0, 3, 1], dtype=np.int64))
    p = tmp_path / "p.txt"
    jv.write_permutation_file(perm, p)
    q = jv.read_permutation_file(p, 4)
    assert np.array_equal(q.perm, perm.perm)
    with pytest.raises(MatrixFormatError):
        jv.read_permutation_file(p, 5)
