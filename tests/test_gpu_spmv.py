"""spmv kernels (csrc/spmv.cu) against the pinned oracle, bitwise: the
CTA-per-tile stream kernel and the persistent bulk-copy kernel on the same
matrices — empty rows (leading, trailing, at tile boundaries), rows longer
than several tiles, nonzero counts that are and are not tile multiples,
unaligned col/val arrays and the row-mapped variant.  Reference semantics:
_kernels.py:28-34 (ascending order, separately rounded products and sums)."""
import os
import sys

import numpy as np
import pytest

import oracle

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
pytestmark = pytest.mark.gpu

from paper_1812_06160_b200 import _lib  # noqa: E402
from paper_1812_06160_b200 import device as dv  # noqa: E402


def _random_csr(rng, n, lens, ncols=None):
    ncols = ncols or n
    rs = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=rs[1:])
    row = np.repeat(np.arange(n), lens)
    col = rng.integers(0, ncols, int(rs[-1]))   # repeated columns in a row are legal here
    col = col[np.lexsort((col, row))].astype(np.int64)
    val = rng.uniform(-1.0, 1.0, col.size)
    return rs, col, val


def _run(impl, rs, col, val, x, row_map=None, offset=0):
    """y through jv_spmv / jv_spmv_rows with the kernel `impl` forced; offset
    shifts col/val off 16-byte alignment (elements)."""
    n = rs.size - 1
    nnz = int(rs[-1])
    lib = _lib.load()
    lib.jv_set_spmv_impl(impl)
    try:
        rsd = dv.i32(rs)
        cold = dv.i32(np.concatenate((np.zeros(offset, dtype=np.int64), col, [0])))[offset:]
        vald = dv.f64(np.concatenate((np.zeros(offset), val, [0.0])))[offset:]
        xd = dv.f64(x)
        nout = n if row_map is None else int(row_map.max()) + 1 if n else 0
        yd = dv.f64(np.full(max(nout, 1), np.nan))
        if row_map is None:
            _lib.call("jv_spmv", n, nnz, dv.ptr(rsd), dv.ptr(cold), dv.ptr(vald), dv.ptr(xd),
                      dv.ptr(yd), None, dv.stream())
        else:
            _lib.call("jv_spmv_rows", n, nnz, dv.ptr(rsd), dv.ptr(cold), dv.ptr(vald), dv.ptr(xd),
                      dv.ptr(yd), None, dv.ptr(dv.i32(row_map)), dv.stream())
        return dv.host_f64(yd, nout)
    finally:
        lib.jv_set_spmv_impl(-1)


def _cases(rng):
    # name, row lengths
    yield "short rows, nnz a tile multiple", np.full(2048, 7)
    n = 3000
    lens = rng.integers(0, 12, n)
    lens[:5] = 0
    lens[-7:] = 0
    yield "ragged with leading/trailing empty rows", lens
    lens = rng.integers(1, 9, 5000)
    lens[100] = 5000       # a row over several tiles
    lens[101] = 0
    lens[2500] = 1024
    lens[4999] = 3333      # long last row
    yield "long rows", lens
    lens = np.zeros(4097, dtype=np.int64)
    lens[::2] = 1024       # every row ends exactly on a tile boundary, empty rows between
    yield "rows on tile boundaries", lens
    yield "all rows empty", np.zeros(100, dtype=np.int64)
    yield "one row", np.array([12345])
    yield "single entry", np.array([1])


@pytest.mark.parametrize("impl", [0, 1])
def test_spmv_kernels_bitwise(impl):
    rng = np.random.default_rng(42)
    for name, lens in _cases(rng):
        n = lens.size
        rs, col, val = _random_csr(rng, n, lens, ncols=max(n, 64))
        x = rng.uniform(-1.0, 1.0, max(n, 64))
        want = oracle.spmv(rs, col, val, x)
        got = _run(impl, rs, col, val, x)
        assert np.array_equal(got, want), (impl, name)


@pytest.mark.parametrize("offset", [1, 2, 3])
def test_persistent_kernel_unaligned_arrays(offset):
    rng = np.random.default_rng(offset)
    lens = rng.integers(0, 20, 4000)
    rs, col, val = _random_csr(rng, lens.size, lens)
    x = rng.uniform(-1.0, 1.0, lens.size)
    want = oracle.spmv(rs, col, val, x)
    assert np.array_equal(_run(1, rs, col, val, x, offset=offset), want)


@pytest.mark.parametrize("impl", [0, 1])
def test_row_mapped_variant(impl):
    rng = np.random.default_rng(5)
    lens = rng.integers(0, 30, 2500)
    rs, col, val = _random_csr(rng, lens.size, lens)
    x = rng.uniform(-1.0, 1.0, lens.size)
    row_map = rng.permutation(3000)[:lens.size].astype(np.int64)
    want = np.full(3000, np.nan)
    want[row_map] = oracle.spmv(rs, col, val, x)
    got = _run(impl, rs, col, val, x, row_map=row_map)
    got = np.concatenate((got, np.full(3000 - got.size, np.nan)))
    assert np.array_equal(got, want, equal_nan=True)


def test_persistent_kernel_many_ctas():
    """More tiles than resident CTAs: chunks of several tiles, rows crossing
    both tile and chunk boundaries."""
    rng = np.random.default_rng(11)
    n = 400_000
    lens = rng.integers(0, 11, n)
    lens[rng.integers(0, n, 40)] = rng.integers(1500, 9000, 40)
    rs, col, val = _random_csr(rng, n, lens)
    x = rng.uniform(-1.0, 1.0, n)
    want = oracle.spmv(rs, col, val, x)
    assert np.array_equal(_run(1, rs, col, val, x), want)
    assert np.array_equal(_run(-1, rs, col, val, x), want)
