"""Symbolic ILU patterns and assembly of the combined L|U storage — the
reference symbolic.py API (/root/reference/pkg/src/ilukit/symbolic.py) with
the diagonal check, the ILU(1) fill pattern, permutation and assembly run on
the GPU (libjv), bit-exact with the reference.

Storage: row i holds its strict-lower part (L, unit diagonal implicit), the
diagonal, then its upper part (U) in one sorted CSR row; diag_pos[i] indexes
the diagonal.
"""

from __future__ import annotations

import ctypes
import sys
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from . import device as dv
from .csr import CsrMatrix, Permutation, SparsityPattern, permute_dev
from .errors import MatrixFormatError, MissingDiagonalError

__all__ = [
    "FillLevelTable",
    "IluFactors",
    "ilu0_pattern",
    "iluk_pattern",
    "assemble_factors",
]


@dataclass
class FillLevelTable:
    """Fill level per stored position, aligned to the pattern's entries."""

    level: np.ndarray


@dataclass
class IluFactors:
    """Combined L/U factor storage over one CSR pattern (symbolic.py:36-67)."""

    n: int
    pattern: SparsityPattern
    val: np.ndarray
    diag_pos: np.ndarray
    perm: Permutation
    drop_tol: float = 0.0
    milu: bool = False
    _dev: object = field(default=None, repr=False, compare=False)

    def row_cols(self, i: int) -> np.ndarray:
        return self.pattern.row_cols(i)

    def row_vals(self, i: int) -> np.ndarray:
        return self.val[self.pattern.row_start[i]:self.pattern.row_start[i + 1]]

    def copy(self) -> "IluFactors":
        return IluFactors(self.n, self.pattern, self._val.copy(), self.diag_pos, self.perm,
                          self.drop_tol, self.milu, self._dev)

    # device mirror of the structure ---------------------------------------
    def device(self) -> dv.DevIlu:
        key = (id(self.pattern.row_start), id(self.pattern.col), id(self.diag_pos), self.n)
        if self._dev is None or self._dev[0] != key:
            pat = self.pattern
            d = dv.DevIlu(
                self.n, dv.i32(pat.row_start),
                dv.i32(pat.col) if pat.nnz else dv.empty_i32(1),
                dv.i32(self.diag_pos) if self.n else dv.empty_i32(1),
            )
            self._dev = (key, d, (pat.row_start, pat.col, self.diag_pos))
        d = self._dev[1]
        d.tau = float(self.drop_tol)
        d.milu = bool(self.milu)
        return d

    # Host values and their device copy.  `val` is the caller's numpy array,
    # as in the reference; the device copy is reused across calls only while
    # the package can prove the host array is unchanged: nobody has read the
    # `val` attribute since the last transfer (a read hands out a reference
    # the caller may write through) and nobody else holds a reference to the
    # array (a kept alias or view).  The reference's Krylov pattern
    # `precond = lambda r: apply_preconditioner(factors, r)` (pipeline.py:300)
    # then moves only the vector per call instead of all factor values.
    def _host(self) -> np.ndarray:
        """The host value array, without marking it as handed out."""
        return self._val

    def _synced(self) -> None:
        """Host array and device copy hold the same values as of now."""
        self._dirty = False

    def device_is_current(self) -> bool:
        d = self._dev[1] if self._dev is not None else None
        return (d is not None and d.holder is self and not self._dirty
                and sys.getrefcount(self._val) <= 2)

    def upload_values(self) -> dv.DevIlu:
        d = self.device()
        if self.device_is_current():
            return d
        if self.pattern.nnz:
            dv.upload_f64(d.val, self._val)
        d.values_changed()
        d.holder = self
        self._dirty = False
        return d


def _get_val(self) -> np.ndarray:
    self._dirty = True
    return self._val


def _set_val(self, v) -> None:
    self._val = v
    self._dirty = True


# (a property over the dataclass field: the generated __init__ assigns
# through the setter)
IluFactors.val = property(_get_val, _set_val)


def _dev_pattern(p: SparsityPattern) -> dv.DevCsr:
    return dv.DevCsr.from_host(p.n, p.row_start, p.col)


def _first_missing_diagonal_dev(d: dv.DevCsr) -> int:
    slot = dv.reset_row_slot()
    _lib.call("jv_check_diagonal", d.n, dv.ptr(d.row_start), dv.ptr(d.col), dv.ptr(slot),
              dv.stream())
    return dv.read_row_slot(slot)


def ilu0_pattern(pattern: SparsityPattern) -> SparsityPattern:
    """ILU(0) keeps the pattern; every row must store its diagonal."""
    if pattern.n:
        row = _first_missing_diagonal_dev(_dev_pattern(pattern))
        if row >= 0:
            raise MissingDiagonalError(row)
    return pattern


def iluk1_dev(d: dv.DevCsr, want_levels: bool = True):
    """ILU(1) pattern on the device: A ∪ pattern(L_A U_A), levels 0/1."""
    out_rs = dv.empty_i32(d.n + 1)
    nnz = ctypes.c_int64(0)
    _lib.call("jv_iluk1_pattern", d.n, dv.ptr(d.row_start), dv.ptr(d.col), dv.ptr(out_rs), None,
              None, ctypes.byref(nnz), dv.stream())
    out_col = dv.empty_i32(nnz.value)
    out_lev = dv.empty_i32(nnz.value) if want_levels else None
    _lib.call("jv_iluk1_pattern", d.n, dv.ptr(d.row_start), dv.ptr(d.col), dv.ptr(out_rs),
              dv.ptr(out_col), dv.ptr(out_lev), ctypes.byref(nnz), dv.stream())
    return dv.DevCsr(d.n, int(nnz.value), out_rs, out_col), out_lev


def iluk_dev(d: dv.DevCsr, k: int):
    """ILU(k) pattern and fill levels on the device for any k >= 1: k rounds
    of the level-of-fill closure (jv_iluk_round) from (A, level 0).  Levels
    are exact by induction on their value, so the result is the reference's
    row-by-row symbolic factorization (symbolic.py:86-138).  Returns
    (DevCsr, int32 level tensor)."""
    t = dv.torch()
    cur = d
    lev = t.zeros(max(d.nnz, 1), dtype=t.int32, device="cuda")
    for _ in range(k):
        out_rs = dv.empty_i32(d.n + 1)
        nnz = ctypes.c_int64(0)
        args = (d.n, dv.ptr(cur.row_start), dv.ptr(cur.col), dv.ptr(lev), int(k), dv.ptr(out_rs))
        _lib.call("jv_iluk_round", *args, None, None, ctypes.byref(nnz), dv.stream())
        out_col = dv.empty_i32(nnz.value)
        out_lev = dv.empty_i32(nnz.value)
        _lib.call("jv_iluk_round", *args, dv.ptr(out_col), dv.ptr(out_lev), ctypes.byref(nnz),
                  dv.stream())
        grown = int(nnz.value) != cur.nnz
        same = (not grown) and bool(t.equal(out_lev[:cur.nnz], lev[:cur.nnz]))
        cur, lev = dv.DevCsr(d.n, int(nnz.value), out_rs, out_col), out_lev
        if same:
            break          # fixed point before round k: nothing more can appear
    return cur, lev


def iluk_pattern(pattern: SparsityPattern, k: int) -> tuple[SparsityPattern, FillLevelTable]:
    """Level-of-fill symbolic factorization (symbolic.py:86-138)."""
    if k < 0:
        raise ValueError("fill level k must be >= 0")
    if pattern.n == 0:
        return pattern, FillLevelTable(np.zeros(0, dtype=np.int64))
    d = _dev_pattern(pattern)
    row = _first_missing_diagonal_dev(d)
    if row >= 0:
        raise MissingDiagonalError(row)
    if k == 0:
        return pattern, FillLevelTable(np.zeros(pattern.nnz, dtype=np.int64))
    if k == 1:
        out, lev = iluk1_dev(d)
        rs, col = out.host_pattern()
        return SparsityPattern(pattern.n, rs, col), FillLevelTable(dv.host_i64(lev, out.nnz))
    if k <= 254:
        try:
            out, lev = iluk_dev(d, k)
        except RuntimeError as e:            # candidate lists beyond int32: host C++ below
            if "too large" not in str(e):
                raise
        else:
            rs, col = out.host_pattern()
            return SparsityPattern(pattern.n, rs, col), FillLevelTable(dv.host_i64(lev, out.nnz))
    return _iluk_host(pattern, k)


def _iluk_host(pattern: SparsityPattern, k: int) -> tuple[SparsityPattern, FillLevelTable]:
    """Row-by-row symbolic factorization in libjv's host C++ (setup; used
    when a round's candidate lists exceed int32, and as the test oracle's
    counterpart for the device rounds)."""
    rs = np.ascontiguousarray(pattern.row_start, dtype=np.int32)
    col = np.ascontiguousarray(pattern.col, dtype=np.int32)
    prs = ctypes.POINTER(ctypes.c_int32)()
    pcol = ctypes.POINTER(ctypes.c_int32)()
    plev = ctypes.POINTER(ctypes.c_int32)()
    lib = _lib.load()
    nnz = lib.jv_iluk_host(pattern.n, rs.ctypes.data_as(ctypes.c_void_p),
                           col.ctypes.data_as(ctypes.c_void_p), int(k), ctypes.byref(prs),
                           ctypes.byref(pcol), ctypes.byref(plev))
    if nnz < 0:
        raise MemoryError("jv_iluk_host failed")
    try:
        out_rs = np.ctypeslib.as_array(prs, shape=(pattern.n + 1,)).astype(np.int64)
        out_col = np.ctypeslib.as_array(pcol, shape=(max(nnz, 1),))[:nnz].astype(np.int64)
        out_lev = np.ctypeslib.as_array(plev, shape=(max(nnz, 1),))[:nnz].astype(np.int64)
    finally:
        for p in (prs, pcol, plev):
            lib.jv_free_host(ctypes.cast(p, ctypes.c_void_p))
    return SparsityPattern(pattern.n, out_rs, out_col), FillLevelTable(out_lev)


def assemble_dev(permuted: dv.DevCsr, fpat: dv.DevCsr):
    """Scatter permuted values into the factor pattern; returns
    (val, diag_pos, bad_cover_row, bad_diag_row)."""
    val = dv.empty_f64(fpat.nnz)
    diag = dv.empty_i32(fpat.n)
    bad_cover = dv.reset_row_slot()
    bad_diag = dv.reset_row_slot()
    _lib.call("jv_assemble", fpat.n, dv.ptr(permuted.row_start), dv.ptr(permuted.col),
              dv.ptr(permuted.val), dv.ptr(fpat.row_start), dv.ptr(fpat.col), dv.ptr(val),
              dv.ptr(diag), dv.ptr(bad_cover), dv.ptr(bad_diag), dv.stream())
    return val, diag, dv.read_row_slot(bad_cover), dv.read_row_slot(bad_diag)


def assemble_factors(
    a: CsrMatrix,
    pattern: SparsityPattern,
    perm: Permutation,
    drop_tol: float = 0.0,
    milu: bool = False,
) -> IluFactors:
    """Place P A Pᵀ into the factor pattern (fill starts at zero) and locate
    the diagonals (symbolic.py:146-181)."""
    if pattern.n != a.n:
        raise MatrixFormatError(
            f"pattern size {pattern.n} does not match matrix size {a.n}"
        )
    n = a.n
    if n == 0:
        return IluFactors(0, pattern, np.zeros(0), np.zeros(0, dtype=np.int64), perm, drop_tol,
                          milu)
    da = dv.DevCsr.from_host(n, a.row_start, a.col, a.val)
    permuted = permute_dev(da, dv.i32(perm.perm), dv.i32(perm.inv))
    fpat = _dev_pattern(pattern)
    val, diag, bad_cover, bad_diag = assemble_dev(permuted, fpat)
    if bad_cover >= 0:
        raise MatrixFormatError("pattern does not cover the permuted matrix")
    if bad_diag >= 0:
        raise MissingDiagonalError(bad_diag)
    return IluFactors(n, pattern, dv.host_f64(val, pattern.nnz), dv.host_i64(diag, n), perm,
                      drop_tol, milu)
