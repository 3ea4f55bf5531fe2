"""Device-resident front end: the reference pipeline's build step
(pipeline.py:151-186 of ilukit: base order -> levels of lower(A+Aᵀ) ->
two-stage partition -> level permutation -> ILU(k) pattern -> assembly)
with every array staying in HBM.  Returns an IluPlan whose `ilu` member
factors / solves in place and whose `permuted` member is P A Pᵀ for spmv.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import device as dv
from .csr import CsrMatrix, permute_dev, sym_lower_dev
from .errors import MatrixFormatError, MissingDiagonalError
from .symbolic import assemble_dev, iluk1_dev


@dataclass
class IluPlan:
    n: int
    base_perm: object        # device int32 (new -> old) of the base order
    level_of: object         # device int32 levels of lower(A+Aᵀ) (base order)
    nlev: int
    cut: int
    n_upper: int
    perm: object             # device int32 total permutation (new -> old)
    permuted: dv.DevCsr      # P A Pᵀ (values included)
    fill: object             # device int32 fill levels (or None for k = 0)
    ilu: dv.DevIlu           # factor storage (values = assembled on return)
    assembled: object        # device copy of the assembled values

    def reset_values(self):
        self.ilu.load_values(self.assembled)


def _inverse(perm_d):
    t = dv.torch()
    inv = t.empty_like(perm_d)
    inv[perm_d.long()] = t.arange(perm_d.numel(), dtype=t.int32, device="cuda")
    return inv


def build_plan(a: CsrMatrix, base_perm=None, k: int = 0, tau: float = 0.0, milu: bool = False,
               min_level_rows: int = 16, density_factor: float = 4.0, cut=None,
               da: dv.DevCsr | None = None) -> IluPlan:
    t = dv.torch()
    n = a.n
    da = da or dv.DevCsr.from_host(n, a.row_start, a.col, a.val)
    if base_perm is not None:
        base = dv.i32(np.asarray(base_perm, dtype=np.int64))
        pa = permute_dev(da, base, _inverse(base))
    else:
        base = t.arange(n, dtype=t.int32, device="cuda")
        pa = da
    src = sym_lower_dev(pa, lower_only=True)
    level_of, nlev = dv.levels_dev(src, backward=False)
    order, level_ptr = dv.level_sort_dev(n, nlev, level_of)
    if cut is None:
        row_nnz = (pa.row_start[1:] - pa.row_start[:-1]).contiguous()
        cut_h, nup_h = ctypes.c_int32(0), ctypes.c_int32(0)
        _lib.call("jv_partition", n, nlev, dv.ptr(level_ptr), dv.ptr(order), dv.ptr(row_nnz),
                  int(min_level_rows), float(density_factor), 1, ctypes.byref(cut_h),
                  ctypes.byref(nup_h), dv.stream())
        cut, n_upper = int(cut_h.value), int(nup_h.value)
    else:
        n_upper = int(level_ptr[cut].item())
    total = base[order.long()].contiguous()
    permuted = permute_dev(da, total, _inverse(total))
    fill = None
    if k == 0:
        slot = dv.reset_row_slot()
        _lib.call("jv_check_diagonal", n, dv.ptr(permuted.row_start), dv.ptr(permuted.col),
                  dv.ptr(slot), dv.stream())
        bad = dv.read_row_slot(slot)
        if bad >= 0:
            raise MissingDiagonalError(bad)
        fpat = dv.DevCsr(n, permuted.nnz, permuted.row_start, permuted.col)
    elif k == 1:
        fpat, fill = iluk1_dev(permuted)
    else:
        from .symbolic import iluk_dev

        fpat, fill = iluk_dev(permuted, k)      # k rounds of jv_iluk_round, all in HBM
    val, diag, bad_cover, bad_diag = assemble_dev(permuted, fpat)
    if bad_cover >= 0:
        raise MatrixFormatError("pattern does not cover the permuted matrix")
    if bad_diag >= 0:
        raise MissingDiagonalError(bad_diag)
    ilu = dv.DevIlu(n, fpat.row_start, fpat.col, diag, val, tau, milu)
    ilu.n_upper = n_upper
    return IluPlan(n, base, level_of, nlev, cut, n_upper, total, permuted, fill, ilu,
                   val.clone())
