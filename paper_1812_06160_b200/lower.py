"""Lower-stage ("second stage") factorization of the rows excluded from
level scheduling — the reference lower.py API
(/root/reference/pkg/src/ilukit/lower.py).

On the CPU the reference offers two methods for the tail (Segmented-Rows
tiles and Even-Rows chunks, then the corner).  On the GPU both become the
same two launches (csrc/tail.cu): the segmented upper-pivot stage over all
tail rows at once (warp per row; DIVIDE over groups of independent pivots,
UPDATE as a segmented reduction with one lane per target position folding
its updates in pivot order), then the corner — the tail rows restricted to
columns >= n_upper — by the sync-free factor kernel on a compact copy.  The
result is bitwise equal to factor_serial either way, exactly as both
reference methods are.  The
layouts (TileLayout, ER chunks) are still built with the reference's rules
because they are part of the API and of the solve setup.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .csr import SparsityPattern
from .errors import ConfigurationError, ZeroPivotError
from .ordering import LOWER_A_PLUS_AT, StagePartition
from .symbolic import IluFactors

__all__ = [
    "SR",
    "ER",
    "AUTO",
    "NONE",
    "DEFAULT_TILE_SIZE",
    "TileLayout",
    "select_lower_method",
    "build_tiles",
    "er_chunks",
    "factor_sr",
    "factor_er",
]

SR = "sr"
ER = "er"
AUTO = "auto"
NONE = "none"

DEFAULT_TILE_SIZE = 256


@dataclass
class TileLayout:
    """Tiles over the excluded rows' storage, grouped by upper level
    (lower.py:60-92).  Segment s covers val[seg_lo[s]:seg_hi[s]] of row
    seg_row[s]; tile t owns segments tile_ptr[t]:tile_ptr[t+1]; the last
    level group holds the corner tiles (columns >= n_upper)."""

    n_upper: int
    tile_size: int
    lptr_cols: np.ndarray
    tile_ptr: np.ndarray
    seg_row: np.ndarray
    seg_lo: np.ndarray
    seg_hi: np.ndarray
    tile_level: np.ndarray
    level_tile_ptr: np.ndarray

    @property
    def num_upper_levels(self) -> int:
        return self.lptr_cols.size - 1

    @property
    def ntiles(self) -> int:
        return self.tile_ptr.size - 1

    def tile_nnz(self, t: int) -> int:
        a, b = self.tile_ptr[t], self.tile_ptr[t + 1]
        return int(np.sum(self.seg_hi[a:b] - self.seg_lo[a:b]))


def select_lower_method(lower_row_count: int, nthreads: int, imbalance: float) -> str:
    """ER with enough evenly weighted rows, otherwise SR; none without rows
    (lower.py:95-103)."""
    if lower_row_count == 0:
        return NONE
    if lower_row_count >= 2 * nthreads and imbalance <= 8.0:
        return ER
    return SR


def _check_level_order(partition: StagePartition, n: int) -> np.ndarray:
    """Require level-ordered indexing; return each upper level's first
    column plus n_upper (lower.py:106-123)."""
    sizes = np.array([len(l) for l in partition.upper_levels], dtype=np.int64)
    lptr = np.zeros(sizes.size + 1, dtype=np.int64)
    np.cumsum(sizes, out=lptr[1:])
    for i, rows in enumerate(partition.upper_levels):
        if not np.array_equal(np.asarray(rows), np.arange(lptr[i], lptr[i + 1])):
            raise ConfigurationError(
                "lower-stage methods require factors assembled in level order"
            )
    if not np.array_equal(np.asarray(partition.lower_rows), np.arange(partition.n_upper, n)):
        raise ConfigurationError("lower-stage methods require excluded rows at the end")
    return lptr


def _check_intra_level_independence(pat: SparsityPattern, lptr: np.ndarray) -> None:
    """No strict-lower entry may join two rows of one upper level
    (lower.py:199-211)."""
    n_upper = int(lptr[-1])
    if n_upper == 0:
        return
    owner = np.repeat(np.arange(pat.n, dtype=np.int64), np.diff(pat.row_start))
    m = (owner < n_upper) & (pat.col < owner)
    if not m.any():
        return
    level_of = np.searchsorted(lptr, np.arange(n_upper), side="right") - 1
    if np.any(level_of[owner[m]] == level_of[pat.col[m]]):
        raise ConfigurationError(
            "intra-level dependency found; levels must come from lower(A+A^T)"
        )


def build_tiles(
    factors: IluFactors,
    partition: StagePartition,
    tile_size: int = DEFAULT_TILE_SIZE,
) -> TileLayout:
    """Greedy row-major packing of each (tail rows x upper level) subblock,
    then of the corner, into tiles of at most tile_size entries
    (lower.py:126-196)."""
    if partition.levels_kind != LOWER_A_PLUS_AT:
        raise ConfigurationError("sr_requires_symmetrized_levels")
    if tile_size < 1:
        raise ConfigurationError("tile_size must be >= 1")
    pat = factors.pattern
    n = pat.n
    n_upper = partition.n_upper
    lptr = _check_level_order(partition, n)
    nlev = lptr.size - 1
    _check_intra_level_independence(pat, lptr)

    rs = pat.row_start
    tail = np.arange(n_upper, n, dtype=np.int64)
    # position of every level boundary column inside every tail row
    bounds = np.empty((tail.size, nlev + 2), dtype=np.int64)
    for k, r in enumerate(tail):
        cols = pat.col[rs[r]:rs[r + 1]]
        bounds[k, :nlev + 1] = rs[r] + np.searchsorted(cols, lptr)
        bounds[k, nlev + 1] = rs[r + 1]

    tile_ptr = [0]
    seg_row, seg_lo, seg_hi, tile_level = [], [], [], []
    level_tile_ptr = np.zeros(nlev + 2, dtype=np.int64)
    for g in range(nlev + 1):
        room = tile_size
        pending = False
        for k in range(tail.size):
            lo, hi = int(bounds[k, g]), int(bounds[k, g + 1])
            while lo < hi:
                take = min(room, hi - lo)
                seg_row.append(int(tail[k]))
                seg_lo.append(lo)
                seg_hi.append(lo + take)
                pending = True
                lo += take
                room -= take
                if room == 0:
                    tile_ptr.append(len(seg_row))
                    tile_level.append(g)
                    room = tile_size
                    pending = False
        if pending:
            tile_ptr.append(len(seg_row))
            tile_level.append(g)
        level_tile_ptr[g + 1] = len(tile_level)

    as64 = lambda v: np.asarray(v, dtype=np.int64)
    return TileLayout(n_upper, tile_size, lptr, as64(tile_ptr), as64(seg_row), as64(seg_lo),
                      as64(seg_hi), as64(tile_level), level_tile_ptr)


def er_chunks(pattern: SparsityPattern, n_upper: int, nthreads: int) -> np.ndarray:
    """Contiguous chunk bounds over the excluded rows balancing the nonzero
    count of their upper-column segments (+1 per row) (lower.py:214-232)."""
    n = pattern.n
    if n_upper >= n:
        return np.full(nthreads + 1, n_upper, dtype=np.int64)
    rs = pattern.row_start
    tail = np.arange(n_upper, n, dtype=np.int64)
    weight = np.empty(tail.size, dtype=np.int64)
    for k, r in enumerate(tail):
        weight[k] = np.searchsorted(pattern.col[rs[r]:rs[r + 1]], n_upper) + 1
    cum = np.zeros(tail.size + 1, dtype=np.int64)
    np.cumsum(weight, out=cum[1:])
    targets = cum[-1] * np.arange(1, nthreads) / nthreads
    cuts = np.searchsorted(cum, targets)
    return np.concatenate(([n_upper], n_upper + cuts, [n])).astype(np.int64)


def _factor_tail(factors: IluFactors, n_upper: int) -> None:
    """Both reference methods (SR tiles, ER chunks) on the GPU: stage 1 is
    the segmented upper-pivot elimination of every tail row (jv_tail_upper:
    warp per row, groups of independent pivots divided in parallel, each
    target's updates folded in pivot order — the SR kernel's DIVIDE/UPDATE
    with per-row groups), stage 2 the corner by the sync-free kernel on its
    compact copy.  Bitwise equal to factor_serial; after a zero pivot the
    later corner rows keep their stage-1 values, as in the reference."""
    from . import device as dv

    d = factors.upload_values()
    bad = d.factor_tail(n_upper)
    from .factor import _host_values

    dv.download_f64(_host_values(factors), d.val, factors.pattern.nnz)
    factors._synced()
    if bad >= 0:
        raise ZeroPivotError(int(bad))


def factor_sr(factors: IluFactors, tiles: TileLayout, nthreads: int = 1) -> None:
    """Segmented-rows lower stage (lower.py:273-295); upper rows must be
    factored already."""
    if tiles.n_upper >= factors.pattern.n:
        return
    _factor_tail(factors, tiles.n_upper)


def factor_er(
    factors: IluFactors,
    partition: StagePartition,
    parallel_corner: bool = False,
    nthreads: int = 1,
) -> None:
    """Even-rows lower stage (lower.py:298-318); upper rows must be factored
    already."""
    n_upper = partition.n_upper
    if n_upper >= factors.pattern.n:
        return
    _check_level_order(partition, factors.pattern.n)
    _factor_tail(factors, n_upper)
