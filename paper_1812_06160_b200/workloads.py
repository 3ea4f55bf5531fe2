"""Synthetic matrices: small stencil/random families for tests and the five
BASELINE.json configurations (SURVEY.md §8d recipes).  The reference's
SuiteSparse matrices are not available; these seeded generators stand in
for them.  All generators build sorted CSR directly (no COO sort), so the
multi-million-row configs take seconds.
"""

from __future__ import annotations

import numpy as np

from .csr import CsrMatrix, Permutation

__all__ = [
    "tridiag",
    "poisson2d",
    "poisson3d",
    "convdiff2d",
    "random_diag_dominant",
    "stencil_csr",
    "config_matrix",
    "CONFIGS",
]


def stencil_csr(dims, offsets):
    """Pattern of a stencil on a box grid with natural (last axis fastest)
    ordering.  offsets: list of integer vectors (including 0 for the
    diagonal).  Returns (row_start, col, offset_id) with columns sorted."""
    dims = tuple(int(d) for d in dims)
    nd = len(dims)
    n = int(np.prod(dims))
    strides = [int(np.prod(dims[a + 1:])) for a in range(nd)]
    offs = sorted((tuple(o) for o in offsets),
                  key=lambda o: sum(o[a] * strides[a] for a in range(nd)))
    coords = np.indices(dims).reshape(nd, n)
    cols = np.full((n, len(offs)), -1, dtype=np.int64)
    idx = np.arange(n, dtype=np.int64)
    for t, o in enumerate(offs):
        ok = np.ones(n, dtype=bool)
        for a in range(nd):
            c = coords[a] + o[a]
            ok &= (c >= 0) & (c < dims[a])
        lin = sum(o[a] * strides[a] for a in range(nd))
        cols[ok, t] = idx[ok] + lin
    valid = cols >= 0
    row_start = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(valid.sum(axis=1), out=row_start[1:])
    offid = np.broadcast_to(np.arange(len(offs)), cols.shape)[valid]
    return row_start, cols[valid], offid, offs


def _diag_mask(row_start, col):
    owner = np.repeat(np.arange(row_start.size - 1), np.diff(row_start))
    return col == owner, owner


def tridiag(n: int) -> CsrMatrix:
    """[-1, 2, -1] chain of length n."""
    rs, col, offid, offs = stencil_csr((n,), [(-1,), (0,), (1,)])
    diag, _ = _diag_mask(rs, col)
    return CsrMatrix(n, rs, col, np.where(diag, 2.0, -1.0))


def poisson2d(k: int) -> CsrMatrix:
    """5-point Laplacian on a k x k grid (diag 4, neighbours -1)."""
    rs, col, _, _ = stencil_csr((k, k), [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)])
    diag, _ = _diag_mask(rs, col)
    return CsrMatrix(k * k, rs, col, np.where(diag, 4.0, -1.0))


def _box_offsets(nd, reach=1):
    rng = range(-reach, reach + 1)
    return [tuple(o) for o in np.array(np.meshgrid(*([list(rng)] * nd), indexing="ij")).reshape(nd, -1).T]


def poisson3d(k: int) -> CsrMatrix:
    """27-point stencil on a k^3 grid: diagonal 26, each neighbour -1."""
    rs, col, _, _ = stencil_csr((k, k, k), _box_offsets(3))
    diag, _ = _diag_mask(rs, col)
    return CsrMatrix(k ** 3, rs, col, np.where(diag, 26.0, -1.0))


def convdiff2d(k: int, seed: int = 0) -> CsrMatrix:
    """Unsymmetric 2-D convection-diffusion, 5-point + first-order upwind,
    wind from the seed."""
    rng = np.random.default_rng(seed)
    h = 1.0 / (k + 1)
    v = rng.uniform(5.0, 25.0, 2) * rng.choice([-1.0, 1.0], 2)
    offs = [(0, 0), (-1, 0), (1, 0), (0, -1), (0, 1)]
    rs, col, offid, offs_sorted = stencil_csr((k, k), offs)
    vals = np.empty(col.size)
    for t, o in enumerate(offs_sorted):
        m = offid == t
        if o == (0, 0):
            vals[m] = 4.0 + (abs(v[0]) + abs(v[1])) * h
            continue
        a = 0 if o[0] else 1
        up = (o[a] < 0 and v[a] > 0) or (o[a] > 0 and v[a] < 0)
        vals[m] = -1.0 - (abs(v[a]) * h if up else 0.0)
    return CsrMatrix(k * k, rs, col, vals)


def random_diag_dominant(n: int, row_nnz: int = 6, seed: int = 0,
                         symmetric_pattern: bool = False) -> CsrMatrix:
    """Random strictly diagonally dominant matrix with a full diagonal."""
    rng = np.random.default_rng(seed)
    rows = [np.arange(n)]
    cols = [np.arange(n)]
    counts = rng.integers(0, max(1, row_nnz), size=n)
    for i in range(n):
        m = min(int(counts[i]), n - 1)
        if m > 0:
            pick = rng.choice(n - 1, size=m, replace=False)
            pick = pick + (pick >= i)
            rows.append(np.full(m, i))
            cols.append(pick)
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    if symmetric_pattern:
        off = r != c
        r, c = np.concatenate([r, c[off]]), np.concatenate([c, r[off]])
    a = CsrMatrix.from_coo(n, r, c, np.ones(r.size))  # dedupes positions
    a.val = rng.uniform(-1.0, 1.0, a.nnz)
    diag, owner = _diag_mask(a.row_start, a.col)
    off_abs = np.bincount(owner[~diag], weights=np.abs(a.val[~diag]), minlength=n)
    a.val[diag] = off_abs + 1.0
    return a


# ------------------------------------------------------------ BASELINE configs

CONFIGS = {
    "c1": dict(name="poisson2d_64", k=0, tau=0.0, order="natural", min_level_rows=16),
    "c2": dict(name="laplace7_128_rcm", k=0, tau=0.0, order="rcm", min_level_rows=16),
    "c3": dict(name="convdiff7_96_ilu1_tau1e-3", k=1, tau=1e-3, order="natural",
               min_level_rows=16),
    # c3 with tau = 1e-2: the variant where drops fire at full size
    # (tau = 1e-3 drops nothing on this matrix)
    "c3t": dict(name="convdiff7_96_ilu1_tau1e-2", k=1, tau=1e-2, order="natural",
                min_level_rows=16),
    "c4": dict(name="stencil27_100_nd", k=0, tau=0.0, order="file", min_level_rows=256),
    "c5": dict(name="rmat18_x64", k=0, tau=0.0, order="natural", min_level_rows=16),
}


def laplace7(k: int, seed: int = 0) -> CsrMatrix:
    """c2: 7-point Laplacian on k^3, off-diagonals -(1 + 0.1 U[-1,1]) per
    stored position (CSR order), diagonal 1.05 x sum |off|."""
    offs = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    rs, col, _, _ = stencil_csr((k, k, k), offs)
    diag, owner = _diag_mask(rs, col)
    rng = np.random.default_rng(seed)
    vals = np.empty(col.size)
    vals[~diag] = -(1.0 + 0.1 * rng.uniform(-1.0, 1.0, int((~diag).sum())))
    vals[diag] = 1.05 * np.bincount(owner[~diag], weights=np.abs(vals[~diag]), minlength=k ** 3)
    return CsrMatrix(k ** 3, rs, col, vals)


def convdiff3d(k: int, seed: int = 0) -> CsrMatrix:
    """c3: 7-point upwind convection-diffusion on k^3; v ~ U[0,5]^3 from the
    seed; upstream neighbour -(1+v_a), downstream -1, diagonal 6 + sum v."""
    rng = np.random.default_rng(seed)
    v = rng.uniform(0.0, 5.0, 3)
    offs = [(0, 0, 0), (1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]
    rs, col, offid, offs_sorted = stencil_csr((k, k, k), offs)
    vals = np.empty(col.size)
    for t, o in enumerate(offs_sorted):
        m = offid == t
        if o == (0, 0, 0):
            vals[m] = 6.0 + float(v.sum())
            continue
        a = int(np.flatnonzero(o)[0])
        vals[m] = -(1.0 + v[a]) if o[a] < 0 else -1.0
    return CsrMatrix(k ** 3, rs, col, vals)


def stencil27(k: int, seed: int = 0) -> CsrMatrix:
    """c4: 27-point stencil on k^3, off-diagonals N(0,1) per position,
    diagonal 1.1 x sum |off|."""
    rs, col, _, _ = stencil_csr((k, k, k), _box_offsets(3))
    diag, owner = _diag_mask(rs, col)
    rng = np.random.default_rng(seed)
    vals = np.empty(col.size)
    vals[~diag] = rng.standard_normal(int((~diag).sum()))
    vals[diag] = 1.1 * np.bincount(owner[~diag], weights=np.abs(vals[~diag]), minlength=k ** 3)
    return CsrMatrix(k ** 3, rs, col, vals)


def nd_permutation(dims, leaf: int = 6) -> Permutation:
    """Geometric nested dissection of a box grid: split the longest axis at
    its midpoint, order left half, right half, then the separator plane;
    boxes with every side <= leaf stay in natural order."""
    dims = tuple(int(d) for d in dims)
    strides = [int(np.prod(dims[a + 1:])) for a in range(len(dims))]
    out = []

    def natural(lo, hi):
        grids = np.meshgrid(*[np.arange(l, h) for l, h in zip(lo, hi)], indexing="ij")
        return sum(g * s for g, s in zip(grids, strides)).ravel()

    def rec(lo, hi):
        ext = [h - l for l, h in zip(lo, hi)]
        if min(ext) <= 0:
            return
        if max(ext) <= leaf:
            out.append(natural(lo, hi))
            return
        a = int(np.argmax(ext))
        mid = lo[a] + ext[a] // 2
        left_hi = list(hi); left_hi[a] = mid
        right_lo = list(lo); right_lo[a] = mid + 1
        sep_lo = list(lo); sep_lo[a] = mid
        sep_hi = list(hi); sep_hi[a] = mid + 1
        rec(lo, tuple(left_hi))
        rec(tuple(right_lo), hi)
        out.append(natural(tuple(sep_lo), tuple(sep_hi)))

    rec(tuple(0 for _ in dims), dims)
    perm = np.concatenate(out).astype(np.int64)
    return Permutation(perm)


def rmat(scale: int, seed: int, edge_factor: int = 8, abcd=(0.57, 0.19, 0.19, 0.05)) -> CsrMatrix:
    """c5: R-MAT graph -> symmetrised, deduplicated, self loops dropped;
    off-diagonals U[-1,1] per stored position (CSR order); diagonal
    1.2 x sum |off|, 1.0 for isolated rows."""
    n = 1 << scale
    m = edge_factor * n
    rng = np.random.default_rng(seed)
    a, b, c, _ = abcd
    r = np.zeros(m, dtype=np.int64)
    q = np.zeros(m, dtype=np.int64)
    for lvl in range(scale):
        u = rng.random(m)
        bit = np.int64(1) << np.int64(scale - 1 - lvl)
        r += np.where(u >= a + b, bit, 0)
        q += np.where(((u >= a) & (u < a + b)) | (u >= a + b + c), bit, 0)
    keep = r != q
    r, q = r[keep], q[keep]
    key = np.unique(np.concatenate([r * n + q, q * n + r]))
    key = np.union1d(key, np.arange(n, dtype=np.int64) * (n + 1))
    rows = key // n
    cols = key % n
    row_start = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_start[1:])
    diag = rows == cols
    vals = np.empty(cols.size)
    vals[~diag] = rng.uniform(-1.0, 1.0, int((~diag).sum()))
    off = np.bincount(rows[~diag], weights=np.abs(vals[~diag]), minlength=n)
    vals[diag] = np.where(off > 0, 1.2 * off, 1.0)
    return CsrMatrix(n, row_start, cols, vals)


def block_diagonal(mats) -> CsrMatrix:
    """Stack independent systems into one block-diagonal CSR (config 5)."""
    n = sum(m.n for m in mats)
    rs = [np.zeros(1, dtype=np.int64)]
    cols, vals = [], []
    roff = 0
    voff = 0
    for m in mats:
        rs.append(m.row_start[1:] + voff)
        cols.append(m.col + roff)
        vals.append(m.val)
        roff += m.n
        voff += m.nnz
    return CsrMatrix(n, np.concatenate(rs), np.concatenate(cols), np.concatenate(vals))


def config_matrix(cfg: str, scale: float = 1.0, rmat_count: int = 64):
    """(matrix, base permutation, settings) of a BASELINE config.  `scale`
    shrinks the grid edge for quick tests (1.0 = the published size)."""
    s = CONFIGS[cfg]
    if cfg == "c1":
        k = max(4, int(round(64 * scale)))
        a, base = poisson2d(k), None
    elif cfg == "c2":
        k = max(4, int(round(128 * scale)))
        a, base = laplace7(k), "rcm"
    elif cfg in ("c3", "c3t"):
        k = max(4, int(round(96 * scale)))
        a, base = convdiff3d(k), None
    elif cfg == "c4":
        k = max(4, int(round(100 * scale)))
        a, base = stencil27(k), nd_permutation((k, k, k))
    elif cfg == "c5":
        sc = max(6, int(round(18 + np.log2(max(scale, 1e-9)))))
        a = block_diagonal([rmat(sc, seed) for seed in range(rmat_count)])
        base = None
    else:
        raise KeyError(cfg)
    return a, base, s


def box_regions(dims, perm, parts):
    """Grid-aligned box decomposition of a box grid, in the numbering of a
    permuted matrix (perm: new -> natural index).  parts = boxes per axis.
    The application-side domain decomposition a PDE code would supply."""
    dims = tuple(int(d) for d in dims)
    nat = np.asarray(perm, dtype=np.int64)
    coords = np.unravel_index(nat, dims)
    rid = np.zeros(nat.size, dtype=np.int64)
    for a, (d, p) in enumerate(zip(dims, parts)):
        rid = rid * p + (coords[a] * p) // d
    return rid.astype(np.int32)
