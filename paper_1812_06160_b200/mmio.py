"""Matrix Market coordinate I/O and permutation files — the reference
mmio.py API (/root/reference/pkg/src/ilukit/mmio.py:33-140): the data
format on the input side of the hot path.

Accepted: `%%MatrixMarket matrix coordinate real|integer
general|symmetric|skew-symmetric`, square.  Pattern files are rejected (the
factorization needs values).  Explicit zeros are kept, duplicates summed
(CsrMatrix.from_coo), symmetric storage mirrored to both triangles
(skew: negated).  The entry block is parsed in bulk with numpy rather than
line by line; malformed input raises MatrixFormatError with the offending
line.  Writing uses %.17g, so a write/read round trip is exact.
"""

from __future__ import annotations

import io
from pathlib import Path

import numpy as np

from .csr import CsrMatrix, Permutation
from .errors import MatrixFormatError

__all__ = [
    "parse_matrix_market",
    "write_matrix_market",
    "read_matrix_market_file",
    "write_matrix_market_file",
    "read_permutation_file",
    "write_permutation_file",
]

_FIELDS = ("real", "integer")
_SYMMETRY = ("general", "symmetric", "skew-symmetric")


def _header(line: str):
    words = line.strip().lower().split()
    if len(words) != 5 or words[0] != "%%matrixmarket" or words[1] != "matrix":
        raise MatrixFormatError(f"malformed MatrixMarket header: {line.strip()!r}")
    layout, field, symmetry = words[2:]
    if layout != "coordinate":
        raise MatrixFormatError(f"unsupported layout {layout!r} (coordinate required)")
    if field == "pattern":
        raise MatrixFormatError("pattern-only files are rejected: numeric values required")
    if field not in _FIELDS:
        raise MatrixFormatError(f"unsupported field {field!r}")
    if symmetry not in _SYMMETRY:
        raise MatrixFormatError(f"unsupported symmetry {symmetry!r}")
    return symmetry


def _data_lines(text: str):
    """Non-blank, non-comment lines of a text block."""
    return [s for s in (ln.strip() for ln in text.splitlines()) if s and not s.startswith("%")]


def _entries(lines, nent, n):
    """0-based rows, cols and values of the entry lines (validated)."""
    if len(lines) > nent:
        raise MatrixFormatError("more entries than declared")
    if len(lines) < nent:
        raise MatrixFormatError(f"declared {nent} entries, found {len(lines)}")
    if nent == 0:
        z = np.zeros(0, dtype=np.int64)
        return z, z.copy(), np.zeros(0)
    toks = " ".join(lines).split()
    if len(toks) != 3 * nent:
        bad = next(s for s in lines if len(s.split()) != 3)
        raise MatrixFormatError(f"malformed entry line: {bad!r}")
    t = np.array(toks, dtype=object).reshape(nent, 3)
    try:
        ij = t[:, :2].astype(np.int64)
        v = t[:, 2].astype(np.float64)
    except (ValueError, OverflowError):
        for s in lines:   # find the first culprit for the message
            a, b, c = s.split()
            try:
                int(a), int(b), float(c)
            except ValueError as exc:
                raise MatrixFormatError(f"malformed entry line: {s!r}") from exc
        raise MatrixFormatError("malformed entry block")
    bad = np.nonzero((ij[:, 0] < 1) | (ij[:, 0] > n) | (ij[:, 1] < 1) | (ij[:, 1] > n))[0]
    if bad.size:
        i, j = ij[bad[0]]
        raise MatrixFormatError(f"entry index ({i},{j}) out of range for n={n}")
    return ij[:, 0] - 1, ij[:, 1] - 1, v


def parse_matrix_market(stream) -> CsrMatrix:
    """Matrix Market coordinate text (str, bytes or a text stream) -> CsrMatrix."""
    if isinstance(stream, bytes):
        stream = stream.decode()
    if isinstance(stream, str):
        stream = io.StringIO(stream)
    symmetry = _header(stream.readline())
    rest = stream.read()
    lines = _data_lines(rest)
    if not lines:
        raise MatrixFormatError("missing size line")
    size = lines[0].split()
    try:
        if len(size) != 3:
            raise ValueError
        nrows, ncols, nent = (int(x) for x in size)
    except ValueError as exc:
        raise MatrixFormatError(f"malformed size line: {lines[0]!r}") from exc
    if nrows != ncols:
        raise MatrixFormatError(f"matrix is not square ({nrows}x{ncols})")
    n = nrows
    rows, cols, vals = _entries(lines[1:], nent, n)
    if symmetry != "general":
        off = rows != cols
        sign = -1.0 if symmetry == "skew-symmetric" else 1.0
        rows, cols, vals = (np.concatenate([rows, cols[off]]), np.concatenate([cols, rows[off]]),
                            np.concatenate([vals, sign * vals[off]]))
    return CsrMatrix.from_coo(n, rows, cols, vals)


def write_matrix_market(a: CsrMatrix, sink) -> None:
    """coordinate / real / general text of `a` (exact round trip)."""
    rows = np.repeat(np.arange(a.n, dtype=np.int64), np.diff(a.row_start)) + 1
    cols = np.asarray(a.col, dtype=np.int64) + 1
    sink.write("%%MatrixMarket matrix coordinate real general\n")
    sink.write(f"{a.n} {a.n} {a.nnz}\n")
    if a.nnz:
        body = "\n".join(f"{i} {j} {v:.17g}" for i, j, v in
                         zip(rows.tolist(), cols.tolist(), np.asarray(a.val).tolist()))
        sink.write(body + "\n")


def read_matrix_market_file(path) -> CsrMatrix:
    with open(path, "r", encoding="ascii") as fh:
        return parse_matrix_market(fh)


def write_matrix_market_file(a: CsrMatrix, path) -> None:
    with open(path, "w", encoding="ascii") as fh:
        write_matrix_market(a, fh)


def read_permutation_file(path, n: int | None = None) -> Permutation:
    """One 0-based index per line; line k is perm[k] (new -> old)."""
    text = Path(path).read_text(encoding="ascii")
    perm = np.array([int(s) for s in text.split()], dtype=np.int64)
    if n is not None and perm.size != n:
        raise MatrixFormatError(f"permutation has {perm.size} entries, expected {n}")
    p = Permutation(perm)
    p.validate()
    return p


def write_permutation_file(p: Permutation, path) -> None:
    Path(path).write_text("".join(f"{int(x)}\n" for x in p.perm), encoding="ascii")
