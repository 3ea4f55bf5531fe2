"""CPU tests of the region plans (regionplan.py / csrc/regions_host.cpp).

* The partition is acyclic (the quotient graph of the regions has a
  topological order) and balanced.
* Replaying a wave stream the way region.cu executes it — regions
  advancing wave by wave, a wave only when its remote dependencies are
  published — reproduces the oracle's factor / forward / backward results
  bit for bit and never deadlocks.
* The ring placement never lets a block overlap a block still in flight
  (static window S, dynamic window D).
"""

import numpy as np
import pytest

import oracle
from paper_1812_06160_b200 import regionplan as RP
from paper_1812_06160_b200 import workloads as W

pytest.importorskip("paper_1812_06160_b200._lib")

BUDGET = 232448 - 2048


def _front(a, k=0, tau=0.0, base_perm=None):
    fe = oracle.front_end(a.n, a.row_start, a.col, a.val, base_perm=base_perm, k=k, tau=tau)
    return fe["row_start"], fe["col"], fe["diag"], fe["val"]


def _cases():
    return {
        "poisson2d_40": (W.poisson2d(40), 0, 0.0),
        "laplace7_12": (W.laplace7(12, 3), 0, 0.0),
        "convdiff3d_10_ilu1": (W.convdiff3d(10, 1), 1, 1e-3),
        "stencil27_9": (W.stencil27(9, 2), 0, 0.0),
        "random_dd": (W.random_diag_dominant(3000, 7, seed=5), 0, 0.0),
    }


def _quotient_is_acyclic(rs, col, diag, region_of, nreg):
    edges = set()
    for r in range(diag.size):
        for p in range(rs[r], diag[r]):
            a, b = region_of[col[p]], region_of[r]
            if a != b:
                edges.add((int(a), int(b)))
    indeg = np.zeros(nreg, np.int64)
    succ = [[] for _ in range(nreg)]
    for a, b in edges:
        succ[a].append(b)
        indeg[b] += 1
    ready = [g for g in range(nreg) if indeg[g] == 0]
    seen = 0
    while ready:
        g = ready.pop()
        seen += 1
        for h in succ[g]:
            indeg[h] -= 1
            if indeg[h] == 0:
                ready.append(h)
    return seen == nreg


@pytest.mark.parametrize("name", list(_cases()))
def test_partition_acyclic_balanced(name):
    a, k, tau = _cases()[name]
    rs, col, diag, _ = _front(a, k, tau)
    part = RP.partition(rs, col, diag, 148)
    assert part is not None
    nreg, region_of = part
    assert 1 <= nreg <= 148 and region_of.min() == 0 and region_of.max() == nreg - 1
    sizes = np.bincount(region_of, minlength=nreg)
    assert sizes.max() - sizes.min() <= max(2, sizes.max() // 2)
    assert _quotient_is_acyclic(rs, col, diag, region_of, nreg)


def _upos(rs, col, diag, r, k):
    """position of u(c_k, r) in val: row c_k's upper entry in column r (-1: none)"""
    c = int(col[rs[r] + k])
    seg = col[diag[c] + 1:rs[c + 1]]
    hit = np.nonzero(seg == r)[0]
    return int(diag[c] + 1 + hit[0]) if hit.size else -1


def _check_pack(ws, rs, diag, val, col=None):
    """The packed copy (val[sidx]) holds, per wave, vals_m[k][i] in the
    layout region.cu reads."""
    packed = np.where(ws.sidx >= 0, val[np.maximum(ws.sidx, 0)], 0.0)
    for w in range(ws.waves):
        _, recs = RP.records(ws, w)
        off = int(ws.table[w, 4]) * 2
        K, cnt = recs[0]["K"], recs[0]["cnt"]
        m = packed[off:off + int(ws.table[w, 5]) // 8]
        for i, rc in enumerate(recs):
            p0, nd = rc["p0"], rc["nd"]
            if ws.kind == 0:
                want = [(k, p0 + k) for k in range(nd)] + [(K, p0 + nd)] + \
                       [(K + 1 + k, _upos(rs, col, diag, rc["r"], k)) for k in range(nd)
                        if _upos(rs, col, diag, rc["r"], k) >= 0]
            elif ws.kind == 1:
                want = [(k, p0 + k) for k in range(nd)]
            else:
                want = [(k, p0 + k) for k in range(nd + 1)]
            for k, pos in want:
                assert m[k * cnt + i] == val[pos]


def _check_vec(ws):
    """The packed per-call vector (x[vidx]) holds, per wave, x[row_i]."""
    for w in range(ws.waves):
        _, recs = RP.records(ws, w)
        off = int(ws.table[w, 6]) * 2
        for i, rc in enumerate(recs):
            assert ws.vidx[off + i] == rc["r"]


def _replay(ws, rs, col, diag, val, vec, tau=0.0, norms=None):
    """Execute the stream on the host: returns the output vector (solves)
    or the factored values (factor)."""
    n = diag.size
    kind = ws.kind
    _check_pack(ws, rs, diag, val, col)
    if ws.kind != 0:
        _check_vec(ws)
    val = val.copy()
    out = np.full(n, np.nan)
    published = {}                      # mailbox slot -> value
    nreg = ws.nreg
    slots = [dict() for _ in range(nreg)]
    ptr = [int(ws.reg_wave[g]) for g in range(nreg)]
    end = [int(ws.reg_wave[g + 1]) for g in range(nreg)]
    decoded = {}
    progress = True
    while progress:
        progress = False
        for g in range(nreg):
            while ptr[g] < end[g]:
                w = ptr[g]
                if w not in decoded:
                    decoded[w] = RP.records(ws, w)
                slot0, recs = decoded[w]
                ready = all(int(s) in published for rc in recs for s in rc["rsl"])
                if not ready:
                    break
                results = []
                for i, rc in enumerate(recs):
                    rem = list(int(x) for x in rc["rsl"])
                    dv = []
                    for ref in rc["refs"]:
                        ref = int(ref)
                        dv.append(slots[g][ref] if ref >= 0 else published[rem.pop(0)])
                    r, p0, nd = rc["r"], rc["p0"], rc["nd"]
                    if kind == 0:
                        d = val[p0 + nd]
                        thresh = tau * norms[r] if tau > 0 else 0.0
                        for kk in range(nd):
                            l = val[p0 + kk] / dv[kk]
                            if tau > 0 and abs(l) < thresh:
                                l = 0.0
                            elif rc["umask"] >> kk & 1:
                                d = d - l * val[_upos(rs, col, diag, r, kk)]
                            val[p0 + kk] = l
                        val[p0 + nd] = d
                        x, key = d, r
                    elif kind == 1:
                        s = vec[r]
                        for kk in range(nd):
                            s = s - val[p0 + kk] * dv[kk]
                        x, key = s, r
                    else:
                        s = vec[r]
                        for kk in range(nd):
                            s = s - val[p0 + 1 + kk] * dv[kk]
                        x, key = s / val[p0], r
                    results.append((i, r, x, key, rc["pub"]))
                # the kernel's threads read every dependency of a wave before
                # any row of it is stored (slot ring: (slot0 + i) % SC)
                for i, r, x, key, pub in results:
                    slots[g][(slot0 + i) % ws.slot_ring] = x
                    out[r] = x
                    if pub:
                        published[key] = x
                ptr[g] += 1
                progress = True
    assert all(ptr[g] == end[g] for g in range(nreg)), "replay deadlocked"
    return val if kind == 0 else out


def _ring_ok(ws):
    """No in-flight block overlap in either ring."""
    for g in range(ws.nreg):
        w0, w1 = int(ws.reg_wave[g]), int(ws.reg_wave[g + 1])
        for kind, win, cap, col_off in (("s", ws.S, ws.CS, 2), ("d", ws.D, ws.CD, 3)):
            blocks = []
            for w in range(w0, w1):
                if kind == "s":
                    size = int(ws.table[w, 1])
                else:
                    npk = int(ws.table[w, 7]) >> 16   # remote values, 8 bytes each
                    size = int(ws.table[w, 5]) + (int(ws.table[w, 7]) & 0xFFFF) + \
                        ((8 * npk + 15) & ~15)
                off = int(ws.table[w, col_off])
                assert off % 16 == 0 and off + size <= cap
                for (o2, s2) in blocks[-win:]:
                    assert not (off < o2 + s2 and o2 < off + size), (g, w, kind)
                blocks.append((off, size))
    return True


@pytest.mark.parametrize("name", list(_cases()))
def test_stream_replay_bitwise(name):
    a, k, tau = _cases()[name]
    rs, col, diag, val = _front(a, k, tau)
    nreg, region_of = RP.partition(rs, col, diag, 148)
    b = np.random.default_rng(0).uniform(-1, 1, diag.size)
    norms = oracle.row_inf_norms(rs, val, tau)
    want, bad = oracle.factor_serial(rs, col, val.copy(), diag, tau, False)
    assert bad < 0
    fs = RP.build_stream("factor", rs, col, diag, region_of, nreg, BUDGET, tau)
    stencil = name in ("poisson2d_40", "laplace7_12")
    assert (fs is not None) == stencil or (fs is not None and k == 0)
    if fs is not None:
        got = _replay(fs, rs, col, diag, val, None, tau, norms)
        assert np.array_equal(got, want)
        assert _ring_ok(fs)
    y_want = oracle.solve_forward(rs, col, want, b)
    x_want, _ = oracle.solve_backward(rs, col, want, diag, y_want)
    ff = RP.build_stream("fwd", rs, col, diag, region_of, nreg, BUDGET)
    fb = RP.build_stream("bwd", rs, col, diag, region_of, nreg, BUDGET)
    assert ff is not None and fb is not None
    y = _replay(ff, rs, col, diag, want, b)
    assert np.array_equal(y, y_want)
    x = _replay(fb, rs, col, diag, want, y)
    assert np.array_equal(x, x_want)
    assert _ring_ok(ff) and _ring_ok(fb)


def test_factor_stream_rejects_non_stencil():
    rs, col, diag, _ = _front(W.stencil27(6, 0))
    nreg, region_of = RP.partition(rs, col, diag, 148)
    assert RP.build_stream("factor", rs, col, diag, region_of, nreg, BUDGET) is None


def test_partition_finds_boxes_on_grid():
    """On a 3D grid the rotated depth-first orders recover the axes: the
    regions are boxes, so few rows have a dependency in another region."""
    a = W.laplace7(24, 0)
    rs, col, diag, _ = _front(a)
    nreg, region_of = RP.partition(rs, col, diag, 64)
    assert nreg == 64
    remote = sum(region_of[col[p]] != region_of[r]
                 for r in range(diag.size) for p in range(rs[r], diag[r]))
    # 4x4x4 boxes of a 24^3 grid: 3 cut planes per axis, 3 * 3 * 24^2 lower edges
    assert remote == 3 * 3 * 24 * 24
