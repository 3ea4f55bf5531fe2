"""CPU test of the hub-row gather plan (jv_hub_plan_host): replaying the
planned stream the way the kernel executes it must reproduce the oracle's
factor row bit for bit."""

import numpy as np
import pytest

import oracle
from paper_1812_06160_b200 import hubplan
from paper_1812_06160_b200 import workloads as W

pytest.importorskip("paper_1812_06160_b200._lib")


def elim_list(rs, col, diag, r):
    """(piv_ptr, q, w) of row r: the matches _factor_row applies, pivot order."""
    a, b = rs[r], rs[r + 1]
    cols = col[a:b]
    pos = {int(c): i for i, c in enumerate(cols)}
    nL = diag[r] - a
    piv_ptr, qs, ws = [0], [], []
    for k in range(nL):
        c = int(cols[k])
        for q in range(diag[c] + 1, rs[c + 1]):
            w = pos.get(int(col[q]))
            if w is not None and w > k:
                qs.append(q)
                ws.append(w)
        piv_ptr.append(len(qs))
    return np.array(piv_ptr, np.int64), np.array(qs, np.int32), np.array(ws, np.int32)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_replay_matches_oracle(seed):
    a = W.rmat(9, seed)
    fe = oracle.front_end(a.n, a.row_start, a.col, a.val)
    rs, col, diag, val = fe["row_start"], fe["col"], fe["diag"], fe["val"]
    want, bad = oracle.factor_serial(rs, col, val.copy(), diag, 0.0, False)
    assert bad < 0
    nL = diag - rs[:-1]
    checked = 0
    for r in np.argsort(nL)[-12:]:
        piv_ptr, q, w = elim_list(rs, col, diag, r)
        L = int(nL[r])
        dslot = diag[col[rs[r]:rs[r] + L]].astype(np.int32)
        plan = hubplan.plan_row(rs[r + 1] - rs[r], L, piv_ptr, q, w, dslot)
        assert plan is not None
        stream, meta = plan
        assert stream.shape[0] == len(q) + L
        av = val[rs[r]:rs[r + 1]].astype(np.float64).copy()
        hubplan.replay(stream, meta, av, L, lambda s: want[s], lambda s: want[s])
        assert np.array_equal(av, want[rs[r]:rs[r + 1]]), r
        checked += 1
    assert checked == 12
