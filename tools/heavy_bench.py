"""Isolated heavy-row cost: rows 0..m-1 hold a diagonal and `ops` upper
entries (no pivots, ready at once); the last row is dense, so it is one
heavy row with m pivots x `ops` updates.  Prints us/pivot and checks the
factor against the oracle.   python tools/heavy_bench.py [m] [ops]"""
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def build(m, ops, seed=0):
    rng = np.random.default_rng(seed)
    n = m + 1
    rows, cols = [], []
    for i in range(m):
        up = np.sort(rng.choice(np.arange(i + 1, n), size=min(ops, n - 1 - i), replace=False))
        c = np.concatenate([[i], up])
        rows.append(np.full(c.size, i)); cols.append(c)
    rows.append(np.full(n, m)); cols.append(np.arange(n))
    r = np.concatenate(rows); c = np.concatenate(cols)
    rs = np.zeros(n + 1, np.int64); np.add.at(rs, r + 1, 1); rs = np.cumsum(rs)
    val = rng.uniform(-1, 1, c.size) * 0.01
    diag = np.array([rs[i] + np.searchsorted(cols[i], i) for i in range(n)])
    val[diag] = 4.0
    val[diag[-1]] = 1e3
    return n, rs, c, val, diag


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
    ops = int(sys.argv[2]) if len(sys.argv) > 2 else 73
    import torch
    import oracle
    from paper_1812_06160_b200 import device as dv
    n, rs, col, val, diag = build(m, ops)
    ilu = dv.DevIlu.from_host(n, rs, col, diag, val)
    el = ilu.elim_lists()
    if os.environ.get("NO_HUB"):
        dv.DevIlu.HUB_MIN_OPS = 1 << 40
    hub = ilu.hub_plans()
    assert el is not None and int(el[0][n - 1].item()) in (2, 4)
    v0 = dv.f64(val)
    ms = []
    for _ in range(5):
        ilu.val.copy_(v0)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); ilu.factor_async(); e1.record(); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    bad = dv.read_row_slot(ilu.err); dv.check_hang()
    want, wbad = oracle.factor_serial(rs, col, val.copy(), diag, 0.0, False)
    same = bool(np.array_equal(ilu.host_val(), want)) and bad == wbad
    best = min(ms[1:])
    prof = {}
    if os.environ.get("JV_TRACE"):
        from paper_1812_06160_b200 import _lib
        sch = ilu.factor_schedule()
        buf = torch.zeros(16 * sch.nbatch, dtype=torch.int64, device="cuda")
        ilu.val.copy_(v0)
        _lib.call("jv_set_trace", dv.ptr(buf), sch.nbatch)
        ilu.factor_async(); torch.cuda.synchronize()
        _lib.call("jv_set_trace", None, 0)
        tr = buf.cpu().numpy().reshape(-1, 16).astype(np.uint64)
        last = tr[-1]
        prof = {"own_or_hub": int(last[7] & 1), "piv_or_steps": int(last[7] >> 1), "adv": int(last[13]) / m,
                "miss": int(last[14]) / m, "div": int(last[15] >> 32) / m,
                "total": int(last[15] & 0xffffffff) / m}
    print(json.dumps({"m": m, "ops_per_pivot": ops, "ms": [round(x, 3) for x in ms],
                      "us_per_pivot": round(1e3 * best / m, 4),
                      "cycles_per_pivot_at_1.96GHz": round(1.96e6 * best / m), "bitwise": same, "hub_rows": hub[4] if hub else 0,
                      "cycles_per_pivot_by_phase": prof}))


if __name__ == "__main__":
    main()
