"""Region-partition experiment on config 2: the automatic partition versus
grid boxes of given shapes (forward/backward region sweeps, CUDA events)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1812_06160_b200 as jv
from paper_1812_06160_b200 import device as dv, workloads as W
from paper_1812_06160_b200.plan import build_plan

a, base, s = W.config_matrix("c2")
bp = jv.rcm_order(a.pattern).perm
plan = build_plan(a, base_perm=bp, k=0, tau=0.0, min_level_rows=s["min_level_rows"])
ilu = plan.ilu
n = ilu.n
ilu.region_mode = "on"
b = dv.f64(np.random.default_rng(0).uniform(-1, 1, n))
y, x = dv.empty_f64(n), dv.empty_f64(n)
nat = dv.host_i64(plan.perm, n)


def timed(fn, reps=5):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
    return float(np.median(ts))


for parts in [None, (6, 6, 4), (12, 12, 1), (1, 12, 12), (4, 6, 6), (8, 6, 3), (37, 4, 1), (2, 8, 9)]:
    if parts is None:
        ilu.region_hint = None
        ilu._regions = None
        ilu._rstreams = {}
    else:
        ilu.set_regions(W.box_regions((128, 128, 128), nat, parts))
    plan.reset_values()
    ilu.factor_async()
    tf = timed(lambda: (plan.reset_values(), ilu.factor_async())) - timed(lambda: plan.reset_values())
    t0 = timed(lambda: ilu.solve_async(0, b, y))
    t1 = timed(lambda: ilu.solve_async(1, y, x))
    dv.check_hang()
    rp = ilu.region_stream("fwd")
    print(json.dumps({"parts": parts, "nreg": rp["nreg"] if rp else None, "factor_us": round(tf, 1),
                      "fwd_us": round(t0, 1), "bwd_us": round(t1, 1),
                      "remote_deps": rp["remote_deps"] if rp else None}), flush=True)
