"""Partition dimensionality per sweep on a config (region path forced)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1812_06160_b200 as jv
from paper_1812_06160_b200 import device as dv, workloads as W
from paper_1812_06160_b200.plan import build_plan

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
a, base, s = W.config_matrix(cfg)
bp = jv.rcm_order(a.pattern).perm if base == "rcm" else (base.perm if base is not None and hasattr(base, "perm") else base)
plan = build_plan(a, base_perm=bp, k=s["k"], tau=s["tau"], min_level_rows=s["min_level_rows"])
ilu = plan.ilu
n = ilu.n
ilu.region_mode = "on"
b = dv.f64(np.random.default_rng(0).uniform(-1, 1, n))
y, x = dv.empty_f64(n), dv.empty_f64(n)


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


combos = [(int(a), int(b)) for a, b in (c.split(',') for c in os.environ.get('JV_COMBOS', '3,0 2,0 2,64 2,36 3,64').split())]
for dims, rmax in combos:
    ilu.region_candidates = {sw: [(dims, rmax)] for sw in ("factor", "fwd", "bwd")}
    ilu._regions = None
    ilu._rstreams = {}
    ilu._rchoice = {}
    out = {"cfg": cfg, "dims": dims, "region_max": rmax}
    if ilu.region_stream("factor") is not None:
        plan.reset_values()
        ilu.factor_async()
        out["factor_us"] = round(timed(lambda: (plan.reset_values(), ilu.factor_async())) - timed(lambda: plan.reset_values()), 1)
    else:
        plan.reset_values()
        ilu.factor_async()
    out["fwd_us"] = round(timed(lambda: ilu.solve_async(0, b, y)), 1)
    out["bwd_us"] = round(timed(lambda: ilu.solve_async(1, y, x)), 1)
    dv.check_hang()
    print(json.dumps(out), flush=True)
