"""Region sweeps with diagnostic flags (8 = no remote waits: every region
runs alone at its own speed; results are wrong): kernel times by CUDA
events.  python tools/region_flags.py c2 [flags...]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1812_06160_b200 as jv
from paper_1812_06160_b200 import _lib, device as dv, workloads as W
from paper_1812_06160_b200.plan import build_plan

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
flag_list = [int(f) for f in sys.argv[2:]] or [0, 8]
a, base, s = W.config_matrix(cfg)
bp = jv.rcm_order(a.pattern).perm if base == "rcm" else (base.perm if base is not None and hasattr(base, "perm") else base)
plan = build_plan(a, base_perm=bp, k=s["k"], tau=s["tau"], min_level_rows=s["min_level_rows"])
ilu = plan.ilu
n = ilu.n
b = dv.f64(np.random.default_rng(0).uniform(-1, 1, n))
y, x = dv.empty_f64(n), dv.empty_f64(n)
plan.reset_values()
ilu.factor_async()
ilu.solve_async(0, b, y)
ilu.solve_async(1, y, x)
torch.cuda.synchronize()
for sw in ("factor", "fwd", "bwd"):
    rp = ilu._region_for(sw)
    if isinstance(rp, dict):
        print(sw, {k: rp[k] for k in ("nreg", "slot_ring", "max_waves", "S", "D", "CS", "CD", "waves", "remote_deps") if k in rp})


def timed(fn, pre=None, reps=10):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(reps + 2):
        if pre:
            pre()
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
    return float(np.median(ts[2:]))


for fl in flag_list:
    _lib.call("jv_set_region_flags", fl)
    out = {"flags": fl}
    out["factor_us"] = timed(ilu.factor_async, plan.reset_values)
    out["fwd_us"] = timed(lambda: ilu.solve_async(0, b, y))
    out["bwd_us"] = timed(lambda: ilu.solve_async(1, y, x))
    print(json.dumps(out), flush=True)
_lib.call("jv_set_region_flags", 0)
