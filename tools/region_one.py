"""Run each region sweep once on a config (for ncu captures):
python tools/region_one.py c2 [fwd|bwd|factor]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1812_06160_b200 as jv
from paper_1812_06160_b200 import device as dv, workloads as W
from paper_1812_06160_b200.plan import build_plan

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
sweeps = sys.argv[2:] or ["fwd"]
a, base, s = W.config_matrix(cfg)
bp = jv.rcm_order(a.pattern).perm if base == "rcm" else (base.perm if base is not None and hasattr(base, "perm") else base)
plan = build_plan(a, base_perm=bp, k=s["k"], tau=s["tau"], min_level_rows=s["min_level_rows"])
ilu = plan.ilu
n = ilu.n
b = dv.f64(np.random.default_rng(0).uniform(-1, 1, n))
y = dv.empty_f64(n)
x = dv.empty_f64(n)
# the autotuned plans (JV_REGIONS unset) or the first candidates (JV_REGIONS=1)
plan.reset_values()
ilu.factor_async()
ilu.solve_async(0, b, y)
ilu.solve_async(1, y, x)
torch.cuda.synchronize()
print({sw: (ilu._region_for(sw) or {}).get("nreg") for sw in ("factor", "fwd", "bwd")})
from paper_1812_06160_b200 import _lib
_lib.call("jv_set_region_flags", int(os.environ.get("JV_RFLAGS", "0")))
for sw in sweeps:
    torch.cuda.nvtx.range_push(sw)
    if sw == "factor":
        plan.reset_values()
        ilu.factor_async()
    elif sw == "fwd":
        ilu.solve_async(0, b, y)
    else:
        ilu.solve_async(0, b, y)
        ilu.solve_async(1, y, x)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
dv.check_hang()
print("ok")
