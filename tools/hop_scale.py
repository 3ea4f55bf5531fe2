"""Factor time per level vs problem size (c2 recipe at smaller grids):
does the per-level hop grow with the mailbox footprint?"""
import json, os, sys
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import torch
import paper_1812_06160_b200 as jv
from paper_1812_06160_b200 import workloads as W, device as dv
from paper_1812_06160_b200.plan import build_plan
for arg in (sys.argv[1:] or ["48", "64", "96", "128"]):
    if arg.startswith("t"):      # tridiagonal chain: one row per level
        k = int(arg[1:])
        a = W.tridiag(k)
        plan = build_plan(a)
    else:
        k = int(arg)
        a = W.laplace7(k)
        plan = build_plan(a, base_perm=jv.rcm_order(a.pattern).perm)
    ilu = plan.ilu
    ms = []
    for _ in range(4):
        plan.reset_values()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); ilu.factor_async(); e1.record(); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = min(ms[1:])
    print(json.dumps({"k": k, "n": a.n, "levels": plan.nlev, "factor_ms": t,
                      "us_per_level": 1e3 * t / plan.nlev, "mbox_MB": 16 * ilu.nnz / 1e6}))
