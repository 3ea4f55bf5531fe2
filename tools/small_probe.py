"""jv_solve_small at config 1: whole sweep vs staging only (nlev = 0)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1812_06160_b200 as jv
from paper_1812_06160_b200 import device as dv, _lib
from paper_1812_06160_b200.plan import build_plan

plan = build_plan(jv.poisson2d(64))
ilu = plan.ilu
ilu.factor()
n = ilu.n
b = dv.f64(np.ones(n)); y = dv.empty_f64(n)


def t(fn, reps=50):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


for which in (0, 1):
    order, lptr, nlev, estart, nent, width = ilu._small_plan(which)
    def run(nl):
        _lib.call("jv_solve_small", which, n, dv.ptr(ilu.row_start), dv.ptr(ilu.col), dv.ptr(ilu.val),
                  dv.ptr(ilu.diag_pos), dv.ptr(order), dv.ptr(lptr), nl, dv.ptr(estart), nent, width,
                  dv.ptr(b), dv.ptr(y), dv.stream())
    print("which", which, "nlev", nlev, "width", width, "nent", nent,
          "full_us %.1f" % t(lambda: run(nlev)), "staging_only_us %.1f" % t(lambda: run(0)),
          "half_levels_us %.1f" % t(lambda: run(nlev // 2)))
