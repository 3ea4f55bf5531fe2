"""Time the c5 factor / solves on one R-MAT matrix (seed argv[1])."""
import sys, time, json
import numpy as np
import torch
from paper_1812_06160_b200 import workloads as W, device as dv
from paper_1812_06160_b200.plan import build_plan

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 0
scale = int(sys.argv[2]) if len(sys.argv) > 2 else 18
a = W.rmat(scale, seed)
t0 = time.time()
plan = build_plan(a, k=0)
ilu = plan.ilu
ilu.factor_schedule(); el = ilu.elim_lists()
torch.cuda.synchronize()
setup = time.time() - t0
res = {"seed": seed, "n": a.n, "nnz": ilu.nnz, "setup_s": round(setup, 2),
       "heavy_ops": el[3] if el else 0,
       "heavy_rows": int(el[0][:a.n].sum().item()) if el else 0}
ms = []
for i in range(3):
    plan.reset_values()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); bad = ilu.factor_async(); e1.record(); torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
bad = dv.read_row_slot(ilu.err); dv.check_hang()
res["factor_ms"] = [round(x, 3) for x in ms]
res["bad"] = bad
b = dv.f64(np.random.default_rng(0).uniform(-1, 1, a.n)); y = dv.empty_f64(a.n); x = dv.empty_f64(a.n)
for which, src, dst in ((0, b, y), (1, y, x)):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    ilu.solve_async(which, src, dst)
    e0.record(); ilu.solve_async(which, src, dst); e1.record(); torch.cuda.synchronize()
    res["fwd_ms" if which == 0 else "bwd_ms"] = round(e0.elapsed_time(e1), 3)
print(json.dumps(res))
