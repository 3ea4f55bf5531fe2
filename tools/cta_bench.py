"""Single-CTA kernels (csrc/cta.cu) vs the other paths: c1 whole matrix and
the c4 corner, per ring depth; device time per sweep (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_1812_06160_b200 import device as dv


def t(fn, reps=20):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


def run(ilu, label):
    n = ilu.n
    b = dv.f64(np.ones(n)); y = dv.empty_f64(n)
    save = ilu.val.clone()
    for rb in (2, 3, 4, 5):
        ilu._cta = None
        ilu.CTA_RINGS = (rb,)
        g = ilu.cta_programs()
        if g["factor"] is None:
            print(label, "rb", rb, "does not fit"); continue
        f = t(lambda: (ilu.val.copy_(save), ilu._factor_cta(False)))
        cp = t(lambda: ilu.val.copy_(save))
        fw = t(lambda: ilu._solve_cta(0, b, y)) if g["fwd"] else None
        bw = t(lambda: ilu._solve_cta(1, b, y)) if g["bwd"] else None
        print(label, "rb", rb, "res", g["factor"]["resident"], "nlev", g["factor"]["nlev"],
              "maxblk", g["factor"]["maxblk"], "factor_us %.1f" % (f - cp), "fwd_us", fw, "bwd_us", bw)
    ilu.val.copy_(save)
    f = t(lambda: (ilu.val.copy_(save), ilu._factor_tickets(0, n, 0, False)))
    print(label, "tickets factor_us %.1f" % (f - cp))


a, plan, s, _ = bench.build_config("c1")
run(plan.ilu, "c1")
a, plan, s, _ = bench.build_config("c4")
ilu = plan.ilu
plan.reset_values()
ilu._factor_tickets(0, plan.n_upper, 0, True)
tp = ilu.tail_plan(plan.n_upper)
_lib = __import__("paper_1812_06160_b200._lib", fromlist=["x"])
_lib.call("jv_tail_upper", tp.h, dv.ptr(ilu.col), dv.ptr(ilu.diag_pos), dv.ptr(ilu.val), dv.ptr(ilu.norms), 0.0, dv.stream())
c = tp.corner
_lib.call("jv_gather", tp.nc, dv.ptr(tp.pos), dv.ptr(ilu.val), dv.ptr(c.val), dv.stream())
run(c, "c4corner")

# per-level clock trace of the c1 factor and forward sweep (thread 0)
from paper_1812_06160_b200 import _lib as L_
a, plan, s, _ = bench.build_config("c1")
ilu = plan.ilu
buf = torch.zeros(16 * 200, dtype=torch.int64, device="cuda")
for sweep in ("factor", "fwd"):
    ilu._cta = None
    ilu.CTA_RINGS = (3,)
    ilu.cta_programs()
    L_.call("jv_set_trace", dv.ptr(buf), 200)
    plan.reset_values()
    if sweep == "factor":
        ilu._factor_cta(False)
    else:
        b = dv.f64(np.ones(ilu.n)); y = dv.empty_f64(ilu.n); ilu._solve_cta(0, b, y)
    torch.cuda.synchronize()
    L_.call("jv_set_trace", None, 0)
    tr = buf.cpu().numpy().reshape(200, 16)[:127]
    clk = tr[:, 8:12].astype(np.int64)
    d = np.diff(clk, axis=1)
    lv = np.diff(clk[:, 0])
    print(sweep, "cycles per level median", np.median(lv), "issue", np.median(d[:, 0]), "compute(thread0)", np.median(d[:, 1]), "wait", np.median(d[:, 2]))
