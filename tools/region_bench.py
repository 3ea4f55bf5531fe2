"""Region kernels vs ticket kernels on one config: bitwise equality and
back-to-back kernel times (CUDA events).  python tools/region_bench.py c2"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1812_06160_b200 as jv
from paper_1812_06160_b200 import device as dv, workloads as W
from paper_1812_06160_b200.plan import build_plan

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
t0 = time.time()
a, base, s = W.config_matrix(cfg)
bp = jv.rcm_order(a.pattern).perm if base == "rcm" else (base.perm if base is not None and hasattr(base, "perm") else base)
plan = build_plan(a, base_perm=bp, k=s["k"], tau=s["tau"], min_level_rows=s["min_level_rows"])
ilu = plan.ilu
n = ilu.n
print(json.dumps({"cfg": cfg, "n": n, "nnz": ilu.nnz, "setup_s": round(time.time() - t0, 1)}), flush=True)
b = dv.f64(np.random.default_rng(0).uniform(-1, 1, n))
y = dv.empty_f64(n)
x = dv.empty_f64(n)


def timed(fn):
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


res = {}
for mode in ("tickets", "regions"):
    ilu.use_regions = mode == "regions"
    t1 = time.time()
    info = {}
    if ilu.use_regions:
        for sw in ("factor", "fwd", "bwd"):
            rp = ilu.region_stream(sw)
            info[sw] = None if rp is None else {k: rp[k] for k in ("nreg", "slot_ring", "max_waves", "S", "D", "CS", "CD", "waves", "remote_deps")}
    plan.reset_values()
    ilu.factor_async()
    torch.cuda.synchronize()
    dv.check_hang()
    fv = ilu.host_val()
    ilu.solve_async(0, b, y)
    ilu.solve_async(1, y, x)
    torch.cuda.synchronize()
    out = (fv, dv.host_f64(y, n), dv.host_f64(x, n))

    def fac():
        plan.reset_values()
    t_reset = timed(fac)
    t_fac = timed(lambda: (plan.reset_values(), ilu.factor_async())) - t_reset
    t_fwd = timed(lambda: ilu.solve_async(0, b, y))
    t_bwd = timed(lambda: ilu.solve_async(1, y, x))
    dv.check_hang()
    res[mode] = out
    print(json.dumps({"mode": mode, "plan_s": round(time.time() - t1, 1), "factor_us": round(t_fac, 1),
                      "fwd_us": round(t_fwd, 1), "bwd_us": round(t_bwd, 1), "info": info}), flush=True)
same = [bool(np.array_equal(res["tickets"][i], res["regions"][i])) for i in range(3)]
from paper_1812_06160_b200 import _lib as _L
for fl in (0, 4, 8, 12):
    _L.call("jv_set_region_flags", fl)
    print(json.dumps({"flags": fl, "factor_us": round(timed(lambda: (plan.reset_values(), ilu.factor_async())) - timed(lambda: plan.reset_values()), 1),
                      "fwd_us": round(timed(lambda: ilu.solve_async(0, b, y)), 1), "bwd_us": round(timed(lambda: ilu.solve_async(1, y, x)), 1)}), flush=True)
_L.call("jv_set_region_flags", 0)
print(json.dumps({"bitwise_factor_fwd_bwd": same}))

# per-wave phase profile of the region kernels (trace marks in region.cu)
from paper_1812_06160_b200 import _lib
ilu.use_regions = True
_L.call("jv_set_region_flags", int(os.environ.get("JV_TRACE_FLAGS", "0")))
for sw, fn in (("factor", lambda: (plan.reset_values(), ilu.factor_async())),
               ("fwd", lambda: ilu.solve_async(0, b, y)), ("bwd", lambda: ilu.solve_async(1, y, x))):
    rp = ilu.region_stream(sw)
    if rp is None:
        continue
    nw = rp["waves"]
    buf = torch.zeros(16 * nw, dtype=torch.int64, device="cuda")
    fn()
    torch.cuda.synchronize()
    _lib.call("jv_set_trace", dv.ptr(buf), nw)
    fn()
    torch.cuda.synchronize()
    _lib.call("jv_set_trace", None, 0)
    tr = buf.cpu().numpy().reshape(nw, 16)
    c = tr[:, 8:16]
    g = tr[:, 0:8]
    ph = np.stack([c[:, 2] - c[:, 1], c[:, 3] - c[:, 2], c[:, 4] - c[:, 3], c[:, 7] - c[:, 4]], 1)
    rw = rp["reg_wave"].cpu().numpy()
    # critical path: span of globaltimer over all waves
    span = (g[:, 7].max() - g[:, 1].min()) / 1e3
    first_start = np.array([g[rw[i], 1] for i in range(len(rw) - 1)]) - g[:, 1].min()
    t0g = g[:, 1].min()
    reg = []
    for i in range(len(rw) - 1):
        a_, b_ = rw[i], rw[i + 1]
        if b_ > a_:
            st = (g[a_:b_, 1] - t0g) / 1e3
            en = (g[a_:b_, 7] - t0g) / 1e3
            dur = en - st
            reg.append((st[0], en[-1], b_ - a_, float(np.median(dur)), float(np.mean(dur))))
    reg.sort()
    print(json.dumps({"sweep": sw, "first_regions(start,end,waves,med_wave_us,mean_wave_us)": [tuple(round(float(v), 2) for v in r) for r in reg[:3]],
                      "last_regions": [tuple(round(float(v), 2) for v in r) for r in reg[-3:]]}), flush=True)
    print(json.dumps({"sweep": sw, "waves": int(nw), "span_us": round(float(span), 1),
                      "median_cycles[wait+pkt,probe,compute,issue+bar]": np.median(ph, 0).tolist(),
                      "p90": np.percentile(ph, 90, 0).tolist(),
                      "mean": np.mean(ph, 0).round(1).tolist(),
                      "region_start_us_p50_max": [float(np.median(first_start) / 1e3), float(first_start.max() / 1e3)]}), flush=True)
