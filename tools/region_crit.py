"""Critical-path analysis of one region sweep on a config: for every level,
the wave that finishes last; the phase breakdown of those waves (trace
marks).  python tools/region_crit.py c2 fwd"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1812_06160_b200 as jv
from paper_1812_06160_b200 import _lib, device as dv, regionplan as RP, workloads as W
from paper_1812_06160_b200.plan import build_plan

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
sweep = sys.argv[2] if len(sys.argv) > 2 else "fwd"
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
rp = ilu._region_for(sweep)
assert rp is not None, "sweep not on the region path"
fn = {"factor": lambda: (plan.reset_values(), ilu.factor_async()),
      "fwd": lambda: ilu.solve_async(0, b, y), "bwd": lambda: ilu.solve_async(1, y, x)}[sweep]
nw = rp["waves"]
buf = torch.zeros(16 * nw, dtype=torch.int64, device="cuda")
fn()
torch.cuda.synchronize()
_lib.call("jv_set_trace", dv.ptr(buf), nw)
_lib.call("jv_set_region_flags", int(os.environ.get("JV_RFLAGS", "0")))
fn()
torch.cuda.synchronize()
_lib.call("jv_set_trace", None, 0)
_lib.call("jv_set_region_flags", 0)
tr = buf.cpu().numpy().reshape(nw, 16)
g = tr[:, 0:8].astype(np.float64)
c = tr[:, 8:16]
t0 = g[:, 1].min()
start, end = (g[:, 1] - t0) / 1e3, (g[:, 7] - t0) / 1e3
ph = np.stack([c[:, 2] - c[:, 1], c[:, 3] - c[:, 2], c[:, 4] - c[:, 3], c[:, 7] - c[:, 4]], 1)
# level of each wave: the level of its first row (host decode of the stream)
rw = rp["reg_wave"].cpu().numpy()
words = rp["words"].cpu().numpy()
table = rp["table"].cpu().numpy().reshape(-1, 8)
rs, col, diag = ilu._host_pattern()
lev = np.zeros(n, np.int64)
if sweep == "bwd":
    for r in range(n - 1, -1, -1):
        u = col[diag[r] + 1:rs[r + 1]]
        lev[r] = lev[u].max() + 1 if u.size else 0
else:
    for r in range(n):
        l = col[rs[r]:diag[r]]
        lev[r] = lev[l].max() + 1 if l.size else 0
wl = np.array([lev[words[int(table[w, 0]) * 4 + 4 + 5]] for w in range(nw)])   # first record's row
L = wl.max() + 1
if os.environ.get("JV_CRIT_DUMP"):
    np.savez_compressed(os.environ["JV_CRIT_DUMP"], g=tr[:, 0:8], c=c,  wl=wl, rw=rw,
                        cnt=np.array([words[int(table[w, 0]) * 4] for w in range(nw)]),
                        npk=table[:, 7] >> 16)
crit = np.array([np.argmax(np.where(wl == l, end, -1)) for l in range(L)])
tl = end[crit]
dt = np.diff(np.concatenate([[0.0], tl]))
cp = ph[crit]
print(json.dumps({"cfg": cfg, "sweep": sweep, "levels": int(L), "span_us": float(end.max()),
                  "per_level_us_median": float(np.median(dt)), "per_level_us_mean": float(dt.mean()),
                  "crit_phase_cycles_median[wait,remote+deps,compute,bar]": np.median(cp, 0).tolist(),
                  "crit_phase_cycles_mean": cp.mean(0).round(1).tolist(),
                  "crit_wave_us_median": float(np.median(end[crit] - start[crit])),
                  "crit_start_minus_prev_end_us_median": float(np.median(start[crit][1:] - tl[:-1])),
                  "region_changes_on_crit": int((np.diff([np.searchsorted(rw, w, side='right') for w in crit]) != 0).sum())}))
