import sys, os, time, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1812_06160_b200 as jv
from paper_1812_06160_b200 import device as dv, workloads as W
from paper_1812_06160_b200.plan import build_plan
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
a, base, s = W.config_matrix(cfg)
bp = jv.rcm_order(a.pattern).perm if base == "rcm" else None
plan = build_plan(a, base_perm=bp, k=s["k"], tau=s["tau"], min_level_rows=s["min_level_rows"])
ilu = plan.ilu
k = {"c1": 64, "c2": 128}[cfg]
dims = (k, k) if cfg == "c1" else (k, k, k)
ref = None
for parts in ([None] + ([(6, 6, 4), (5, 5, 5), (6, 5, 4), (4, 4, 4), (8, 6, 3)] if cfg == "c2" else [(12, 12), (10, 10), (8, 8)])):
    if parts is not None and np.prod(parts) > 148:
        continue
    if parts is None:
        ilu.region_hint = None
        ilu._rplan = None
    else:
        ilu.set_regions(W.box_regions(dims, dv.host_i64(plan.perm, ilu.n), parts))
    ts = []
    for rep in range(4):
        plan.reset_values()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ilu.factor_async()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    dv.check_hang()
    v = ilu.host_val()
    if ref is None:
        ref = v
    rp = ilu.region_plan() if parts is not None else None
    print(json.dumps({"parts": parts, "ms": [round(x * 1e3, 3) for x in ts], "bitwise": bool(np.array_equal(v, ref)),
                      "crossing": rp["crossing"] if rp else None, "max_region": rp["max_region"] if rp else None}))

# trace one run with the best partition
if cfg == "c2":
    ilu.set_regions(W.box_regions(dims, dv.host_i64(plan.perm, ilu.n), (6, 6, 4)))
else:
    ilu.set_regions(W.box_regions(dims, dv.host_i64(plan.perm, ilu.n), (8, 8)))
rp = ilu.region_plan()
nw = int(rp["wave_ptr"][-1].item())
from paper_1812_06160_b200 import _lib
buf = torch.zeros(16 * nw, dtype=torch.int64, device="cuda")
plan.reset_values()
_lib.call("jv_set_trace", dv.ptr(buf), nw)
ilu.factor_async()
torch.cuda.synchronize()
_lib.call("jv_set_trace", None, 0)
tr = buf.cpu().numpy().reshape(nw, 16)
c = tr[:, 8:16]
wp = rp["wave_ptr"].cpu().numpy()
# per-wave cycles: top(1->2), remote(2->3), compute(3->4), sync(4->7), and next-top gap
ph = np.stack([c[:, 2] - c[:, 1], c[:, 3] - c[:, 2], c[:, 4] - c[:, 3], c[:, 7] - c[:, 4]], 1)
print(json.dumps({"cfg": cfg, "waves": nw, "median_cycles[top,remote,compute,sync]": np.median(ph, 0).tolist(),
                  "p90": np.percentile(ph, 90, 0).tolist()}))
g0 = slice(wp[0], wp[1])
print("region0 first 12 waves:", ph[g0][:12].tolist())
mid = len(wp) // 2
print("region mid first 12 waves:", ph[wp[mid]:wp[mid+1]][:12].tolist())
