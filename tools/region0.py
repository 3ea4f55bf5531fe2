"""Per-region wave cadence from the light trace (end-of-wave marks only):
python tools/region0.py c2 factor|fwd|bwd   (JV_RFLAGS, JV_REGION_D apply)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1812_06160_b200 as jv
from paper_1812_06160_b200 import _lib, device as dv, workloads as W
from paper_1812_06160_b200.plan import build_plan

cfg = sys.argv[1]
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
for flags in [int(f) for f in os.environ.get("JV_RFLAGS_LIST", "16").split(",")]:
    for sweep in sys.argv[2:]:
        rp = ilu._region_for(sweep)
        fn = {"factor": lambda: (plan.reset_values(), ilu.factor_async()),
              "fwd": lambda: ilu.solve_async(0, b, y), "bwd": lambda: ilu.solve_async(1, y, x)}[sweep]
        nw = rp["waves"]
        buf = torch.zeros(16 * nw, dtype=torch.int64, device="cuda")
        fn()
        torch.cuda.synchronize()
        _lib.call("jv_set_trace", dv.ptr(buf), nw)
        _lib.call("jv_set_region_flags", flags)
        fn()
        torch.cuda.synchronize()
        _lib.call("jv_set_trace", None, 0)
        _lib.call("jv_set_region_flags", 0)
        tr = buf.cpu().numpy().reshape(nw, 16)
        c = tr[:, 15]
        g = tr[:, 7] if tr[:, 7].any() else c / 1.965
        rw = rp["reg_wave"].cpu().numpy()
        med = []
        for r in range(len(rw) - 1):
            med.append(np.median(np.diff(c[rw[r]:rw[r + 1]])))
        if flags & 256:
            a0, b0 = rw[0], rw[1]
            cc = tr[a0:b0, 8:16]
            # marks: 1 top (after probed wait), 3 deps loaded, 2 next operands loaded, 4 computed, 5 after barrier
            print("  region0 phases (median cycles): deps", np.median(cc[:, 3] - cc[:, 1]),
                  "fetch", np.median(cc[:, 2] - cc[:, 3]), "compute", np.median(cc[:, 4] - cc[:, 2]),
                  "barrier", np.median(cc[:, 5] - cc[:, 4]), "loop", np.median(cc[1:, 1] - cc[:-1, 5]))
        print(sweep, "flags", flags, "D", min(rp["D"], dv._REGION_D_CAP), "span_us", (g.max() - g.min()) / 1e3,
              "region0 cyc/wave", med[0], "median over regions", np.median(med), flush=True)
