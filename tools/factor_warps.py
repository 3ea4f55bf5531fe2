"""Ticket factorization time on a config with the library libjv or
JV_LIB (e.g. a JV_FACTOR_WARPS=16 build): python tools/factor_warps.py c4"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1812_06160_b200 as jv
from paper_1812_06160_b200 import device as dv, workloads as W
from paper_1812_06160_b200.plan import build_plan

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
a, base, s = W.config_matrix(cfg)
bp = jv.rcm_order(a.pattern).perm if base == "rcm" else (base.perm if base is not None and hasattr(base, "perm") else base)
plan = build_plan(a, base_perm=bp, k=s["k"], tau=s["tau"], min_level_rows=s["min_level_rows"])
ilu = plan.ilu
ilu.region_mode = "off"
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ts = []
for rep in range(6):
    plan.reset_values()
    ev[0].record()
    ilu.factor_async()
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
dv.check_hang()
v = ilu.host_val()
print(json.dumps({"cfg": cfg, "lib": os.environ.get("JV_LIB", "libjv.so"), "factor_us": round(float(np.median(ts[1:])), 1),
                  "digest": int(np.frombuffer(v.tobytes(), np.uint64).sum() % (1 << 61))}), flush=True)
