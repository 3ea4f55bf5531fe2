"""Why a region plan does (not) build: for every candidate partition and
wave width the status and sizes of jv_rstream_build.
python tools/region_fit.py c4 bwd"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1812_06160_b200 as jv
from paper_1812_06160_b200 import _lib, device as dv, regionplan as RP, workloads as W
from paper_1812_06160_b200.plan import build_plan

cfg, sweep = sys.argv[1], sys.argv[2]
a, base, s = W.config_matrix(cfg)
bp = jv.rcm_order(a.pattern).perm if base == "rcm" else (base.perm if base is not None and hasattr(base, "perm") else base)
plan = build_plan(a, base_perm=bp, k=s["k"], tau=s["tau"], min_level_rows=s["min_level_rows"])
ilu = plan.ilu
rs, col, diag = ilu._host_pattern()
props = torch.cuda.get_device_properties(0)
budget = props.shared_memory_per_block_optin - 2048
lib = _lib.load()
for cand in ilu.region_candidates[sweep]:
    reg = ilu.regions(*cand)
    if reg is None:
        print(cand, "no partition")
        continue
    nreg, region_of = reg
    for t in (512, 256, 128):
        sizes = np.zeros(13, np.int64)
        r, c, d, ro = (np.ascontiguousarray(x, np.int32) for x in (rs, col, diag, region_of))
        h = lib.jv_rstream_build(RP.KINDS[sweep], d.size, RP._p(r), RP._p(c), RP._p(d), RP._p(ro),
                                 int(nreg), t, int(budget), int(ilu.tau > 0), RP._p(sizes))
        print(cand, "nreg", nreg, "threads", t, "status", h,
              dict(zip(["static", "waves", "nreg", "SC", "max_waves", "S", "D", "CS", "CD", "remote",
                        "m", "mv", "max_rows"], sizes.tolist())) if h > 0 else "")
