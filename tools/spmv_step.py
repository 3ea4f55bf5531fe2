"""spmv timed back to back versus right after a region / ticket backward
sweep (as in the bench step): python tools/spmv_step.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1812_06160_b200 as jv
from paper_1812_06160_b200 import device as dv, workloads as W
from paper_1812_06160_b200.plan import build_plan

a, base, s = W.config_matrix("c2")
plan = build_plan(a, base_perm=jv.rcm_order(a.pattern).perm, k=0, tau=0.0,
                  min_level_rows=s["min_level_rows"])
ilu = plan.ilu
n = ilu.n
b = dv.f64(np.random.default_rng(0).uniform(-1, 1, n))
y, x, sy = dv.empty_f64(n), dv.empty_f64(n), dv.empty_f64(n)
plan.reset_values()
ilu.factor_async()
ilu.solve_async(0, b, y)
ilu.solve_async(1, y, x)
plan.permuted.tile_rows()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]


def span(fn, reps=20):
    """Average time of fn() over `reps` back-to-back calls (one event pair:
    single-launch event times are quantised to ~2 us)."""
    fn()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) * 1e3 / reps


def med(fn, n=5):
    return float(np.median([fn() for _ in range(n)]))


def spmv():
    dv.spmv_dev(plan.permuted, b, sy)


def bwd():
    ilu.solve_async(1, y, x)


def bwd_spmv():
    bwd()
    spmv()


t_b2b = med(lambda: span(spmv))
t_bwd = med(lambda: span(bwd))
t_pair = med(lambda: span(bwd_spmv))
print({"spmv_b2b_us": round(t_b2b, 2), "spmv_after_bwd_us": round(t_pair - t_bwd, 2),
       "bwd_us": round(t_bwd, 2), "impl": os.environ.get("JV_SPMV_IMPL"),
       "cfg": os.environ.get("JV_SPMV_CFG")})
