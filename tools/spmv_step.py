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


def med(fn, reps=10):
    ts = []
    for _ in range(reps):
        t = fn()
        ts.append(t)
    return float(np.median(ts))


def b2b():
    dv.spmv_dev(plan.permuted, b, sy)
    ev[0].record()
    dv.spmv_dev(plan.permuted, b, sy)
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) * 1e3


def after_bwd():
    ilu.solve_async(1, y, x)
    ev[0].record()
    dv.spmv_dev(plan.permuted, b, sy)
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) * 1e3


def after_bwd_gap():
    ilu.solve_async(1, y, x)
    ev[2].record()
    torch.cuda._sleep(20000)
    ev[0].record()
    dv.spmv_dev(plan.permuted, b, sy)
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) * 1e3


print({"spmv_b2b_us": med(b2b), "spmv_after_bwd_us": med(after_bwd),
       "spmv_after_bwd_and_sleep_us": med(after_bwd_gap), "bwd_impl_region": ilu._region_for("bwd") is not None})
