"""GPU diagnostics: per-phase timing of the hot path on one config.

    python tools/diag.py --config c2 [--backoff 256] [--spin 22] [--reps 5]
Env JV_BLOCKS_PER_SM caps resident CTAs per SM.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--backoff", type=int, default=None)
    ap.add_argument("--spin", type=int, default=24)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--rmat-seed", type=int, default=-1)
    ap.add_argument("--gate", type=int, default=None)
    ap.add_argument("--poll", type=int, default=None)
    ap.add_argument("--group", type=int, default=None)
    ap.add_argument("--staged", type=int, default=None)
    args = ap.parse_args()
    import torch
    import paper_1812_06160_b200 as jv
    from paper_1812_06160_b200 import _lib, device as dv, workloads as W
    from paper_1812_06160_b200.plan import build_plan

    torch.cuda.init()
    _lib.call("jv_set_spin_limit", 1 << args.spin)
    if args.backoff is not None:
        _lib.call("jv_set_backoff", args.backoff)
    if args.gate is not None:
        _lib.call("jv_set_gate", args.gate)
    if args.poll is not None:
        _lib.call("jv_set_poll", args.poll)
    if args.group is not None:
        _lib.call("jv_set_sfp_group", args.group)
    if args.staged is not None:
        _lib.call("jv_set_solve_staged", args.staged)
    t0 = time.time()
    if args.rmat_seed >= 0:
        a, base, s = W.rmat(18, args.rmat_seed), None, W.CONFIGS["c5"]
    else:
        a, base, s = W.config_matrix(args.config)
    tg = time.time() - t0
    base_perm = None
    if base == "rcm":
        base_perm = jv.rcm_order(a.pattern).perm
    elif base is not None:
        base_perm = base.perm
    t0 = time.time()
    plan = build_plan(a, base_perm=base_perm, k=s["k"], tau=s["tau"],
                      min_level_rows=s["min_level_rows"])
    torch.cuda.synchronize()
    dv.check_hang()
    tp = time.time() - t0
    ilu = plan.ilu
    t0 = time.time()
    ilu.factor_schedule(); ilu.fwd_schedule(); ilu.bwd_schedule(); torch.cuda.synchronize(); dv.check_hang()
    ts = time.time() - t0
    out = {"config": args.config, "gen_s": tg, "plan_s": tp, "sched_s": ts, "n": ilu.n,
           "nnz_f": ilu.nnz, "fac_nbatch": ilu._fsched.nbatch, "fwd_nbatch": ilu._fwd.nbatch, "bwd_nbatch": ilu._bwd.nbatch,
           "blocks_per_sm": os.environ.get("JV_BLOCKS_PER_SM"), "backoff": args.backoff}
    b = dv.f64(np.ones(ilu.n))
    y = dv.empty_f64(ilu.n)
    x = dv.empty_f64(ilu.n)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    fs, fw, bw = [], [], []
    for rep in range(args.reps):
        plan.reset_values()
        ev[0].record()
        ilu.factor_async()
        ev[1].record()
        ilu.solve_async(0, b, y)
        ev[2].record()
        ilu.solve_async(1, y, x)
        ev[3].record()
        torch.cuda.synchronize()
        fs.append(ev[0].elapsed_time(ev[1]))
        fw.append(ev[1].elapsed_time(ev[2]))
        bw.append(ev[2].elapsed_time(ev[3]))
        try:
            dv.check_hang()
        except RuntimeError as e:
            out["hang_rep"] = rep
            break
    out.update(factor_ms=fs, fwd_ms=fw, bwd_ms=bw, err=dv.read_row_slot(ilu.err))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
