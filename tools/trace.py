"""Per-batch timeline of one factorization (globaltimer stamps) -> level stats.

    python tools/trace.py --config c1|c2|... [--rmat-seed S]
"""

import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--rmat-seed", type=int, default=-1)
    ap.add_argument("--backoff", type=int, default=None)
    ap.add_argument("--tridiag", type=int, default=0)
    ap.add_argument("--tag", default="")
    args = ap.parse_args()
    import torch
    import paper_1812_06160_b200 as jv
    from paper_1812_06160_b200 import _lib, device as dv, workloads as W
    from paper_1812_06160_b200.plan import build_plan

    if args.backoff is not None:
        _lib.call("jv_set_backoff", args.backoff)
    if args.tridiag:
        a, base, s = W.tridiag(args.tridiag), None, dict(k=0, tau=0.0, min_level_rows=16)
    elif args.rmat_seed >= 0:
        a, base, s = W.rmat(18, args.rmat_seed), None, W.CONFIGS["c5"]
    else:
        a, base, s = W.config_matrix(args.config)
    base_perm = jv.rcm_order(a.pattern).perm if base == "rcm" else (
        None if base is None else base.perm)
    plan = build_plan(a, base_perm=base_perm, k=s["k"], tau=s["tau"],
                      min_level_rows=s["min_level_rows"])
    ilu = plan.ilu
    sch = ilu.factor_schedule()
    nb = sch.nbatch
    buf = torch.zeros(16 * nb, dtype=torch.int64, device="cuda")
    for rep in range(3):
        plan.reset_values()
        _lib.call("jv_set_trace", dv.ptr(buf), nb if rep == 2 else 0)
        ilu.factor_async()
        torch.cuda.synchronize()
    _lib.call("jv_set_trace", None, 0)
    tr = buf.cpu().numpy().reshape(nb, 16).astype(np.int64)
    bp = dv.host_i64(sch.batch_ptr, nb + 1)
    order = dv.host_i64(sch.order, ilu.n)
    keys = dv.host_i64(sch.keys, ilu.n)
    first = order[bp[:-1]]
    tag = args.tag or (f"rmat{args.rmat_seed}" if args.rmat_seed >= 0 else
                       (f"tridiag{args.tridiag}" if args.tridiag else args.config))
    os.makedirs(os.path.join(REPO, "gpurun_out"), exist_ok=True)
    np.savez_compressed(os.path.join(REPO, "gpurun_out", f"trace_{tag}.npz"), tr=tr, bp=bp,
                        first=first, key=keys[first],
                        rs=dv.host_i64(ilu.row_start, ilu.n + 1), diag=dv.host_i64(ilu.diag_pos, ilu.n),
                        heavy=(ilu.elim_lists()[0][:ilu.n].cpu().numpy() if ilu.elim_lists()
                               else np.zeros(ilu.n, np.int8)))
    ncls = len(getattr(sch, "steps", (32, 1)))
    lev = keys[first] // ncls
    cls = keys[first] % ncls
    t = tr[:, :5] - tr[:, 0].min()
    nlev = int(lev.max()) + 1
    lev_end = np.array([t[lev == L, 4].max() for L in range(nlev)])
    hop = np.diff(lev_end)
    busy = (t[:, 4] - t[:, 0]).sum()
    nwarps = len(np.unique(tr[:, 5]))
    out = {
        "tag": tag, "batches": int(nb), "levels": nlev, "warps": nwarps,
        "total_us": float(t[:, 4].max()) / 1e3,
        "busy_frac": float(busy / (nwarps * t[:, 4].max())),
        "claim_us_median": float(np.median(t[:, 1] - t[:, 0])) / 1e3,
        "struct_us_median": float(np.median(t[:, 2] - t[:, 1])) / 1e3,
        "gatewait_us_median": float(np.median(t[:, 3] - t[:, 2])) / 1e3,
        "finish_us_median": float(np.median(t[:, 4] - t[:, 3])) / 1e3,
        "finish_us_p90": float(np.percentile(t[:, 4] - t[:, 3], 90)) / 1e3,
        "level_hop_us_median": float(np.median(hop)) / 1e3 if hop.size else None,
        "warp_class_batches": int((cls == 1).sum()),
    }
    # time per level: where the makespan goes
    lev_start = np.array([t[lev == L, 0].min() for L in range(nlev)])
    sizes = np.bincount(lev, minlength=nlev)
    span = lev_end - np.concatenate([[0], lev_end[:-1]])
    top = np.argsort(-span)[:8]
    out["top_levels(level,batches,us_added)"] = [(int(L), int(sizes[L]), float(span[L]) / 1e3) for L in top]
    out["busy_warps_frac_by_quartile"] = [float(x) for x in np.percentile(span, [25, 50, 75, 100]) / 1e3]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
