"""spmv timing on a config's permuted matrix (CUDA events, back-to-back),
bitwise check against the oracle.   python tools/spmv_bench.py [c2] [reps]"""
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    import torch
    import oracle
    from bench import build_config, alg_bytes, peaks
    from paper_1812_06160_b200 import device as dv
    a, plan, s, _ = build_config(cfg)
    A = plan.permuted
    x = np.random.default_rng(0).uniform(-1, 1, A.n)
    xd, yd = dv.f64(x), dv.empty_f64(A.n)
    A.tile_rows()
    for _ in range(3):
        dv.spmv_dev(A, xd, yd)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        dv.spmv_dev(A, xd, yd)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    rs, col = A.host_pattern()
    want = oracle.spmv(rs, col, dv.host_f64(A.val, A.nnz), x)
    got = dv.host_f64(yd, A.n)
    b = alg_bytes(A.n, A.nnz, 0)["spmv"]
    peak, _ = peaks()
    print(json.dumps({"cfg": cfg, "us": us, "GBps": b / us / 1e3, "frac": b / us / 1e3 / peak,
                      "bitwise": bool(np.array_equal(got, want)),
                      "maxrel": float(np.max(np.abs(got - want)) / np.max(np.abs(want)))}))


if __name__ == "__main__":
    main()
