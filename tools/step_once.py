"""Two warm steps, then ONE bench step (refresh + factor + forward + backward
+ spmv) between cudaProfilerStart/Stop, for targeted ncu captures:

    ncu --profile-from-start off --set full --clock-control none \
        --import-source on -o out python tools/step_once.py c2
"""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    count = int(sys.argv[2]) if len(sys.argv) > 2 else 4   # c5: R-MAT systems
    import torch
    from bench import build_config, rhs
    from paper_1812_06160_b200 import device as dv

    a, plan, s, blocks = build_config(cfg, rmat_count=count)
    ilu = plan.ilu
    n = ilu.n
    b = dv.f64(np.asarray(rhs(n, blocks))[dv.host_i64(plan.perm, n)])
    y, x, sy = dv.empty_f64(n), dv.empty_f64(n), dv.empty_f64(n)
    plan.permuted.tile_rows()

    def step():
        plan.reset_values()
        ilu.factor_async()
        ilu.solve_async(0, b, y)
        ilu.solve_async(1, y, x)
        dv.spmv_dev(plan.permuted, b, sy)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    dv.check_hang()
    torch.cuda.profiler.start()
    step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("step_once", cfg, "impl", getattr(ilu, "impl", None))


if __name__ == "__main__":
    main()
