"""Device time of the sync-free factor kernel over row sub-ranges of a config
(the streamed factor_serial's chunks): python tools/range_cost.py c3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1812_06160_b200 import device as dv

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
a, plan, s, blocks = bench.build_config(cfg)
ilu = plan.ilu
n = ilu.n


def timed(lo, hi, reps=3):
    ts = []
    for _ in range(reps):
        plan.reset_values()
        if lo > 0:
            ilu._factor_tickets(0, lo, 0, True)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        ilu._factor_tickets(lo, hi, lo, False, reset=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return round(sorted(ts)[len(ts) // 2])


print("full", timed(0, n))
for frac in (2, 4, 16, 64, 256, 4096):
    m = n // frac
    sched = ilu.factor_schedule()
    print("rows [0, n/%d)" % frac, timed(0, m), "us;  middle range", timed(n // 2, n // 2 + m), "us",
          "batches", ilu._sub[1][(0, m)].nbatch if (0, m) in ilu._sub[1] else None)
