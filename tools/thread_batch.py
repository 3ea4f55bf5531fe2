import sys, json
sys.path.insert(0, '/root/repo')
import torch
from paper_1812_06160_b200 import device as dv
from bench import build_config
for tb in (32, 24, 16, 8):
    dv.DevIlu.THREAD_BATCH = tb
    a, plan, s, _ = build_config("c2")
    ilu = plan.ilu
    ms = []
    for _ in range(5):
        plan.reset_values()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); ilu.factor_async(); e1.record(); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    print(json.dumps({"thread_batch": tb, "factor_ms": min(ms[1:])}))
