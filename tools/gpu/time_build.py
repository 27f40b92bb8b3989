"""Plan construction: host (native C++) vs device builders, per stage."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2202_04894_b200 import FmmConfig, FmmPlan
from paper_2202_04894_b200.workloads import make_workload
for name in sys.argv[1:] or ["cfg2", "cfg3", "cfg5", "cfg4"]:
    pts, q, kappa, w = make_workload(name)
    cfg = FmmConfig(order=w.order, ncrit=w.ncrit, kappa=kappa, dtype=w.dtype)
    res = {}
    for b in ("host", "gpu", "host", "gpu", "host", "gpu"):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        plan = FmmPlan(pts, None, cfg, charges=q, build=b)
        torch.cuda.synchronize(); res[b] = (round(time.perf_counter() - t0, 3), {k: round(v, 3) for k, v in plan.timings.items()})
        counts = plan.plan.counts
        del plan
    print(name, res, counts["m2l_events"], flush=True)
