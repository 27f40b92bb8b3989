import sys, time, os, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2202_04894_b200 import FmmConfig, FmmPlan
from paper_2202_04894_b200.workloads import make_workload
name = sys.argv[1]
pts, q, kappa, w = make_workload(name)
cfg = FmmConfig(order=w.order, ncrit=w.ncrit, kappa=kappa, dtype=w.dtype)
for b in ("host", "gpu"):
    plan = FmmPlan(pts, None, cfg, charges=q, build=b); del plan
pr = cProfile.Profile(); pr.enable()
plan = FmmPlan(pts, None, cfg, charges=q, build="gpu")
torch.cuda.synchronize(); pr.disable()
print(plan.timings)
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
