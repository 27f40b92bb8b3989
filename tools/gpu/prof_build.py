"""cProfile of one FmmPlan construction (device builders) after a warm-up build."""
import sys, os, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2202_04894_b200 import FmmConfig, FmmPlan
from paper_2202_04894_b200.workloads import make_workload
name = sys.argv[1]
pts, q, kappa, w = make_workload(name)
cfg = FmmConfig(order=w.order, ncrit=w.ncrit, kappa=kappa, dtype=w.dtype)
plan = FmmPlan(pts, None, cfg, charges=q); del plan
pr = cProfile.Profile(); pr.enable()
plan = FmmPlan(pts, None, cfg, charges=q)
torch.cuda.synchronize(); pr.disable()
print(plan.timings)
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
