"""Per-line wall time (CUDA-synchronised) of the plan-construction functions
during one warm FmmPlan build: python tools/gpu/line_time.py cfg4 [func ...]"""
import sys, os, time, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2202_04894_b200 import FmmConfig, FmmPlan
from paper_2202_04894_b200.workloads import make_workload

name = sys.argv[1]
funcs = set(sys.argv[2:] or ["build_plan", "__init__", "_host_lists", "build_tree_gpu", "_local_slots",
                             "p2p_mutual_lists", "dense_levels"])
pts, q, kappa, w = make_workload(name)
cfg = FmmConfig(order=w.order, ncrit=w.ncrit, kappa=kappa, dtype=w.dtype)
plan = FmmPlan(pts, None, cfg, charges=q); del plan
acc = collections.defaultdict(float)
last = {}


def local(frame, event, arg):
    key = id(frame)
    now = None
    if event in ("line", "return"):
        torch.cuda.synchronize()
        now = time.perf_counter()
        if key in last:
            ln, t = last[key]
            acc[(frame.f_code.co_filename.rsplit("/", 1)[-1], frame.f_code.co_name, ln)] += now - t
        if event == "line":
            last[key] = (frame.f_lineno, now)
        else:
            last.pop(key, None)
    return local


def tracer(frame, event, arg):
    if event == "call" and frame.f_code.co_name in funcs and "paper_2202" in frame.f_code.co_filename:
        return local
    return None


sys.settrace(tracer)
t0 = time.perf_counter()
plan = FmmPlan(pts, None, cfg, charges=q)
torch.cuda.synchronize()
sys.settrace(None)
print("total", time.perf_counter() - t0, plan.timings)
for (f, fn, ln), t in sorted(acc.items(), key=lambda kv: -kv[1])[:45]:
    print(f"{t:7.3f}s  {f}:{ln} ({fn})")
