"""Where the end-to-end matvec's time goes: H2D, charge gather, graph replay, D2H (events per phase)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2202_04894_b200 import FmmConfig, FmmPlan
from paper_2202_04894_b200.workloads import make_workload

pts, q, kappa, w = make_workload(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
cfg = FmmConfig(order=w.order, ncrit=w.ncrit, kappa=kappa, dtype=w.dtype)
plan = FmmPlan(pts, None, cfg, charges=q)
dev = plan.device
st = torch.cuda.current_stream(dev)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
q_src = torch.as_tensor(q).to(plan.cdtype)
q_host = q_src.clone().pin_memory()
REFRESH = os.environ.get("REFRESH", "0") == "1"
out_host = torch.empty(q_host.shape[0], dtype=plan.cdtype).pin_memory()
for _ in range(3):
    plan.set_charges(q_host.to(dev, non_blocking=True)); out_host.copy_(plan.apply(), non_blocking=True)
torch.cuda.synchronize()
for rep in range(6):
    acc = np.zeros(5)
    n = 20
    for _ in range(n):
        flush.zero_()
        if REFRESH:
            q_host.copy_(q_src)  # the step's input written by the host, as a solver would
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record(st)
        qd = q_host.to(dev, non_blocking=True); ev[1].record(st)
        plan.set_charges(qd); ev[2].record(st)
        o = plan.apply(); ev[3].record(st)
        out_host.copy_(o, non_blocking=True); ev[4].record(st)
        torch.cuda.synchronize()
        acc += [ev[i].elapsed_time(ev[i + 1]) for i in range(4)] + [ev[0].elapsed_time(ev[4])]
    print("h2d %.3f  gather %.3f  apply %.3f  d2h %.3f  total %.3f" % tuple(acc / n), flush=True)
