"""GPU probe: does the P2P on the side stream overlap the far-field launches?"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2202_04894_b200 import FmmConfig
from paper_2202_04894_b200.fmm import FmmPlan
from paper_2202_04894_b200.workloads import make_workload

pts, q, kappa, w = make_workload(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
plan = FmmPlan(pts, None, FmmConfig(order=w.order, ncrit=w.ncrit, kappa=kappa, dtype=w.dtype), charges=q)
print("current stream handle", torch.cuda.current_stream().cuda_stream, "side", plan.side_stream.cuda_stream)


def timed(fn, stream, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(n):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


ms = torch.cuda.current_stream()
for fp in (False, True):
    plan.far_priority = fp
    for grid in (0, 592):
        plan.p2p_grid = grid
        res = {}
        for ov in ("upward", "full"):
            plan.p2p_overlap = ov
            res[ov] = timed(lambda: plan.apply(), ms)
        def p2p_only():
            plan._near_field(None)
            ms.wait_stream(plan.side_stream)
        t_p2p = timed(p2p_only, ms)
        print(f"far_priority={fp} grid={grid}: " + " ".join(f"{k}={v:.3f}" for k, v in res.items()) + f" p2p alone={t_p2p:.3f} ms")
