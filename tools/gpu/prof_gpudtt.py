import sys, time, os, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from paper_2202_04894_b200.workloads import make_workload
from paper_2202_04894_b200.tree import build_tree, TreeConfig
from paper_2202_04894_b200.directions import generate_direction_tree
from paper_2202_04894_b200.gpu_build import GpuDtt
from paper_2202_04894_b200.plan import NativeDtt, _traversal_tables, hf_max_level
name = sys.argv[1]
pts, q, kappa, w = make_workload(name)
tt, _ = build_tree(pts, q, TreeConfig(ncrit=w.ncrit))
hf = hf_max_level(tt, tt.depth, kappa, 2.0)
dt = generate_direction_tree(hf)
dir_off = np.concatenate([[0], np.cumsum([d.shape[0] for d in dt.levels])]).astype(np.int64)
tabs = _traversal_tables(tt, tt.depth, hf, dt, dir_off, kappa, 1.0)
GpuDtt(tt, tt, 2, *tabs)
t0 = time.perf_counter(); n = NativeDtt(tt, tt, tt.depth, *tabs); print("native", time.perf_counter() - t0)
torch.cuda.synchronize(); t0 = time.perf_counter(); g = GpuDtt(tt, tt, tt.depth, *tabs); torch.cuda.synchronize(); print("gpu", time.perf_counter() - t0)
pr = cProfile.Profile(); pr.enable(); g = GpuDtt(tt, tt, tt.depth, *tabs); torch.cuda.synchronize(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
