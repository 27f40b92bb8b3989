cd $GRAFT_REPO_ROOT
O=gpurun_out/r15; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_build.py -m gpu -q -x > $O/tests.log 2>&1
echo "tests rc=$?" >> $O/rc.txt
python - > $O/time_tree.log 2>&1 <<'PY'
import time, numpy as np, torch
from paper_2202_04894_b200.workloads import make_workload
from paper_2202_04894_b200.tree import build_tree, TreeConfig
from paper_2202_04894_b200.gpu_build import build_tree_gpu
for name in ("cfg2", "cfg3", "cfg4"):
    pts, q, kappa, w = make_workload(name)
    cfg = TreeConfig(ncrit=w.ncrit)
    t0 = time.perf_counter(); th, ph = build_tree(pts, q, cfg); t1 = time.perf_counter()
    build_tree_gpu(pts[:1000], q[:1000], cfg)
    torch.cuda.synchronize(); t2 = time.perf_counter(); tg, pg = build_tree_gpu(pts, q, cfg); torch.cuda.synchronize(); t3 = time.perf_counter()
    same = all(np.array_equal(getattr(tg, k), getattr(th, k)) for k in ("level", "coords", "start", "stop", "parent")) and np.array_equal(pg.original_index, ph.original_index)
    print(name, "N", pts.shape[0], "cells", th.n_cells, "host s", round(t1 - t0, 3), "gpu s", round(t3 - t2, 3), "equal", same, flush=True)
PY
