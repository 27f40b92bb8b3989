"""Small matvecs for compute-sanitizer (memcheck / racecheck): one golden case
through every M2L kernel family and both P2P paths, checked against the
reference potentials.  usage: compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import load_case  # noqa: E402
from paper_2202_04894_b200 import FmmConfig, FmmPlan  # noqa: E402

g = load_case(sys.argv[1] if len(sys.argv) > 1 else "sphere3000")
for dtype, tol in (("c128", 1e-11), ("c64", 2e-5)):
    cfg = FmmConfig(**{**g["config"], "dtype": dtype})
    base = None
    for mode in ("auto", "rows", "blocked_all", "pairs_all", "quartets_all", "staged_all"):
        plan = FmmPlan(g["points"], None, cfg, charges=g["charges"], reuse=base, m2l=mode)
        base = base or plan
        pot = plan.apply().cpu().numpy().astype(complex)
        rel = np.linalg.norm(pot - g["pot"]) / np.linalg.norm(g["pot"])
        assert rel <= tol, (dtype, mode, rel)
        print(dtype, mode, f"{rel:.2e}", flush=True)
os.environ["DEFMM_P2P_MUTUAL"] = "0"
plan = FmmPlan(g["points"], None, FmmConfig(**g["config"]), charges=g["charges"])
pot = plan.apply().cpu().numpy()
print("one-directional P2P", np.linalg.norm(pot - g["pot"]) / np.linalg.norm(g["pot"]))
