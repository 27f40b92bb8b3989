"""c64 vs the north-star bar (1e-2 eps_ref) on every small golden case."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tests"))
import numpy as np
from conftest import golden_cases, load_case
from oracle import defmm_oracle as O
from paper_2202_04894_b200 import FmmConfig, run_fmm_full
from paper_2202_04894_b200.geometry import compute_root_box
for c in golden_cases():
    g = load_case(c)
    pts, q = g["points"], g["charges"]
    kap = g["config"].get("kappa", 0.0)
    side = compute_root_box(pts).side
    d = O.direct_sum(pts, pts, q, kap, 1e-12 * side)
    eps_ref = np.linalg.norm(g["pot"] - d) / np.linalg.norm(d)
    out = {"case": c, "L": g["config"].get("order"), "eps_ref": eps_ref, "bar": 1e-2 * eps_ref}
    for dt in ("c64", "c128"):
        pot, _ = run_fmm_full(pts, pts, q, FmmConfig(dtype=dt, **g["config"]))
        out[dt] = float(np.linalg.norm(pot - g["pot"]) / np.linalg.norm(g["pot"]))
    print(json.dumps(out), flush=True)
