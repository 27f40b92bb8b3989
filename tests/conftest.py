import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libdefmm_b200.so")


def golden_cases():
    return sorted(os.path.basename(p)[4:-4] for p in glob.glob(os.path.join(GOLDEN, "fmm_*.npz")))


def load_case(name):
    d = np.load(os.path.join(GOLDEN, f"fmm_{name}.npz"))
    return {
        "points": d["points"],
        "charges": d["charges"],
        "config": json.loads(str(d["config"])),
        "pot": d["pot"],
        "counts": json.loads(str(d["counts"])),
        "hf_max": int(d["hf_max"]),
        "m2l": d["m2l"],
        "p2p": d["p2p"],
    }


def load_ref(name):
    path = os.path.join(GOLDEN, f"ref_{name}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    d = np.load(path)
    out = {k: d[k] for k in d.files}
    out["counts"] = json.loads(str(d["counts"]))
    out["timings"] = json.loads(str(d["timings"]))
    return out


@pytest.fixture(scope="session")
def operators():
    return np.load(os.path.join(GOLDEN, "operators.npz"))


def two_tree_cases():
    return sorted(os.path.basename(p)[4:-4] for p in glob.glob(os.path.join(GOLDEN, "two_*.npz")))


def load_two_tree(name):
    d = np.load(os.path.join(GOLDEN, f"two_{name}.npz"))
    return {
        "targets": d["targets"],
        "sources": d["sources"],
        "charges": d["charges"],
        "config": json.loads(str(d["config"])),
        "pot": d["pot"],
        "counts": json.loads(str(d["counts"])),
        "hf_max": int(d["hf_max"]),
        "m2l": d["m2l"],
        "p2p": d["p2p"],
    }
