"""Generate small golden fixtures by running the REFERENCE (helmfmm) itself.

Runs only in the build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/fmm_<case>.npz (end-to-end potentials, counts, hf_max,
event lists keyed by (level, Morton code)) and tests/golden/operators.npz
(kernel values, directions + nearest-direction ties, canonical translations,
symbols, M2F/F2L, P2M/L2P, M2M factors).  These pin the CPU oracle
(oracle/defmm_oracle.py) and, through it and directly, the B200 path.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")

from helmfmm import interpolation as I  # noqa: E402
from helmfmm.directions import generate_direction_tree, nearest_direction  # noqa: E402
from helmfmm.distributions import Distribution, generate_distribution, random_charges  # noqa: E402
from helmfmm.fourier import (  # noqa: E402
    FourierWorkspace,
    canonicalize_translation,
    frequency_permutation,
    precompute_symbol,
)
from helmfmm.geometry import CellFrame, compute_root_box  # noqa: E402
from helmfmm.kernel import HelmholtzKernel  # noqa: E402
from helmfmm.traversal import FmmConfig, run_fmm_full  # noqa: E402

from paper_2202_04894_b200.workloads import make_charges, make_points  # noqa: E402


def _cases():
    """(name, points, charges, FmmConfig kwargs)."""
    out = []
    rng = np.random.default_rng(1)
    pts = rng.uniform(size=(500, 3))
    q = rng.uniform(size=500) + 1j * rng.uniform(size=500)
    out.append(("laplace500", pts, q, dict(order=5, ncrit=32, kappa=0.0)))

    rng = np.random.default_rng(0)
    a = rng.uniform(0.01, 0.23, size=(20, 3))
    b = rng.uniform(0.01, 0.23, size=(20, 3))
    b[:, 0] += 0.76
    pts = np.vstack([a, b])
    q = rng.normal(size=40) + 1j * rng.normal(size=40)
    out.append(("twocluster", pts, q, dict(order=7, ncrit=10, kappa=10.0)))

    pts = generate_distribution(Distribution("uniform-cube", 2000, 0))
    q = random_charges(2000, 1)
    for kd in (8.0, 16.0):
        out.append((f"c1_kd{int(kd)}", pts, q, dict(order=6, ncrit=64, kappa=kd / compute_root_box(pts).side)))

    def synth(kind, n, kd, order, ncrit):
        p = make_points(kind, n, 0)
        return p, make_charges(n, 1), dict(order=order, ncrit=ncrit, kappa=kd / compute_root_box(p).side)

    out.append(("sphere3000", *synth("sphere", 3000, 16.0, 4, 64)))
    out.append(("cubesurf4000", *synth("cube-surface", 4000, 32.0, 4, 32)))
    out.append(("ellipsoid3000", *synth("ellipsoid", 3000, 24.0, 5, 32)))
    out.append(("refined3000", *synth("refined-cube", 3000, 32.0, 6, 32)))
    out.append(("volume3000", *synth("volume", 3000, 12.0, 4, 32)))
    out.append(("flat50", np.random.default_rng(2).uniform(size=(50, 3)), np.random.default_rng(3).normal(size=50) + 0j, dict(order=3, ncrit=64, kappa=3.0)))
    return out


def _event_arrays(events):
    m2l, p2p = [], []
    for ev in events:
        t, s = ev.target, ev.source
        if ev.kind == "M2L":
            e, i = ev.direction if ev.direction is not None else (-1, -1)
            m2l.append((t.level, t.key.code, s.key.code, e, i))
        else:
            p2p.append((t.level, t.key.code, s.level, s.key.code))
    return np.array(m2l, np.int64).reshape(-1, 5), np.array(p2p, np.int64).reshape(-1, 4)


def _two_tree_cases():
    """(name, targets, sources, charges, FmmConfig kwargs) -- traversal.py:453-461."""
    out = []
    rng = np.random.default_rng(3)
    sources = rng.uniform(size=(400, 3))
    targets = rng.uniform(size=(150, 3)) * [1.0, 1.0, 0.2] + [0.0, 0.0, 1.5]
    q = rng.uniform(size=400) + 1j * rng.uniform(size=400)
    out.append(("tt_distinct400", targets, sources, q, dict(order=5, ncrit=32, kappa=0.0)))
    src = make_points("sphere", 2500, 0)
    tgt = make_points("cube-surface", 1200, 5) * 0.7
    qq = make_charges(2500, 1)
    box = compute_root_box(np.vstack([tgt, src]))
    out.append(("tt_hf_sphere", tgt, src, qq, dict(order=4, ncrit=32, kappa=24.0 / box.side)))
    return out


def two_tree_cases():
    for name, tgt, src, q, kw in _two_tree_cases():
        cfg = FmmConfig(**kw)
        events = []
        pot, info = run_fmm_full(tgt, src, q, cfg, events=events)
        m2l = []
        p2p = []
        for ev in events:
            t, s_ = ev.target, ev.source
            if ev.kind == "M2L":
                e, i = ev.direction if ev.direction is not None else (-1, -1)
                m2l.append((t.level, t.key.code, s_.key.code, e, i))
            else:
                p2p.append((t.level, t.key.code, s_.level, s_.key.code))
        np.savez_compressed(
            os.path.join(HERE, f"two_{name}.npz"),
            targets=tgt,
            sources=src,
            charges=q,
            config=json.dumps(kw),
            pot=pot,
            counts=json.dumps(info.counts),
            hf_max=info.hf_max_level,
            m2l=np.array(m2l, np.int64).reshape(-1, 5),
            p2p=np.array(p2p, np.int64).reshape(-1, 4),
        )
        print(name, info.counts, "hf_max", info.hf_max_level)


def harness_cases():
    """Reference generators (distributions.py) and one harness record."""
    from helmfmm.harness import ExperimentConfig, run_experiment

    out = {}
    for kind in ("uniform-cube", "sphere", "refined-cube", "ellipse"):
        out[f"dist_{kind}"] = generate_distribution(Distribution(kind, 257, 3))
    out["charges_257_4"] = random_charges(257, 4)
    cfg = ExperimentConfig(distribution="refined-cube", n=1500, kappa_d=12.0, order=4, ncrit=32,
                           check_error=60, seed=1)
    rec = run_experiment(cfg)
    out["record"] = json.dumps(rec.to_json_dict())
    out["record_pot"] = rec.potentials
    np.savez_compressed(os.path.join(HERE, "harness.npz"), **out)
    print("harness", rec.counts, rec.errors)


def fmm_cases():
    for name, pts, q, kw in _cases():
        cfg = FmmConfig(**kw)
        events = []
        pot, info = run_fmm_full(pts, pts, q, cfg, events=events)
        m2l, p2p = _event_arrays(events)
        np.savez_compressed(
            os.path.join(HERE, f"fmm_{name}.npz"),
            points=pts,
            charges=q,
            config=json.dumps(kw),
            pot=pot,
            counts=json.dumps(info.counts),
            hf_max=info.hf_max_level,
            m2l=m2l,
            p2p=p2p,
        )
        print(name, info.counts, "hf_max", info.hf_max_level)


def operators():
    out = {}
    k2 = HelmholtzKernel(kappa=2.0)
    out["g1_k0"] = HelmholtzKernel(kappa=0.0).of_distance(1.0)
    out["gpi_k2"] = k2.of_distance(np.pi)
    # directions and nearest-direction decisions (ties included)
    dt = generate_direction_tree(4)
    for e in range(5):
        out[f"dirs_{e}"] = dt.levels[e]
        if e:
            out[f"fathers_{e}"] = dt.fathers[e]
    g = np.arange(-7, 8)
    tv = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    tv = tv[np.any(tv != 0, axis=1)]
    out["near_t"] = tv
    for e in range(4):
        out[f"near_{e}"] = np.array([nearest_direction(dt, e, t / np.linalg.norm(t)) for t in tv])
    # canonical translations
    canon = [canonicalize_translation(t) for t in tv]
    out["canon"] = np.array([c for c, _ in canon])
    out["canon_rid"] = np.array([r for _, r in canon])
    for L in (2, 3, 4, 5, 6, 8):
        out[f"fperm_L{L}"] = np.stack([frequency_permutation(L, r) for r in range(48)])
    # symbols, M2F/F2L
    rng = np.random.default_rng(7)
    for L in (4, 6):
        ws = FourierWorkspace(L)
        v = rng.normal(size=L**3) + 1j * rng.normal(size=L**3)
        w = rng.normal(size=(2 * L - 1) ** 3) + 1j * rng.normal(size=(2 * L - 1) ** 3)
        out[f"m2f_in_L{L}"], out[f"m2f_out_L{L}"] = v, ws.m2f(v)
        out[f"f2l_in_L{L}"], out[f"f2l_out_L{L}"] = w, ws.f2l(w)
        ker = HelmholtzKernel(kappa=7.5, singularity_tol=1e-12)
        for t in ((3, 1, 0), (2, 2, 2), (5, 3, 1)):
            out[f"sym_L{L}_{t[0]}{t[1]}{t[2]}"] = precompute_symbol(ker, 3, t, 0.25, L).diagonal
        # P2M / L2P with and without a direction
        fr = CellFrame(alpha=np.array([0.1, -0.2, 0.3]), beta=0.125)
        pos = fr.alpha + fr.beta * rng.uniform(size=(37, 3))
        qq = rng.normal(size=37) + 1j * rng.normal(size=37)
        u = np.array([1.0, 2.0, -2.0]) / 3.0
        out[f"p2m_pos_L{L}"], out[f"p2m_q_L{L}"] = pos, qq
        out[f"p2m_lf_L{L}"] = I.p2m(fr, L, pos, qq)
        out[f"p2m_hf_L{L}"] = I.p2m(fr, L, pos, qq, 40.0, u)
        loc = rng.normal(size=L**3) + 1j * rng.normal(size=L**3)
        out[f"l2p_loc_L{L}"] = loc
        out[f"l2p_lf_L{L}"] = I.l2p(fr, L, pos, loc)
        out[f"l2p_hf_L{L}"] = I.l2p(fr, L, pos, loc, 40.0, u)
        for o in range(8):
            oc = ((o >> 2) & 1, (o >> 1) & 1, o & 1)
            out[f"m2m_L{L}_{o}"] = np.stack(I.m2m_factors(L, oc))
    np.savez_compressed(os.path.join(HERE, "operators.npz"), **out)
    print("operators", len(out))


if __name__ == "__main__":
    import sys as _sys

    if "--two-tree-only" in _sys.argv:
        two_tree_cases()
    elif "--harness-only" in _sys.argv:
        harness_cases()
    else:
        operators()
        fmm_cases()
        two_tree_cases()
        harness_cases()
