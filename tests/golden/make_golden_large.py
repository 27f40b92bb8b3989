"""Run the REFERENCE (helmfmm, /root/reference) on a BASELINE config and save
full-size parity data under tests/golden/.

Only runnable in the build container (the reference tree does not travel to
the GPU box).  Output ``ref_<name>.npz`` holds: counts, hf_max, kappa, the
sampled check targets (default_rng(2), harness.py:152-154), the reference
potentials at those targets, the FP64 direct sum there, eps_ref (rel-L2 of the
reference vs direct), the SHA-256 of the full potential vector, staged
timings, and (for N <= 20k) the full potential vector.

usage: PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
       python tests/golden/make_golden_large.py cfg1 [cfg2 ...]
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")

from helmfmm import traversal as T  # noqa: E402
from helmfmm.kernel import HelmholtzKernel, direct_sum, relative_errors  # noqa: E402

from paper_2202_04894_b200.workloads import make_workload, sample_targets  # noqa: E402


def staged_run(pts, q, cfg):
    """run_fmm_full's pipeline with the staged timers of SURVEY.md §8(d)."""
    from helmfmm.tree import TreeConfig, accumulate_potentials, build_tree

    t = {}
    t0 = time.perf_counter()
    tree, pset = build_tree(pts, q, TreeConfig(ncrit=cfg.ncrit, hard_depth_cap=cfg.hard_depth_cap))
    t["tree"] = time.perf_counter() - t0
    kernel = HelmholtzKernel(kappa=cfg.kappa, singularity_tol=1e-12 * tree.root_box.side)
    ctx = T._Context(cfg, kernel, tree, tree, pset, pset)
    t0 = time.perf_counter()
    T.blank_dtt(tree.root, tree.root, ctx)
    T.blank_downward_pass(tree.root, ctx)
    t["blank"] = time.perf_counter() - t0
    pre_blank = ctx.precompute_time
    t0 = time.perf_counter()
    T._upward(ctx, tree)
    t["upward"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    T.dtt(tree.root, tree.root, ctx)
    t["m2l_p2p"] = time.perf_counter() - t0
    pre_dtt = ctx.precompute_time - pre_blank
    t0 = time.perf_counter()
    T._downward(ctx, tree)
    t["downward"] = time.perf_counter() - t0
    t["precompute"] = ctx.precompute_time
    t["matvec"] = t["upward"] + (t["m2l_p2p"] - pre_dtt) + t["downward"]
    n_exp = sum(len(c.multipole) for lv in tree.levels for c in lv)
    counts = {
        "cells": tree.n_cells,
        "leaves": len(tree.leaves),
        "symbols": ctx.cache.n_canonical,
        "effective_expansions": n_exp,
        "p2p_pairs": ctx.n_p2p_pairs,
        "m2l_events": ctx.n_m2l,
        "translations": ctx.cache.n_translations,
    }
    return accumulate_potentials(pset), counts, ctx.hf_max_level, t


def main(name: str, order: int | None = None):
    pts, q, kappa, w = make_workload(name)
    L = order or w.order
    cfg = T.FmmConfig(order=L, ncrit=w.ncrit, kappa=kappa)
    t0 = time.perf_counter()
    pot, counts, hf_max, timings = staged_run(pts, q, cfg)
    timings["end_to_end"] = time.perf_counter() - t0
    sample = sample_targets(pts.shape[0])
    from paper_2202_04894_b200.geometry import compute_root_box

    side = compute_root_box(pts).side
    kern = HelmholtzKernel(kappa=kappa, singularity_tol=1e-12 * side)
    t0 = time.perf_counter()
    blk = 512 if pts.shape[0] <= 100_000 else 16
    direct = direct_sum(kern, pts[sample], pts, q, block=blk)
    timings["direct"] = time.perf_counter() - t0
    err = relative_errors(direct, pot[sample])
    out = dict(
        name=name,
        order=L,
        kappa=kappa,
        hf_max=hf_max,
        sample=sample,
        pot_sample=pot[sample],
        direct_sample=direct,
        eps_ref=err.rel_l2,
        eps_ref_linf=err.rel_linf,
        sha256=hashlib.sha256(pot.tobytes()).hexdigest(),
        counts=json.dumps(counts),
        timings=json.dumps(timings),
    )
    if pts.shape[0] <= 20_000:
        out["pot"] = pot
    tag = name if order is None else f"{name}_L{L}"
    np.savez_compressed(os.path.join(HERE, f"ref_{tag}.npz"), **out)
    print(tag, json.dumps(counts), json.dumps(timings), "eps_ref", err.rel_l2, flush=True)


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        if ":" in arg:
            nm, lo = arg.split(":")
            main(nm, int(lo))
        else:
            main(arg)
