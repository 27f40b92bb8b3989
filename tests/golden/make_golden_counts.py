"""Counts-only run of the REFERENCE (helmfmm) on a BASELINE config too large
for its full matvec here (cfg4: 16M points; the reference's spectra alone
would need > 62 GB): the reference's own tree build, blank passes and dual
tree traversal (traversal.py:432-506) with the per-event arithmetic stubbed
out -- the Hadamard product is a no-op, the P2P only counts pairs and the
upward pass only creates the (cell, key) expansion slots _p2m_cell/_m2m_cell
would fill (traversal.py:224-296).  Every decision (tree, MAC, directions,
marks, symbol cache) is the reference's, so FmmInfo.counts are exact.  Also
stores the FP64 direct sums on the 1,000 check targets (kernel.py:58-75,
harness.py:151-165) for the accuracy check.

usage: PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
       python tests/golden/make_golden_counts.py cfg4
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")

from helmfmm import traversal as T  # noqa: E402
from helmfmm.kernel import HelmholtzKernel, direct_sum  # noqa: E402
from helmfmm.tree import TreeConfig, build_tree  # noqa: E402

from paper_2202_04894_b200.workloads import make_workload, sample_targets  # noqa: E402


class _Tiny:
    fourier_size = 1  # local_hat accumulators are never used (Hadamard stubbed)


def _count_p2p(ctx, t, s):
    ctx.n_p2p_pairs += (t.stop - t.start) * (s.stop - s.start)


def main(name: str):
    pts, q, kappa, w = make_workload(name)
    cfg = T.FmmConfig(order=w.order, ncrit=w.ncrit, kappa=kappa)
    tm = {}
    t0 = time.perf_counter()
    tree, pset = build_tree(pts, q, TreeConfig(ncrit=cfg.ncrit, hard_depth_cap=cfg.hard_depth_cap))
    tm["tree"] = time.perf_counter() - t0
    kernel = HelmholtzKernel(kappa=cfg.kappa, singularity_tol=1e-12 * tree.root_box.side)
    ctx = T._Context(cfg, kernel, tree, tree, pset, pset)
    ctx.workspace = _Tiny()
    t0 = time.perf_counter()
    T.blank_dtt(tree.root, tree.root, ctx)
    T.blank_downward_pass(tree.root, ctx)
    tm["blank"] = time.perf_counter() - t0
    # expansion slots exactly as _p2m_cell / _m2m_cell create them
    for level in range(tree.depth, -1, -1):
        for c in tree.levels[level]:
            if ctx.is_hf(c.level):
                keys = sorted(c.marks) if (c.is_leaf or c.marks) else []
            else:
                keys = [None]
            for k in keys:
                c.multipole[k] = 0
                c.multipole_hat[k] = 0
    T.m2l_hadamard = lambda acc, src, diag: None
    T._p2p = _count_p2p
    t0 = time.perf_counter()
    T.dtt(tree.root, tree.root, ctx)
    tm["dtt"] = time.perf_counter() - t0
    counts = {
        "cells": tree.n_cells,
        "leaves": len(tree.leaves),
        "symbols": ctx.cache.n_canonical,
        "effective_expansions": sum(len(c.multipole) for lv in tree.levels for c in lv),
        "p2p_pairs": ctx.n_p2p_pairs,
        "m2l_events": ctx.n_m2l,
        "translations": ctx.cache.n_translations,
    }
    print(name, json.dumps(counts), json.dumps(tm), flush=True)
    sample = sample_targets(pts.shape[0])
    t0 = time.perf_counter()
    direct = direct_sum(kernel, pts[sample], pts, q, block=16)
    tm["direct"] = time.perf_counter() - t0
    np.savez_compressed(os.path.join(HERE, f"ref_{name}_counts.npz"), name=name, order=w.order, kappa=kappa,
                        hf_max=ctx.hf_max_level, sample=sample, direct_sample=direct, counts=json.dumps(counts),
                        timings=json.dumps(tm))
    print(name, "direct done", json.dumps(tm), flush=True)


if __name__ == "__main__":
    for arg in sys.argv[1:]:
        main(arg)
