"""GPU plan construction (gpu_build.py, csrc/plan_gpu.cu) against the host
builders, bit for bit: the octree of tree.py:132-213 and the dual-tree-traversal
lists of traversal.py:182-200, 320-348."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from conftest import load_case  # noqa: E402
from paper_2202_04894_b200.config import TreeConfig  # noqa: E402
from paper_2202_04894_b200.tree import build_tree  # noqa: E402
from paper_2202_04894_b200.workloads import make_points  # noqa: E402


def _same_tree(a, b):
    for k in ("level", "coords", "start", "stop", "parent", "first_son", "n_sons", "level_offsets"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert np.array_equal(a.alpha, b.alpha) and a.depth == b.depth
    assert np.array_equal(a.root_box.lower, b.root_box.lower) and a.root_box.side == b.root_box.side


def _points(kind):
    rng = np.random.default_rng(7)
    if kind == "clustered":  # deep, very uneven tree
        c = rng.uniform(-1, 1, (5, 3))
        return np.vstack([c[i] + 10.0 ** (-i - 1) * rng.normal(size=(3000, 3)) for i in range(5)])
    if kind == "duplicates":  # coincident points: splitting stops at the depth cap
        x = rng.uniform(-1, 1, (500, 3))
        return np.vstack([x, np.repeat(x[:7], 40, axis=0)])
    if kind == "grid":  # points exactly on cell centres: the >= ties of every level
        g = np.linspace(-1, 1, 17)
        return np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    return make_points(kind, 20000, 3)


@pytest.mark.parametrize("ncrit,cap", [(64, 30), (8, 30), (16, 6)])
@pytest.mark.parametrize("kind", ["sphere", "cube-surface", "volume", "clustered", "duplicates", "grid"])
def test_gpu_tree_equals_host_tree(kind, ncrit, cap):
    from paper_2202_04894_b200.gpu_build import build_tree_gpu

    pts = _points(kind)
    q = np.arange(pts.shape[0]) + 0j
    cfg = TreeConfig(ncrit=ncrit, hard_depth_cap=cap)
    if kind == "duplicates" and cap > 21 and ncrit < 41:  # 41 coincident points per cluster
        with pytest.raises(NotImplementedError):
            build_tree_gpu(pts, q, cfg)
        return
    th, ph = build_tree(pts, q, cfg)
    tg, pg = build_tree_gpu(pts, q, cfg)
    _same_tree(tg, th)
    assert np.array_equal(pg.original_index, ph.original_index)
    assert np.array_equal(pg.positions, ph.positions) and np.array_equal(pg.charges, ph.charges)


def test_gpu_tree_root_box_edge_cases():
    """One particle and coincident particles take the reference's 0.5 half width
    (geometry.py:92-95); a non-finite coordinate is refused."""
    from paper_2202_04894_b200.gpu_build import build_tree_gpu

    for pts in (np.array([[0.3, -1.2, 4.0]]), np.tile([[1.0, 2.0, 3.0]], (5, 1))):
        q = np.ones(pts.shape[0], complex)
        th, _ = build_tree(pts, q, TreeConfig(ncrit=8, hard_depth_cap=4))
        tg, _ = build_tree_gpu(pts, q, TreeConfig(ncrit=8, hard_depth_cap=4))
        _same_tree(tg, th)
    bad = np.array([[0.0, 0.0, 0.0], [1.0, np.inf, 0.0]])
    with pytest.raises(ValueError):
        build_tree_gpu(bad, np.ones(2, complex), TreeConfig())


@pytest.mark.parametrize("case", ["cubesurf4000", "refined3000", "c1_kd8"])
def test_gpu_tree_on_golden_cases(case):
    from paper_2202_04894_b200.gpu_build import build_tree_gpu

    g = load_case(case)
    cfg = TreeConfig(ncrit=g["config"]["ncrit"])
    th, ph = build_tree(g["points"], g["charges"], cfg)
    tg, pg = build_tree_gpu(g["points"], g["charges"], cfg)
    _same_tree(tg, th)
    assert np.array_equal(pg.original_index, ph.original_index)


def _dtt_pair(tt, st, order, kappa):
    from paper_2202_04894_b200.directions import generate_direction_tree
    from paper_2202_04894_b200.gpu_build import GpuDtt
    from paper_2202_04894_b200.plan import NativeDtt, _traversal_tables, hf_max_level

    depth = max(tt.depth, st.depth)
    hf = hf_max_level(tt, depth, kappa, 2.0)
    dt = generate_direction_tree(hf) if hf >= 0 else None
    dir_off = np.concatenate([[0], np.cumsum([d.shape[0] for d in dt.levels])]).astype(np.int64) if dt else np.zeros(1, np.int64)
    tabs = _traversal_tables(tt, depth, hf, dt, dir_off, kappa, 1.0)
    return NativeDtt(tt, st, depth, *tabs), GpuDtt(tt, st, depth, *tabs)


def _same_lists(nat, gpu):
    for k in ("ev_s", "ev_trans", "row_ptr", "row_t", "row_key", "row_lev", "grp_rows", "grp_p", "grp_key", "grp_lev",
              "grp_ptr", "blk_trans", "blk_mask", "p_t", "p_s", "trans_dense"):
        assert nat[k].shape == gpu[k].shape, k
        assert np.array_equal(nat[k], gpu[k]), k
    # blk_src names an event of the block's source cell b: the same cell in both
    a, b = nat["blk_src"], gpu["blk_src"]
    assert np.array_equal(a >= 0, b >= 0)
    assert np.array_equal(nat["ev_s"][a[a >= 0]], gpu["ev_s"][b[b >= 0]])
    rk = np.repeat(np.arange(nat["row_t"].shape[0]), np.diff(nat["row_ptr"]))
    assert np.array_equal(nat["row_key"][rk[a[a >= 0]]], gpu["row_key"][rk[b[b >= 0]]])


@pytest.mark.parametrize("case", ["cubesurf4000", "volume3000", "c1_kd16", "laplace500", "refined3000", "twocluster"])
def test_gpu_dtt_lists_equal_native_lists(case):
    g = load_case(case)
    kw = g["config"]
    tr, _ = build_tree(g["points"], g["charges"], TreeConfig(ncrit=kw["ncrit"]))
    nat, gpu = _dtt_pair(tr, tr, kw["order"], kw.get("kappa", 0.0))
    assert nat["ev_s"].shape[0] == g["counts"]["m2l_events"]
    _same_lists(nat, gpu)


def test_gpu_dtt_two_trees():
    from conftest import load_two_tree, two_tree_cases
    from paper_2202_04894_b200.geometry import compute_root_box

    for case in two_tree_cases():
        g = load_two_tree(case)
        kw = g["config"]
        box = compute_root_box(np.vstack([g["targets"], g["sources"]]))
        cfg = TreeConfig(ncrit=kw["ncrit"])
        st, _ = build_tree(g["sources"], g["charges"], cfg, root_box=box)
        tt, _ = build_tree(g["targets"], np.zeros(len(g["targets"])), cfg, root_box=box)
        nat, gpu = _dtt_pair(tt, st, kw["order"], kw.get("kappa", 0.0))
        _same_lists(nat, gpu)


@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("case", ["cubesurf4000", "c1_kd16"])
def test_device_sibling_groups_equal_host_lists(case, K):
    """fmm.m2l_groups_dev (per-event merging on the device) == fmm.m2l_groups."""
    from paper_2202_04894_b200.fmm import m2l_groups, m2l_groups_dev
    from paper_2202_04894_b200.plan import build_plan

    g = load_case(case)
    kw = g["config"]
    tr, _ = build_tree(g["points"], g["charges"], TreeConfig(ncrit=kw["ncrit"]))
    p = build_plan(tr, tr, kw["order"], kw["kappa"], 1.0, 2.0)
    rows, ptr, ent = p.m2l_row_slot, p.m2l_row_ptr, p.m2l_rows_entries
    ids = np.arange(rows.shape[0])
    a = m2l_groups(ids, rows, ptr, ent, p.l_cell, p.l_dir, tr.level, tr.parent, K)
    b = m2l_groups_dev(ids, rows, ptr, torch.as_tensor(ent).cuda(), p.l_cell, p.l_dir, tr.level, tr.parent, K, "cuda")
    assert a["n"] == b["n"]
    for k in ("grp_slot", "grp_ptr", "ent"):
        assert np.array_equal(np.asarray(a[k]).reshape(-1), b[k].cpu().numpy().reshape(-1)), k


@pytest.mark.parametrize("ns_cap", [16, 48])
@pytest.mark.parametrize("case", ["cubesurf4000", "c1_kd16", "volume3000"])
def test_device_stage_lists_equal_host_lists(case, ns_cap):
    """fmm.m2l_stage_lists_dev (per-event work on the device) == fmm.m2l_stage_lists."""
    from paper_2202_04894_b200.fmm import m2l_stage_lists, m2l_stage_lists_dev
    from paper_2202_04894_b200.plan import build_plan

    g = load_case(case)
    kw = g["config"]
    tr, _ = build_tree(g["points"], g["charges"], TreeConfig(ncrit=kw["ncrit"]))
    p = build_plan(tr, tr, kw["order"], kw["kappa"], 1.0, 2.0)
    rows, ptr, ent = p.m2l_row_slot, p.m2l_row_ptr, p.m2l_rows_entries
    ids = np.arange(rows.shape[0])
    hc = tr.coords[p.m_cell[p.hat_slot]]
    a = m2l_stage_lists(ids, rows, ptr, ent, p.l_cell, p.l_dir, tr.level, tr.parent, tr.coords, hc, ns_cap)
    b = m2l_stage_lists_dev(ids, rows, ptr, torch.as_tensor(ent).cuda(), p.l_cell, p.l_dir, tr.level, tr.parent,
                            tr.coords, hc, ns_cap, "cuda")
    assert a["n"] == b["n"]
    for k in ("row_slot", "cta_stage", "cta_went", "stage_slot_ptr", "slot_sym", "stage_wend", "ent", "cta_rows"):
        bv = b[k].cpu().numpy() if torch.is_tensor(b[k]) else b[k]
        assert np.array_equal(np.asarray(a[k]).reshape(-1), np.asarray(bv).reshape(-1)), k


@pytest.mark.parametrize("max_pairs,chunk", [(1 << 16, 128), (700, 3)])
@pytest.mark.parametrize("case", ["cubesurf4000", "volume3000", "refined3000"])
def test_device_mutual_p2p_lists_equal_host_lists(case, max_pairs, chunk, monkeypatch):
    """plan.p2p_mutual_lists on the device (torch ops) == on the host (numpy)."""
    from paper_2202_04894_b200 import plan as plan_mod
    from paper_2202_04894_b200.plan import build_plan, p2p_mutual_lists

    monkeypatch.setattr(plan_mod, "P2P_GATHER_CHUNK", chunk)
    g = load_case(case)
    kw = g["config"]
    tr, _ = build_tree(g["points"], g["charges"], TreeConfig(ncrit=kw["ncrit"]))
    p = build_plan(tr, tr, kw["order"], kw["kappa"], 1.0, 2.0)
    args = (p.p2p_ptr, p.p2p_lo, p.p2p_hi, tr.start[p.leaf_cells], tr.stop[p.leaf_cells], p.counts["p2p_pairs"],
            max_pairs)
    a, b = p2p_mutual_lists(*args), p2p_mutual_lists(*args, device="cuda")
    for k in ("ptr", "lo", "hi", "item_leaf", "item_f0", "item_f1", "item_row", "item_col"):
        assert np.array_equal(a[k], b[k]), k
    assert a["partial_size"] == b["partial_size"] and len(a["gather"]) == len(b["gather"])
    for ga, gb in zip(a["gather"], b["gather"]):
        for k in ga:
            assert np.array_equal(ga[k], gb[k].cpu().numpy()), k
