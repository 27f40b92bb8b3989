"""Host plan (tree, level-synchronous DTT, marks, slots, CSR lists) against
the reference's own decisions: exact tree, exact FmmInfo.counts, exact M2L
(with direction keys) and P2P event sets (tests/golden, from helmfmm)."""

import numpy as np
import pytest

from conftest import golden_cases, load_case, load_ref
from oracle import defmm_oracle as O
from paper_2202_04894_b200.config import FmmConfig, TreeConfig
from paper_2202_04894_b200.directions import generate_direction_tree, nearest_directions
from paper_2202_04894_b200.plan import GROUP48, build_plan, canonicalize_many
from paper_2202_04894_b200.tree import build_tree
from paper_2202_04894_b200.workloads import make_workload


def _plan(g):
    kw = g["config"]
    tr, ps = build_tree(g["points"], g["charges"], TreeConfig(ncrit=kw["ncrit"]))
    pl = build_plan(tr, tr, kw["order"], kw["kappa"], 1.0, 2.0, keep_events=True)
    return tr, ps, pl


@pytest.mark.parametrize("case", golden_cases())
def test_tree_matches_reference(case):
    g = load_case(case)
    tr, ps = build_tree(g["points"], g["charges"], TreeConfig(ncrit=g["config"]["ncrit"]))
    ot = O.Tree(g["points"], g["config"]["ncrit"])
    assert np.array_equal(ps.original_index, ot.perm)
    assert np.array_equal(ps.positions, g["points"][ot.perm])
    mine = sorted(zip(tr.level.tolist(), map(tuple, tr.coords.tolist()), tr.start.tolist(), tr.stop.tolist()))
    ref = sorted(zip(ot.level, [tuple(c) for c in ot.coords], ot.start, ot.stop))
    assert mine == ref


@pytest.mark.parametrize("case", golden_cases())
def test_plan_counts_and_event_lists_match_reference(case):
    g = load_case(case)
    tr, ps, pl = _plan(g)
    assert pl.hf_max == g["hf_max"]
    assert {k: pl.counts[k] for k in g["counts"]} == g["counts"]
    codes = tr.morton_code(np.arange(tr.n_cells)).astype(np.int64)
    mt, ms, ed = pl.m2l_events
    e = np.where(ed >= 0, pl.hf_max - tr.level[mt], -1)
    i = np.where(ed >= 0, ed - pl.dir_off[np.maximum(e, 0)], -1)
    mine = sorted(zip(tr.level[mt].tolist(), codes[mt].tolist(), codes[ms].tolist(), e.tolist(), i.tolist()))
    assert mine == sorted(map(tuple, g["m2l"].tolist()))
    pt, pss = pl.p2p_events
    mp = sorted(zip(tr.level[pt].tolist(), codes[pt].tolist(), tr.level[pss].tolist(), codes[pss].tolist()))
    assert mp == sorted(map(tuple, g["p2p"].tolist()))


@pytest.mark.parametrize("case", ["volume3000", "cubesurf4000", "laplace500"])
def test_p2p_runs_cover_every_pair_once(case):
    """test_traversal.py:190-201 analogue: near + far lists partition all N^2 pairs."""
    g = load_case(case)
    tr, ps, pl = _plan(g)
    n = ps.n
    cov = np.zeros((n, n), np.int8)
    for li, leaf in enumerate(pl.leaf_cells):
        for k in range(pl.p2p_ptr[li], pl.p2p_ptr[li + 1]):
            cov[tr.start[leaf] : tr.stop[leaf], pl.p2p_lo[k] : pl.p2p_hi[k]] += 1
    mt, ms, _ = pl.m2l_events
    for t, s in zip(mt, ms):
        cov[tr.start[t] : tr.stop[t], tr.start[s] : tr.stop[s]] += 1
    assert np.all(cov == 1)


def test_m2l_rows_are_target_major_and_complete():
    g = load_case("cubesurf4000")
    tr, ps, pl = _plan(g)
    assert np.all(np.diff(pl.m2l_row_slot) > 0)
    assert pl.m2l_row_ptr[-1] == pl.counts["m2l_events"]
    assert np.all(np.diff(pl.m2l_row_ptr) > 0)
    assert pl.m2l_src.max() < pl.n_hat and pl.m2l_sym.max() < pl.n_sym


def test_batched_nearest_direction_ties(operators):
    dt = generate_direction_tree(3)
    for e in range(4):
        assert np.array_equal(nearest_directions(dt.levels[e], operators["near_t"]), operators[f"near_{e}"])


def test_batched_canonicalization(operators):
    c, r = canonicalize_many(operators["near_t"])
    assert np.array_equal(c, operators["canon"])
    assert np.array_equal(r, operators["canon_rid"])


def test_closed_form_rotation_matches_frequency_permutation(operators):
    """The device gathers D_canon[idx(j, rid)] with mapped[perm[a]] = sign[a] f[a]
    mod P; check that closed form against fourier.py:123-143."""
    import itertools

    perms = list(itertools.permutations(range(3)))
    for L in (2, 4, 5, 6, 8):
        P = 2 * L - 1
        f = np.stack(np.meshgrid(*([np.arange(P)] * 3), indexing="ij"), -1).reshape(-1, 3)
        W = (P * P, P, 1)
        for rid in range(48):
            pi, sb = rid >> 3, rid & 7
            idx = np.zeros(P**3, np.int64)
            for a in range(3):
                neg = (sb >> (2 - a)) & 1
                v = (P - f[:, a]) % P if neg else f[:, a]
                idx += W[perms[pi][a]] * v
            assert np.array_equal(idx, operators[f"fperm_L{L}"][rid])


def test_cfg1_plan_counts_match_reference_run():
    ref = load_ref("cfg1")
    pts, q, k, w = make_workload("cfg1")
    assert abs(k - float(ref["kappa"])) == 0.0
    tr, ps = build_tree(pts, q, TreeConfig(ncrit=w.ncrit))
    pl = build_plan(tr, tr, w.order, k, 1.0, 2.0)
    assert pl.counts == ref["counts"]
    assert pl.hf_max == int(ref["hf_max"])


@pytest.mark.parametrize("name,workload", [("cfg2", "cfg2"), ("cfg3", "cfg3"), ("cfg5", "cfg5"), ("cfg4_counts", "cfg4")])
def test_full_size_plan_counts_match_reference_run(name, workload):
    """Host plan (tree + native DTT) at BASELINE size: FmmInfo.counts and
    hf_max equal the reference's own run (tests/golden/ref_*.npz)."""
    ref = load_ref(name)
    pts, q, k, w = make_workload(workload)
    assert abs(k - float(ref["kappa"])) == 0.0
    tr, ps = build_tree(pts, q, TreeConfig(ncrit=w.ncrit))
    pl = build_plan(tr, tr, int(ref["order"]), k, 1.0, 2.0)
    assert pl.counts == ref["counts"]
    assert pl.hf_max == int(ref["hf_max"])


def test_config_validation():
    with pytest.raises(ValueError):
        FmmConfig(order=1)
    # boundary deviation: orders above 8 are refused (the reference accepts any order >= 2)
    with pytest.raises(ValueError, match="orders 2..8"):
        FmmConfig(order=9)
    assert FmmConfig(order=8).order == 8
    with pytest.raises(ValueError):
        FmmConfig(strategy="dense")
    with pytest.raises(ValueError):
        FmmConfig(eta=0.0)
    with pytest.raises(ValueError):
        FmmConfig(kappa=-2.0)
    with pytest.raises(ValueError):
        build_tree(np.zeros((0, 3)), np.zeros(0))
    with pytest.raises(ValueError):
        build_tree(np.array([[0.0, np.nan, 0.0]]), np.ones(1))


def test_mac_violation_raises():
    """fourier.py:179-180 / test_fourier.py:181-184: a stencil that touches the
    singularity (adjacent cells) raises ValueError."""
    from paper_2202_04894_b200.plan import _check_stencils

    g = load_case("laplace500")
    tr, ps = build_tree(g["points"], g["charges"], TreeConfig(ncrit=32))
    _check_stencils(np.array([[2, 0, 0]]), np.array([2]), tr, 4, 1e-12)
    with pytest.raises(ValueError):
        _check_stencils(np.array([[1, 0, 0]]), np.array([2]), tr, 4, 1e-12)


@pytest.mark.parametrize("case", __import__("conftest").two_tree_cases())
def test_two_tree_plan_matches_reference(case):
    """targets is not sources: two trees on one root box (traversal.py:453-461);
    counts and both event lists equal the reference's."""
    from conftest import load_two_tree
    from paper_2202_04894_b200.geometry import compute_root_box

    g = load_two_tree(case)
    kw = g["config"]
    box = compute_root_box(np.vstack([g["targets"], g["sources"]]))
    cfg = TreeConfig(ncrit=kw["ncrit"])
    st, sp = build_tree(g["sources"], g["charges"], cfg, root_box=box)
    tt, tp = build_tree(g["targets"], np.zeros(len(g["targets"])), cfg, root_box=box)
    pl = build_plan(tt, st, kw["order"], kw["kappa"], 1.0, 2.0, keep_events=True)
    assert pl.hf_max == g["hf_max"]
    assert {k: pl.counts[k] for k in g["counts"]} == g["counts"]
    tc = tt.morton_code(np.arange(tt.n_cells)).astype(np.int64)
    sc = st.morton_code(np.arange(st.n_cells)).astype(np.int64)
    mt, ms, ed = pl.m2l_events
    e = np.where(ed >= 0, pl.hf_max - tt.level[mt], -1)
    i = np.where(ed >= 0, ed - pl.dir_off[np.maximum(e, 0)], -1)
    mine = sorted(zip(tt.level[mt].tolist(), tc[mt].tolist(), sc[ms].tolist(), e.tolist(), i.tolist()))
    assert mine == sorted(map(tuple, g["m2l"].tolist()))
    pt, pss = pl.p2p_events
    mp = sorted(zip(tt.level[pt].tolist(), tc[pt].tolist(), st.level[pss].tolist(), sc[pss].tolist()))
    assert mp == sorted(map(tuple, g["p2p"].tolist()))


def test_p2p_work_items_cover_each_leaf_source_list_once():
    from paper_2202_04894_b200.plan import p2p_work_items

    rng = np.random.default_rng(0)
    nleaf = 200
    runs = rng.integers(1, 6, nleaf)
    ptr = np.concatenate([[0], np.cumsum(runs)])
    run_len = rng.integers(1, 5000, ptr[-1])
    nt = rng.integers(1, 65, nleaf)
    wi = p2p_work_items(ptr, run_len, nt, max_pairs=20000)
    cs = np.concatenate([[0], np.cumsum(run_len)])
    ns = cs[ptr[1:]] - cs[ptr[:-1]]
    covered = np.zeros(nleaf, np.int64)
    for l, a, b in zip(wi["item_leaf"], wi["item_f0"], wi["item_f1"]):
        assert 0 <= a < b <= ns[l]
        assert nt[l] * (b - a) <= 20000 + nt[l] * 5000  # bounded (one chunk of rounding)
        covered[l] += b - a
    assert np.array_equal(covered, ns)
    # split leaves: partial blocks are disjoint and exactly k * nt long
    seen = set()
    for l, base, k in zip(wi["split_leaf"], wi["split_base"], wi["split_n"]):
        outs = sorted(o for ll, o in zip(wi["item_leaf"], wi["item_out"]) if ll == l)
        assert outs == [base + m * nt[l] for m in range(k)]
        assert not (set(range(base, base + k * nt[l])) & seen)
        seen |= set(range(base, base + k * nt[l]))
    single = set(range(nleaf)) - set(wi["split_leaf"].tolist())
    assert all(o == -1 for l, o in zip(wi["item_leaf"], wi["item_out"]) if l in single)


@pytest.mark.parametrize("case", ["cubesurf4000", "volume3000", "c1_kd16"])
def test_m2l_blocks_reconstruct_the_event_list(case):
    """Every M2L event appears in exactly one parent-pair block with its row,
    source spectrum and derived symbol (K7 v3 input)."""
    g = load_case(case)
    tr, ps, pl = _plan(g)
    rows_ev = []
    for gi in range(pl.blk_group_rows.shape[0]):
        for bi in range(pl.blk_group_ptr[gi], pl.blk_group_ptr[gi + 1]):
            m = int(pl.blk_mask[bi])
            for bit in range(64):
                if (m >> bit) & 1:
                    a, b = divmod(bit, 8)
                    row = pl.blk_group_rows[gi, a]
                    src = pl.blk_src[bi, b]
                    # child offset index from the octants
                    av = np.array([(a >> 2) & 1, (a >> 1) & 1, a & 1])
                    bv = np.array([(b >> 2) & 1, (b >> 1) & 1, b & 1])
                    dv = av - bv
                    d = (dv[0] + 1) * 9 + (dv[1] + 1) * 3 + (dv[2] + 1)
                    tr_id = pl.blk_trans[bi, d]
                    assert row >= 0 and src >= 0 and tr_id >= 0
                    rows_ev.append((int(row), int(src), int(tr_id)))
    ref = []
    for r in range(len(pl.m2l_row_slot)):
        for e in range(pl.m2l_row_ptr[r], pl.m2l_row_ptr[r + 1]):
            ref.append((int(pl.m2l_row_slot[r]), int(pl.m2l_rows_entries[e, 0]), int(pl.m2l_rows_entries[e, 1])))
    assert sorted(rows_ev) == sorted(ref)
    # planar classification: every pair of a planar block lies in its plane
    for bi, k in enumerate(pl.blk_kind):
        if k < 0:
            continue
        p_, v = divmod(int(k), 2)
        m = int(pl.blk_mask[bi]) & ((1 << 64) - 1)
        for bit in range(64):
            if (m >> bit) & 1:
                a, b = divmod(bit, 8)
                assert ((a >> (2 - p_)) & 1) == v and ((b >> (2 - p_)) & 1) == v


# ---- native traversal (csrc/dtt_build.cpp) against the numpy restatement ----

def _event_sets(mt, ms, pt, ps):
    return sorted(zip(mt.tolist(), ms.tolist())), sorted(zip(pt.tolist(), ps.tolist()))


@pytest.mark.parametrize(
    "kind,n,kd,ncrit",
    [("sphere", 3000, 32.0, 32), ("cube-surface", 5000, 96.0, 24), ("volume", 4000, 16.0, 16),
     ("refined-cube", 4000, 128.0, 20), ("ellipsoid", 3000, 0.0, 32)],
)
def test_native_traversal_equals_numpy_dtt(kind, n, kd, ncrit):
    """defmm_dtt_build (threshold MAC, dense key tables, target-major sweep)
    visits exactly the pairs of the per-pair numpy traversal, with the same keys."""
    from paper_2202_04894_b200.plan import dtt_numpy
    from paper_2202_04894_b200.workloads import kappa_for, make_points

    pts = make_points(kind, n, 3)
    kappa = kappa_for(pts, kd) if kd else 0.0
    tr, _ = build_tree(pts, np.ones(n), TreeConfig(ncrit=ncrit))
    pl = build_plan(tr, tr, 4, kappa, 1.0, 2.0, keep_events=True)
    mt, ms, mlev, pt, ps = dtt_numpy(tr, tr, kappa, 1.0, 2.0)
    nm, npp = _event_sets(*pl.m2l_events[:2], *pl.p2p_events)
    rm, rp = _event_sets(mt, ms, pt, ps)
    assert nm == rm and npp == rp
    # keys: nearest direction of each event's translation (directions.py:78-89)
    hf = pl.hf_max
    if hf >= 0:
        dt = generate_direction_tree(hf)
        m_t, m_s, key = pl.m2l_events
        lev = tr.level[m_t]
        for l in np.unique(lev[lev <= hf]):
            sel = lev == l
            e = hf - int(l)
            ref = pl.dir_off[e] + nearest_directions(dt.levels[e], tr.coords[m_t[sel]] - tr.coords[m_s[sel]])
            assert np.array_equal(key[sel], ref)
        assert np.all(key[lev > hf] == -1)


def test_native_traversal_two_trees_equals_numpy_dtt():
    from paper_2202_04894_b200.geometry import compute_root_box
    from paper_2202_04894_b200.plan import dtt_numpy

    rng = np.random.default_rng(5)
    src = rng.random((3000, 3))
    tgt = rng.random((2000, 3)) * 0.5 + 0.25
    box = compute_root_box(np.vstack([tgt, src]))
    cfg = TreeConfig(ncrit=20)
    st, _ = build_tree(src, np.ones(3000), cfg, root_box=box)
    tt, _ = build_tree(tgt, np.zeros(2000), cfg, root_box=box)
    kappa = 40.0
    pl = build_plan(tt, st, 4, kappa, 1.0, 2.0, keep_events=True)
    mt, ms, mlev, pt, ps = dtt_numpy(tt, st, kappa, 1.0, 2.0)
    assert _event_sets(*pl.m2l_events[:2], *pl.p2p_events) == _event_sets(mt, ms, pt, ps)


@pytest.mark.parametrize("kappa", [0.0, 3.0, 25.0, 80.0, 300.0])
@pytest.mark.parametrize("eta", [0.5, 1.0, 2.0])
def test_mac_threshold_equals_per_gap_mac(kappa, eta):
    """The integer threshold reproduces the reference MAC (traversal.py:100-113)
    for every gap^2 of every level (the HF test is an up-set in gap^2)."""
    from paper_2202_04894_b200.plan import _mac_lut, mac_threshold

    for level in range(0, 7):
        span = (1 << level) - 1
        gmax = 3 * max(span - 1, 0) ** 2
        g = np.arange(gmax + 1)
        beta = 2.0 / (1 << level)
        for hf in (False, True):
            if hf and kappa == 0.0:
                continue
            thr = mac_threshold(level, hf, beta, kappa, eta, gmax)
            assert np.array_equal(g >= thr, _mac_lut(g, level, hf, beta, kappa, eta))


def test_native_traversal_is_independent_of_thread_count(monkeypatch):
    g = load_case("cubesurf4000")
    kw = g["config"]
    tr, _ = build_tree(g["points"], g["charges"], TreeConfig(ncrit=kw["ncrit"]))
    outs = []
    for nthr in ("1", "3", "8"):
        monkeypatch.setenv("DEFMM_PLAN_THREADS", nthr)
        pl = build_plan(tr, tr, kw["order"], kw["kappa"], 1.0, 2.0)
        outs.append(pl)
    for pl in outs[1:]:
        for name in ("m2l_row_slot", "m2l_row_ptr", "m2l_rows_entries", "blk_group_rows", "blk_group_ptr",
                     "blk_src", "blk_trans", "blk_mask", "p2p_ptr", "p2p_lo", "p2p_hi", "hat_slot"):
            assert np.array_equal(getattr(pl, name), getattr(outs[0], name)), name


@pytest.mark.parametrize("L", [2, 3, 4, 5, 6, 7, 8])
def test_spectral_layout_slices_are_closed_under_the_cube_group(L):
    """Device spectra are stored in orbit order (defmm_spectral_layout); every
    slice of <= 128 positions is a union of orbits of the 48 rotations
    (fourier.py:90-143)."""
    from paper_2202_04894_b200.fmm import spectral_layout

    P = 2 * L - 1
    forder, starts = spectral_layout(L)
    assert np.array_equal(np.sort(forder), np.arange(P**3))
    assert starts[0] == 0 and starts[-1] == P**3 and np.all(np.diff(starts) > 0) and np.diff(starts).max() <= 128
    f = np.stack([forder // (P * P), (forder // P) % P, forder % P], 1)
    pos_of = np.empty(P**3, np.int64)
    pos_of[forder] = np.arange(P**3)
    slice_of = np.searchsorted(starts, np.arange(P**3), side="right") - 1
    for g in GROUP48:
        img = (f @ g.T) % P  # signed permutation of the frequency vector mod P
        j = img[:, 0] * P * P + img[:, 1] * P + img[:, 2]
        assert np.array_equal(slice_of[pos_of[j]], slice_of)


@pytest.mark.parametrize("case", ["cubesurf4000", "volume3000", "refined3000"])
def test_m2l_level_policy(case):
    """Per-level M2L kernel choice (fmm.m2l_level_kinds): dense levels ->
    blocked; "auto" moves sparse levels with >= PAIR_MIN_ROWS rows to the
    sibling-group kernel (quartets at L <= 4, pairs above), the rest to the
    row kernel; overrides (dict or env string) win; bad names raise."""
    from paper_2202_04894_b200.fmm import PAIR_MIN_ROWS, block_levels, dense_levels, m2l_level_kinds, sibling_kind

    tr, _, p = _plan(load_case(case))
    levels = np.unique(p.m2l_level)
    dense = dense_levels(p, tr)
    blev, ev, _, _ = block_levels(p, tr)
    for lv in np.unique(blev):
        assert (int(lv) in dense) == (ev[blev == lv].mean() >= 32.0)
    # row counts per level scaled up so that some levels cross PAIR_MIN_ROWS
    rpl = {int(lv): int(c) * (PAIR_MIN_ROWS // 2) for lv, c in zip(*np.unique(p.m2l_level, return_counts=True))}
    for order in (4, 6):
        for dt in ("c64", "c128"):
            k = m2l_level_kinds("auto", dt, levels, dense, rows_per_level=rpl, order=order)
            for lv in levels:
                lv = int(lv)
                big = rpl.get(lv, 0) >= PAIR_MIN_ROWS
                assert k[lv] == ("blocked" if lv in dense else sibling_kind(dt, order) if big else "rows")
    assert sibling_kind("c64", 4) == "quartet" and sibling_kind("c64", 6) == "pair" and sibling_kind("c128", 7) == "pair"
    assert sibling_kind("c128", 4) == "staged" and sibling_kind("c128", 6) == "staged" and sibling_kind("c64", 5) == "staged"
    assert set(m2l_level_kinds("auto", "c64", levels, dense).values()) <= {"blocked", "rows"}
    assert set(m2l_level_kinds("hybrid_rows", "c64", levels, dense).values()) <= {"blocked", "rows"}
    lv0 = int(levels[0])
    assert m2l_level_kinds("auto", "c64", levels, dense, {lv0: "pair"})[lv0] == "pair"
    assert m2l_level_kinds("rows", "c64", levels, dense, env=f"{lv0}:quartet")[lv0] == "quartet"
    for gone in ("quad", "slice", "tile"):  # variants measured slower and removed (profiles/r02)
        with pytest.raises(ValueError):
            m2l_level_kinds("auto", "c64", levels, dense, override={lv0: gone})
    with pytest.raises(ValueError):
        m2l_level_kinds("auto", "c64", levels, dense, override={lv0: "nope"})
    with pytest.raises(ValueError):
        m2l_level_kinds("nope", "c64", levels, dense)


@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("case", ["cubesurf4000", "volume3000", "c1_kd16"])
def test_m2l_groups_reconstruct_every_row(case, K):
    """fmm.m2l_pairs (pair M2L lists): rows are paired only with a sibling of
    the same level and key, every row appears once, and each row's (source,
    symbol) events are exactly its entries in the merged per-source lists."""
    from paper_2202_04894_b200.fmm import m2l_groups

    tr, _, p = _plan(load_case(case))
    ptr, ent, rows = p.m2l_row_ptr, p.m2l_rows_entries, p.m2l_row_slot
    ids = np.arange(rows.shape[0])
    pr = m2l_groups(ids, rows, ptr, ent, p.l_cell, p.l_dir, tr.level, tr.parent, K)
    ps = pr["grp_slot"].reshape(-1, K)
    assert sorted(ps[ps >= 0].tolist()) == sorted(rows.tolist())
    row_of_slot = {int(s): i for i, s in enumerate(rows)}
    for g in range(pr["n"]):
        members = [int(x) for x in ps[g] if x >= 0]
        assert all(x < 0 for x in ps[g][len(members):])  # rows fill the group from the front
        cells = p.l_cell[members]
        assert len(set(tr.parent[cells].tolist())) == 1 and len(set(p.l_dir[members].tolist())) == 1
        e = pr["ent"][pr["grp_ptr"][g]:pr["grp_ptr"][g + 1]]
        assert len(np.unique(e[:, 0])) == len(e)
        for col, slot in enumerate(ps[g], start=1):
            if slot < 0:
                assert np.all(e[:, col] == -1)
                continue
            r = row_of_slot[int(slot)]
            got = sorted(zip(e[e[:, col] >= 0, 0].tolist(), e[e[:, col] >= 0, col].tolist()))
            want = sorted(zip(ent[ptr[r]:ptr[r + 1], 0].tolist(), ent[ptr[r]:ptr[r + 1], 1].tolist()))
            assert got == want


@pytest.mark.parametrize("ns_cap", [16, 48])
@pytest.mark.parametrize("case", ["cubesurf4000", "volume3000", "c1_kd16", "tt_hf_sphere"])
def test_m2l_stage_lists_replay_every_event(case, ns_cap):
    """fmm.m2l_stage_lists (staged M2L, K7 v13): walking the lists the way the
    kernel does -- per CTA its stages, per warp unit the entries up to the
    stage's end, per row byte the stage's slot -> symbol -- visits every row's
    (source, symbol) events exactly once; warp units hold sibling rows of one
    key, stages stay within ns_cap slots."""
    from paper_2202_04894_b200.fmm import STAGE_ENT_PAD, STAGE_K, STAGE_NW, m2l_stage_lists

    if case.startswith("tt_"):
        from conftest import load_two_tree
        from paper_2202_04894_b200.geometry import compute_root_box

        g = load_two_tree(case)
        kw = g["config"]
        box = compute_root_box(np.vstack([g["targets"], g["sources"]]))
        st, _ = build_tree(g["sources"], g["charges"], TreeConfig(ncrit=kw["ncrit"]), root_box=box)
        tr, _ = build_tree(g["targets"], np.zeros(g["targets"].shape[0]), TreeConfig(ncrit=kw["ncrit"]), root_box=box)
        p = build_plan(tr, st, kw["order"], kw["kappa"], 1.0, 2.0)
    else:
        tr, _, p = _plan(load_case(case))
        st = tr
    ptr, ent, rows = p.m2l_row_ptr, p.m2l_rows_entries, p.m2l_row_slot
    ids = np.arange(rows.shape[0])
    hc = st.coords[p.m_cell[p.hat_slot]]
    sg = m2l_stage_lists(ids, rows, ptr, ent, p.l_cell, p.l_dir, tr.level, tr.parent, tr.coords, hc, ns_cap)
    K, NW = STAGE_K, STAGE_NW
    assert sorted(sg["row_slot"].tolist()) == sorted(rows.tolist())
    assert sg["ent"].shape[0] == sg["stage_wend"].max() + STAGE_ENT_PAD
    assert np.diff(sg["stage_slot_ptr"]).max() <= ns_cap and np.diff(sg["stage_slot_ptr"]).min() >= 1
    got = {}
    e32 = sg["ent"]
    for c in range(sg["n"]):
        for w in range(NW):
            cw = c * NW + w
            lrows = sg["cta_rows"][cw * K:(cw + 1) * K]
            members = sg["row_slot"][lrows[lrows >= 0]]
            if members.size:
                cells = p.l_cell[members]
                assert len(set(tr.parent[cells].tolist())) == 1 and len(set(p.l_dir[members].tolist())) == 1
            i = int(sg["cta_went"][cw])
            s0, s1 = int(sg["cta_stage"][c]), int(sg["cta_stage"][c + 1])
            for s in range(s0, s1):
                end = int(sg["stage_wend"][s0 * NW + w * (s1 - s0) + (s - s0)])
                base = int(sg["stage_slot_ptr"][s])
                nslot = int(sg["stage_slot_ptr"][s + 1]) - base
                while i < end:
                    src, packed = int(e32[i, 0]), int(e32[i, 1]) & 0xFFFFFFFF
                    for k in range(K):
                        b = (packed >> (8 * k)) & 0xFF
                        if b != ns_cap:
                            assert b < nslot and lrows[k] >= 0
                            got.setdefault(int(sg["row_slot"][lrows[k]]), []).append((src, int(sg["slot_sym"][base + b])))
                    i += 1
            nxt = int(sg["cta_went"][cw + 1]) if cw + 1 < sg["n"] * NW else int(sg["stage_wend"].max())
            assert i == nxt
    for r, slot in enumerate(rows.tolist()):
        want = sorted(zip(ent[ptr[r]:ptr[r + 1], 0].tolist(), ent[ptr[r]:ptr[r + 1], 1].tolist()))
        assert sorted(got[slot]) == want


@pytest.mark.parametrize("max_pairs,chunk", [(1 << 16, 128), (700, 3)])
@pytest.mark.parametrize("case", ["cubesurf4000", "volume3000", "c1_kd16", "flat50", "twocluster"])
def test_p2p_mutual_lists_reproduce_the_near_field(case, max_pairs, chunk, monkeypatch):
    """plan.p2p_mutual_lists (mutual P2P, K1 v2): evaluating every item the way
    the kernel does (rows over its whole clipped range, columns past the
    leaf's own particles) and gathering the contributor segments gives the
    one-directional near-field sums, with a symmetric stand-in kernel."""
    from paper_2202_04894_b200 import plan as plan_mod
    from paper_2202_04894_b200.plan import p2p_mutual_lists

    monkeypatch.setattr(plan_mod, "P2P_GATHER_CHUNK", chunk)  # 3: several pre-sum passes
    tr, ps, p = _plan(load_case(case))
    tlo, thi = tr.start[p.leaf_cells], tr.stop[p.leaf_cells]
    ml = p2p_mutual_lists(p.p2p_ptr, p.p2p_lo, p.p2p_hi, tlo, thi, p.counts["p2p_pairs"], max_pairs)
    assert ml is not None
    n = ps.n
    rng = np.random.default_rng(5)
    q = rng.normal(size=n) + 1j * rng.normal(size=n)
    x = ps.positions
    G = 1.0 / (1.0 + np.linalg.norm(x[:, None, :] - x[None, :, :], axis=2))  # symmetric
    want = np.zeros(n, complex)
    for l in range(tlo.shape[0]):
        for e in range(p.p2p_ptr[l], p.p2p_ptr[l + 1]):
            a, b = p.p2p_lo[e], p.p2p_hi[e]
            want[tlo[l]:thi[l]] += G[tlo[l]:thi[l], a:b] @ q[a:b]
    part = np.full(ml["partial_size"], np.nan + 0j)
    for i in range(ml["item_leaf"].shape[0]):
        l = int(ml["item_leaf"][i])
        src = np.concatenate([np.arange(ml["lo"][e], ml["hi"][e]) for e in range(ml["ptr"][l], ml["ptr"][l + 1])])
        assert np.array_equal(src[: thi[l] - tlo[l]], np.arange(tlo[l], thi[l]))
        f0, f1 = int(ml["item_f0"][i]), int(ml["item_f1"][i])
        sl = src[f0:f1]
        t = np.arange(tlo[l], thi[l])
        part[ml["item_row"][i]: ml["item_row"][i] + t.size] = G[np.ix_(t, sl)] @ q[sl]
        part[ml["item_col"][i]: ml["item_col"][i] + sl.size] = G[np.ix_(sl, t)] @ q[t]
    got = np.full(n, np.nan + 0j)
    part = np.concatenate([part, np.full(ml["partial_size"] - part.shape[0], np.nan + 0j)])
    assert ml["gather"][-1]["task_leaf"].shape[0] == tlo.shape[0] and np.all(ml["gather"][-1]["task_out"] == -1)
    for gp in ml["gather"]:
        assert np.diff(gp["cptr"]).max() <= chunk
        for j, l in enumerate(gp["task_leaf"].tolist()):
            acc = np.zeros(thi[l] - tlo[l], complex)
            for c in range(gp["cptr"][j], gp["cptr"][j + 1]):
                xs = np.arange(gp["cxlo"][c], gp["cxhi"][c])
                assert 0 <= gp["cxlo"][c] < gp["cxhi"][c] <= thi[l] - tlo[l]
                acc[xs] += part[gp["cbase"][c] + xs]
            if gp["task_out"][j] < 0:
                got[tlo[l]:thi[l]] = acc
            else:
                part[gp["task_out"][j]: gp["task_out"][j] + acc.size] = acc
    assert np.all(np.isfinite(got))
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


@pytest.mark.parametrize("case", ["cubesurf4000", "volume3000", "c1_kd16", "laplace500"])
def test_m_mark_pruning_keeps_every_multipole_that_is_read(case):
    """P2M/M2M run only on the multipoles an M2L reads and, top-down, on the
    sons a needed father's M2M reads (plan.m_used); the reference's count of
    expansions (the union of marks, traversal.py:190-192, 229-236) is unchanged."""
    g = load_case(case)
    tr, _, p = _plan(g)
    used = p.m_used
    assert p.counts["effective_expansions"] == g["counts"]["effective_expansions"] == p.n_mult
    assert used[p.hat_slot].all() and p.n_mult_used == used.sum() <= p.n_mult
    produced = np.zeros(p.n_mult, bool)
    produced[p.p2m_idx] = True
    for lev, slots, son in p.m2m_levels:  # deepest level first: sons are produced before their father
        ok = son >= 0
        assert produced[son[ok]].all() and used[son[ok]].all()
        assert not produced[slots].any()
        produced[slots] = True
    assert np.array_equal(produced, used)  # every needed multipole is produced exactly once, nothing else


def test_p2p_overlap_policy():
    """P2P beside the M2L (high-priority far field) only when every M2L level
    runs the quartet kernel (measured, profiles/r01_summary_v9.md)."""
    from paper_2202_04894_b200.fmm import p2p_overlap_policy

    assert p2p_overlap_policy({4: "quartet", 5: "quartet", 6: "quartet", 7: "quartet"}) == ("m2l", True)
    assert p2p_overlap_policy({4: "rows", 5: "pair"}) == ("upward", False)
    assert p2p_overlap_policy({3: "pair", 4: "blocked"}) == ("upward", False)
    assert p2p_overlap_policy({4: "quartet", 5: "blocked"}) == ("upward", False)
    assert p2p_overlap_policy({}) == ("upward", False)


def test_plan_deferred_lists_materialise_once():
    """Plan lists handed over as device-resident handles (gpu_build.Deferred) are
    downloaded on first read and then behave as plain host arrays."""
    from paper_2202_04894_b200.plan import Plan

    class Handle:
        calls = 0

        def __init__(self, a):
            self.dev, self._a = "device tensor", a

        def host(self):
            Handle.calls += 1
            return self._a

    pl = Plan(order=4, kappa=1.0, tol=0.0, hf_max=-1, same=True, dirs=np.zeros((0, 3)), dir_off=np.zeros(1, np.int64))
    ent = np.arange(10, dtype=np.int32).reshape(5, 2)
    pl.m2l_rows_entries = Handle(ent)
    pl.blk_trans = np.zeros((0, 27), np.int32)
    assert pl.on_device("m2l_rows_entries") == "device tensor" and pl.on_device("blk_trans") is None
    assert np.array_equal(pl.m2l_src, ent[:, 0]) and np.array_equal(pl.m2l_rows_entries, ent)
    assert Handle.calls == 1 and pl.on_device("m2l_rows_entries") is None
    pl.blk_mask = np.array([0x0101, 0x1], np.int64)
    assert pl.blk_kind.shape == (2,) and pl.blk_kind is pl.blk_kind
