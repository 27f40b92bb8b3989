"""Host "precompute": the reference's blank passes + DTT as flat CSR lists.

The reference decides everything recursively, one Python frame per visited
cell pair (traversal.py:182-213 blank passes, :320-348 DTT).  Since every
visited pair is same-level, the recursion is equivalent to a level-
synchronous sweep: at level l each candidate pair is M2L (MAC holds), P2P
(either cell is a leaf) or expands into sons x sons.  This module performs
that sweep with vectorised numpy and emits the device plan:

* MAC per level as a lookup on the integer gap^2 (the MAC depends on
  (level, gap^2) only), each entry evaluated with the reference's exact FP64
  expression ``max(kappa*w*w, 2.0*w) <= eta*(beta*sqrt(gap2))``
  (traversal.py:107-113) or ``gap2 >= 1`` (:100-104);
* HF M2L keys = nearest direction of each distinct translation
  (directions.nearest_directions, bit-exact with directions.py:78-89);
* canonical symbols + rotation ids per distinct (level, translation)
  (fourier.py:104-120, 211-247);
* marks (traversal.py:190-192) and their downward propagation (:203-213);
* dense expansion slots: multipoles keyed (cell, key) on the source tree,
  locals on the target tree, sorted by (cell, key) -- the reference's
  per-cell dicts (tree.py:75-78) made contiguous;
* CSR lists for P2M, M2M (son slot per octant), M2F, M2L rows (target-major),
  L2L (gather per son slot), L2P (slot range per leaf) and P2P (merged
  source runs per target leaf).

Integer counts reproduce FmmInfo.counts exactly (traversal.py:495-505).
"""

from __future__ import annotations

import ctypes as C
import itertools
import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .directions import generate_direction_tree, nearest_directions
from .tree import SQRT3, ClusterTree

__all__ = ["Plan", "build_plan", "hf_max_level", "canonicalize_many", "GROUP48", "p2p_work_items"]

# upper bound of target x source pairs per P2P work item (cfg2's largest leaf
# has 4e4 pairs; cfg3's coarse leaves next to huge source cells up to 1.6e7)
P2P_ITEM_PAIRS = 1 << 16


def _group48() -> np.ndarray:
    """fourier.py:90-101's signed permutation matrices, same order."""
    mats = []
    for perm in itertools.permutations(range(3)):
        for signs in itertools.product((1, -1), repeat=3):
            m = np.zeros((3, 3), dtype=np.int64)
            for a in range(3):
                m[a, perm[a]] = signs[a]
            mats.append(m)
    return np.stack(mats)


GROUP48 = _group48()


_PERMS = list(itertools.permutations(range(3)))  # GROUP48[8 p + s]: permutation p, sign pattern s


def canonicalize_many(t: np.ndarray):
    """(canonical (m,3), rotation id (m,)) -- fourier.py:104-120 batched: the
    canonical translation is |t| sorted descending and the rotation id the FIRST
    group element g (fourier.py:90-101's order: permutations x sign patterns,
    (g c)[a] = signs[a] c[perm[a]]) with g canon = t.  Closed form of that
    first hit: the first permutation matching |t| (ties between equal entries),
    signs[a] = -1 iff t[a] < 0 (a zero entry matches +1 first)."""
    t = np.asarray(t, np.int64)
    if np.any(np.all(t == 0, axis=1)):
        raise ValueError("zero translation cannot be canonicalized")
    at = np.abs(t)
    canon = -np.sort(-at, axis=1)
    pid = np.full(t.shape[0], -1, np.int64)
    for p in range(5, -1, -1):  # the smallest matching permutation index wins
        perm = _PERMS[p]
        hit = (canon[:, perm[0]] == at[:, 0]) & (canon[:, perm[1]] == at[:, 1]) & (canon[:, perm[2]] == at[:, 2])
        pid[hit] = p
    sid = ((t[:, 0] < 0).astype(np.int64) << 2) | ((t[:, 1] < 0).astype(np.int64) << 1) | (t[:, 2] < 0)
    return canon, (pid * 8 + sid).astype(np.int8)


def hf_max_level(tree: ClusterTree, depth: int, kappa: float, hf_switch: float) -> int:
    """traversal.py:145-157 (w = sqrt(3) * side / 2 >= hf_switch / kappa)."""
    hf = -1
    if kappa > 0:
        for level in range(depth + 1):
            w = np.sqrt(3.0) * tree.side_at(level) / 2.0
            if kappa * w >= hf_switch:
                hf = level
            else:
                break
    return hf


def _mac_lut(g2: np.ndarray, level: int, hf: bool, beta: float, kappa: float, eta: float) -> np.ndarray:
    uniq, inv = np.unique(g2, return_inverse=True)
    if hf:
        w = SQRT3 * beta / 2.0
        lhs = max(kappa * w * w, 2.0 * w)
        vals = np.array([lhs <= eta * (beta * np.sqrt(float(g))) for g in uniq], dtype=bool)
    else:
        vals = uniq >= 1
    return vals[inv]


def _expand_pairs(ft, nt, fs, ns):
    """sons(t) x sons(s) for each pair, t-major (traversal.py:345-348)."""
    cnt = nt * ns
    tot = int(cnt.sum())
    if tot == 0:
        z = np.zeros(0, np.int64)
        return z, z
    rep = np.repeat(np.arange(cnt.shape[0]), cnt)
    k = np.arange(tot) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    nsr = ns[rep]
    return ft[rep] + k // nsr, fs[rep] + k % nsr


def _csr(keys: np.ndarray, n: int) -> np.ndarray:
    """Row pointer of sorted ``keys`` over rows 0..n-1."""
    return np.searchsorted(keys, np.arange(n + 1)).astype(np.int64)


def _deferred_list(name: str, doc: str):
    """A Plan list that may be handed over as a device-resident
    gpu_build.Deferred: reading the attribute downloads it once."""
    slot = "_d_" + name

    def get(self):
        v = self.__dict__.get(slot)
        if hasattr(v, "host"):
            v = self.__dict__[slot] = v.host()
        return v

    def put(self, v):
        self.__dict__[slot] = v

    return property(get, put, doc=doc)


@dataclass
class Plan:
    """Everything the device matvec needs, as host numpy arrays (the device
    builders leave the per-event and per-block lists on the device:
    ``on_device``)."""

    order: int
    kappa: float
    tol: float
    hf_max: int
    same: bool
    dirs: np.ndarray  # (ndir, 3) all refinements concatenated
    dir_off: np.ndarray  # refinement e -> first global id
    counts: dict = field(default_factory=dict)
    # symbols
    sym_tvec: np.ndarray = None  # (nsym, 3) int32 canonical translations
    sym_beta: np.ndarray = None  # (nsym,)
    sym_level: np.ndarray = None  # (nsym,) level; symbols are sorted by (level, canonical t)
    # multipole slots (source tree)
    m_cell: np.ndarray = None
    m_dir: np.ndarray = None  # global dir id or -1
    p2m_idx: np.ndarray = None  # slots computed by P2M
    m2m_levels: list = None  # [(level, slots, son_slot (k,8))] deepest first
    hat_slot: np.ndarray = None  # mult slot of each spectrum
    m_used: np.ndarray = None  # per multipole slot: computed by P2M/M2M (an M2L reads it or a needed father does)
    n_mult_used: int = 0
    # locals (target tree)
    l_cell: np.ndarray = None
    l_dir: np.ndarray = None
    m2l_row_slot: np.ndarray = None
    m2l_row_ptr: np.ndarray = None
    m2l_level: np.ndarray = None  # per row
    m2l_rows_entries = _deferred_list("m2l_rows_entries",
                                      "(n_m2l, 2) int32 {hat, derived symbol} in row order")
    l2l_levels: list = None  # [(son level, out_slot, octant, ptr, src_slot, src_dir)]
    leaf_cells: np.ndarray = None  # target-tree leaves
    leaf_slot_lo: np.ndarray = None
    leaf_slot_hi: np.ndarray = None
    # near field (target leaves)
    p2p_ptr: np.ndarray = None
    p2p_lo: np.ndarray = None
    p2p_hi: np.ndarray = None
    # derived symbols (one per distinct (level, translation))
    trans_canon: np.ndarray = None  # canonical symbol id
    trans_rid: np.ndarray = None  # cube-group rotation id
    # parent-pair blocks of the blocked M2L (K7 v3)
    blk_group_rows: np.ndarray = None  # (ngroups, 8) local slots of the group's rows, -1 absent
    blk_group_ptr: np.ndarray = None  # block range per group
    blk_src_ev = _deferred_list("blk_src_ev", "(nblocks, 8) an event of each source child (its spectrum: "
                                "entries[ev, 0]), -1 absent")
    blk_trans = _deferred_list("blk_trans", "(nblocks, 27) derived symbol per child offset, -1 unused")
    blk_mask: np.ndarray = None  # (nblocks,) int64: bit 8a+b = (a, b) is an M2L event
    # event logs (optional, for the events= API)
    m2l_events: tuple = None
    p2p_events: tuple = None

    @property
    def blk_kind(self):
        """(nblocks,) int8: -1 general, 2p+v planar (from blk_mask, on first use)."""
        if getattr(self, "_blk_kind", None) is None:
            self._blk_kind = planar_kind(self.blk_mask)
        return self._blk_kind

    def on_device(self, name: str):
        """The device tensor of a list the host has not read yet, else None."""
        v = self.__dict__.get("_d_" + name)
        return v.dev if hasattr(v, "host") else None

    @property
    def blk_src(self):
        """(nblocks, 8) spectrum index per source child, -1 absent (mapped on
        first use: only plans with blocked levels need it)."""
        if getattr(self, "_blk_src", None) is None:
            bs = self.blk_src_ev
            hat = self.m2l_rows_entries[:, 0]
            self._blk_src = np.where(bs >= 0, hat[np.maximum(bs, 0)] if hat.size else 0, -1).astype(np.int32)
        return self._blk_src

    @property
    def n_mult(self):
        return int(self.m_cell.shape[0])

    @property
    def n_local(self):
        return int(self.l_cell.shape[0])

    @property
    def n_hat(self):
        return int(self.hat_slot.shape[0])

    @property
    def n_sym(self):
        return int(self.sym_tvec.shape[0])

    # per-event views in row order (derived from the entries table)
    @property
    def m2l_src(self):  # spectrum index
        return self.m2l_rows_entries[:, 0]

    @property
    def m2l_sym(self):  # canonical symbol id
        return self.trans_canon[self.m2l_rows_entries[:, 1]]

    @property
    def m2l_rid(self):  # cube-group rotation id
        return self.trans_rid[self.m2l_rows_entries[:, 1]]


def build_plan(tt: ClusterTree, st: ClusterTree, order: int, kappa: float, eta: float, hf_switch: float,
               keep_events: bool = False, dtt: str = "native", device="cuda") -> Plan:
    """``dtt``: "native" = the multi-threaded host traversal (csrc/dtt_build.cpp),
    "gpu" = the level-synchronous device traversal (gpu_build.GpuDtt); both
    produce the same lists (tests/test_gpu_build.py)."""
    same = tt is st
    depth = max(tt.depth, st.depth)
    hf = hf_max_level(tt, depth, kappa, hf_switch)
    dt = generate_direction_tree(hf) if hf >= 0 else None
    if dt is not None:
        dirs = np.concatenate(dt.levels)
        dir_off = np.concatenate([[0], np.cumsum([d.shape[0] for d in dt.levels])]).astype(np.int64)
    else:
        dirs = np.zeros((0, 3))
        dir_off = np.zeros(1, np.int64)
    tol = 1e-12 * st.root_box.side  # traversal.py:465-467
    plan = Plan(order=order, kappa=kappa, tol=tol, hf_max=hf, same=same, dirs=dirs, dir_off=dir_off)

    # ---- dual tree traversal (native, traversal.py:320-348) ----------------
    g2min, R, tab_off, key_tab = _traversal_tables(tt, depth, hf, dt, dir_off, kappa, eta)
    if dtt == "gpu":
        from .gpu_build import GpuDtt

        nat = GpuDtt(tt, st, depth, g2min, R, tab_off, key_tab, device=device)
    elif dtt == "native":
        nat = NativeDtt(tt, st, depth, g2min, R, tab_off, key_tab)
    else:
        raise ValueError(f"unknown traversal builder {dtt!r}")
    row_ptr, row_t, row_key, row_lev = nat["row_ptr"], nat["row_t"], nat["row_key"], nat["row_lev"]
    on_dev = hasattr(nat, "deferred")  # the device traversal keeps the per-event lists on the device
    pt, ps = nat["p_t"].astype(np.int64), nat["p_s"].astype(np.int64)
    n_m2l = int(nat.n_events)
    n_rows = int(row_t.shape[0])
    row_cnt = np.diff(row_ptr)
    # events are level-contiguous (rows are ordered (level, target, key))
    lev_rows = np.searchsorted(row_lev, np.arange(depth + 2)).astype(np.int64)
    lev_ev = row_ptr[lev_rows]
    row_loc = np.where(row_key >= 0, row_key - dir_off[np.maximum(hf - row_lev, 0)], -1).astype(np.int64)

    # ---- distinct (level, t): the used entries of the dense tables ---------
    uniq = nat["trans_dense"]  # used dense-table entries == (level, t) lexicographic order
    u_lev = np.searchsorted(tab_off, uniq, side="right") - 1
    rel = uniq - tab_off[u_lev]
    w = 2 * R[u_lev].astype(np.int64) + 1
    u_tv = np.stack([rel // (w * w), (rel // w) % w, rel % w], 1) - R[u_lev].astype(np.int64)[:, None]
    # canonical symbol classes (fourier.py:233-247)
    if uniq.shape[0]:
        canon, rid = canonicalize_many(u_tv)
    else:
        canon, rid = np.zeros((0, 3), np.int64), np.zeros(0, np.int8)
    Rc = int(canon.max()) + 1 if canon.size else 1
    cpack = ((u_lev * Rc + canon[:, 0]) * Rc + canon[:, 1]) * Rc + canon[:, 2]
    cuniq, cinv = np.unique(cpack, return_inverse=True)
    sym_lev = np.empty(cuniq.shape[0], np.int64)
    sym_lev[cinv] = u_lev
    sym_t = np.empty((cuniq.shape[0], 3), np.int64)
    sym_t[cinv] = canon
    plan.sym_tvec = sym_t.astype(np.int32)
    plan.sym_beta = tt.root_box.side / np.left_shift(np.int64(1), sym_lev)  # ClusterTree.side_at per symbol
    plan.sym_level = sym_lev
    _check_stencils(sym_t, sym_lev, tt, order, tol)

    # ---- marks (traversal.py:190-192) + downward propagation (:203-213) ---
    # mark key = cell * KD + local direction index (refinement e = hf - level)
    KD = int(dirs.shape[0]) + 1
    t_marks = [[] for _ in range(depth + 1)]
    s_marks = [[] for _ in range(depth + 1)] if not same else t_marks
    for lev in range(min(hf, depth) + 1):
        r0, r1 = lev_rows[lev], lev_rows[lev + 1]
        if r1 == r0:
            continue
        t_marks[lev].append(row_t[r0:r1].astype(np.int64) * KD + row_loc[r0:r1])
        sm = nat.source_marks(lev) if hasattr(nat, "source_marks") else None
        if sm is not None:  # distinct (source cell, key) of the level's events, found on the device
            s_marks[lev].append(sm[0] * KD + (sm[1] - dir_off[hf - lev]))
        else:
            loc_ev = np.repeat(row_loc[r0:r1], row_cnt[r0:r1])
            s_marks[lev].append(_unique_cell_keys(nat["ev_s"][lev_ev[lev] : lev_ev[lev + 1]], loc_ev, st, lev,
                                                  dt.levels[hf - lev].shape[0], KD))
    marks_t = _propagate_marks(tt, t_marks, hf, dt, KD)
    marks_s = marks_t if same else _propagate_marks(st, s_marks, hf, dt, KD)

    # ---- multipole slots on the source tree --------------------------------
    m_cell, m_loc, m_dir = [], [], []
    for lev in range(st.depth + 1):
        if lev <= hf:
            mk = marks_s[lev]
            c, i = mk // KD, mk % KD
            m_dir.append(dir_off[hf - lev] + i)
        else:
            c = np.arange(st.level_offsets[lev], st.level_offsets[lev + 1])
            i = np.full(c.shape[0], -1, np.int64)
            m_dir.append(i)
        m_cell.append(c)
        m_loc.append(i)
    m_cell = np.concatenate(m_cell)
    m_loc = np.concatenate(m_loc)
    m_dir = np.concatenate(m_dir)
    plan.m_cell, plan.m_dir = m_cell, m_dir
    # slot lookup key: cell*(KD+1) + (local dir + 1), 0 for LF; sorted by construction
    mkey = m_cell * (KD + 1) + (m_loc + 1)
    assert np.all(np.diff(mkey) > 0)

    def mslot(cells, loc_dirs):
        k = cells * (KD + 1) + (loc_dirs + 1)
        j = np.searchsorted(mkey, k)
        ok = (j < mkey.shape[0]) & (mkey[np.minimum(j, mkey.shape[0] - 1)] == k)
        return np.where(ok, j, -1)

    leaf_m = st.is_leaf[m_cell]
    plan.p2m_idx = np.nonzero(leaf_m)[0]
    # M2M per level, deepest first (traversal.py:283-289)
    m2m_levels = []
    mlevel = st.level[m_cell]
    for lev in range(st.depth - 1, -1, -1):
        slots = np.nonzero((mlevel == lev) & ~leaf_m)[0]
        if slots.size == 0:
            continue
        c = m_cell[slots]
        son_slot = np.full((slots.shape[0], 8), -1, np.int64)
        for k in range(8):
            has = st.n_sons[c] > k
            if not has.any():
                continue
            sons = st.first_son[c[has]] + k
            octv = st.coords[sons] - 2 * st.coords[c[has]]
            oct_ = octv[:, 0] * 4 + octv[:, 1] * 2 + octv[:, 2]
            if lev + 1 <= hf:
                e = hf - lev
                li = m_dir[slots[has]] - dir_off[e]
                sk = dt.fathers[e][li]
            else:
                sk = np.full(sons.shape[0], -1, np.int64)
            ss = mslot(sons, sk)
            if np.any(ss < 0):
                raise RuntimeError("missing son expansion: blank-pass inconsistency")
            son_slot[np.nonzero(has)[0], oct_] = ss
        m2m_levels.append((lev, slots, son_slot))
    plan.m2m_levels = m2m_levels

    # ---- M2L sources -> spectra (M2F only for used multipoles) -------------
    nd_s, base_s = _dense_space(st, hf, dt)
    m_dense = np.full(int(base_s[-1]), -1, np.int64)
    m_dense[_dense_index(st, nd_s, base_s, m_cell, m_loc)] = np.arange(m_cell.shape[0])
    key_base = np.zeros(depth + 1, np.int32)
    for lev in range(min(hf, depth) + 1):
        key_base[lev] = dir_off[hf - lev]
    src_hat, hat_slot = nat.source_hats(m_dense, base_s, nd_s, st.level_offsets, key_base, m_cell.shape[0])
    nat.close()
    plan.hat_slot = hat_slot
    # M-mark pruning: the reference creates an expansion for every mark (the union of target
    # and source marks in single-tree mode, traversal.py:190-192, 229-236 -- that is what
    # counts["effective_expansions"] reports); only the multipoles an M2L reads, and the
    # sons the M2M of such a multipole reads (top-down closure), are ever used.  P2M and
    # M2M run on those; the other slots keep their place (layout unchanged) and stay unread.
    needed = np.zeros(m_cell.shape[0], bool)
    needed[hat_slot] = True
    for lev, slots, son_slot in reversed(m2m_levels):  # coarsest level first
        ss = son_slot[needed[slots]]
        needed[ss[ss >= 0]] = True
    plan.m_used = needed
    plan.n_mult_used = int(needed.sum())
    plan.p2m_idx = plan.p2m_idx[needed[plan.p2m_idx]]
    plan.m2m_levels = [(lev, slots[needed[slots]], son_slot[needed[slots]]) for lev, slots, son_slot in m2m_levels
                       if needed[slots].any()]

    # ---- local slots on the target tree -------------------------------------
    rt64 = row_t.astype(np.int64)
    l_cell, l_loc, l2l = _local_slots(tt, rt64, row_loc, hf, dt, dir_off, KD)
    plan.l_cell = l_cell
    plan.l_dir = np.where(l_loc >= 0, dir_off[np.maximum(hf - tt.level[l_cell], 0)] + l_loc, -1)
    lkey = l_cell * (KD + 1) + (l_loc + 1)
    assert np.all(np.diff(lkey) > 0)

    def lslot(cells, loc_dirs):
        k = cells * (KD + 1) + (loc_dirs + 1)
        j = np.searchsorted(lkey, k)
        assert np.all(lkey[j] == k)
        return j

    tslot = lslot(rt64, row_loc)  # rows are (level, cell, key)-ordered: increasing
    plan.m2l_row_slot = tslot.astype(np.int64)
    plan.m2l_row_ptr = row_ptr
    if on_dev:
        plan.m2l_rows_entries = nat.entries(src_hat)
    else:
        ent = np.empty((n_m2l, 2), np.int32)
        ent[:, 0] = src_hat
        ent[:, 1] = nat["ev_trans"]  # translation id per event
        plan.m2l_rows_entries = ent
    plan.m2l_level = row_lev.astype(np.int64)
    # derived-symbol table: one per distinct (level, t)
    plan.trans_canon = cinv.astype(np.int32)
    plan.trans_rid = rid
    # parent-pair blocks of the blocked M2L (K7 v3), from the traversal
    gr = nat["grp_rows"]
    plan.blk_group_rows = np.where(gr >= 0, tslot[np.maximum(gr, 0)], -1) if n_rows else gr
    plan.blk_group_ptr = nat["grp_ptr"]
    plan.blk_src_ev = nat.deferred("blk_src") if on_dev else nat["blk_src"]
    plan.blk_trans = nat.deferred("blk_trans") if on_dev else nat["blk_trans"]
    plan.blk_mask = nat["blk_mask"]

    # L2L gather lists per son level
    l2l_levels = []
    if l2l[0].size:
        f_slot = lslot(l2l[0], l2l[1])
        s_slot = lslot(l2l[2], l2l[3])
        f_dir = plan.l_dir[f_slot]
        o = np.lexsort((f_slot, s_slot))
        f_slot, s_slot, f_dir = f_slot[o], s_slot[o], f_dir[o]
        outs, first = np.unique(s_slot, return_index=True)
        ptr = np.concatenate([first, [s_slot.shape[0]]]).astype(np.int64)
        son_cells = l_cell[outs]
        fathers = tt.parent[son_cells]
        octv = tt.coords[son_cells] - 2 * tt.coords[fathers]
        octant = (octv[:, 0] * 4 + octv[:, 1] * 2 + octv[:, 2]).astype(np.int8)
        son_lev = tt.level[son_cells]
        for lev in np.unique(son_lev):
            sel = np.nonzero(son_lev == lev)[0]
            a, b = ptr[sel[0]], ptr[sel[-1] + 1]
            l2l_levels.append((int(lev), outs[sel], octant[sel], ptr[sel[0] : sel[-1] + 2] - a, f_slot[a:b], f_dir[a:b].astype(np.int32)))
    plan.l2l_levels = l2l_levels

    # L2P: every target leaf (also writes near + far, un-permuted)
    leaves = np.nonzero(tt.is_leaf)[0]
    leaves = leaves[np.argsort(tt.start[leaves], kind="stable")]  # Morton (particle) order
    plan.leaf_cells = leaves
    plan.leaf_slot_lo = np.searchsorted(l_cell, leaves, side="left").astype(np.int64)
    plan.leaf_slot_hi = np.searchsorted(l_cell, leaves, side="right").astype(np.int64)

    # ---- P2P lists: split non-leaf targets into leaves, merge runs ---------
    n_pairs = int(nat.n_pairs) if on_dev else int(((tt.stop[pt] - tt.start[pt]) * (st.stop[ps] - st.start[ps])).sum())
    run_leaf, run_lo, run_hi = _p2p_runs(pt, ps, tt, st, leaves, device if dtt == "gpu" else None)
    plan.p2p_ptr = _csr(run_leaf, leaves.shape[0])
    plan.p2p_lo, plan.p2p_hi = run_lo.astype(np.int64), run_hi.astype(np.int64)

    n_exp = int(m_cell.shape[0])
    plan.counts = {
        "cells": tt.n_cells if same else tt.n_cells + st.n_cells,
        "leaves": tt.n_leaves if same else tt.n_leaves + st.n_leaves,
        "symbols": int(cuniq.shape[0]),
        "effective_expansions": n_exp,
        "p2p_pairs": n_pairs,
        "m2l_events": int(n_m2l),
        "translations": int(uniq.shape[0]),
    }
    if keep_events:
        plan.m2l_events = (np.repeat(rt64, row_cnt), nat["ev_s"].astype(np.int64),
                           np.repeat(row_key.astype(np.int64), row_cnt))
        plan.p2p_events = (pt, ps)
    return plan


def mac_threshold(level: int, hf: bool, beta: float, kappa: float, eta: float, gmax: int) -> int:
    """Smallest integer gap^2 in [0, gmax] satisfying the reference MAC at this
    level (gmax + 1 if none): ``gap2 >= 1`` at LF levels (traversal.py:100-104),
    ``max(kappa*w*w, 2.0*w) <= eta*(beta*sqrt(gap2))`` at HF levels (:107-113),
    evaluated with the same FP64 expression.  The HF test is an up-set in gap2
    (sqrt and multiplication by positive constants are monotone under
    round-to-nearest), so the threshold reproduces the per-pair test exactly."""
    if not hf:
        return 1 if gmax >= 1 else gmax + 1
    w = SQRT3 * beta / 2.0
    lhs = max(kappa * w * w, 2.0 * w)

    def ok(g):
        return bool(lhs <= eta * (beta * np.sqrt(float(g))))

    if not ok(gmax):
        return gmax + 1
    lo, hi = 0, gmax
    while lo < hi:
        mid = (lo + hi) // 2
        if ok(mid):
            hi = mid
        else:
            lo = mid + 1
    return lo


_TABLE_CACHE: dict = {}


def _traversal_tables(tt, depth, hf, dt, dir_off, kappa, eta):
    """Cached per (depth, hf, kappa, eta, root side): see _traversal_tables_build."""
    key = (int(depth), int(hf), float(kappa), float(eta), float(tt.root_box.side))
    if key not in _TABLE_CACHE:
        if len(_TABLE_CACHE) >= 8:
            _TABLE_CACHE.pop(next(iter(_TABLE_CACHE)))
        _TABLE_CACHE[key] = _traversal_tables_build(tt, depth, hf, dt, dir_off, kappa, eta)
    return _TABLE_CACHE[key]


def _traversal_tables_build(tt, depth, hf, dt, dir_off, kappa, eta):
    """Per-level MAC thresholds and dense HF key tables for defmm_dtt_build.

    Level l's candidate translations are bounded by R_l = min(2^l - 1,
    2 D_{l-1} + 1), D_{l-1} the largest |t|_inf of a non-admissible pair one
    level up.  key_tab holds the global nearest-direction id of every
    admissible translation of an HF level (directions.nearest_directions,
    bit-exact with directions.py:78-89), -1 elsewhere."""
    g2min = np.zeros(depth + 1, np.int64)
    R = np.zeros(depth + 1, np.int32)
    tabs = []
    for lev in range(depth + 1):
        span = (1 << lev) - 1
        gmax = 3 * max(span - 1, 0) ** 2
        g2min[lev] = mac_threshold(lev, lev <= hf, tt.side_at(lev), kappa, eta, gmax)
        if lev == 0:
            r = 0
        else:
            pspan = (1 << (lev - 1)) - 1
            gp = int(g2min[lev - 1])
            dp = pspan if gp > 3 * max(pspan - 1, 0) ** 2 else min(pspan, math.isqrt(max(gp - 1, 0)) + 1)
            r = min(span, 2 * dp + 1)
        R[lev] = r
        w = 2 * r + 1
        tab = np.full(w**3, -1, np.int32)
        if lev <= hf and g2min[lev] <= gmax:
            ax = np.arange(-r, r + 1, dtype=np.int64)
            tv = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), -1).reshape(-1, 3)
            g = np.maximum(np.abs(tv) - 1, 0)
            adm = np.nonzero((g * g).sum(1) >= g2min[lev])[0]
            e = hf - lev
            tab[adm] = dir_off[e] + nearest_directions(dt.levels[e], tv[adm])
        tabs.append(tab)
    tab_off = np.concatenate([[0], np.cumsum([t.shape[0] for t in tabs])]).astype(np.int64)
    if tab_off[-1] >= 2**31:
        raise ValueError("translation tables exceed the int32 index range")
    return g2min, R, tab_off, np.concatenate(tabs)


class NativeDtt:
    """Lists of defmm_dtt_build (csrc/dtt_build.cpp); the handle stays open
    for the source-spectrum pass (defmm_dtt_source_hats) until close()."""

    _NAMES = ["ev_s", "ev_trans", "row_ptr", "row_t", "row_key", "row_lev", "grp_rows", "grp_p", "grp_key",
              "grp_lev", "grp_ptr", "blk_src", "blk_trans", "blk_mask", "p_t", "p_s"]

    def __init__(self, tt: ClusterTree, st: ClusterTree, depth, g2min, R, tab_off, key_tab):
        self.lib = lib = _lib.load()

        def arrs(tree):
            return [np.ascontiguousarray(tree.level_offsets, np.int64), np.ascontiguousarray(tree.coords, np.int64),
                    np.ascontiguousarray(tree.first_son, np.int64), np.ascontiguousarray(tree.n_sons, np.int64),
                    np.ascontiguousarray(tree.parent, np.int64)]

        ta = arrs(tt)
        sa = ta if st is tt else arrs(st)
        g2min = np.ascontiguousarray(g2min, np.int64)
        R = np.ascontiguousarray(R, np.int32)
        tab_off = np.ascontiguousarray(tab_off, np.int64)
        key_tab = np.ascontiguousarray(key_tab, np.int32)
        self.h = C.c_void_p()
        rc = lib.defmm_dtt_build(ta[0].ctypes.data, tt.depth, *[a.ctypes.data for a in ta[1:]],
                                 sa[0].ctypes.data, st.depth, *[a.ctypes.data for a in sa[1:]],
                                 int(depth), g2min.ctypes.data, R.ctypes.data, tab_off.ctypes.data,
                                 key_tab.ctypes.data, C.byref(self.h))
        if rc == -4:
            raise RuntimeError("defmm_dtt_build: a translation fell outside its level's key table")
        if rc != 0:
            raise RuntimeError(f"defmm_dtt_build failed ({rc})")
        sz = np.zeros(6, np.int64)
        _lib.check(lib.defmm_dtt_sizes(self.h, sz.ctypes.data), "defmm_dtt_sizes")
        ne, nr, ng, nb, npp, ntr = (int(x) for x in sz)
        self.n_events = ne
        shapes = {
            "ev_s": (ne, np.int32), "ev_trans": (ne, np.int32), "row_ptr": (nr + 1, np.int64),
            "row_t": (nr, np.int32), "row_key": (nr, np.int32), "row_lev": (nr, np.int32),
            "grp_rows": ((ng, 8), np.int64), "grp_p": (ng, np.int32), "grp_key": (ng, np.int32),
            "grp_lev": (ng, np.int32), "grp_ptr": (ng + 1, np.int64), "blk_src": ((nb, 8), np.int64),
            "blk_trans": ((nb, 27), np.int32), "blk_mask": (nb, np.int64), "p_t": (npp, np.int32),
            "p_s": (npp, np.int32),
        }
        self.a = {k: np.empty(*shapes[k]) for k in self._NAMES}
        _lib.check(lib.defmm_dtt_fetch(self.h, *[self.a[k].ctypes.data for k in self._NAMES]), "defmm_dtt_fetch")
        self.a["trans_dense"] = np.empty(ntr, np.int64)
        _lib.check(lib.defmm_dtt_translations(self.h, self.a["trans_dense"].ctypes.data), "defmm_dtt_translations")

    def __getitem__(self, k):
        return self.a[k]

    def source_hats(self, m_dense, base, nd, level_off, key_base, n_mult):
        """(src_hat per event int32, hat_slot) -- see defmm_dtt_source_hats."""
        args = [np.ascontiguousarray(x, np.int64) for x in (m_dense, base, nd, level_off)]
        kb = np.ascontiguousarray(key_base, np.int32)
        src_hat = np.empty(self.n_events, np.int32)
        hat = np.empty(max(int(n_mult), 1), np.int64)
        nh = C.c_int64(0)
        rc = self.lib.defmm_dtt_source_hats(self.h, *[x.ctypes.data for x in args], kb.ctypes.data, int(n_mult),
                                            src_hat.ctypes.data, hat.ctypes.data, C.byref(nh))
        if rc == -6:
            raise RuntimeError("missing source expansion: blank-pass bug")
        _lib.check(rc, "defmm_dtt_source_hats")
        return src_hat, hat[: nh.value].copy()

    def close(self):
        if self.h:
            self.lib.defmm_dtt_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dtt_numpy(tt: ClusterTree, st: ClusterTree, kappa: float, eta: float, hf_switch: float):
    """Vectorised level-synchronous restatement of traversal.py:320-348 with
    the per-pair MAC (cross-check of dtt_native in tests/test_plan.py).
    Returns (m2l_t, m2l_s, m2l_level, p2p_t, p2p_s)."""
    depth = max(tt.depth, st.depth)
    hf = hf_max_level(tt, depth, kappa, hf_switch)
    m2l_t, m2l_s, m2l_lev, p2p_t, p2p_s = [], [], [], [], []
    T = np.zeros(1, np.int64)
    S = np.zeros(1, np.int64)
    for lev in range(depth + 1):
        if T.size == 0:
            break
        d = tt.coords[T] - st.coords[S]
        g = np.maximum(np.abs(d) - 1, 0)
        g2 = (g * g).sum(axis=1)
        mac = _mac_lut(g2, lev, lev <= hf, tt.side_at(lev), kappa, eta)
        m2l_t.append(T[mac])
        m2l_s.append(S[mac])
        m2l_lev.append(np.full(int(mac.sum()), lev, np.int64))
        rest = ~mac
        leafy = tt.is_leaf[T] | st.is_leaf[S]
        sel = rest & leafy
        p2p_t.append(T[sel])
        p2p_s.append(S[sel])
        sel = rest & ~leafy
        rt, rs = T[sel], S[sel]
        T, S = _expand_pairs(tt.first_son[rt], tt.n_sons[rt], st.first_son[rs], st.n_sons[rs])
    cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.int64)  # noqa: E731
    return cat(m2l_t), cat(m2l_s), cat(m2l_lev), cat(p2p_t), cat(p2p_s)


def _p2p_runs(pt, ps, tt, st, leaves, device=None):
    """P2P events (target cell, source cell) -> per target LEAF (Morton order) the
    merged source particle runs: non-leaf targets are split into their leaves, each
    leaf's source ranges sorted by start and contiguous ranges merged (the source
    cells of one leaf are disjoint).  Returns (leaf index, run start, run stop),
    ordered by (leaf, start).  ``device``: run the expansion and the sort there."""
    X = _NumpyOps if device is None else _TorchOps(device)
    n_part = int(st.stop[0]) if st.stop.size else 0
    lstart = X.arr(tt.start[leaves])
    pt_, ps_ = X.arr(pt), X.arr(ps)
    l0 = X.searchsorted(lstart, X.arr(tt.start)[pt_])
    l1 = X.searchsorted(lstart, X.arr(tt.stop)[pt_])
    cnt = l1 - l0
    tot = int(cnt.sum())
    rep = X.repeat(X.arange(pt_.shape[0]), cnt)
    lidx = X.repeat(l0, cnt) + (X.arange(tot) - X.repeat(X.cumsum(cnt) - cnt, cnt))
    slo = X.arr(st.start)[ps_][rep]
    shi = X.arr(st.stop)[ps_][rep]
    o = X.argsort_stable(lidx * (n_part + 1) + slo)
    lidx, slo, shi = lidx[o], slo[o], shi[o]
    # a run continues while the next range of the same leaf starts where this one stops
    cont = (lidx[1:] == lidx[:-1]) & (slo[1:] == shi[:-1])
    first = X.cat([X.full(min(tot, 1), 1) > 0, ~cont])
    last = X.cat([~cont, X.full(min(tot, 1), 1) > 0])
    return tuple(X.to_host(a) for a in (lidx[first], slo[first], shi[last]))


def _dense_space(tree, hf, dt):
    """Per-level dense index space over (cell, local direction): nd[l] slots
    per cell (directions of refinement hf - l at HF levels, 1 at LF levels)."""
    nd = np.ones(tree.depth + 1, np.int64)
    for lev in range(min(hf, tree.depth) + 1):
        nd[lev] = dt.levels[hf - lev].shape[0]
    ncell = np.diff(tree.level_offsets)[: tree.depth + 1]
    base = np.concatenate([[0], np.cumsum(ncell * nd)]).astype(np.int64)
    return nd, base


def _dense_index(tree, nd, base, cells, loc):
    lev = tree.level[cells]
    return base[lev] + (cells - tree.level_offsets[lev]) * nd[lev] + np.maximum(loc, 0)


def _unique_cell_keys(cells, loc, tree, lev, nd, KD):
    """Sorted distinct cell*KD + loc of one level's (cell, loc) list (bitmap)."""
    off = int(tree.level_offsets[lev])
    bm = np.zeros(int(tree.level_offsets[lev + 1] - off) * nd, bool)
    bm[(cells.astype(np.int64) - off) * nd + loc] = True
    nz = np.nonzero(bm)[0]
    return (off + nz // nd) * KD + nz % nd


def _planar_masks():
    """allowed[2p+v]: pair bits 8a+b with a_p == b_p == v."""
    out = []
    for p in range(3):
        for v in range(2):
            m = 0
            for a in range(8):
                for b in range(8):
                    if ((a >> (2 - p)) & 1) == v and ((b >> (2 - p)) & 1) == v:
                        m |= 1 << (8 * a + b)
            out.append(np.uint64(m))
    return out


_PLANAR = _planar_masks()


def planar_kind(mask: np.ndarray) -> np.ndarray:
    """-1 for a general block, 2p+v when every pair lies in the plane a_p = b_p = v."""
    m = np.asarray(mask).view(np.uint64)
    kind = np.full(m.shape[0], -1, np.int8)
    for k in range(5, -1, -1):
        kind[(m & ~_PLANAR[k]) == 0] = k
    return kind


def p2p_work_items(ptr, run_len, nt, max_pairs: int = P2P_ITEM_PAIRS) -> dict:
    """Cut every target leaf's flattened source list into work items of at
    most ~max_pairs pairs (defmm_p2p_*: item_leaf/f0/f1/out + split lists).
    Items are ordered by decreasing work so the heavy ones start first."""
    ptr = np.asarray(ptr, np.int64)
    cs = np.concatenate([[0], np.cumsum(np.asarray(run_len, np.int64))])
    ns = cs[ptr[1:]] - cs[ptr[:-1]]
    nt = np.asarray(nt, np.int64)
    work = nt * ns
    k = np.maximum(1, -(-work // max_pairs))
    k = np.minimum(k, np.maximum(ns, 1))
    chunk = -(-ns // k)
    k = np.where(ns > 0, -(-ns // np.maximum(chunk, 1)), 1)  # drop empty tail items
    leaf = np.repeat(np.arange(ns.shape[0]), k)
    m = np.arange(leaf.shape[0]) - np.repeat(np.cumsum(k) - k, k)
    f0 = m * chunk[leaf]
    f1 = np.minimum(ns[leaf], f0 + chunk[leaf])
    split = k > 1
    base = np.zeros(ns.shape[0], np.int64)
    base[split] = np.concatenate([[0], np.cumsum((k * nt)[split])[:-1]]) if split.any() else []
    out = np.where(split[leaf], base[leaf] + m * nt[leaf], -1)
    order = np.argsort(-(nt[leaf] * (f1 - f0)), kind="stable")
    return {
        "item_leaf": leaf[order].astype(np.int32),
        "item_f0": f0[order].astype(np.int64),
        "item_f1": f1[order].astype(np.int64),
        "item_out": out[order].astype(np.int64),
        "split_leaf": np.nonzero(split)[0].astype(np.int32),
        "split_base": base[split].astype(np.int64),
        "split_n": k[split].astype(np.int32),
        "partial_size": int((k * nt)[split].sum()),
    }


P2P_MUTUAL_MAX_LEAF = 256  # particles per leaf the mutual kernel handles (2 per thread)
P2P_GATHER_CHUNK = 128  # contributor segments one gather task sums


class _NumpyOps:
    """The array operations p2p_mutual_lists needs, on numpy (host) ..."""

    @staticmethod
    def arr(a):
        return np.asarray(a, np.int64)

    arange = staticmethod(lambda n: np.arange(n, dtype=np.int64))
    zeros = staticmethod(lambda n: np.zeros(n, np.int64))
    full = staticmethod(lambda n, v: np.full(n, v, np.int64))
    cat = staticmethod(lambda xs: np.concatenate(xs))
    repeat = staticmethod(lambda a, c: np.repeat(a, c))
    cumsum = staticmethod(lambda a: np.cumsum(a))
    maximum = staticmethod(np.maximum)
    minimum = staticmethod(np.minimum)
    where = staticmethod(np.where)
    searchsorted = staticmethod(lambda a, v, right=False: np.searchsorted(a, v, side="right" if right else "left"))
    argsort_stable = staticmethod(lambda a: np.argsort(a, kind="stable"))
    to_host = staticmethod(lambda a: np.asarray(a))

    @staticmethod
    def unique_inverse(a):
        u, inv = np.unique(a, return_inverse=True)
        return u, inv.reshape(-1)


class _TorchOps:
    """... and on torch device tensors (the same index arithmetic on the GPU)."""

    def __init__(self, device):
        import torch

        self.t, self.dev = torch, device

    def arr(self, a):
        return self.t.as_tensor(np.ascontiguousarray(a, np.int64)).to(self.dev) if not self.t.is_tensor(a) else a

    def arange(self, n):
        return self.t.arange(int(n), dtype=self.t.int64, device=self.dev)

    def zeros(self, n):
        return self.t.zeros(int(n), dtype=self.t.int64, device=self.dev)

    def full(self, n, v):
        return self.t.full((int(n),), int(v), dtype=self.t.int64, device=self.dev)

    def cat(self, xs):
        return self.t.cat([self.arr(x) for x in xs])

    def repeat(self, a, c):
        return self.t.repeat_interleave(a, c)

    def cumsum(self, a):
        return self.t.cumsum(a, 0)

    def maximum(self, a, b):
        return self.t.maximum(a, b if self.t.is_tensor(b) else self.t.as_tensor(b, device=self.dev))

    def minimum(self, a, b):
        return self.t.minimum(a, b if self.t.is_tensor(b) else self.t.as_tensor(b, device=self.dev))

    def where(self, c, a, b):
        a = a if self.t.is_tensor(a) else self.t.as_tensor(a, dtype=self.t.int64, device=self.dev)
        b = b if self.t.is_tensor(b) else self.t.as_tensor(b, dtype=self.t.int64, device=self.dev)
        return self.t.where(c, a, b)

    def searchsorted(self, a, v, right=False):
        return self.t.searchsorted(a.contiguous(), v.contiguous(), right=right)

    def argsort_stable(self, a):
        return self.t.sort(a, stable=True)[1]

    def to_host(self, a):
        return a.cpu().numpy() if self.t.is_tensor(a) else np.asarray(a)

    def unique_inverse(self, a):
        return self.t.unique(a, return_inverse=True)


def p2p_mutual_lists(ptr, lo, hi, tlo, thi, n_pairs=None, max_pairs: int = P2P_ITEM_PAIRS, device=None):
    """Lists of the mutual P2P (K1 v2, defmm_p2p_mutual_* / defmm_p2p_gather_*)
    for a single-tree plan.  Target leaf l (Morton order, particles
    [tlo[l], thi[l])) has the merged source runs [lo[e], hi[e]), e in
    [ptr[l], ptr[l+1]).  Each list is clipped to particles >= tlo[l] -- the
    leaf itself first, then the later leaves, whose pairs are evaluated once
    for both directions -- and cut into work items.  Returns the clipped CSR,
    the items (leaf, f0, f1, row/col offsets into the partial buffer), the
    partial size, and the gather passes: lists of tasks (task_leaf, task_out:
    offset into partial, or -1 = the leaf's slice of near) with their
    contributor segments (cbase, xlo, xhi) in fixed order, out[x] = sum_c
    partial[cbase[c] + x]; the last pass writes near for every leaf, earlier
    passes pre-sum the longest lists in chunks.  None if the relation is not
    symmetric (n_pairs check) or a leaf is too large.

    ``device``: None = numpy arrays; a torch device = the segment expansion,
    sorts and gather passes run there and the gather lists are returned as
    device tensors (same values, tests/test_gpu_build.py)."""
    ptr = np.asarray(ptr, np.int64)
    lo, hi = np.asarray(lo, np.int64), np.asarray(hi, np.int64)
    tlo, thi = np.asarray(tlo, np.int64), np.asarray(thi, np.int64)
    nl = tlo.shape[0]
    nt = thi - tlo
    if nl == 0 or nt.max() > P2P_MUTUAL_MAX_LEAF:
        return None
    run_leaf = np.repeat(np.arange(nl), np.diff(ptr))
    clo = np.maximum(lo, tlo[run_leaf])
    keep = hi > clo
    c_leaf, c_lo, c_hi = run_leaf[keep], clo[keep], hi[keep]
    c_ptr = np.searchsorted(c_leaf, np.arange(nl + 1)).astype(np.int64)
    # every list starts with the leaf's own particles
    first = c_ptr[:-1]
    if np.any(np.diff(c_ptr) == 0) or np.any(c_lo[first] != tlo) or np.any(c_hi[first] < thi):
        return None
    c_len = c_hi - c_lo
    cs = np.concatenate([[0], np.cumsum(c_len)])
    ns = cs[c_ptr[1:]] - cs[c_ptr[:-1]]
    if n_pairs is not None and int((nt * (2 * (ns - nt) + nt)).sum()) != int(n_pairs):
        return None  # not a symmetric relation: keep the one-directional kernel
    wi = p2p_work_items(c_ptr, c_len, nt, max_pairs)
    il, f0, f1 = wi["item_leaf"].astype(np.int64), wi["item_f0"], wi["item_f1"]
    ni = il.shape[0]
    size = nt[il] + (f1 - f0)
    off = np.concatenate([[0], np.cumsum(size)])
    row, col = off[:-1], off[:-1] + nt[il]
    # ---- from here on host (numpy) or device (torch): X holds the array operations ----
    X = _NumpyOps if device is None else _TorchOps(device)
    cs_, c_lo_, tlo_, thi_, nt_, il_, f0_, col_ = (X.arr(v) for v in (cs, c_lo, tlo, thi, nt, il, f0, col))
    # column segments: the item's flattened range past the leaf's own particles,
    # cut at run boundaries, then at leaf boundaries
    base_i = X.arr(cs[c_ptr[il]])
    F0 = base_i + X.maximum(f0_, nt_[il_])
    F1 = base_i + X.arr(f1)
    has = F1 > F0
    r0 = X.searchsorted(cs_, F0, right=True) - 1
    r1 = X.searchsorted(cs_, X.maximum(F1 - 1, F0), right=True) - 1
    cnt = X.where(has, r1 - r0 + 1, 0)
    it = X.repeat(X.arange(ni), cnt)
    r = X.repeat(r0, cnt) + (X.arange(int(cnt.sum())) - X.repeat(X.cumsum(cnt) - cnt, cnt))
    sF0 = X.maximum(F0[it], cs_[r])
    sF1 = X.minimum(F1[it], cs_[r + 1])
    g0 = c_lo_[r] + (sF0 - cs_[r])
    g1 = g0 + (sF1 - sF0)
    b0 = X.searchsorted(tlo_, g0, right=True) - 1
    b1 = X.searchsorted(tlo_, g1 - 1, right=True) - 1
    bc = b1 - b0 + 1
    sg = X.repeat(X.arange(it.shape[0]), bc)
    B = X.repeat(b0, bc) + (X.arange(int(bc.sum())) - X.repeat(X.cumsum(bc) - bc, bc))
    xlo = X.maximum(g0[sg], tlo_[B]) - tlo_[B]
    xhi = X.minimum(g1[sg], thi_[B]) - tlo_[B]
    # partial index of particle tlo[B] + x: col + (F - (cs[c_ptr] + f0)), F = sF0 + (g - g0)
    ii = it[sg]
    cb = col_[ii] + (sF0[sg] - (base_i[ii] + f0_[ii])) + (tlo_[B] - g0[sg])
    # contributors per leaf: its own items' rows (item order), then the column segments
    leaf_all = X.cat([il_, B])
    base_all = X.cat([X.arr(row), cb])
    xlo_all = X.cat([X.zeros(ni), xlo])
    xhi_all = X.cat([nt_[il_], xhi])
    o = X.argsort_stable(leaf_all)
    c_leaf_s, c_base, c_xlo, c_xhi = leaf_all[o], base_all[o], xlo_all[o], xhi_all[o]
    # gather passes: a leaf listed by very many items (particles of a large cell next
    # to many small target leaves: cfg3) is summed in chunks of <= P2P_GATHER_CHUNK
    # segments into extra partial rows first, so that no gather task is long
    total = int(off[-1])
    passes = []
    leaves = X.arange(nl + 1)
    while True:
        cptr = X.searchsorted(c_leaf_s, leaves)
        cnt_l = cptr[1:] - cptr[:-1]
        cmax = int(cnt_l.max())
        if cmax <= P2P_GATHER_CHUNK:
            break
        heavy = cnt_l > P2P_GATHER_CHUNK
        hv = heavy[c_leaf_s]
        j = X.arange(c_leaf_s.shape[0]) - cptr[c_leaf_s]
        nchunk = cmax // P2P_GATHER_CHUNK + 2
        key = c_leaf_s[hv] * nchunk + j[hv] // P2P_GATHER_CHUNK
        tk, tinv = X.unique_inverse(key)  # tasks = (leaf, chunk), in (leaf, chunk) order
        t_leaf = tk // nchunk
        t_nt = nt_[t_leaf]
        t_out = total + X.cumsum(t_nt) - t_nt
        total += int(t_nt.sum())
        t_ptr = X.searchsorted(tinv, X.arange(tk.shape[0] + 1))
        passes.append({"task_leaf": t_leaf, "task_out": t_out, "cptr": t_ptr, "cbase": c_base[hv], "cxlo": c_xlo[hv],
                       "cxhi": c_xhi[hv]})
        # the heavy leaves now read their chunk sums (full range) instead
        leaf2 = X.cat([c_leaf_s[~hv], t_leaf])
        base2 = X.cat([c_base[~hv], t_out])
        xlo2 = X.cat([c_xlo[~hv], X.zeros(t_leaf.shape[0])])
        xhi2 = X.cat([c_xhi[~hv], t_nt])
        o2 = X.argsort_stable(leaf2)
        c_leaf_s, c_base, c_xlo, c_xhi = leaf2[o2], base2[o2], xlo2[o2], xhi2[o2]
    passes.append({"task_leaf": X.arange(nl), "task_out": X.full(nl, -1), "cptr": cptr, "cbase": c_base,
                   "cxlo": c_xlo, "cxhi": c_xhi})
    if device is None:  # the documented dtypes of the host lists
        passes = [{k: v.astype(np.int32 if k in ("task_leaf", "cxlo", "cxhi") else np.int64) for k, v in g.items()}
                  for g in passes]
    return {
        "ptr": c_ptr, "lo": c_lo, "hi": c_hi,
        "item_leaf": il.astype(np.int32), "item_f0": f0.astype(np.int64), "item_f1": f1.astype(np.int64),
        "item_row": row.astype(np.int64), "item_col": col.astype(np.int64), "partial_size": total,
        "gather": passes,
    }


def _check_stencils(sym_t, sym_lev, tree, order, tol):
    """fourier.py:179-180: a symbol stencil touching r < tol means the MAC is
    violated -> ValueError (same expression as precompute_symbol)."""
    if sym_t.shape[0] == 0:
        return
    P = 2 * order - 1
    off = np.arange(P)
    off = np.where(off < order, off, off - P) * (1.0 / (order - 1))
    # min over the grid of r is attained per axis at the smallest |t_a + off|
    for lev in np.unique(sym_lev):
        beta = tree.side_at(int(lev))
        t = sym_t[sym_lev == lev].astype(np.float64)
        z = t[:, :, None] + off[None, None, :]
        zmin = np.min(np.abs(z), axis=2)
        r = beta * np.sqrt(zmin[:, 0] ** 2 + zmin[:, 1] ** 2 + zmin[:, 2] ** 2)
        if np.any(r < tol * 4):  # conservative pre-screen, then exact check
            for tv in t[r < tol * 4]:
                zx, zy, zz = np.meshgrid(tv[0] + off, tv[1] + off, tv[2] + off, indexing="ij")
                if np.min(beta * np.sqrt(zx**2 + zy**2 + zz**2)) < tol:
                    raise ValueError("kernel singularity inside the M2L stencil: MAC violated")


def _propagate_marks(tree, own, hf, dt, KD):
    """blank_downward_pass (traversal.py:203-213): per HF level the sorted,
    unique mark keys cell*KD + i, fathers' marks (e > 0) pushed to all sons."""
    out = [np.zeros(0, np.int64) for _ in range(tree.depth + 1)]
    carry = np.zeros(0, np.int64)
    for lev in range(min(hf, tree.depth) + 1):
        parts = own[lev] + [carry]
        mk = np.unique(np.concatenate(parts)) if parts else np.zeros(0, np.int64)
        out[lev] = mk
        e = hf - lev
        if e > 0 and mk.size:
            c = mk // KD
            i = mk % KD
            ns = tree.n_sons[c]
            rep = np.repeat(np.arange(c.shape[0]), ns)
            k = np.arange(rep.shape[0]) - np.repeat(np.cumsum(ns) - ns, ns)
            sons = tree.first_son[c][rep] + k
            carry = sons * KD + dt.fathers[e][i[rep]]
        else:
            carry = np.zeros(0, np.int64)
    return out


def _local_slots(tree, cells, loc, hf, dt, dir_off, KD):
    """Local expansion keys per target cell: M2L targets plus everything the
    L2L pass pushes down (traversal.py:355-391), top-down.

    Returns (l_cell, l_loc sorted by (cell, loc)) and the L2L relation
    (father cell, father loc, son cell, son loc)."""
    lev_of = tree.level[cells]
    keys_all = []
    rel = ([], [], [], [])
    carry = np.zeros(0, np.int64)
    for lev in range(tree.depth + 1):
        sel = lev_of == lev
        k = np.unique(np.concatenate([cells[sel] * (KD + 1) + (loc[sel] + 1), carry]))
        keys_all.append(k)
        c = k // (KD + 1)
        li = k % (KD + 1) - 1
        nonleaf = ~tree.is_leaf[c]
        c, li = c[nonleaf], li[nonleaf]
        ns = tree.n_sons[c]
        rep = np.repeat(np.arange(c.shape[0]), ns)
        kk = np.arange(rep.shape[0]) - np.repeat(np.cumsum(ns) - ns, ns)
        sons = tree.first_son[c][rep] + kk
        fl = li[rep]
        if lev + 1 <= hf:
            e = hf - lev
            sl = dt.fathers[e][fl]
        else:
            sl = np.full(sons.shape[0], -1, np.int64)
        rel[0].append(c[rep])
        rel[1].append(fl)
        rel[2].append(sons)
        rel[3].append(sl)
        carry = sons * (KD + 1) + (sl + 1)
    keys = np.concatenate(keys_all)
    l_cell = keys // (KD + 1)
    l_loc = keys % (KD + 1) - 1
    return l_cell, l_loc, tuple(np.concatenate(r) if r else np.zeros(0, np.int64) for r in rel)
