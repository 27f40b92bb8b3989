"""Device plan + matvec driver (drop-in for helmfmm.traversal's run_fmm*).

``FmmPlan`` = tree + lists + symbols resident in HBM (the reusable
"precompute" the reference recomputes every call); ``FmmPlan.apply`` is the
matvec: P2M -> M2M (per level) -> M2F -> Hadamard M2L + F2L -> L2L (per level)
-> L2P (+ near field, un-permute), with the P2P near field on a second CUDA
stream overlapping the far field (traversal.py:283-418).  Every operator is a
libdefmm_b200 kernel called through the C-ABI; there is no CPU path.
"""

from __future__ import annotations

import os
import time

import numpy as np
import torch

from . import _lib
from .config import FmmConfig, FmmInfo, InteractionEvent, TreeConfig
from .geometry import compute_root_box
from .plan import build_plan, p2p_work_items
from .tree import build_tree

__all__ = ["FmmPlan", "run_fmm", "run_fmm_full"]


def _dev(a, dtype, device):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).to(device)


def _quad_tables():
    """Per (p, V, W): pair-bit mask of the quad, and per in-plane (ia, ib) the
    block pair bit 8a+b, per in-plane offset e its block child offset d."""
    def embed2(i, pp, v):
        return (v << 2) | i if pp == 0 else (((i >> 1) & 1) << 2) | (v << 1) | (i & 1) if pp == 1 else (i << 1) | v

    def d3(a, b):
        return ((((a >> 2) & 1) - ((b >> 2) & 1)) + 1) * 9 + ((((a >> 1) & 1) - ((b >> 1) & 1)) + 1) * 3 + \
            (((a & 1) - (b & 1)) + 1)

    out = {}
    for pp in range(3):
        for v in range(2):
            for w in range(2):
                bit = np.zeros((4, 4), np.int64)
                qm = 0
                d_of_e = np.zeros(9, np.int64)
                for ia in range(4):
                    for ib in range(4):
                        a, b = embed2(ia, pp, v), embed2(ib, pp, w)
                        bit[ia, ib] = 8 * a + b
                        qm |= 1 << (8 * a + b)
                        e = (((ia >> 1) & 1) - ((ib >> 1) & 1) + 1) * 3 + ((ia & 1) - (ib & 1) + 1)
                        d_of_e[e] = d3(a, b)
                out[(pp, v, w)] = (np.uint64(qm), bit, d_of_e, [embed2(ib, pp, w) for ib in range(4)])
    return out


_QUAD_TABLES = None


def _quads(bsrc, btr, bmask, gptr):
    """Quad descriptors (defmm_m2l_quad_*) of every block: split along the axis
    giving the fewest non-empty quads; quads ordered (block, V, W)."""
    global _QUAD_TABLES
    if _QUAD_TABLES is None:
        _QUAD_TABLES = _quad_tables()
    T = _QUAD_TABLES
    nb = bmask.shape[0]
    m = bmask.view(np.uint64)
    cnt = np.stack([sum(((m & T[(pp, v, w)][0]) != 0).astype(np.int64) for v in range(2) for w in range(2))
                    for pp in range(3)]) if nb else np.zeros((3, 0), np.int64)
    best = np.argmin(cnt, axis=0) if nb else np.zeros(0, np.int64)
    parts, keys = [], []
    for pp in range(3):
        bsel = np.nonzero(best == pp)[0]
        if bsel.size == 0:
            continue
        mb = m[bsel]
        for v in range(2):
            for w in range(2):
                qm, bit, d_of_e, b_of = T[(pp, v, w)]
                ne = (mb & qm) != 0
                blk = bsel[ne]
                if blk.size == 0:
                    continue
                mm = mb[ne]
                q = np.full((blk.shape[0], 16), -1, np.int32)
                m16 = np.zeros(blk.shape[0], np.int64)
                for ia in range(4):
                    for ib in range(4):
                        m16 |= ((mm >> np.uint64(bit[ia, ib])) & np.uint64(1)).astype(np.int64) << (4 * ia + ib)
                for ib in range(4):
                    used = (m16 >> ib) & 0x1111
                    q[:, ib] = np.where(used != 0, bsrc[blk, b_of[ib]], -1)
                for e in range(9):
                    du, dw = e // 3 - 1, e % 3 - 1
                    em = 0
                    for ia in range(4):
                        for ib in range(4):
                            if ((ia >> 1) & 1) - ((ib >> 1) & 1) == du and (ia & 1) - (ib & 1) == dw:
                                em |= 1 << (4 * ia + ib)
                    q[:, 4 + e] = np.where((m16 & em) != 0, btr[blk, d_of_e[e]], -1)
                q[:, 13] = m16
                q[:, 14] = 4 * pp + 2 * v + w
                q[:, 15] = 0
                parts.append(q)
                keys.append(blk * 4 + 2 * v + w)
    if not parts:
        return np.zeros((0, 16), np.int32), np.zeros(gptr.shape[0], np.int64)
    q = np.concatenate(parts)
    k = np.concatenate(keys)
    o = np.argsort(k, kind="stable")
    q, k = q[o], k[o]
    qblk = k // 4
    qptr = np.searchsorted(qblk, gptr).astype(np.int64)  # block range per group -> quad range
    return q, qptr


def m2l_tiles(order, row_ptr, ent, n_hat: int, n_trans: int, u_max: int, k_max: int, e_max: int = 1 << 30) -> dict:
    """Host tiling of M2L rows for the tile kernel (defmm_m2l_tiles, native):
    tiles of consecutive rows of ``order`` whose operand union (spectra +
    derived symbols) has <= u_max entries and <= k_max rows."""
    import ctypes as C

    lib = _lib.load()
    ptr = np.ascontiguousarray(row_ptr, np.int64)
    ent = np.ascontiguousarray(ent, np.int32)
    order = np.ascontiguousarray(order, np.int64)
    n = order.shape[0]
    n_ev = int((ptr[order + 1] - ptr[order]).sum()) if n else 0
    tile_ptr = np.zeros(n + 1, np.int64)
    tile_rows = np.zeros(max(n, 1), np.int64)
    op_ptr = np.zeros(n + 1, np.int64)
    ops = np.zeros(max(2 * n_ev, 1), np.int32)
    ev_ptr = np.zeros(n + 1, np.int64)
    ev = np.zeros(max(n_ev, 1), np.uint32)
    counts = np.zeros(5, np.int64)

    def a(x):
        return x.ctypes.data_as(C.c_void_p)

    _lib.check(lib.defmm_m2l_tiles(n, a(order), a(ptr), a(ent), int(n_hat), int(n_trans), int(u_max), int(k_max),
                                   int(e_max), a(tile_ptr), a(tile_rows), a(op_ptr), a(ops), a(ev_ptr), a(ev), a(counts)),
               "defmm_m2l_tiles")
    nt, nr, no, ne = (int(x) for x in counts[:4])
    return {"n_tiles": nt, "tile_ptr": tile_ptr[: nt + 1], "rows": tile_rows[:nr], "op_ptr": op_ptr[: nt + 1],
            "ops": ops[:no], "ev_ptr": ev_ptr[: nr + 1], "ev": ev[:ne], "untiled": int(counts[4])}


def m2l_groups(ids, rows, row_ptr, ent, l_cell, l_dir, level, parent, K: int = 2) -> dict:
    """Sibling-group lists of the group M2L (K7 v8, defmm_m2l_group_*, K = 2 or
    4): the rows ``ids`` (indices into ``rows``, the local slots) grouped by
    (level, key, target parent), consecutive siblings packed K per CTA group;
    each group's events merged per source spectrum into {s, symbol of row k or
    -1 (k < K)} padded to 4 (K = 2) / 8 (K = 4) ints."""
    S = 4 if K <= 3 else 8
    if ids.size == 0:
        return {"n": 0, "K": K, "grp_slot": np.zeros(0, np.int64), "grp_ptr": np.zeros(1, np.int64),
                "ent": np.zeros((0, S), np.int32)}
    slots = rows[ids]
    cell = l_cell[slots]
    key = l_dir[slots].astype(np.int64)
    lev = level[cell].astype(np.int64)
    par = parent[cell].astype(np.int64)
    o = np.lexsort((cell, par, key, lev))
    ids, slots, key, lev, par = ids[o], slots[o], key[o], lev[o], par[o]
    n = ids.shape[0]
    new = np.ones(n, bool)
    new[1:] = (lev[1:] != lev[:-1]) | (key[1:] != key[:-1]) | (par[1:] != par[:-1])
    gstart = np.nonzero(new)[0]
    pos = np.arange(n) - gstart[np.cumsum(new) - 1]
    side = pos % K  # row index within its CTA group
    gid = np.cumsum(side == 0) - 1
    ng = int(gid[-1]) + 1
    grp_slot = np.full((ng, K), -1, np.int64)
    grp_slot[gid, side] = slots
    cnt = row_ptr[ids + 1] - row_ptr[ids]
    rep = np.repeat(np.arange(n), cnt)
    sel = np.repeat(row_ptr[ids] - np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt) + np.arange(int(cnt.sum()))
    ev = ent[sel]
    eg, es, et, eside = gid[rep], ev[:, 0].astype(np.int64), ev[:, 1], side[rep]
    so = np.lexsort((eside, es, eg))
    eg, es, et, eside = eg[so], es[so], et[so], eside[so]
    first = np.ones(eg.shape[0], bool)
    first[1:] = (eg[1:] != eg[:-1]) | (es[1:] != es[:-1])
    eid = np.cumsum(first) - 1
    m = int(eid[-1]) + 1 if eid.size else 0
    out = np.full((m, S), -1, np.int32)
    out[:, K + 1:] = 0
    out[eid, 0] = es
    out[eid, 1 + eside] = et
    grp_ptr = np.searchsorted(eg[first], np.arange(ng + 1)).astype(np.int64)
    return {"n": ng, "K": K, "grp_slot": grp_slot.reshape(-1), "grp_ptr": grp_ptr, "ent": out}


def m2l_pairs(ids, rows, row_ptr, ent, l_cell, l_dir, level, parent) -> dict:
    """K = 2 sibling groups (m2l_groups)."""
    return m2l_groups(ids, rows, row_ptr, ent, l_cell, l_dir, level, parent, 2)


def _rows_to_ids(slots, rows):
    """Local slots -> index into the sorted row-slot list ``rows`` (-1 if absent)."""
    slots = np.asarray(slots)
    j = np.searchsorted(rows, np.maximum(slots, 0))
    j = np.minimum(j, max(rows.shape[0] - 1, 0))
    ok = (slots >= 0) & (rows.shape[0] > 0)
    if rows.shape[0]:
        ok &= rows[j] == slots
    return np.where(ok, j, -1).astype(np.int64)


def _sub_csr(ptr, keep):
    """Rows ``keep`` of a CSR: (row ids, new row pointer, selected entry ids)."""
    ptr = np.asarray(ptr)
    starts = ptr[:-1][keep]
    lens = (ptr[1:] - ptr[:-1])[keep]
    new_ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    sel = np.repeat(starts - new_ptr[:-1], lens) + np.arange(int(new_ptr[-1]))
    return np.nonzero(keep)[0], new_ptr, sel.astype(np.int64)


# ---- per-level M2L kernel policy (host; pure functions, CPU-tested) --------

# M2L kernel per level for each mode: (dense level, sparse level)
M2L_MODE_KINDS = {
    "auto": ("blocked", "rows"), "hybrid_rows": ("blocked", "rows"), "hybrid": ("blocked", "quad"),
    "rows": ("rows", "rows"), "blocked_all": ("blocked", "blocked"), "quad_all": ("quad", "quad"),
    "tiles": ("blocked", "tile"), "tiles_all": ("tile", "tile"), "slice_all": ("slice", "slice"),
    "pairs": ("blocked", "pair"), "pairs_all": ("pair", "pair"), "quartets": ("blocked", "quartet"),
    "quartets_all": ("quartet", "quartet"), "triples_all": ("triple", "triple"),
}
M2L_KERNELS = ("rows", "blocked", "quad", "tile", "slice", "pair", "triple", "quartet")
# events per parent-pair block above which a level counts as dense (blocked kernel)
BLOCKED_MIN_EVENTS_PER_BLOCK = 32.0
# "auto": a complex64 sparse level runs the quad kernel when its quads are this
# full: cfg2 L6 (cube faces, 13.3 events/quad) wins 6% of the M2L; 7-9
# events/quad (cfg2 L4-5, cfg3) and every complex128 level lose
# (profiles/r01_summary_v5.md)
QUAD_MIN_EVENTS_PER_QUAD = 12.0
# ... and only up to this order: at L = 6 the pair kernel beats the quads on
# the same cfg2 level (10.2 vs 11.1 ms, profiles/r01_summary_v7.md).  Since
# the pair kernel keeps three entries in flight it also wins cfg2's planar
# level 6 at L = 4 (2.445 vs 2.48 ms, r01_summary_v8.md): QUAD_MAX_ORDER = 0
# takes the quads out of "auto" (they stay selectable per level)
QUAD_MAX_ORDER = 0
# "auto": other sparse levels with at least this many rows run the pair kernel
# (sibling rows merged per source: cfg2 M2L -9%, cfg3 -10%); small levels
# (cfg1) keep the row kernel (profiles/r01_summary_v7.md)
PAIR_MIN_ROWS = 2048
# rows per sibling group, measured (r01_summary_v8.md): at L <= 4 quartets
# (one entry in flight, 56-register cap) beat pairs (cfg2 M2L c64 2.445 ->
# 2.377 ms, c128 4.71 -> 4.39); from L = 5 their larger spectra make them lose
# (cfg3 9.35 -> 9.63, cfg2 L6 8.64 -> 11.7 ms) and the pair kernel (three
# entries in flight, 56 registers) is best; triples never win
def sibling_kind(dtype: str, order: int) -> str:
    return "quartet" if order <= 4 else "pair"


def block_levels(plan, tt):
    """(level of each parent-pair block, events per block, level of each group,
    blocks per group) of the plan's blocked-M2L lists."""
    g_rows = plan.blk_group_rows
    first = np.where(g_rows >= 0, g_rows, np.iinfo(np.int64).max).min(axis=1)
    glev = tt.level[plan.l_cell[first]] if first.size else np.zeros(0, np.int64)
    nblk = np.diff(plan.blk_group_ptr)
    ev = np.bitwise_count(plan.blk_mask.view(np.uint64)).astype(np.int64) if plan.blk_mask.size else \
        np.zeros(0, np.int64)
    return np.repeat(glev, nblk), ev, glev, nblk


def dense_levels(plan, tt, threshold: float = BLOCKED_MIN_EVENTS_PER_BLOCK) -> set:
    """Levels whose parent-pair blocks hold >= threshold events on average."""
    blev, ev, _, _ = block_levels(plan, tt)
    return {int(lv) for lv in np.unique(blev) if ev[blev == lv].mean() >= threshold}


def quad_fill(plan, tt, levels) -> dict:
    """level -> mean M2L events per in-plane quad of its parent-pair blocks."""
    blev, _, glev, nblk = block_levels(plan, tt)
    out = {}
    for lv in levels:
        gsel = np.nonzero(glev == lv)[0]
        if gsel.size == 0:
            continue
        bsel = np.nonzero(blev == lv)[0]
        bptr = np.concatenate([[0], np.cumsum(nblk[gsel])]).astype(np.int64)
        qd, _ = _quads(plan.blk_src[bsel], plan.blk_trans[bsel], plan.blk_mask[bsel], bptr)
        if qd.shape[0]:
            out[int(lv)] = float(np.bitwise_count(qd[:, 13].astype(np.uint64)).mean())
    return out


def p2p_overlap_policy(level_kinds: dict) -> tuple:
    """(p2p_overlap, far_priority) for a plan's M2L level kinds, measured
    (profiles/r01_summary_v9.md): when every M2L level runs the quartet
    kernel (L <= 4 sparse data: cfg2 c64 / c128), the M2L is bound by the
    L2 -> SM fabric and co-runs well with the FP/XU-bound P2P under a
    high-priority far-field stream (cfg2 c64 3.38 -> 3.28 ms, c128 6.73 ->
    6.68); elsewhere (pairs, rows, blocked levels: cfg3, cfg5, cfg2 L6) the
    P2P beside the upward pass is 0.6-2% faster."""
    if level_kinds and all(k == "quartet" for k in level_kinds.values()):
        return "m2l", True
    return "upward", False


def m2l_level_kinds(mode: str, dtype: str, levels, dense, fill=None, override=None, env: str = "",
                    rows_per_level=None, order: int = 4) -> dict:
    """level -> M2L kernel: the mode's (dense, sparse) choice; in "auto" a
    complex64 sparse level with quad fill >= QUAD_MIN_EVENTS_PER_QUAD runs
    quads, another sparse level with >= PAIR_MIN_ROWS rows the pair kernel;
    then the per-level overrides (dict, or "4:quad,6:rows")."""
    if mode not in M2L_MODE_KINDS:
        raise ValueError(f"unknown M2L mode {mode!r}")
    kd, ks = M2L_MODE_KINDS[mode]
    kinds = {int(lv): (kd if int(lv) in dense else ks) for lv in levels}
    if mode == "auto":
        for lv in list(kinds):
            if kinds[lv] != "rows":
                continue
            if dtype == "c64" and order <= QUAD_MAX_ORDER and (fill or {}).get(lv, 0.0) >= QUAD_MIN_EVENTS_PER_QUAD:
                kinds[lv] = "quad"
            elif (rows_per_level or {}).get(lv, 0) >= PAIR_MIN_ROWS:
                kinds[lv] = sibling_kind(dtype, order)
    over = dict(override or {})
    for tok in filter(None, env.split(",")):
        lv, k = tok.split(":")
        over[int(lv)] = k
    for lv, k in over.items():
        if k not in M2L_KERNELS:
            raise ValueError(f"unknown M2L kernel {k!r} for level {lv}")
        if int(lv) in kinds:
            kinds[int(lv)] = k
    return kinds


class FmmPlan:
    """Reusable device plan for one particle geometry (targets is sources, or
    a target/source pair sharing one root box, traversal.py:449-461)."""

    def __init__(self, targets, sources=None, config: FmmConfig = FmmConfig(), device="cuda",
                 keep_events: bool = False, charges=None, reuse: "FmmPlan | None" = None,
                 shard=None, allreduce=None, m2l: str = "auto", m2l_levels: dict | None = None):
        """``reuse``: share the host tree + lists of an existing plan built for
        the same geometry and (order, ncrit, eta, kappa) -- e.g. to run the same
        lists at another storage precision.

        ``shard``: (rank, world) or a ``parallel.Shard`` -- this process then
        computes only its Morton chunk (parallel.py); ``allreduce(tensor)``
        must sum a device tensor over the ranks in place (NCCL
        ``torch.distributed.all_reduce``), it completes the multipoles."""
        if not torch.cuda.is_available():
            raise RuntimeError("the defmm B200 path needs a CUDA device (no CPU fallback)")
        _lib.load()
        self.config = config
        self.device = torch.device(device)
        self._shard_arg = shard
        self.allreduce = allreduce
        # "hybrid" (per-level choice), "blocked_all" (every level blocked) or
        # "rows" (no level blocked) -- decides the lists built for the hybrid path
        self.m2l_variant_default = m2l
        self.m2l_level_override = m2l_levels
        if reuse is not None:
            rc = reuse.config
            if (rc.order, rc.ncrit, rc.eta, rc.kappa, rc.hf_switch, rc.hard_depth_cap) != (
                    config.order, config.ncrit, config.eta, config.kappa, config.hf_switch, config.hard_depth_cap):
                raise ValueError("reuse= needs a plan built with the same list parameters")
            self.same = reuse.same
            self.tt, self.st, self.tp, self.sp = reuse.tt, reuse.st, reuse.tp, reuse.sp
            self.plan = reuse.plan
            self.timings = dict(reuse.timings)
            t2 = time.perf_counter()
            self._make_shard()
            self._upload()
            self._symbols()
            torch.cuda.synchronize(self.device)
            self.timings["precompute"] = time.perf_counter() - t2
            if charges is not None:
                self.set_charges(charges)
            return
        t0 = time.perf_counter()
        tree_cfg = TreeConfig(ncrit=config.ncrit, hard_depth_cap=config.hard_depth_cap)
        same = sources is None or targets is sources
        src = targets if same else sources
        n_src = np.atleast_2d(np.asarray(src)).shape[0]
        qs = np.zeros(n_src, complex) if charges is None else charges
        if same:
            st, sp = build_tree(src, qs, tree_cfg)
            tt, tp = st, sp
        else:
            both = np.vstack([np.atleast_2d(targets), np.atleast_2d(sources)])
            box = compute_root_box(both)
            st, sp = build_tree(sources, qs, tree_cfg, root_box=box)
            tt, tp = build_tree(targets, np.zeros(np.atleast_2d(targets).shape[0]), tree_cfg, root_box=box)
        self.same = same
        self.tt, self.st, self.tp, self.sp = tt, st, tp, sp
        t1 = time.perf_counter()
        self.plan = build_plan(tt, st, config.order, config.kappa, config.eta, config.hf_switch,
                               keep_events=keep_events)
        t2 = time.perf_counter()
        self.timings = {"tree": t1 - t0, "blank": t2 - t1}
        self._make_shard()
        self._upload()
        self._symbols()
        torch.cuda.synchronize(self.device)
        self.timings["precompute"] = time.perf_counter() - t2
        if charges is not None:
            self.set_charges(charges)

    # ------------------------------------------------------------------
    def _upload(self):
        p, d = self.plan, self.device
        self.cdtype = torch.complex128 if self.config.dtype == "c128" else torch.complex64
        L = self.config.order
        i64, i32, f64 = torch.int64, torch.int32, torch.float64
        tt, st = self.tt, self.st
        self.L, self.L3, self.P3 = L, L**3, (2 * L - 1) ** 3
        # HBM stride of one spectrum (even-padded for complex64 vector loads)
        self.SS = int(_lib.load().defmm_spectrum_stride(L, int(self.config.dtype == "c64")))
        # particles (sorted order), SoA
        self.s_xyz = [_dev(self.sp.positions[:, k], f64, d) for k in range(3)]
        self.t_xyz = self.s_xyz if self.same else [_dev(self.tp.positions[:, k], f64, d) for k in range(3)]
        self.s_perm = _dev(self.sp.original_index, i64, d)
        self.t_perm = self.s_perm if self.same else _dev(self.tp.original_index, i64, d)
        self.n_src = self.sp.n
        self.n_tgt = self.tp.n

        def geom(tree):
            return dict(start=_dev(tree.start, i64, d), stop=_dev(tree.stop, i64, d),
                        alpha=_dev(tree.alpha, f64, d), level=_dev(tree.level, i32, d),
                        beta=_dev(tree.level_beta, f64, d))

        self.sg = geom(st)
        self.tg = self.sg if self.same else geom(tt)
        self.dirs = _dev(p.dirs if p.dirs.size else np.zeros((1, 3)), f64, d)
        h = self._host_lists()
        # upward lists
        self.p2m_cell = _dev(p.m_cell[h["p2m_idx"]], i32, d)
        self.p2m_dir = _dev(p.m_dir[h["p2m_idx"]], i32, d)
        self.p2m_slot = _dev(h["p2m_idx"], i64, d)
        self.m2m = []
        for lev, slots, son_slot in h["m2m"]:
            self.m2m.append((float(st.side_at(lev + 1)), _dev(slots, i64, d), _dev(p.m_dir[slots], i32, d),
                             _dev(son_slot, i64, d), int(slots.shape[0])))
        self.hat_slot = _dev(h["hat_slot"], i64, d)
        self.n_hat = int(h["hat_slot"].shape[0])
        # M2L, all rows (target-major CSR): reference variants "derived" / "canonical"
        self.row_slot = _dev(h["rows"], i64, d)
        self.row_ptr = _dev(h["row_ptr"], i64, d)
        self._ent_canon = None  # per-event (src, sym, rid) of the canonical variant, on first use
        self.row_entries = _dev(h["ent"].reshape(-1), i32, d)
        # M2L product path ("hybrid"): sparse levels -> row kernel, dense -> blocked
        self.rk_rows = _dev(h["rk_rows"], i64, d)
        self.rk_ptr = _dev(h["rk_ptr"], i64, d)
        self.rk_ent = _dev(h["rk_ent"].reshape(-1), i32, d)
        self.bk_rows = _dev(h["bk_rows"], i64, d)
        self.n_groups = int(h["grp_rows"].shape[0])
        self.grp_ptr = _dev(h["grp_ptr"], i64, d)
        self.grp_rows = _dev(h["grp_rows"].reshape(-1), i64, d)
        self.blk_src = _dev(h["blk_src"].reshape(-1), i32, d)
        self.blk_trans = _dev(h["blk_trans"].reshape(-1), i32, d)
        self.blk_mask = _dev(h["blk_mask"], i64, d)
        self.blk_kind = _dev(h["blk_kind"], torch.int8, d)
        self.n_qgroups = int(h["qd_rows"].shape[0])
        self.qd_ptr = _dev(h["qd_ptr"], i64, d)
        self.qd_rows = _dev(h["qd_rows"].reshape(-1), i64, d)
        self.quads = _dev(h["quads"].reshape(-1), i32, d)
        self.sib_groups = []  # (K, n, slots, ptr, entries) of the pair / quartet kernels
        for kind in ("pair", "triple", "quartet"):
            gr = h[kind]
            if gr["n"]:
                self.sib_groups.append((gr["K"], int(gr["n"]), _dev(gr["grp_slot"], i64, d),
                                        _dev(gr["grp_ptr"], i64, d), _dev(gr["ent"].reshape(-1), i32, d)))
        self.n_pairs = sum(x[1] for x in self.sib_groups)
        tl = h["tl"]
        self.n_tiles = int(tl["n_tiles"]) if tl is not None else 0
        if self.n_tiles:
            self.tl_ptr = _dev(tl["tile_ptr"], i64, d)
            self.tl_op_ptr = _dev(tl["op_ptr"], i64, d)
            self.tl_ops = _dev(tl["ops"], i32, d)
            self.tl_ev_ptr = _dev(tl["ev_ptr"], i64, d)
            self.tl_ev = _dev(tl["ev"].view(np.int32), i32, d)
            self.tl_base = int(tl["lhat_base"])
        sl = h["slice"]
        self.n_slice_batch = int(sl["n_batch"])
        self.sl_batch = _dev(sl["batch"].reshape(-1), i32, d)
        self.sl_seg = _dev(sl["seg"], i64, d)
        self.sl_ent = _dev(sl["ent"].reshape(-1), i32, d)
        self.sl_ngs, self.sl_row_base = int(sl["ngs"]), int(sl["row_base"])
        # downward
        self.l2l = []
        for lev, outs, octant, ptr, src, sdir in h["l2l"]:
            self.l2l.append((float(tt.side_at(lev)), _dev(outs, i64, d), _dev(octant, torch.int8, d),
                             _dev(ptr, i64, d), _dev(src, i64, d), _dev(sdir, i32, d), int(outs.shape[0])))
        lv = h["leaves"]
        self.n_leaves = int(lv.sum())
        self.leaf_cell = _dev(p.leaf_cells[lv], i32, d)
        self.leaf_lo = _dev(p.leaf_slot_lo[lv], i64, d)
        self.leaf_hi = _dev(p.leaf_slot_hi[lv], i64, d)
        self.slot_dir = _dev(p.l_dir, i32, d)
        self.tgt_lo = _dev(tt.start[p.leaf_cells[lv]], i64, d)
        self.tgt_hi = _dev(tt.stop[p.leaf_cells[lv]], i64, d)
        self.p2p_ptr = _dev(h["p2p_ptr"], i64, d)
        p2p_lo, p2p_hi = p.p2p_lo[h["p2p_sel"]], p.p2p_hi[h["p2p_sel"]]
        self.p2p_lo = _dev(p2p_lo, i64, d)
        self.p2p_hi = _dev(p2p_hi, i64, d)
        wi = p2p_work_items(h["p2p_ptr"], p2p_hi - p2p_lo, tt.stop[p.leaf_cells[lv]] - tt.start[p.leaf_cells[lv]])
        self.n_items = int(wi["item_leaf"].shape[0])
        self.p2p_items = [_dev(wi[k], torch.int32 if k == "item_leaf" else i64, d)
                          for k in ("item_leaf", "item_f0", "item_f1", "item_out")]
        self.n_split = int(wi["split_leaf"].shape[0])
        self.p2p_split = [_dev(wi["split_leaf"], i32, d), _dev(wi["split_base"], i64, d), _dev(wi["split_n"], i32, d)]
        self._partial_size = wi["partial_size"]
        # workspaces (storage precision per FmmConfig.dtype)
        cd = self.cdtype
        self.mult = torch.empty((max(p.n_mult, 1), self.L3), dtype=cd, device=d)
        self.hat = torch.empty((max(self.n_hat, 1), self.SS), dtype=cd, device=d)
        self.local = torch.empty((max(p.n_local, 1), self.L3), dtype=cd, device=d)
        self.lhat = torch.empty((max(int(self.bk_rows.shape[0]), 1), self.SS), dtype=cd, device=d)
        self.near = torch.empty(self.n_tgt, dtype=cd, device=d)
        # late near field: with the P2P still running beside the M2L, the L2P
        # starts from a zero near field and add_near folds the P2P in after
        # the join (DEFMM_LATE_NEAR=1; measured slower on cfg2: 3.304 vs 3.282 ms)
        self.late_near = os.environ.get("DEFMM_LATE_NEAR", "0") == "1"
        self.zero_near = torch.zeros(self.n_tgt, dtype=cd, device=d)
        self.p2p_partial = torch.empty(max(self._partial_size, 1), dtype=cd, device=d)
        self.q = torch.zeros(self.n_src, dtype=cd, device=d)
        self.out = torch.empty(self.n_tgt, dtype=cd, device=d)
        lo, hi = torch.cuda.Stream.priority_range()  # (lowest, highest) priority numbers
        self.side_stream = torch.cuda.Stream(device=d, priority=lo)
        self.far_stream = torch.cuda.Stream(device=d, priority=hi)
        self.m2l_variant = "hybrid"
        # "upward": P2P concurrent with P2M/M2M/M2F, joined before the M2L (clean
        # M2L stage timer); "m2l": P2P launched after the upward pass on the
        # low-priority side stream, concurrent with the M2L; "full": P2P spans
        # the upward pass and the M2L (optionally on a persistent grid of
        # p2p_grid CTAs).  far_priority: far field on the high-priority stream.
        self.p2p_overlap, self.far_priority = p2p_overlap_policy(getattr(self, "level_kinds", {}))
        # sibling-group M2L fed by bulk copies into a shared-memory ring (K7 v9)
        # instead of per-thread global loads; DEFMM_GROUP_TMA=0/1 overrides
        self.group_tma = os.environ.get("DEFMM_GROUP_TMA", "0") == "1"
        # sibling groups claimed per SM from contiguous chunks (K7 v10): CTAs
        # sharing an SM work on neighbouring groups -> L1 reuse of spectra and
        # symbols; DEFMM_GROUP_SMQ=0/1 overrides
        self.group_smq = os.environ.get("DEFMM_GROUP_SMQ", "0") == "1"
        self.smq_chunk = int(os.environ.get("DEFMM_GROUP_SMQ_CHUNK", "8"))
        self.n_sm = torch.cuda.get_device_properties(d).multi_processor_count
        self.qcnt = torch.zeros(self.n_sm, dtype=torch.int32, device=d)
        self.p2p_grid = 0
        # c64 near-field coordinates: hi/lo float pairs where the order's
        # accuracy bar needs them (defmm_b200.h, K1)
        self.p2p_hilo = self.L >= 6

    def _make_shard(self):
        from .parallel import Shard, make_shard

        sa = self._shard_arg
        if sa is None or isinstance(sa, Shard):
            self.shard = sa
        else:
            rank, world = sa
            self.shard = make_shard(self.plan, self.tt, self.st, int(rank), int(world)) if int(world) > 1 else None
        self.halo = None
        if self.shard is not None and self.shard.world > 1 and self.allreduce is None:
            # halo exchange over torch.distributed (NCCL between GPUs)
            import torch.distributed as dist

            from .parallel import make_halo

            if not (dist.is_available() and dist.is_initialized()):
                raise ValueError("a sharded plan needs torch.distributed initialised (or allreduce=)")
            self.halo = make_halo(self.plan, self.tt, self.shard.cuts, self.shard.rank, self.shard.world)

    # events per parent-pair block above which a level's M2L runs blocked
    BLOCKED_MIN_EVENTS_PER_BLOCK = BLOCKED_MIN_EVENTS_PER_BLOCK

    def _host_lists(self) -> dict:
        """Per-level M2L kernel choice: levels whose parent-pair blocks are
        dense (volume-like, >= BLOCKED_MIN_EVENTS_PER_BLOCK events per block)
        run the blocked kernel (K7 v3, operand reuse in registers), sparse
        (surface-like) levels the row kernel by default (their blocks would be
        mostly predicated-off pairs) -- profiles/r01_summary_v3.md, v4.md.
        lhat rows: grouped (blocked + quad) rows, then slice rows, then tile
        rows (one F2L launch over all of them)."""
        h = self._host_lists_all()
        p, tt = self.plan, self.tt
        rows = h["rows"]
        rlev = tt.level[p.l_cell[rows]] if rows.size else np.zeros(0, np.int64)
        # density per level from the full plan (identical on every rank)
        dense = dense_levels(p, tt, self.BLOCKED_MIN_EVENTS_PER_BLOCK)
        levels = np.unique(rlev)
        fill = None
        if self.m2l_variant_default == "auto" and self.config.dtype == "c64" and self.L <= QUAD_MAX_ORDER:
            fill = quad_fill(p, tt, [lv for lv in levels if int(lv) not in dense])
        self.quad_fill = fill
        # rows per level from the full plan (identical on every rank)
        flev = tt.level[p.l_cell[p.m2l_row_slot]] if p.m2l_row_slot.size else np.zeros(0, np.int64)
        rpl = {int(lv): int(c) for lv, c in zip(*np.unique(flev, return_counts=True))}
        kinds = m2l_level_kinds(self.m2l_variant_default, self.config.dtype, levels, dense, fill,
                                self.m2l_level_override, os.environ.get("DEFMM_M2L_LEVELS", ""), rpl, self.L)
        self.level_kinds = kinds
        rkind = np.array([kinds[int(lv)] for lv in rlev], dtype=object) if rows.size else np.zeros(0, object)
        z = np.zeros(0, np.int64)

        def pick(*ks):
            return np.isin(rkind, list(ks)) if rows.size else np.zeros(0, bool)

        # row kernel
        is_rows = pick("rows")
        # tiles (rows whose own operands exceed a tile fall back to the row kernel)
        h["tl"] = None
        is_tile = pick("tile")
        if is_tile.any():
            t_ids = np.nonzero(is_tile)[0]
            slot = rows[t_ids]
            order = t_ids[np.lexsort((p.l_cell[slot], p.l_dir[slot], rlev[t_ids]))]
            tl = self._tile_lists(order, h)
            h["tl"] = tl
            is_rows = is_rows.copy()
            is_rows[np.setdiff1d(t_ids, tl["rows"])] = True
        _, rptr, rsel = _sub_csr(h["row_ptr"], is_rows)
        h["rk_rows"], h["rk_ptr"], h["rk_ent"] = rows[is_rows], rptr, h["ent"][rsel]
        # sibling pairs (K7 v8)
        h["pair"] = m2l_groups(np.nonzero(pick("pair"))[0], rows, h["row_ptr"], h["ent"], p.l_cell, p.l_dir,
                               tt.level, tt.parent, 2)
        h["triple"] = m2l_groups(np.nonzero(pick("triple"))[0], rows, h["row_ptr"], h["ent"], p.l_cell, p.l_dir,
                                 tt.level, tt.parent, 3)
        h["quartet"] = m2l_groups(np.nonzero(pick("quartet"))[0], rows, h["row_ptr"], h["ent"], p.l_cell, p.l_dir,
                                  tt.level, tt.parent, 4)
        # grouped rows (blocked + quad)
        is_grp = pick("blocked", "quad")
        grp_rows = rows[is_grp]
        # slice rows
        is_slice = pick("slice")
        n_grp = int(grp_rows.shape[0])
        if is_slice.any():
            _, sptr, ssel = _sub_csr(h["row_ptr"], is_slice)
            h["slice"] = self._slice_lists(sptr, h["ent"][ssel], rlev[is_slice], n_grp)
        else:
            h["slice"] = self._slice_lists(np.zeros(1, np.int64), np.zeros((0, 2), np.int32), z, 0)
        # lhat rows: grouped, slice, tile
        parts = [grp_rows, rows[is_slice]]
        if h["tl"] is not None:
            h["tl"]["lhat_base"] = n_grp + int(is_slice.sum())
            parts.append(rows[h["tl"]["rows"]])
        h["bk_rows"] = np.concatenate(parts) if parts else z
        # groups of grouped levels, rows renumbered into lhat
        gr = h["grp_rows"]
        gr_slots = np.where(gr >= 0, rows[np.maximum(gr, 0)] if rows.size else -1, -1)
        gid = _rows_to_ids(gr_slots, grp_rows)
        gkeep = np.any(gid >= 0, axis=1)
        _, gptr, bsel = _sub_csr(h["grp_ptr"], gkeep)
        grows = gid[gkeep]
        bsrc, btr, bmask, bkind = h["blk_src"][bsel], h["blk_trans"][bsel], h["blk_mask"][bsel], h["blk_kind"][bsel]
        # groups of quad levels -> quad kernel, the others -> blocked kernel
        first = np.where(grows >= 0, grows, np.iinfo(np.int64).max).min(axis=1) if grows.size else z
        glev = tt.level[p.l_cell[grp_rows[first]]] if grows.size else z
        gq = np.array([kinds[int(lv)] == "quad" for lv in glev], bool) if grows.size else np.zeros(0, bool)
        if gq.any():
            _, dptr, dsel = _sub_csr(gptr, ~gq)
            _, qgptr, qsel = _sub_csr(gptr, gq)
            quads, qptr = _quads(bsrc[qsel], btr[qsel], bmask[qsel], qgptr)
            h["qd_ptr"], h["qd_rows"], h["quads"] = qptr, grows[gq], quads
            gptr, grows = dptr, grows[~gq]
            bsrc, btr, bmask, bkind = bsrc[dsel], btr[dsel], bmask[dsel], bkind[dsel]
        else:
            h["qd_ptr"], h["qd_rows"], h["quads"] = np.zeros(1, np.int64), np.zeros((0, 8), np.int64), \
                np.zeros((0, 16), np.int32)
        h["grp_ptr"], h["grp_rows"] = gptr, grows
        h["blk_src"], h["blk_trans"], h["blk_mask"], h["blk_kind"] = bsrc, btr, bmask, bkind
        self.dense_levels = sorted(lv for lv, k in kinds.items() if k == "blocked")
        return h

    # tile kernel (K7 v6): operand slices of 128 B (c64: 16 x 8 B, c128:
    # 8 x 16 B), double-buffered: 2 x 352 x 128 B + 4096 events ~ 107 KB of
    # shared memory -> 2 CTAs per SM
    TILE_U_MAX = 352
    TILE_E_MAX = 4096

    def _tile_lists(self, order, h) -> dict:
        """Greedy operand-union tiles over the rows ``order`` (indices into
        h["rows"], sorted (level, key, Morton target)): defmm_m2l_tiles."""
        return m2l_tiles(order, h["row_ptr"], h["ent"], int(h["hat_slot"].shape[0]),
                         int(self.plan.trans_canon.shape[0]), int(self.TILE_U_MAX),
                         16 if self.config.dtype == "c64" else 32, int(self.TILE_E_MAX))

    # rows per slice-kernel batch: enough events per batch to amortise the
    # shared-memory symbol loads (G symbols per group), one row per warp at least
    SLICE_MIN_BATCH_ROWS = 16
    SLICE_MAX_BATCH_ROWS = 512

    def _slice_lists(self, rptr, ent, rlev, lhat_base) -> dict:
        """Lists of the slice M2L (K7 v4, defmm_m2l_slice_*): per row, events
        sorted by canonical-symbol group (G per group, the level's canonical
        symbols are contiguous in the symbol table); entries {spectrum,
        (canonical-in-group << 6) | rotation}; seg[r, g] = first event of group
        g; batches of rows of one level {row0, row1, first symbol, count}."""
        p = self.plan
        n = int(rlev.shape[0])
        G = int(_lib.load().defmm_slice_group(int(self.config.dtype == "c64")))
        if n == 0:
            return {"n_batch": 0, "batch": np.zeros((0, 4), np.int32), "seg": np.zeros(1, np.int64),
                    "ent": np.zeros((0, 2), np.int32), "ngs": 1, "row_base": lhat_base}
        cnt = np.diff(rptr)
        lev_lo = np.searchsorted(p.sym_level, rlev, side="left")
        lev_nc = np.searchsorted(p.sym_level, rlev, side="right") - lev_lo
        ngs = int(max(1, (-(-lev_nc // G)).max()))
        tid = ent[:, 1].astype(np.int64)
        clocal = p.trans_canon[tid].astype(np.int64) - np.repeat(lev_lo, cnt)
        grp = clocal // G
        meta = ((clocal % G) << 6) | p.trans_rid[tid].astype(np.int64)
        key = np.repeat(np.arange(n, dtype=np.int64), cnt) * ngs + grp
        if ngs > 1:
            order = np.argsort(key, kind="stable")
            key, meta, src = key[order], meta[order], ent[order, 0]
        else:
            src = ent[:, 0]
        sent = np.empty((key.shape[0], 2), np.int32)
        sent[:, 0] = src
        sent[:, 1] = meta
        probe = (np.arange(n, dtype=np.int64)[:, None] * ngs + np.arange(ngs + 1)[None, :]).reshape(-1)
        seg = np.searchsorted(key, probe, side="left").astype(np.int64)
        # batches: rows of one level (contiguous: rows are slot-sorted, level-major)
        batches = []
        brk = np.nonzero(np.diff(rlev))[0] + 1
        for a, b in zip(np.concatenate([[0], brk]), np.concatenate([brk, [n]])):
            ev_row = max(float(cnt[a:b].mean()), 1.0)
            ngl = -(-int(lev_nc[a]) // G)
            br = int(np.clip(16 * G * ngl / ev_row, self.SLICE_MIN_BATCH_ROWS, self.SLICE_MAX_BATCH_ROWS))
            br = -(-br // 16) * 16
            for r0 in range(int(a), int(b), br):
                batches.append((lhat_base + r0, lhat_base + min(int(b), r0 + br), int(lev_lo[a]), int(lev_nc[a])))
        return {"n_batch": len(batches), "batch": np.asarray(batches, np.int32).reshape(-1, 4), "seg": seg,
                "ent": sent, "ngs": ngs, "row_base": lhat_base}

    def _host_lists_all(self) -> dict:
        """The plan's lists, restricted to this rank's chunk when sharded
        (parallel.py); spectra are renumbered compactly."""
        p, sh = self.plan, self.shard
        n_ent = p.m2l_rows_entries.shape[0]
        h = {
            "p2m_idx": p.p2m_idx,
            "m2m": [(lev, sl, ss) for lev, sl, ss in p.m2m_levels],
            "hat_slot": p.hat_slot,
            "rows": p.m2l_row_slot,
            "row_ptr": p.m2l_row_ptr,
            "ent": p.m2l_rows_entries,
            "l2l": list(p.l2l_levels),
            "leaves": np.ones(p.leaf_cells.shape[0], bool),
            "p2p_ptr": p.p2p_ptr,
            "p2p_sel": np.arange(p.p2p_lo.shape[0]),
        }
        # blocked M2L: group rows as indices into h["rows"] (lhat rows)
        blk = {"grp_ptr": p.blk_group_ptr, "grp_rows": p.blk_group_rows, "blk_src": p.blk_src,
               "blk_trans": p.blk_trans, "blk_mask": p.blk_mask, "blk_kind": p.blk_kind}
        if sh is None:
            h.update(blk)
            h["grp_rows"] = _rows_to_ids(blk["grp_rows"], h["rows"])
            return h
        h["p2m_idx"] = sh.p2m_idx
        h["m2m"] = [(lev, sl[k], ss[k]) for (lev, sl, ss), k in zip(p.m2m_levels, sh.m2m_keep) if k.any()]
        rows, ptr, sel = _sub_csr(p.m2l_row_ptr, sh.row_keep)
        h["rows"], h["row_ptr"] = p.m2l_row_slot[sh.row_keep], ptr
        hat_ids = np.nonzero(sh.hat_keep)[0]
        remap = np.full(p.n_hat, -1, np.int64)
        remap[hat_ids] = np.arange(hat_ids.shape[0])
        ent = p.m2l_rows_entries[sel].copy()
        ent[:, 0] = remap[ent[:, 0]]
        h["ent"], h["hat_slot"] = ent, p.hat_slot[hat_ids]
        gr = _rows_to_ids(p.blk_group_rows, h["rows"])  # -1 for rows of other ranks
        gkeep = np.any(gr >= 0, axis=1)
        _, gptr, bsel = _sub_csr(p.blk_group_ptr, gkeep)
        bsrc = p.blk_src[bsel]
        h.update({"grp_ptr": gptr, "grp_rows": gr[gkeep], "blk_trans": p.blk_trans[bsel],
                  "blk_mask": p.blk_mask[bsel], "blk_kind": p.blk_kind[bsel],
                  "blk_src": np.where(bsrc >= 0, remap[np.maximum(bsrc, 0)], -1).astype(np.int32)})
        l2l = []
        for (lev, outs, octant, lptr, src, sdir), k in zip(p.l2l_levels, sh.l2l_keep):
            if not k.any():
                continue
            _, nptr, lsel = _sub_csr(lptr, k)
            l2l.append((lev, outs[k], octant[k], nptr, src[lsel], sdir[lsel]))
        h["l2l"] = l2l
        h["leaves"] = sh.leaf_keep
        _, h["p2p_ptr"], h["p2p_sel"] = _sub_csr(p.p2p_ptr, sh.leaf_keep)
        return h

    def _symbols(self):
        p = self.plan
        self.sym = torch.empty((max(p.n_sym, 1), self.SS), dtype=self.cdtype, device=self.device)
        st = torch.cuda.current_stream(self.device).cuda_stream
        if p.n_sym:
            tv = _dev(p.sym_tvec.reshape(-1), torch.int32, self.device)
            beta = _dev(p.sym_beta, torch.float64, self.device)
            _lib.call(self._op("symbols"), self.L, p.n_sym, tv, beta, float(p.kappa), self.sym, st)
        n_tr = int(p.trans_canon.shape[0])
        self.sym_derived = torch.empty((max(n_tr, 1), self.SS), dtype=self.cdtype, device=self.device)
        if n_tr:
            _lib.call(self._op("expand_symbols"), self.L, n_tr, _dev(p.trans_canon, torch.int32, self.device),
                      _dev(p.trans_rid, torch.int8, self.device), self.sym, self.sym_derived, st)

    def _op(self, name: str) -> str:
        return f"defmm_{name}_{self.config.dtype}"

    # ------------------------------------------------------------------
    def set_charges(self, charges):
        """Load charges (caller order) into the sorted device buffer."""
        q = torch.as_tensor(np.asarray(charges, dtype=complex)) if not torch.is_tensor(charges) else charges
        q = q.to(device=self.device, dtype=self.cdtype)
        torch.index_select(q, 0, self.s_perm, out=self.q)  # one gather into the sorted buffer

    def set_charges_sorted(self, q_sorted):
        self.q.copy_(q_sorted)

    def apply(self, out=None, stage_events=None):
        """One matvec with the charges currently loaded; returns potentials in
        the caller's target order (device tensor; when sharded only this
        rank's targets are non-zero).  ``stage_events`` (list) receives
        (name, start_event, end_event) for the stage timers.  After
        ``capture_graph()`` a plain ``apply()`` replays the captured graph."""
        if (out is None and stage_events is None and getattr(self, "graph", None) is not None
                and not getattr(self, "_capturing", False)):
            self.graph.replay()
            return self.out
        if self.far_priority and self.shard is None:
            # far field on a HIGH-priority stream, P2P on the low-priority side
            # stream: the block scheduler then dispatches the latency-bound
            # far-field chain first and the P2P fills the remaining SM slots
            cur = torch.cuda.current_stream(self.device)
            fs = self.far_stream
            fs.wait_stream(cur)
            with torch.cuda.stream(fs):
                res = self._apply(out, stage_events)
            cur.wait_stream(fs)
            return res
        return self._apply(out, stage_events)

    def _apply(self, out=None, stage_events=None):
        self.apply_upward(stage_events)
        if self.shard is not None:
            if self.allreduce is not None:
                # M2M is linear: summing the partial multipoles over the ranks
                # completes every multipole
                self.allreduce(self.mult)
            else:
                from .parallel import halo_exchange

                halo_exchange(self.mult, self._halo_dev())
        return self.apply_rest(out, stage_events)

    def _halo_dev(self):
        if getattr(self, "_halo_t", None) is None:
            h = self.halo
            dev = self.mult.device
            idx = lambda a: torch.as_tensor(a, dtype=torch.int64, device=dev)  # noqa: E731
            self._halo_t = (idx(h.span), idx(h.send), list(h.send_counts), idx(h.recv), list(h.recv_counts),
                            bool(h.active))
        return self._halo_t

    def _near_field(self, stage_events):
        """P2P on the side stream (FP-pipe bound), concurrent with the far field."""
        p = self.plan
        stream = torch.cuda.current_stream(self.device)
        side = self.side_stream
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            if stage_events is not None:
                e0 = torch.cuda.Event(enable_timing=True)
                e0.record(side)
            _lib.call(self._op("p2p"), self.n_items, *self.p2p_items, self.tgt_lo, self.tgt_hi, self.p2p_ptr,
                      self.p2p_lo, self.p2p_hi, *self.t_xyz, *self.s_xyz, self.q, float(p.kappa), float(p.tol),
                      self.near, self.p2p_partial, self.n_split, *self.p2p_split, int(self.p2p_grid),
                      int(self.p2p_hilo), side.cuda_stream)
            if stage_events is not None:
                e1 = torch.cuda.Event(enable_timing=True)
                e1.record(side)
                stage_events.append(("p2p", e0, e1))

    def apply_upward(self, stage_events=None):
        """Phase 1: (P2P launch on the side stream,) P2M and M2M -- partial
        multipoles of the active cells when sharded."""
        L, kappa, sg = self.L, float(self.plan.kappa), self.sg
        stream = torch.cuda.current_stream(self.device)
        sh = stream.cuda_stream
        if self.p2p_overlap in ("upward", "full"):
            self._near_field(stage_events)
        if stage_events is not None:
            self._ev_a = torch.cuda.Event(enable_timing=True)
            self._ev_a.record(stream)
        if self.shard is not None:
            self.mult.zero_()  # multipoles of other ranks' cells stay 0 -> partial sums
        _lib.call(self._op("p2m"), L, self.p2m_slot.shape[0], self.p2m_cell, self.p2m_dir, self.p2m_slot,
                  sg["start"], sg["stop"], sg["alpha"], sg["level"], sg["beta"], self.dirs, *self.s_xyz, self.q,
                  kappa, self.mult, sh)
        if self.p2p_overlap == "m2m":  # P2P queued behind the P2M (far field keeps priority)
            self._near_field(stage_events)
        for son_beta, slots, mdir, son_slot, n in self.m2m:
            _lib.call(self._op("m2m"), L, n, slots, mdir, son_slot, son_beta, self.dirs, kappa, self.mult, sh)

    def apply_rest(self, out=None, stage_events=None):
        """Phase 2 (multipoles complete): M2F, M2L + F2L, L2L, L2P (+ near, un-permute)."""
        L, kappa, tg = self.L, float(self.plan.kappa), self.tg
        stream = torch.cuda.current_stream(self.device)
        sh = stream.cuda_stream
        out = self.out if out is None else out
        ev = (lambda: torch.cuda.Event(enable_timing=True)) if stage_events is not None else None
        _lib.call(self._op("m2f"), L, self.n_hat, self.hat_slot, self.mult, self.hat, sh)
        if self.p2p_overlap == "m2l":
            self._near_field(stage_events)
        elif self.p2p_overlap == "upward":
            stream.wait_stream(self.side_stream)  # M2L runs alone (clean roofline timing)
        # "full": P2P spans the upward pass and the M2L, joined before L2P
        if stage_events is not None:
            b = ev()
            b.record(stream)
            stage_events.append(("upward", self._ev_a, b))
        # M2L (+ fused F2L) into the local slots
        self.local.zero_()
        if self.m2l_variant == "hybrid":
            _lib.call(self._op("m2l_rows"), L, self.rk_rows.shape[0], self.rk_rows, self.rk_ptr, self.rk_ent,
                      self.hat, self.sym_derived, self.local, sh)
            for K, ng, gslot, gptr, gent in self.sib_groups:
                if self.group_smq:
                    _lib.call(self._op("m2l_group_smq"), L, K, ng, gslot, gptr, gent, self.hat, self.sym_derived,
                              self.local, self.n_sm, self.smq_chunk, self.qcnt, sh)
                else:
                    _lib.call(self._op("m2l_group_tma" if self.group_tma else "m2l_group"), L, K, ng, gslot, gptr,
                              gent, self.hat, self.sym_derived, self.local, sh)
            _lib.call(self._op("m2l_blocked"), L, self.n_groups, self.grp_ptr, self.grp_rows, self.blk_src,
                      self.blk_trans, self.blk_mask, self.blk_kind, self.hat, self.sym_derived, self.lhat, sh)
            _lib.call(self._op("m2l_quad"), L, self.n_qgroups, self.qd_ptr, self.qd_rows, self.quads, self.hat,
                      self.sym_derived, self.lhat, sh)
            if self.n_tiles:
                _lib.call(self._op("m2l_tile"), L, self.n_tiles, self.tl_ptr, self.tl_op_ptr, self.tl_ops,
                          self.tl_ev_ptr, self.tl_ev, self.tl_base, int(self.TILE_U_MAX),
                          int(self.TILE_E_MAX), self.hat,
                          self.sym_derived, self.lhat, sh)
            _lib.call(self._op("m2l_slice"), L, self.n_slice_batch, self.sl_batch, self.sl_row_base, self.sl_seg,
                      self.sl_ngs, self.sl_ent, self.hat, self.sym, self.lhat, sh)
            _lib.call(self._op("f2l_rows"), L, self.bk_rows.shape[0], self.bk_rows, self.lhat, self.local, sh)
        elif self.m2l_variant == "derived":
            _lib.call(self._op("m2l_rows"), L, self.row_slot.shape[0], self.row_slot, self.row_ptr,
                      self.row_entries, self.hat, self.sym_derived, self.local, sh)
        elif self.m2l_variant == "canonical" and self.config.dtype == "c128":
            if self._ent_canon is None:
                ent = self.row_entries.view(-1, 2)
                tid = ent[:, 1].long()
                self._ent_canon = (ent[:, 0].contiguous(),
                                   torch.as_tensor(self.plan.trans_canon, device=ent.device)[tid].to(torch.int32),
                                   torch.as_tensor(self.plan.trans_rid, device=ent.device)[tid].to(torch.int8))
            e_src, e_sym, e_rid = self._ent_canon
            _lib.call("defmm_m2l_canon_c128", L, self.row_slot.shape[0], self.row_slot, self.row_ptr, e_src,
                      e_sym, e_rid, self.hat, self.sym, self.local, sh)
        else:
            raise ValueError(f"unknown M2L variant {self.m2l_variant!r} for dtype {self.config.dtype}")
        if stage_events is not None:
            c = ev()
            c.record(stream)
            stage_events.append(("m2l", b, c))
        # downward: L2L per level top-down, then L2P + near + un-permute
        for son_beta, outs, octant, ptr, src, sdir, n in self.l2l:
            _lib.call(self._op("l2l"), L, n, outs, octant, ptr, src, sdir, son_beta, self.dirs, kappa,
                      self.local, sh)
        late = self.late_near and self.shard is None and self.p2p_overlap != "upward"
        if not late:
            stream.wait_stream(self.side_stream)
        if self.shard is not None:
            out.zero_()  # this rank writes only its own targets
        _lib.call(self._op("l2p"), L, self.n_leaves, self.leaf_cell, self.leaf_lo, self.leaf_hi, self.slot_dir,
                  tg["start"], tg["stop"], tg["alpha"], tg["level"], tg["beta"], self.dirs, *self.t_xyz, kappa,
                  self.local, self.zero_near if late else self.near, self.t_perm, out, sh)
        if late:  # P2P joined after the L2P: out[perm] += near
            stream.wait_stream(self.side_stream)
            _lib.call(self._op("add_near"), self.n_tgt, self.t_perm, self.near, out, sh)
        if stage_events is not None:
            e = ev()
            e.record(stream)
            stage_events.append(("downward", c, e))
        return out

    def capture_graph(self):
        """Record one matvec (all launches on both streams, the memsets) into a
        CUDA graph; ``replay()`` then re-executes it with whatever charges are
        in ``self.q``.  Not for sharded plans (the NCCL all-reduce stays eager)."""
        if self.shard is not None:
            raise ValueError("CUDA-graph replay is for single-GPU plans")
        torch.cuda.synchronize(self.device)
        self._capturing = True
        try:
            s = torch.cuda.Stream(device=self.device)
            s.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(s):
                self.apply()  # warm-up on the capture stream
            torch.cuda.current_stream(self.device).wait_stream(s)
            torch.cuda.synchronize(self.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.apply()
            torch.cuda.synchronize(self.device)
        finally:
            self._capturing = False
        self.graph = g
        return self.graph

    def replay(self):
        """Matvec via the captured CUDA graph; returns ``self.out``."""
        self.graph.replay()
        return self.out

    def m2l_kernels(self) -> list:
        """Names of the M2L-stage kernels one matvec launches (with their levels)."""
        R = "float" if self.config.dtype == "c64" else "double"
        if self.m2l_variant != "hybrid":
            return [f"m2l_rows_kernel<{R}, {self.L}> (all levels, {self.m2l_variant})"]
        kinds = getattr(self, "level_kinds", {})

        def lv(k):
            return sorted(l for l, x in kinds.items() if x == k)

        out = []
        gk = "m2l_group_tma_kernel" if self.group_tma and not self.group_smq else "m2l_group_kernel"
        for n, name, k in ((self.rk_rows.shape[0], "m2l_rows_kernel", "rows"),
                           (sum(x[1] for x in self.sib_groups if x[0] == 2), f"{gk}<2>", "pair"),
                           (sum(x[1] for x in self.sib_groups if x[0] == 3), f"{gk}<3>", "triple"),
                           (sum(x[1] for x in self.sib_groups if x[0] == 4), f"{gk}<4>", "quartet"),
                           (self.n_groups, "m2l_blocked_kernel", "blocked"),
                           (self.n_qgroups, "m2l_quad_kernel", "quad"), (self.n_tiles, "m2l_tile_kernel", "tile"),
                           (self.n_slice_batch, "m2l_slice_kernel", "slice"), (self.bk_rows.shape[0], "f2l_rows_kernel", None)):
            if n:
                out.append(f"{name}<{R}, {self.L}>" + (f" (levels {lv(k)})" if k is not None else ""))
        return out

    @property
    def launches_per_apply(self) -> int:
        """Kernels of one matvec: p2p (+ split reduce), p2m, m2m per level, m2f,
        the M2L kernels with work, l2l per level, l2p."""
        if self.m2l_variant == "hybrid":
            m2l = len(self.sib_groups) + sum(int(n > 0) for n in (self.rk_rows.shape[0], self.n_groups, self.n_qgroups, self.n_tiles,
                                           self.n_slice_batch, self.bk_rows.shape[0]))
        else:
            m2l = 1
        late = self.late_near and self.shard is None and self.p2p_overlap != "upward"
        return 4 + (1 if self.n_split else 0) + len(self.m2m) + len(self.l2l) + m2l + int(late)

    def events(self):
        """InteractionEvent list (traversal.py:80-85) with Cell views."""
        p = self.plan
        if p.m2l_events is None:
            raise RuntimeError("plan was built without keep_events=True")
        tl = {c.index: c for lv in self.tt.levels for c in lv}
        sl = tl if self.same else {c.index: c for lv in self.st.levels for c in lv}
        out = []
        mt, ms, md = p.m2l_events
        for t, s, dd in zip(mt.tolist(), ms.tolist(), md.tolist()):
            key = None
            if dd >= 0:
                e = p.hf_max - int(self.tt.level[t])
                key = (e, dd - int(p.dir_off[e]))
            out.append(InteractionEvent("M2L", tl[t], sl[s], key))
        pt, ps = p.p2p_events
        for t, s in zip(pt.tolist(), ps.tolist()):
            out.append(InteractionEvent("P2P", tl[t], sl[s]))
        return out


def spectral_layout(L: int):
    """(forder, slice_start): storage position -> natural frequency index
    f0 P^2 + f1 P + f2 of every device spectrum, and the orbit-closed slices
    (defmm_spectral_layout, host call)."""
    import ctypes as C

    P3 = (2 * L - 1) ** 3
    forder = np.empty(P3, np.int32)
    starts = np.empty(P3 + 1, np.int32)
    ns = C.c_int32(0)
    _lib.check(_lib.load().defmm_spectral_layout(int(L), forder.ctypes.data, starts.ctypes.data, C.byref(ns)),
               "defmm_spectral_layout")
    return forder, starts[: ns.value + 1].copy()


def run_fmm_full(targets, sources, charges, config: FmmConfig = FmmConfig(), events: list | None = None):
    """traversal.py:432-506 on the B200: (potentials, FmmInfo)."""
    info = FmmInfo()
    t_start = time.perf_counter()
    same = targets is sources
    plan = FmmPlan(targets, None if same else sources, config, keep_events=events is not None,
                   charges=np.asarray(charges, dtype=complex))
    info.hf_max_level = plan.plan.hf_max
    stages = []
    out = plan.apply(stage_events=stages)
    pot = out.cpu().numpy().astype(np.complex128)  # fresh complex128 array (tree.py:224-228)
    for k, v in plan.timings.items():
        info.timings[k] = v
    el = {name: a.elapsed_time(b) / 1e3 for name, a, b in stages}
    info.timings["upward"] = el["upward"]
    info.timings["m2l_p2p"] = el["m2l"] + el["p2p"]
    info.timings["downward"] = el["downward"]
    info.timings["total"] = time.perf_counter() - t_start
    info.counts = {k: v for k, v in plan.plan.counts.items() if k != "translations"}
    if events is not None:
        events.extend(plan.events())
    return pot, info


def run_fmm(targets, sources, charges, config: FmmConfig = FmmConfig()):
    """traversal.py:509-516."""
    return run_fmm_full(targets, sources, charges, config)[0]
