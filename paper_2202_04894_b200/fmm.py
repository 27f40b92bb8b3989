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
from .plan import build_plan, p2p_mutual_lists, p2p_work_items, planar_kind
from .tree import build_tree

__all__ = ["FmmPlan", "run_fmm", "run_fmm_full"]


def _on_device(fn):
    """Run a plan method with the plan's device current: the C-ABI launches
    go to the current device (and ensure_twiddles fills that device's tables)."""
    import functools

    @functools.wraps(fn)
    def wrapped(self, *a, **k):
        with torch.cuda.device(self.device):
            return fn(self, *a, **k)

    return wrapped


def _dev(a, dtype, device):
    if torch.is_tensor(a):  # a list built on the device already
        return a.to(device=device, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).to(device)


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


def m2l_groups_dev(ids, rows, row_ptr, ent_dev, l_cell, l_dir, level, parent, K: int, device) -> dict:
    """m2l_groups with the per-event work (gather, sort by (group, source, row),
    merge per source) on the device; the row-level grouping (a few 1e4..1e6
    rows) stays on the host.  ``ent_dev``: the (n, 2) int32 event table on the
    device.  Returns device tensors; equal to m2l_groups bit for bit
    (tests/test_gpu_build.py)."""
    S = 4 if K <= 3 else 8
    i64, i32 = torch.int64, torch.int32
    if ids.size == 0:
        return {"n": 0, "K": K, "grp_slot": torch.zeros(0, dtype=i64, device=device),
                "grp_ptr": torch.zeros(1, dtype=i64, device=device),
                "ent": torch.zeros((0, S), dtype=i32, device=device)}
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
    side = pos % K
    gid = np.cumsum(side == 0) - 1
    ng = int(gid[-1]) + 1
    grp_slot = np.full((ng, K), -1, np.int64)
    grp_slot[gid, side] = slots
    cnt = row_ptr[ids + 1] - row_ptr[ids]
    with torch.cuda.device(device):
        up = lambda a: torch.as_tensor(np.ascontiguousarray(a, np.int64)).to(device)  # noqa: E731
        cnt_d, start_d, gid_d, side_d = up(cnt), up(row_ptr[ids]), up(gid), up(side)
        tot = int(cnt.sum())
        rep = torch.repeat_interleave(torch.arange(n, device=device), cnt_d, output_size=tot)
        sel = (start_d - (torch.cumsum(cnt_d, 0) - cnt_d))[rep] + torch.arange(tot, device=device)
        ev = ent_dev[sel]
        es, et = ev[:, 0].to(i64), ev[:, 1]
        eg, eside = gid_d[rep], side_d[rep]
        nh = int(es.max().item()) + 1 if tot else 1
        comp = (eg * nh + es) * K + eside  # distinct per event
        comp, so = torch.sort(comp)
        et, eside = et[so], eside[so]
        gs = comp // K  # (group, source)
        first = torch.ones(tot, dtype=torch.bool, device=device)
        first[1:] = gs[1:] != gs[:-1]
        eid = torch.cumsum(first, 0) - 1
        m = int(eid[-1].item()) + 1 if tot else 0
        out = torch.full((m, S), -1, dtype=i32, device=device)
        out[:, K + 1:] = 0
        out[eid, 0] = (gs % nh).to(i32)
        out[eid, 1 + eside] = et
        grp_ptr = torch.searchsorted((gs[first] // nh).contiguous(), torch.arange(ng + 1, device=device))
        return {"n": ng, "K": K, "grp_slot": up(grp_slot.reshape(-1)), "grp_ptr": grp_ptr, "ent": out}


def m2l_pairs(ids, rows, row_ptr, ent, l_cell, l_dir, level, parent) -> dict:
    """K = 2 sibling groups (m2l_groups)."""
    return m2l_groups(ids, rows, row_ptr, ent, l_cell, l_dir, level, parent, 2)


# the mutual P2P (K1 v2) pays from ~1e8 near-field pairs on (cfg1, 1.4e7 pairs: 0.19 ms one-directional
# against 0.28 ms mutual + gather; cfg2, 3.8e8: 0.47 -> 0.43 ms; cfg5, 2.7e9, c128: 9.85 -> 7.2 ms)
P2P_MUTUAL_MIN_PAIRS = 100_000_000

STAGE_NW, STAGE_K = 8, 4  # warp units per CTA, rows per warp unit (STG_NW, STG_K of the kernel)
STAGE_SLOTS = 48  # symbol slices per shared-memory stage (ns_cap)
STAGE_DEPTH = 3  # shared-memory ring stages
STAGE_ENT_PAD = 64  # readable entries past the end (STG_ENT_PAD)


def _stage_units(ids, rows, l_cell, l_dir, level, parent):
    """Row-level grouping of the staged M2L: rows sorted by (level, key, parent,
    cell); warp units of <= STAGE_K sibling rows; STAGE_NW consecutive units of
    one (level, key) per CTA.  Returns (ids, slots, par, k of each row, unit of
    each row, warp of each unit, CTA of each unit, CTA count, cta_rows)."""
    K, NW = STAGE_K, STAGE_NW
    i32 = np.int32
    slots = rows[ids]
    cell = l_cell[slots]
    key = l_dir[slots].astype(np.int64)
    lev = level[cell].astype(np.int64)
    par = parent[cell].astype(np.int64)
    o = np.lexsort((cell, par, key, lev))
    ids, slots, key, lev, par = ids[o], slots[o], key[o], lev[o], par[o]
    n = ids.shape[0]
    newp = np.ones(n, bool)
    newp[1:] = (lev[1:] != lev[:-1]) | (key[1:] != key[:-1]) | (par[1:] != par[:-1])
    pstart = np.nonzero(newp)[0]
    pos = np.arange(n) - pstart[np.cumsum(newp) - 1]
    kk = pos % K  # row index within its warp unit
    wu = np.cumsum(kk == 0) - 1  # warp unit of each row
    first = np.nonzero(kk == 0)[0]
    nwu = first.shape[0]
    w_lev, w_key = lev[first], key[first]
    newc = np.ones(nwu, bool)  # new (level, key) chunk of warp units
    newc[1:] = (w_lev[1:] != w_lev[:-1]) | (w_key[1:] != w_key[:-1])
    cstart = np.nonzero(newc)[0]
    posw = np.arange(nwu) - cstart[np.cumsum(newc) - 1]
    ww = posw % NW  # warp of each warp unit
    cta_of_wu = np.cumsum(ww == 0) - 1
    ncta = int(cta_of_wu[-1]) + 1
    cta_rows = np.full((ncta * NW, K), -1, i32)
    cta_rows[cta_of_wu[wu] * NW + ww[wu], kk] = np.arange(n)  # lhat row = position in the sorted order
    return ids, slots, par, kk, wu, ww, cta_of_wu, ncta, cta_rows


def m2l_stage_lists(ids, rows, row_ptr, ent, l_cell, l_dir, level, parent, coords, hat_coords,
                    ns_cap: int = STAGE_SLOTS) -> dict:
    """Lists of the staged M2L (K7 v13, defmm_m2l_stage_*).  The rows ``ids``
    (indices into ``rows``) are grouped by (level, key, target parent) into warp
    units of <= STAGE_K sibling rows; STAGE_NW consecutive warp units of one
    (level, key) form a CTA.  An event (row, source s) belongs to the class
    u = coords(s) - 2 coords(parent): within a CTA the symbols of a class are
    shared by every warp unit.  Classes are packed in order into stages of <=
    ns_cap distinct symbols; per (warp unit, class) one entry {source spectrum,
    4 bytes: stage slot of row k's symbol or 0xff}.  ``hat_coords``: (n_hat, 3)
    grid coordinates of each spectrum's source cell."""
    K, NW = STAGE_K, STAGE_NW
    i32 = np.int32
    if ids.size == 0:
        return {"n": 0, "ns_cap": ns_cap, "row_slot": np.zeros(0, np.int64), "cta_stage": np.zeros(1, i32),
                "cta_went": np.zeros(0, i32), "stage_slot_ptr": np.zeros(1, i32), "slot_sym": np.zeros(0, i32),
                "stage_wend": np.zeros(0, i32), "ent": np.zeros((STAGE_ENT_PAD, 2), i32),
                "cta_rows": np.zeros(0, i32)}
    ids, slots, par, kk, wu, ww, cta_of_wu, ncta, cta_rows = _stage_units(ids, rows, l_cell, l_dir, level, parent)
    n = ids.shape[0]
    # events
    cnt = row_ptr[ids + 1] - row_ptr[ids]
    rep = np.repeat(np.arange(n), cnt)
    sel = np.repeat(row_ptr[ids] - np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt) + np.arange(int(cnt.sum()))
    e_src = ent[sel, 0].astype(np.int64)
    e_tr = ent[sel, 1].astype(np.int64)
    e_wu = wu[rep]
    e_cw = cta_of_wu[e_wu] * NW + ww[e_wu]  # (CTA, warp)
    e_cta = cta_of_wu[e_wu]
    u = hat_coords[e_src] - 2 * coords[par[rep]]
    off = int(np.abs(u).max()) + 1 if u.size else 1
    nbit = max(int(2 * off + 1).bit_length(), 1)
    # classes = distinct (CTA, u) in Morton order of u: classes that follow
    # each other then read neighbouring translations, i.e. largely the same
    # symbols (sym(o - u) = sym(o' - u') whenever o - u = o' - u')
    ucode = np.zeros(u.shape[0], np.int64)
    for b in range(nbit):
        for a in range(3):
            ucode |= (((u[:, a] + off) >> b) & 1) << (3 * b + 2 - a)
    span3 = np.int64(1) << (3 * nbit)
    ckey = e_cta * span3 + ucode
    cuniq, e_cls = np.unique(ckey, return_inverse=True)
    e_cls = e_cls.reshape(-1)
    ncls = cuniq.shape[0]
    cls_cta = cuniq // span3
    n_tr = int(e_tr.max()) + 1
    su = np.unique(e_cls * n_tr + e_tr)  # (class, symbol) pairs
    su_cls, su_tr = su // n_tr, su % n_tr
    nsym_cls = np.bincount(su_cls, minlength=ncls)
    if nsym_cls.max() > 8:
        raise RuntimeError("staged M2L: a class with more than 8 symbols")
    # stages: greedy in class order, a stage holds <= ns_cap DISTINCT symbols
    # (symbols shared between its classes are staged once)
    cls_ptr = np.concatenate([[0], np.cumsum(nsym_cls)]).astype(np.int64)
    st_rel = np.empty(ncls, np.int64)
    cls_cta = np.ascontiguousarray(cls_cta, np.int64)
    su_tr = np.ascontiguousarray(su_tr, np.int64)
    _lib.check(_lib.load().defmm_stage_pack(ncls, cls_cta.ctypes.data, cls_ptr.ctypes.data, su_tr.ctypes.data,
                                            n_tr, int(ns_cap), st_rel.ctypes.data), "defmm_stage_pack")
    nst_cta = np.zeros(ncta, np.int64)
    np.maximum.at(nst_cta, cls_cta, st_rel + 1)
    cta_stage = np.concatenate([[0], np.cumsum(nst_cta)])
    cls_stage = cta_stage[cls_cta] + st_rel
    nstage = int(cta_stage[-1])
    # slots: distinct (stage, symbol)
    e_stage = cls_stage[e_cls]
    skey = e_stage * n_tr + e_tr
    suniq, e_slotg = np.unique(skey, return_inverse=True)
    e_slotg = e_slotg.reshape(-1)
    slot_stage = suniq // n_tr
    slot_sym = (suniq % n_tr).astype(i32)
    stage_slot_ptr = np.searchsorted(slot_stage, np.arange(nstage + 1))
    if np.diff(stage_slot_ptr).max() > ns_cap:
        raise RuntimeError("staged M2L: stage over capacity")
    e_slot = e_slotg - stage_slot_ptr[e_stage]
    # entries = distinct (CTA, warp, class), ordered by (CTA, warp, stage, class)
    ekey = e_cw * ncls + e_cls  # class ids increase with the stage inside a CTA
    euniq, e_ent = np.unique(ekey, return_inverse=True)
    e_ent = e_ent.reshape(-1)
    nent = euniq.shape[0]
    ent_cw = euniq // ncls
    ent_stage = cls_stage[euniq % ncls]
    # slot bytes: ns_cap (the zero slot) where row k has no event in the class; each (entry, k)
    # holds at most one event, so the bytes add up exactly (values < 2^32)
    ent32 = np.zeros((nent + STAGE_ENT_PAD, 2), i32)
    ent32[e_ent, 0] = e_src
    none = int(ns_cap) * 0x01010101  # every byte = ns_cap: the ring's zero slot
    y = np.bincount(e_ent, weights=((e_slot - int(ns_cap)) << (8 * kk[rep])).astype(np.float64), minlength=nent)
    ent32[:nent, 1] = (y.astype(np.int64) + none).astype(np.uint32).view(i32)
    ent32[nent:, 1] = np.uint32(none).view(i32)
    cta_went = np.searchsorted(ent_cw, np.arange(ncta * NW)).astype(i32)
    # end of warp w's entries of stage s: entries with (cw, stage) <= (cta(s) NW + w, s)
    st_cta = np.repeat(np.arange(ncta), nst_cta)
    q_cw = (st_cta[:, None] * NW + np.arange(NW)[None, :]).reshape(-1)
    q_st = np.repeat(np.arange(nstage), NW)
    ent_k2 = ent_cw * (nstage + 1) + ent_stage
    stage_wend = np.searchsorted(ent_k2, q_cw * (nstage + 1) + q_st, side="right").astype(i32)
    # stored per CTA as [warp][stage]: a warp reads its stage ends contiguously
    q_w = np.tile(np.arange(NW), nstage)
    pos = cta_stage[st_cta[q_st]] * NW + q_w * nst_cta[st_cta[q_st]] + (q_st - cta_stage[st_cta[q_st]])
    wend_t = np.empty_like(stage_wend)
    wend_t[pos] = stage_wend
    stage_wend = wend_t
    return {"n": ncta, "ns_cap": ns_cap, "row_slot": slots.astype(np.int64), "cta_stage": cta_stage.astype(i32),
            "cta_went": cta_went, "stage_slot_ptr": stage_slot_ptr.astype(i32), "slot_sym": slot_sym,
            "stage_wend": stage_wend, "ent": ent32,
            "cta_rows": cta_rows.reshape(-1)}


def m2l_stage_lists_dev(ids, rows, row_ptr, ent_dev, l_cell, l_dir, level, parent, coords, hat_coords,
                        ns_cap: int, device) -> dict:
    """m2l_stage_lists with the per-event work on the device (sorts, uniques,
    scatters on torch tensors; the greedy stage packer stays the native host
    routine over the (class, symbol) pairs).  Same lists bit for bit
    (tests/test_gpu_build.py); returns device tensors except row_slot."""
    K, NW = STAGE_K, STAGE_NW
    i32, i64 = torch.int32, torch.int64
    if ids.size == 0:
        h = m2l_stage_lists(ids, rows, row_ptr, np.zeros((0, 2), np.int32), l_cell, l_dir, level, parent, coords,
                            hat_coords, ns_cap)
        return {k: (torch.as_tensor(v).to(device) if isinstance(v, np.ndarray) and k != "row_slot" else v)
                for k, v in h.items()}
    ids, slots, par, kk, wu, ww, cta_of_wu, ncta, cta_rows = _stage_units(ids, rows, l_cell, l_dir, level, parent)
    n = ids.shape[0]
    cnt = row_ptr[ids + 1] - row_ptr[ids]
    with torch.cuda.device(device):
        up = lambda a: torch.as_tensor(np.ascontiguousarray(a, np.int64)).to(device)  # noqa: E731
        cnt_d, start_d = up(cnt), up(row_ptr[ids])
        tot = int(cnt.sum())
        rep = torch.repeat_interleave(torch.arange(n, device=device), cnt_d, output_size=tot)
        sel = (start_d - (torch.cumsum(cnt_d, 0) - cnt_d))[rep] + torch.arange(tot, device=device)
        ev = ent_dev[sel]
        e_src, e_tr = ev[:, 0].to(i64), ev[:, 1].to(i64)
        e_wu = up(wu)[rep]
        cw_d, ww_d = up(cta_of_wu), up(ww)
        e_cta = cw_d[e_wu]
        e_cw = e_cta * NW + ww_d[e_wu]
        u = up(hat_coords)[e_src] - 2 * up(coords[par])[rep]
        off = int(u.abs().max().item()) + 1
        nbit = max(int(2 * off + 1).bit_length(), 1)
        ucode = torch.zeros(tot, dtype=i64, device=device)
        for b in range(nbit):
            for a in range(3):
                ucode |= (((u[:, a] + off) >> b) & 1) << (3 * b + 2 - a)
        span3 = 1 << (3 * nbit)
        cuniq, e_cls = torch.unique(e_cta * span3 + ucode, return_inverse=True)
        ncls = int(cuniq.numel())
        cls_cta = cuniq // span3
        n_tr = int(e_tr.max().item()) + 1
        su = torch.unique(e_cls * n_tr + e_tr)
        su_cls_h = (su // n_tr).cpu().numpy()
        su_tr_h = np.ascontiguousarray((su % n_tr).cpu().numpy(), np.int64)
        nsym_cls = np.bincount(su_cls_h, minlength=ncls)
        if nsym_cls.max() > 8:
            raise RuntimeError("staged M2L: a class with more than 8 symbols")
        cls_ptr = np.concatenate([[0], np.cumsum(nsym_cls)]).astype(np.int64)
        st_rel_h = np.empty(ncls, np.int64)
        cls_cta_h = np.ascontiguousarray(cls_cta.cpu().numpy(), np.int64)
        _lib.check(_lib.load().defmm_stage_pack(ncls, cls_cta_h.ctypes.data, cls_ptr.ctypes.data,
                                                su_tr_h.ctypes.data, n_tr, int(ns_cap), st_rel_h.ctypes.data),
                   "defmm_stage_pack")
        nst_cta_h = np.zeros(ncta, np.int64)
        np.maximum.at(nst_cta_h, cls_cta_h, st_rel_h + 1)
        cta_stage_h = np.concatenate([[0], np.cumsum(nst_cta_h)])
        nstage = int(cta_stage_h[-1])
        cta_stage, nst_cta = up(cta_stage_h), up(nst_cta_h)
        cls_stage = cta_stage[cls_cta] + up(st_rel_h)
        e_stage = cls_stage[e_cls]
        suniq, e_slotg = torch.unique(e_stage * n_tr + e_tr, return_inverse=True)
        slot_stage = suniq // n_tr
        stage_slot_ptr = torch.searchsorted(slot_stage.contiguous(), torch.arange(nstage + 1, device=device))
        if int((stage_slot_ptr[1:] - stage_slot_ptr[:-1]).max().item()) > ns_cap:
            raise RuntimeError("staged M2L: stage over capacity")
        e_slot = e_slotg - stage_slot_ptr[e_stage]
        euniq, e_ent = torch.unique(e_cw * ncls + e_cls, return_inverse=True)
        nent = int(euniq.numel())
        ent_cw = euniq // ncls
        ent_stage = cls_stage[euniq % ncls]
        none = int(ns_cap) * 0x01010101
        y = torch.full((nent + STAGE_ENT_PAD,), none, dtype=i64, device=device)
        y.index_add_(0, e_ent, (e_slot - int(ns_cap)) << (8 * up(kk)[rep]))
        ent32 = torch.zeros((nent + STAGE_ENT_PAD, 2), dtype=i32, device=device)
        ent32[e_ent, 0] = e_src.to(i32)
        ent32[:, 1] = torch.where(y >= (1 << 31), y - (1 << 32), y).to(i32)  # the uint32 bit pattern
        cta_went = torch.searchsorted(ent_cw.contiguous(), torch.arange(ncta * NW, device=device)).to(i32)
        st_cta = torch.repeat_interleave(torch.arange(ncta, device=device), nst_cta, output_size=nstage)
        q_cw = (st_cta[:, None] * NW + torch.arange(NW, device=device)[None, :]).reshape(-1)
        q_st = torch.repeat_interleave(torch.arange(nstage, device=device), NW)
        wend = torch.searchsorted((ent_cw * (nstage + 1) + ent_stage).contiguous(), q_cw * (nstage + 1) + q_st,
                                  right=True).to(i32)
        q_w = torch.arange(NW, device=device).repeat(nstage)
        qc = st_cta[q_st]
        pos = cta_stage[qc] * NW + q_w * nst_cta[qc] + (q_st - cta_stage[qc])
        stage_wend = torch.empty_like(wend)
        stage_wend[pos] = wend
        return {"n": ncta, "ns_cap": ns_cap, "row_slot": slots.astype(np.int64), "cta_stage": cta_stage.to(i32),
                "cta_went": cta_went, "stage_slot_ptr": stage_slot_ptr.to(i32), "slot_sym": (suniq % n_tr).to(i32),
                "stage_wend": stage_wend, "ent": ent32,
                "cta_rows": torch.as_tensor(cta_rows.reshape(-1)).to(device)}


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
    "auto": ("blocked", "rows"), "hybrid_rows": ("blocked", "rows"),
    "rows": ("rows", "rows"), "blocked_all": ("blocked", "blocked"),
    "pairs": ("blocked", "pair"), "pairs_all": ("pair", "pair"), "quartets": ("blocked", "quartet"),
    "quartets_all": ("quartet", "quartet"), "triples_all": ("triple", "triple"),
    "staged": ("blocked", "staged"), "staged_all": ("staged", "staged"),
}
M2L_KERNELS = ("rows", "blocked", "pair", "triple", "quartet", "staged")
# events per parent-pair block above which a level counts as dense (blocked kernel)
BLOCKED_MIN_EVENTS_PER_BLOCK = 32.0
# "auto": other sparse levels with at least this many rows run the pair kernel
# (sibling rows merged per source: cfg2 M2L -9%, cfg3 -10%); small levels
# (cfg1) keep the row kernel (profiles/r01_summary_v7.md)
PAIR_MIN_ROWS = 2048
# rows per sibling group, measured (r01_summary_v8.md): at L <= 4 quartets
# (one entry in flight, 56-register cap) beat pairs (cfg2 M2L c64 2.445 ->
# 2.377 ms, c128 4.71 -> 4.39); from L = 5 their larger spectra make them lose
# (cfg3 9.35 -> 9.63, cfg2 L6 8.64 -> 11.7 ms) and the pair kernel (three
# entries in flight, 56 registers) is best; triples never win
# Sparse-level kernel by storage type and order, measured (M2L stage alone, ms; profiles/r02/
# summary_v3.md): staged (K7 v13, symbols staged once per 8 warp units in shared memory) against
# the sibling groups --
#   complex128: L=4 cfg2 3.79 vs 4.36 (quartets), L=5 cfg3 14.15 vs 14.55 (pairs), L=6 cfg2
#               15.0 vs 19.3 (pairs) -> staged up to L = 6 (larger orders unmeasured: pairs);
#   complex64:  L=4 cfg2 2.44 vs 2.39 (quartets), L=5 cfg3 8.59 vs 9.37 (pairs), L=6 cfg2 8.91
#               vs 8.69, cfg4 91.9 vs 87.6 (pairs) -> quartets at L <= 4, staged at L = 5, pairs above
def sibling_kind(dtype: str, order: int) -> str:
    if dtype == "c128":
        return "staged" if order <= 6 else "pair"
    if order <= 4:
        return "quartet"
    return "staged" if order == 5 else "pair"


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
    cnt = np.bincount(blev)
    tot = np.bincount(blev, weights=ev)  # integer sums below 2^53: exact
    return {int(lv) for lv in np.nonzero(cnt)[0] if tot[lv] / cnt[lv] >= threshold}


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


def m2l_level_kinds(mode: str, dtype: str, levels, dense, override=None, env: str = "",
                    rows_per_level=None, order: int = 4) -> dict:
    """level -> M2L kernel: the mode's (dense, sparse) choice; in "auto" a
    sparse level with >= PAIR_MIN_ROWS rows runs the sibling-group kernel
    (sibling_kind); then the per-level overrides (dict, or "4:pair,6:rows")."""
    if mode not in M2L_MODE_KINDS:
        raise ValueError(f"unknown M2L mode {mode!r}")
    kd, ks = M2L_MODE_KINDS[mode]
    kinds = {int(lv): (kd if int(lv) in dense else ks) for lv in levels}
    if mode == "auto":
        for lv in list(kinds):
            if kinds[lv] != "rows":
                continue
            if (rows_per_level or {}).get(lv, 0) >= PAIR_MIN_ROWS:
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
                 shard=None, allreduce=None, m2l: str = "auto", m2l_levels: dict | None = None,
                 build: str | None = None):
        """``reuse``: share the host tree + lists of an existing plan built for
        the same geometry and (order, ncrit, eta, kappa) -- e.g. to run the same
        lists at another storage precision.

        ``build``: "gpu" builds the octree and the dual-tree-traversal lists on
        the device (gpu_build.py; same trees and lists bit for bit), "host" on
        the CPU (native C++); default: env DEFMM_PLAN_BUILD, else "gpu".

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
        self.build = build or os.environ.get("DEFMM_PLAN_BUILD", "gpu")
        if self.build not in ("gpu", "host"):
            raise ValueError(f"unknown plan builder {self.build!r}")

        def tree_of(pts, q, box=None):
            if self.build == "gpu":
                from .gpu_build import build_tree_gpu

                try:
                    return build_tree_gpu(pts, q, tree_cfg, root_box=box, device=self.device)
                except (NotImplementedError, torch.cuda.OutOfMemoryError):
                    pass  # deeper than the 21-level device keys / no room on the device: host build
            return build_tree(pts, q, tree_cfg, root_box=box)

        if same:
            st, sp = tree_of(src, qs)
            tt, tp = st, sp
        else:
            both = np.vstack([np.atleast_2d(targets), np.atleast_2d(sources)])
            box = compute_root_box(both)
            st, sp = tree_of(sources, qs, box)
            tt, tp = tree_of(targets, np.zeros(np.atleast_2d(targets).shape[0]), box)
        self.same = same
        self.tt, self.st, self.tp, self.sp = tt, st, tp, sp
        t1 = time.perf_counter()
        try:
            self.plan = build_plan(tt, st, config.order, config.kappa, config.eta, config.hf_switch,
                                   keep_events=keep_events, dtt="gpu" if self.build == "gpu" else "native",
                                   device=self.device)
        except torch.cuda.OutOfMemoryError:
            # the device traversal keeps a level's candidate pairs and events in HBM; a GPU
            # already filled by other plans builds the same lists with the host traversal
            if self.build != "gpu":
                raise
            torch.cuda.empty_cache()
            self.build = "host"
            self.plan = build_plan(tt, st, config.order, config.kappa, config.eta, config.hf_switch,
                                   keep_events=keep_events, dtt="native", device=self.device)
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
        def particles(ps):  # a device-built tree left the sorted positions and the permutation in HBM
            dv = getattr(ps, "dev", None)
            if dv is not None and dv["positions"].device == torch.empty(0, device=d).device:
                return [dv["positions"][:, k].contiguous() for k in range(3)], dv["perm"]
            return [_dev(ps.positions[:, k], f64, d) for k in range(3)], _dev(ps.original_index, i64, d)

        self.s_xyz, self.s_perm = particles(self.sp)
        self.t_xyz, self.t_perm = (self.s_xyz, self.s_perm) if self.same else particles(self.tp)
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
        self.sib_groups = []  # (K, n, slots, ptr, entries) of the pair / quartet kernels
        for kind in ("pair", "triple", "quartet"):
            gr = h[kind]
            if gr["n"]:
                self.sib_groups.append((gr["K"], int(gr["n"]), gr["grp_slot"], gr["grp_ptr"],
                                        gr["ent"].reshape(-1).contiguous()))
        self.n_pairs = sum(x[1] for x in self.sib_groups)
        sg = h["staged"]
        self.staged = None
        self.stage_depth = int(os.environ.get("DEFMM_STAGE_DEPTH", STAGE_DEPTH))
        if sg["n"]:
            self.staged = (int(sg["n"]), int(sg["ns_cap"])) + tuple(
                sg[k].reshape(-1).contiguous() for k in ("cta_stage", "cta_went", "stage_slot_ptr", "slot_sym",
                                                         "stage_wend", "ent", "cta_rows"))
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
        # mutual P2P (K1 v2): single-tree, unsharded plans evaluate every near-field
        # pair once for both directions (DEFMM_P2P_MUTUAL=0 keeps the one-directional kernel)
        self.p2p_mut = None
        self.n_items, self.p2p_items, self.n_split, self.p2p_split, self._partial_size = 0, None, 0, None, 0
        mut = os.environ.get("DEFMM_P2P_MUTUAL", "auto")  # "1" / "0" force, "auto": large near fields
        if self.same and self.shard is None and (mut == "1" or (mut == "auto" and
                                                                p.counts["p2p_pairs"] >= P2P_MUTUAL_MIN_PAIRS)):
            ml = p2p_mutual_lists(p.p2p_ptr, p.p2p_lo, p.p2p_hi, tt.start[p.leaf_cells], tt.stop[p.leaf_cells],
                                  p.counts["p2p_pairs"], device=d)  # segment lists and gather passes on the device
            if ml is not None:
                self.p2p_mut = {k: _dev(ml[k], i32 if k == "item_leaf" else i64, d)
                                for k in ("item_leaf", "item_f0", "item_f1", "item_row", "item_col", "ptr", "lo",
                                          "hi")}
                self.p2p_mut["n_items"] = int(ml["item_leaf"].shape[0])
                self.p2p_mut["gather"] = [
                    (int(g["task_leaf"].shape[0]), _dev(g["task_leaf"], i32, d), _dev(g["task_out"], i64, d),
                     _dev(g["cptr"], i64, d), _dev(g["cbase"], i64, d), _dev(g["cxlo"], i32, d),
                     _dev(g["cxhi"], i32, d)) for g in ml["gather"]]
                self._partial_size = ml["partial_size"]
        if self.p2p_mut is None:  # one-directional work items (K1)
            wi = p2p_work_items(h["p2p_ptr"], p2p_hi - p2p_lo,
                                tt.stop[p.leaf_cells[lv]] - tt.start[p.leaf_cells[lv]])
            self.n_items = int(wi["item_leaf"].shape[0])
            self.p2p_items = [_dev(wi[k], torch.int32 if k == "item_leaf" else i64, d)
                              for k in ("item_leaf", "item_f0", "item_f1", "item_out")]
            self.n_split = int(wi["split_leaf"].shape[0])
            self.p2p_split = [_dev(wi["split_leaf"], i32, d), _dev(wi["split_base"], i64, d),
                              _dev(wi["split_n"], i32, d)]
            self._partial_size = wi["partial_size"]
        # workspaces (storage precision per FmmConfig.dtype)
        cd = self.cdtype
        self.mult = torch.empty((max(p.n_mult, 1), self.L3), dtype=cd, device=d)
        self.hat = torch.empty((max(self.n_hat, 1), self.SS), dtype=cd, device=d)
        self.local = torch.empty((max(p.n_local, 1), self.L3), dtype=cd, device=d)
        self.lhat = torch.empty((max(int(self.bk_rows.shape[0]), 1), self.SS), dtype=cd, device=d)
        self.near = torch.empty(self.n_tgt, dtype=cd, device=d)
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
        self.qhalo = None
        if self.shard is not None and self.shard.world > 1 and self.allreduce is None:
            # halo exchange over torch.distributed (NCCL between GPUs)
            import torch.distributed as dist

            from .parallel import make_halo

            if not (dist.is_available() and dist.is_initialized()):
                raise ValueError("a sharded plan needs torch.distributed initialised (or allreduce=)")
            self.halo = make_halo(self.plan, self.tt, self.shard.cuts, self.shard.rank, self.shard.world)
            # near-field halo: this rank holds its own chunk's charges, the
            # P2P's other-chunk sources arrive per matvec (parallel.charge_exchange)
            from .parallel import make_charge_halo

            self.qhalo = make_charge_halo(self.plan, self.tt, self.shard.cuts, self.shard.rank, self.shard.world)

    # events per parent-pair block above which a level's M2L runs blocked
    BLOCKED_MIN_EVENTS_PER_BLOCK = BLOCKED_MIN_EVENTS_PER_BLOCK

    def _host_lists(self) -> dict:
        """Per-level M2L kernel choice: levels whose parent-pair blocks are
        dense (volume-like, >= BLOCKED_MIN_EVENTS_PER_BLOCK events per block)
        run the blocked kernel (K7 v3, operand reuse in registers), sparse
        (surface-like) levels the row kernel by default (their blocks would be
        mostly predicated-off pairs) -- profiles/r01_summary_v3.md, v4.md.
        lhat rows: the blocked rows (one F2L launch over all of them)."""
        h = self._host_lists_all()
        p, tt = self.plan, self.tt
        rows = h["rows"]
        rlev = tt.level[p.l_cell[rows]] if rows.size else np.zeros(0, np.int64)
        # density per level from the full plan (identical on every rank)
        dense = dense_levels(p, tt, self.BLOCKED_MIN_EVENTS_PER_BLOCK)
        levels = np.unique(rlev)
        # rows per level from the full plan (identical on every rank)
        flev = tt.level[p.l_cell[p.m2l_row_slot]] if p.m2l_row_slot.size else np.zeros(0, np.int64)
        rpl = {int(lv): int(c) for lv, c in zip(*np.unique(flev, return_counts=True))}
        kinds = m2l_level_kinds(self.m2l_variant_default, self.config.dtype, levels, dense,
                                self.m2l_level_override, os.environ.get("DEFMM_M2L_LEVELS", ""), rpl, self.L)
        self.level_kinds = kinds
        kind_of = np.full(int(levels.max()) + 1 if levels.size else 1, "", dtype=object)
        for lv, k in kinds.items():
            if int(lv) < kind_of.shape[0]:
                kind_of[int(lv)] = k
        rkind = kind_of[rlev] if rows.size else np.zeros(0, object)
        z = np.zeros(0, np.int64)

        def pick(*ks):
            return np.isin(rkind, list(ks)) if rows.size else np.zeros(0, bool)

        # row kernel
        is_rows = pick("rows")
        _, rptr, rsel = _sub_csr(h["row_ptr"], is_rows)

        def take(x, idx):  # rows of a host array or of a device-resident list
            return x[torch.as_tensor(idx, dtype=torch.int64, device=x.device)] if torch.is_tensor(x) else x[idx]

        h["rk_rows"], h["rk_ptr"], h["rk_ent"] = rows[is_rows], rptr, take(h["ent"], rsel)
        # sibling pairs (K7 v8)
        # sibling groups (K7 v8): per-event merging on the device (m2l_groups_dev)
        ent_dev = _dev(h["ent"], torch.int32, self.device) if any(pick("pair", "triple", "quartet")) else None
        for kind, K in (("pair", 2), ("triple", 3), ("quartet", 4)):
            h[kind] = m2l_groups_dev(np.nonzero(pick(kind))[0], rows, h["row_ptr"], ent_dev, p.l_cell, p.l_dir,
                                     tt.level, tt.parent, K, self.device)
        # staged M2L (K7 v13): warp units of sibling rows sharing staged symbols
        hat_coords = self.st.coords[p.m_cell[h["hat_slot"]]] if h["hat_slot"].size else np.zeros((0, 3), np.int64)
        if ent_dev is None and any(pick("staged")):
            ent_dev = _dev(h["ent"], torch.int32, self.device)
        h["staged"] = m2l_stage_lists_dev(np.nonzero(pick("staged"))[0], rows, h["row_ptr"], ent_dev, p.l_cell,
                                          p.l_dir, tt.level, tt.parent, tt.coords, hat_coords,
                                          int(os.environ.get("DEFMM_STAGE_SLOTS", STAGE_SLOTS)), self.device)
        # lhat rows = the blocked rows, then the staged rows
        is_grp = pick("blocked")
        grp_rows = rows[is_grp]
        h["bk_rows"] = np.concatenate([grp_rows, h["staged"]["row_slot"]])
        cr = h["staged"]["cta_rows"]  # lhat rows of the staged kernel follow the blocked rows
        h["staged"]["cta_rows"] = torch.where(cr >= 0, cr + int(grp_rows.shape[0]), cr).to(torch.int32)
        # groups of blocked levels, rows renumbered into lhat
        gr = h["grp_rows"]
        gr_slots = np.where(gr >= 0, rows[np.maximum(gr, 0)] if rows.size else -1, -1)
        gid = _rows_to_ids(gr_slots, grp_rows)
        gkeep = np.any(gid >= 0, axis=1)
        _, gptr, bsel = _sub_csr(h["grp_ptr"], gkeep)
        h["grp_ptr"], h["grp_rows"] = gptr, gid[gkeep]
        if "blk_src_ev" in h:  # unsharded: spectrum of the selected blocks' events only
            bs = take(h.pop("blk_src_ev"), bsel)
            if torch.is_tensor(bs) or torch.is_tensor(h["ent"]):
                ent_dev = _dev(h["ent"], torch.int32, self.device) if ent_dev is None else ent_dev
                bs = _dev(bs, torch.int64, self.device)
                src = ent_dev[bs.clamp(min=0), 0] if ent_dev.shape[0] else torch.zeros_like(bs, dtype=torch.int32)
                h["blk_src"] = torch.where(bs >= 0, src, torch.full_like(src, -1))
            else:
                hat = h["ent"][:, 0]
                h["blk_src"] = np.where(bs >= 0, hat[np.maximum(bs, 0)] if hat.size else 0, -1).astype(np.int32)
        else:
            h["blk_src"] = h["blk_src"][bsel]
        h["blk_trans"], h["blk_mask"] = take(h["blk_trans"], bsel), h["blk_mask"][bsel]
        h["blk_kind"] = h["blk_kind"][bsel] if "blk_kind" in h else planar_kind(h["blk_mask"])
        self.dense_levels = sorted(lv for lv, k in kinds.items() if k == "blocked")
        return h

    def _host_lists_all(self) -> dict:
        """The plan's lists, restricted to this rank's chunk when sharded
        (parallel.py); spectra are renumbered compactly."""
        p, sh = self.plan, self.shard
        # lists the device builders left on the device are used there (unsharded plans)
        ent_dev = p.on_device("m2l_rows_entries") if sh is None else None
        h = {
            "p2m_idx": p.p2m_idx,
            "m2m": [(lev, sl, ss) for lev, sl, ss in p.m2m_levels],
            "hat_slot": p.hat_slot,
            "rows": p.m2l_row_slot,
            "row_ptr": p.m2l_row_ptr,
            "ent": ent_dev if ent_dev is not None else p.m2l_rows_entries,
            "l2l": list(p.l2l_levels),
            "leaves": np.ones(p.leaf_cells.shape[0], bool),
            "p2p_ptr": p.p2p_ptr,
            "p2p_sel": np.arange(p.p2p_lo.shape[0]),
        }
        # blocked M2L: group rows as indices into h["rows"] (lhat rows)
        if sh is None:
            def dev_or_host(name):
                t = p.on_device(name)
                return t if t is not None else getattr(p, name)

            h.update({"grp_ptr": p.blk_group_ptr, "grp_rows": _rows_to_ids(p.blk_group_rows, h["rows"]),
                      "blk_src_ev": dev_or_host("blk_src_ev"), "blk_trans": dev_or_host("blk_trans"),
                      "blk_mask": p.blk_mask})
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

    @_on_device
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
    @_on_device
    def set_charges(self, charges):
        """Load charges (caller order) into the sorted device buffer."""
        q = torch.as_tensor(np.asarray(charges, dtype=complex)) if not torch.is_tensor(charges) else charges
        q = q.to(device=self.device, dtype=self.cdtype)
        torch.index_select(q, 0, self.s_perm, out=self.q)  # one gather into the sorted buffer
        if self.qhalo is not None:  # a rank owns its chunk's charges only
            self.q[: self.shard.lo].zero_()
            self.q[self.shard.hi:].zero_()

    def set_charges_sorted(self, q_sorted):
        self.q.copy_(q_sorted)

    @_on_device
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
        # NVTX ranges per stage (the reference's stage timers, traversal.py:445-493)
        nvtx = torch.cuda.nvtx
        nvtx.range_push("defmm.matvec")
        try:
            return self._apply_stages(out, stage_events)
        finally:
            nvtx.range_pop()

    def _apply_stages(self, out=None, stage_events=None):
        nvtx = torch.cuda.nvtx
        if self.qhalo is not None:  # near-field source charges of the other chunks
            from .parallel import charge_exchange

            nvtx.range_push("defmm.charge_halo")
            charge_exchange(self.q, self._qhalo_dev())
            nvtx.range_pop()
        nvtx.range_push("defmm.upward")
        self.apply_upward(stage_events)
        nvtx.range_pop()
        if self.shard is not None:
            if self.allreduce is not None:
                # M2M is linear: summing the partial multipoles over the ranks
                # completes every multipole
                self.allreduce(self.mult)
            else:
                from .parallel import halo_exchange

                nvtx.range_push("defmm.multipole_halo")
                halo_exchange(self.mult, self._halo_dev())
                nvtx.range_pop()
        nvtx.range_push("defmm.m2l_downward")
        try:
            return self.apply_rest(out, stage_events)
        finally:
            nvtx.range_pop()

    def halo_bytes(self) -> int:
        """Bytes this rank moves per matvec: the spanning multipoles it
        all-reduces, the nodal multipoles it sends and receives in the
        all_to_all, and the near-field source charges it sends and receives
        (0 unsharded)."""
        if self.shard is None:
            return 0
        per = self.L3 * self.mult.element_size()
        if self.halo is None:  # allreduce= exchange: the whole multipole array
            return int(self.mult.numel() * self.mult.element_size())
        h = self.halo
        qb = 0
        if self.qhalo is not None:
            qb = self.q.element_size() * (int(sum(self.qhalo.send_counts)) + int(sum(self.qhalo.recv_counts)))
        return int(per * (len(h.span) + int(sum(h.send_counts)) + int(sum(h.recv_counts))) + qb)

    def _qhalo_dev(self):
        if getattr(self, "_qhalo_t", None) is None:
            h = self.qhalo
            idx = lambda a: torch.as_tensor(a, dtype=torch.int64, device=self.q.device)  # noqa: E731
            self._qhalo_t = (idx(h.send), list(h.send_counts), idx(h.recv), list(h.recv_counts), bool(h.active))
        return self._qhalo_t

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
            m = self.p2p_mut
            if m is not None:
                _lib.call(self._op("p2p_mutual"), m["n_items"], m["item_leaf"], m["item_f0"], m["item_f1"],
                          m["item_row"], m["item_col"], self.tgt_lo, self.tgt_hi, m["ptr"], m["lo"], m["hi"],
                          *self.s_xyz, self.q, float(p.kappa), float(p.tol), self.p2p_partial,
                          int(self.p2p_grid), int(self.p2p_hilo), side.cuda_stream)
                for nt_, tleaf, tout, cptr, cbase, cxlo, cxhi in m["gather"]:
                    _lib.call(self._op("p2p_gather"), nt_, tleaf, tout, self.tgt_lo, self.tgt_hi, cptr, cbase,
                              cxlo, cxhi, self.p2p_partial, self.near, side.cuda_stream)
            else:
                _lib.call(self._op("p2p"), self.n_items, *self.p2p_items, self.tgt_lo, self.tgt_hi, self.p2p_ptr,
                          self.p2p_lo, self.p2p_hi, *self.t_xyz, *self.s_xyz, self.q, float(p.kappa),
                          float(p.tol), self.near, self.p2p_partial, self.n_split, *self.p2p_split,
                          int(self.p2p_grid), int(self.p2p_hilo), side.cuda_stream)
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
        self._m2l(sh)
        if stage_events is not None:
            c = ev()
            c.record(stream)
            stage_events.append(("m2l", b, c))
        # downward: L2L per level top-down, then L2P + near + un-permute
        for son_beta, outs, octant, ptr, src, sdir, n in self.l2l:
            _lib.call(self._op("l2l"), L, n, outs, octant, ptr, src, sdir, son_beta, self.dirs, kappa,
                      self.local, sh)
        stream.wait_stream(self.side_stream)
        if self.shard is not None:
            out.zero_()  # this rank writes only its own targets
        _lib.call(self._op("l2p"), L, self.n_leaves, self.leaf_cell, self.leaf_lo, self.leaf_hi, self.slot_dir,
                  tg["start"], tg["stop"], tg["alpha"], tg["level"], tg["beta"], self.dirs, *self.t_xyz, kappa,
                  self.local, self.near, self.t_perm, out, sh)
        if stage_events is not None:
            e = ev()
            e.record(stream)
            stage_events.append(("downward", c, e))
        return out

    def _m2l(self, sh):
        """The M2L stage (K7 + K8) on stream handle ``sh``: zero the locals, the
        per-level M2L kernels, the F2L of the blocked rows."""
        L = self.L
        self.local.zero_()
        if self.m2l_variant == "hybrid":
            _lib.call(self._op("m2l_rows"), L, self.rk_rows.shape[0], self.rk_rows, self.rk_ptr, self.rk_ent,
                      self.hat, self.sym_derived, self.local, sh)
            for K, ng, gslot, gptr, gent in self.sib_groups:
                _lib.call(self._op("m2l_group"), L, K, ng, gslot, gptr, gent, self.hat, self.sym_derived, self.local,
                          sh)
            _lib.call(self._op("m2l_blocked"), L, self.n_groups, self.grp_ptr, self.grp_rows, self.blk_src,
                      self.blk_trans, self.blk_mask, self.blk_kind, self.hat, self.sym_derived, self.lhat, sh)
            if self.staged is not None:
                _lib.call(self._op("m2l_stage"), L, self.staged[0], self.staged[1], self.stage_depth,
                          *self.staged[2:], self.hat, self.sym_derived, self.lhat, sh)
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

    @_on_device
    def time_isolated(self, reps: int = 5, flush=None) -> dict:
        """Kernel times with nothing running beside them (ms, CUDA events on the
        launching stream, mean of ``reps``): the M2L stage (memset + M2L kernels
        + F2L) on the current stream after a full matvec, and the P2P alone on
        its side stream.  These are the roofline denominators of bench.py."""
        dev = self.device
        stream = torch.cuda.current_stream(dev)
        self._apply()  # spectra of the loaded charges
        torch.cuda.synchronize(dev)
        t = {"m2l": 0.0, "p2p": 0.0}
        for _ in range(reps):
            if flush is not None:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            a.record(stream)
            self._m2l(stream.cuda_stream)
            b.record(stream)
            torch.cuda.synchronize(dev)
            t["m2l"] += a.elapsed_time(b)
            if flush is not None:
                flush.zero_()
            torch.cuda.synchronize(dev)
            ev = []
            self._near_field(ev)
            torch.cuda.synchronize(dev)
            t["p2p"] += ev[0][1].elapsed_time(ev[0][2])
        return {k: v / max(reps, 1) for k, v in t.items()}

    @_on_device
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
        gk = "m2l_group_kernel"
        for n, name, k in ((self.rk_rows.shape[0], "m2l_rows_kernel", "rows"),
                           (sum(x[1] for x in self.sib_groups if x[0] == 2), f"{gk}<2>", "pair"),
                           (sum(x[1] for x in self.sib_groups if x[0] == 3), f"{gk}<3>", "triple"),
                           (sum(x[1] for x in self.sib_groups if x[0] == 4), f"{gk}<4>", "quartet"),
                           (self.n_groups, "m2l_blocked_kernel", "blocked"),
                           (self.staged[0] if self.staged else 0, "m2l_stage_kernel", "staged"),
                           (self.bk_rows.shape[0], "f2l_rows_kernel", None)):
            if n:
                out.append(f"{name}<{R}, {self.L}>" + (f" (levels {lv(k)})" if k is not None else ""))
        return out

    @property
    def launches_per_apply(self) -> int:
        """Kernels of one matvec: p2p (+ split reduce), p2m, m2m per level, m2f,
        the M2L kernels with work, l2l per level, l2p."""
        if self.m2l_variant == "hybrid":
            m2l = len(self.sib_groups) + sum(int(n > 0) for n in (self.rk_rows.shape[0], self.n_groups,
                                                                   self.bk_rows.shape[0])) + int(bool(self.staged))
        else:
            m2l = 1
        p2p_extra = len(self.p2p_mut["gather"]) if self.p2p_mut is not None else int(bool(self.n_split))
        return 4 + p2p_extra + len(self.m2m) + len(self.l2l) + m2l

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
