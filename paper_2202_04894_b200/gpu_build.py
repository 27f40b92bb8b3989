"""Plan construction on the GPU: the octree and the
dual-tree-traversal lists, built from device sorts / scans (torch, the
plumbing) around two decision kernels of libdefmm_b200 (csrc/plan_gpu.cu)
that keep the reference's FP64 octant tests and integer MAC bit-identical.

``build_tree_gpu`` returns the same (ClusterTree, ParticleSet) as
``tree.build_tree`` (tree.py:132-213): the tree arrays, the permutation and the
sorted positions are equal bit for bit (tests/test_gpu_build.py).
``GpuDtt`` produces the lists of ``plan.NativeDtt`` (traversal.py:182-200,
320-348) with the same ordering conventions.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .config import TreeConfig
from .geometry import BoundingBox
from .tree import ClusterTree, ParticleSet

__all__ = ["build_tree_gpu", "GpuDtt", "Deferred", "DeviceParticleSet"]

KEY_DEPTH = 21  # 3 bits per level in one int64 key


def _run_info(sorted_prefix: torch.Tensor):
    """(run id of every element, run lengths) of a sorted 1-D tensor."""
    uniq, inv, cnt = torch.unique_consecutive(sorted_prefix, return_inverse=True, return_counts=True)
    return inv, cnt


def build_tree_gpu(points, charges, config: TreeConfig = TreeConfig(), root_box: BoundingBox | None = None,
                   device="cuda"):
    """tree.build_tree on the GPU.  Every particle's octant path comes from
    defmm_tree_keys; a cell is split while it holds more than ncrit particles
    (and its level is below the depth cap); particles are ordered by the path
    truncated at their leaf's level, stably (= the reference's recursive stable
    partition: inside a leaf the original order survives)."""
    points = np.atleast_2d(np.asarray(points, dtype=float))
    charges = np.asarray(charges, dtype=complex)
    if points.shape[0] == 0:
        raise ValueError("at least one particle is required")
    if points.shape[0] != charges.shape[0]:
        raise ValueError("points and charges length mismatch")
    dev = torch.device(device)
    n = points.shape[0]
    ncrit, cap = int(config.ncrit), int(config.hard_depth_cap)
    D = min(cap, KEY_DEPTH)
    with torch.cuda.device(dev):
        pts = torch.as_tensor(np.ascontiguousarray(points, dtype=np.float64)).to(dev)
        if not bool(torch.isfinite(pts).all()):
            raise ValueError("particle coordinates must be finite")
        if root_box is None:
            root_box = _root_box(points, pts)
        keys = torch.empty(n, dtype=torch.int64, device=dev)
        lower = np.ascontiguousarray(root_box.lower, dtype=np.float64)
        _lib.check(_lib.load().defmm_tree_keys(n, pts.data_ptr(), lower.ctypes.data, float(root_box.side), D,
                                               keys.data_ptr(), torch.cuda.current_stream(dev).cuda_stream),
                   "defmm_tree_keys")
        sk, order0 = torch.sort(keys, stable=True)
        # leaf level of every particle (Morton order): the first level whose cell holds <= ncrit
        leaf = torch.full((n,), D, dtype=torch.int64, device=dev)
        undecided = torch.ones(n, dtype=torch.bool, device=dev)
        depth = 0
        for lev in range(D + 1):
            inv, cnt = _run_info(sk >> (3 * (D - lev)))
            small = (cnt <= ncrit)[inv]
            if lev == D:
                if cap > D and bool((undecided & ~small).any()):
                    raise NotImplementedError("tree deeper than 21 levels: use the host build (tree.build_tree)")
                small = torch.ones(n, dtype=torch.bool, device=dev)  # the depth cap ends the splitting
            hit = undecided & small
            leaf[hit] = lev
            undecided &= ~small
            if bool(hit.any()):
                depth = lev
            if not bool(undecided.any()):
                break
        # truncated keys in the ORIGINAL particle order, then the stable sort
        sh = 3 * (D - leaf)
        tk_sorted = (sk >> sh) << sh
        tk = torch.empty_like(tk_sorted)
        tk[order0] = tk_sorted
        lf = torch.empty_like(leaf)
        lf[order0] = leaf
        tks, perm = torch.sort(tk, stable=True)
        lfs = lf[perm]
        # cells of level l: the distinct prefixes among particles whose leaf is at level >= l
        pos = torch.arange(n, device=dev)
        lv_l, co_l, st_l, sp_l = [], [], [], []
        for lev in range(depth + 1):
            m = lfs >= lev
            pm = pos[m]
            pref = tks[m] >> (3 * (D - lev))
            uq, cnt = torch.unique_consecutive(pref, return_counts=True)
            first = torch.cumsum(cnt, 0) - cnt
            start = pm[first]
            c = torch.zeros((uq.shape[0], 3), dtype=torch.int64, device=dev)
            for b in range(lev):  # de-interleave: level-b octant sits at bits 3 (lev - 1 - b) ..
                o = (uq >> (3 * (lev - 1 - b))) & 7
                c[:, 0] = 2 * c[:, 0] + ((o >> 2) & 1)
                c[:, 1] = 2 * c[:, 1] + ((o >> 1) & 1)
                c[:, 2] = 2 * c[:, 2] + (o & 1)
            lv_l.append(torch.full((uq.shape[0],), lev, dtype=torch.int64, device=dev))
            co_l.append(c)
            st_l.append(start)
            sp_l.append(start + cnt)
        level = torch.cat(lv_l)
        coords = torch.cat(co_l)
        start = torch.cat(st_l)
        stop = torch.cat(sp_l)
        # parent = the level l-1 cell whose particle range holds the cell's first particle
        offs = np.concatenate([[0], np.cumsum([x.shape[0] for x in st_l])])
        parent = torch.full((level.shape[0],), -1, dtype=torch.int64, device=dev)
        for lev in range(1, depth + 1):
            ps = st_l[lev - 1]
            j = torch.searchsorted(ps, st_l[lev], right=True) - 1
            parent[offs[lev]:offs[lev + 1]] = offs[lev - 1] + j
        h = _to_host({"perm": perm, "level": level, "coords": coords, "start": start, "stop": stop,
                      "parent": parent}, dev)
        tree = ClusterTree(root_box, config, h["level"], h["coords"], h["start"], h["stop"], h["parent"])
        pset = DeviceParticleSet(h["perm"], pts[perm], perm, charges)
    return tree, pset


class DeviceParticleSet(ParticleSet):
    """The ParticleSet (tree.py:48-59) of a device-built tree.  The sorted
    positions and the permutation stay on the device (``dev``) where FmmPlan
    uses them; the host arrays of the reference's record -- sorted positions,
    permuted charges, zeroed potentials -- are produced when first read."""

    def __init__(self, original_index: np.ndarray, positions_dev: torch.Tensor, perm_dev: torch.Tensor,
                 charges: np.ndarray):
        self.original_index = original_index
        self.dev = {"positions": positions_dev, "perm": perm_dev}
        self._late = {
            "positions": lambda: _to_host({"x": positions_dev}, positions_dev.device)["x"],
            "charges": lambda: charges[original_index].copy(),
            "potentials": lambda: np.zeros(original_index.shape[0], dtype=complex),
        }

    @property
    def n(self) -> int:
        return int(self.original_index.shape[0])


def _late_field(name):
    def get(self):
        v = self._late[name]
        if callable(v):
            v = self._late[name] = v()
        return v

    def put(self, v):
        self._late[name] = v

    return property(get, put)


for _name in ("positions", "charges", "potentials"):
    setattr(DeviceParticleSet, _name, _late_field(_name))


def _root_box(points: np.ndarray, pts: torch.Tensor) -> BoundingBox:
    """geometry.compute_root_box (geometry.py:82-97) with the extremes found on
    the device: the centre is the same numpy mean; max |x - c| is attained at a
    coordinate extreme because the rounded difference is monotone in x, so the
    half width (and the box) is bit-identical."""
    center = points.mean(axis=0)
    half = 0.5
    if points.shape[0] > 1:
        lo, hi = torch.aminmax(pts, dim=0)
        lo, hi = lo.cpu().numpy(), hi.cpu().numpy()
        half = np.max(np.maximum(hi - center, center - lo))
    if half == 0.0:
        half = 0.5
    return BoundingBox(center=center, half_width=half * (1.0 + 1e-6))


def _to_host(tensors: dict, dev) -> dict:
    """Device tensors -> numpy arrays in pinned host memory (the pageable path
    moves these lists at ~1.5 GB/s; a second copy out of the staging buffer
    cost as much as the transfer).  The arrays keep their buffers alive."""
    staged = {}
    for k, v in tensors.items():
        h = torch.empty(v.shape, dtype=v.dtype, device="cpu", pin_memory=True)
        h.copy_(v, non_blocking=True)
        staged[k] = h
    torch.cuda.synchronize(dev)
    return {k: h.numpy() for k, h in staged.items()}


class Deferred:
    """A plan list that stays on the device until host code asks for it (the
    per-event lists are hundreds of MB at the large workloads and the device
    matvec never needs them on the host)."""

    def __init__(self, tensor: torch.Tensor):
        self.dev = tensor
        self.shape = tuple(tensor.shape)

    def host(self) -> np.ndarray:
        return _to_host({"x": self.dev}, self.dev.device)["x"]


def _octant(coords, parent, cells):
    d = coords[cells] - 2 * coords[parent[cells]]
    return d[:, 0] * 4 + d[:, 1] * 2 + d[:, 2]


class GpuDtt:
    """The lists of plan.NativeDtt (csrc/dtt_build.cpp), built on the GPU: a
    level-synchronous sweep over target-major candidate lists.  Per level the
    pairs are classified by defmm_dtt_classify (M2L / P2P / expand); M2L events
    are ordered into rows (target, key) by a stable sort, so a row keeps the
    reference's traversal order; the sons x sons of the expanding pairs, stably
    sorted by target son, are the next level's candidates.  Parent-pair groups
    and blocks come from the same events by stable sorts and scatters.  Same
    keys and conventions as NativeDtt (ids, orders; blk_src may name another
    event of the same source cell)."""

    def __init__(self, tt: ClusterTree, st: ClusterTree, depth, g2min, R, tab_off, key_tab, device="cuda"):
        dev = torch.device(device)
        lib = _lib.load()
        i64, i32 = torch.int64, torch.int32

        def up(a, dt=i64):
            return torch.as_tensor(np.ascontiguousarray(a)).to(dev, dt)

        with torch.cuda.device(dev):
            stream = torch.cuda.current_stream(dev).cuda_stream
            tco, tns, tfs, tpa = up(tt.coords), up(tt.n_sons), up(tt.first_son), up(tt.parent)
            same = st is tt
            sco, sns, sfs, spa = (tco, tns, tfs, tpa) if same else (up(st.coords), up(st.n_sons), up(st.first_son),
                                                                    up(st.parent))
            ktab = up(key_tab, i32)
            status = torch.zeros(1, dtype=i32, device=dev)
            pt = torch.zeros(1, dtype=i64, device=dev)
            ps = torch.zeros(1, dtype=i64, device=dev)
            pq = torch.zeros(1, dtype=i64, device=dev)
            KS = int(ktab.max().item()) + 3 if ktab.numel() else 3
            out = {k: [] for k in ("ev_s", "ev_dense", "row_t", "row_key", "row_lev", "row_cnt", "grp_rows", "grp_p",
                                   "grp_key", "grp_lev", "grp_nblk", "blk_src", "blk_dense", "blk_mask", "p_t", "p_s")}
            n_ev = n_row = 0
            smarks = {}
            for lev in range(int(depth) + 1):
                if lev > tt.depth or lev > st.depth or pt.numel() == 0:
                    break
                n = pt.numel()
                kind = torch.empty(n, dtype=torch.int8, device=dev)
                key = torch.empty(n, dtype=i32, device=dev)
                dense = torch.empty(n, dtype=i64, device=dev)
                nexp = torch.empty(n, dtype=i64, device=dev)
                _lib.check(lib.defmm_dtt_classify(n, pt.data_ptr(), ps.data_ptr(), tco.data_ptr(), sco.data_ptr(),
                                                  tns.data_ptr(), sns.data_ptr(), int(g2min[lev]), int(R[lev]),
                                                  int(tab_off[lev]), ktab.data_ptr(), kind.data_ptr(),
                                                  key.data_ptr(), dense.data_ptr(), nexp.data_ptr(),
                                                  status.data_ptr(), stream), "defmm_dtt_classify")
                # ---- M2L events -> rows (t, key), candidate order inside a row ----
                mi = torch.nonzero(kind == 0).reshape(-1)
                if mi.numel():
                    if lev == 0:
                        raise RuntimeError("defmm_dtt_build failed (-5)")  # an M2L between the roots
                    et, es, ek, ed, eq = pt[mi], ps[mi], key[mi].to(i64), dense[mi], pq[mi]
                    o = torch.sort(et * KS + (ek + 1), stable=True)[1]
                    et, es, ek, ed, eq = et[o], es[o], ek[o], ed[o], eq[o]
                    rkey, rinv, rcnt = torch.unique_consecutive(et * KS + (ek + 1), return_inverse=True,
                                                                return_counts=True)
                    nr = rkey.numel()
                    out["ev_s"].append(es.to(i32))
                    out["ev_dense"].append(ed)
                    sm = torch.unique(es * KS + (ek + 1))  # distinct (source cell, key): the source marks
                    smarks[lev] = (sm // KS, sm % KS - 1)
                    out["row_t"].append((rkey // KS).to(i32))
                    out["row_key"].append((rkey % KS - 1).to(i32))
                    out["row_lev"].append(torch.full((nr,), lev, dtype=i32, device=dev))
                    out["row_cnt"].append(rcnt)
                    # ---- groups (key, target parent) and blocks (group, source parent) ----
                    ne = et.numel()
                    P, Q = tpa[et], spa[es]
                    a, b = _octant(tco, tpa, et), _octant(sco, spa, es)
                    dd = ((((a >> 2) & 1) - ((b >> 2) & 1)) + 1) * 9 + ((((a >> 1) & 1) - ((b >> 1) & 1)) + 1) * 3 + \
                        ((a & 1) - (b & 1)) + 1
                    np_l = int(tt.level_offsets[lev] - tt.level_offsets[lev - 1])
                    gk = (ek + 1) * np_l + (P - int(tt.level_offsets[lev - 1]))
                    go = torch.sort(gk, stable=True)[1]  # group-scan order: (key, P), then row order
                    guq, ginv, gcnt = torch.unique_consecutive(gk[go], return_inverse=True, return_counts=True)
                    ng = guq.numel()
                    j = torch.arange(ne, device=dev)
                    qmax = int(eq.max().item()) + 1
                    bk = ginv * qmax + eq[go]
                    buq, binv = torch.unique(bk, return_inverse=True)
                    nb = buq.numel()
                    first_use = torch.full((nb,), ne, dtype=i64, device=dev).scatter_reduce(0, binv, j, "amin")
                    bgrp = buq // qmax
                    border = torch.sort(bgrp * (ne + 1) + first_use)[1]  # blocks by (group, first use)
                    brank = torch.empty(nb, dtype=i64, device=dev)
                    brank[border] = torch.arange(nb, device=dev)
                    eb = brank[binv]  # block of every event (group-scan order)
                    ev_id = n_ev + go  # global event id
                    ag, bg, dg = a[go], b[go], dd[go]
                    blk_src = torch.full((nb * 8,), -1, dtype=i64, device=dev).scatter_reduce(
                        0, eb * 8 + bg, ev_id, "amax")
                    blk_dense = torch.full((nb * 27,), -1, dtype=i64, device=dev).scatter_reduce(
                        0, eb * 27 + dg, ed[go], "amax")
                    blk_mask = torch.zeros(nb, dtype=i64, device=dev).index_add_(0, eb, torch.ones_like(eb) << (8 * ag + bg))
                    grp_rows = torch.full((ng * 8,), -1, dtype=i64, device=dev).scatter_reduce(
                        0, ginv * 8 + ag, n_row + rinv[go], "amax")
                    out["grp_rows"].append(grp_rows.reshape(ng, 8))
                    out["grp_p"].append((guq % np_l + int(tt.level_offsets[lev - 1])).to(i32))
                    out["grp_key"].append((guq // np_l - 1).to(i32))
                    out["grp_lev"].append(torch.full((ng,), lev, dtype=i32, device=dev))
                    out["grp_nblk"].append(torch.bincount(bgrp, minlength=ng))
                    out["blk_src"].append(blk_src.reshape(nb, 8))
                    out["blk_dense"].append(blk_dense.reshape(nb, 27))
                    out["blk_mask"].append(blk_mask)
                    n_ev += ne
                    n_row += nr
                # ---- near field ----
                pi = torch.nonzero(kind == 1).reshape(-1)
                out["p_t"].append(pt[pi].to(i32))
                out["p_s"].append(ps[pi].to(i32))
                # ---- next level: sons x sons of the expanding pairs, target-major ----
                xi = torch.nonzero(kind == 2).reshape(-1)
                if xi.numel() == 0:
                    pt = pt[:0]
                    continue
                xt, xs, cnt = pt[xi], ps[xi], nexp[xi]
                tu, tinv, tcnt = torch.unique_consecutive(xt, return_inverse=True, return_counts=True)
                rank = torch.arange(xt.numel(), device=dev) - (torch.cumsum(tcnt, 0) - tcnt)[tinv]
                tot = int(cnt.sum().item())
                rep = torch.repeat_interleave(torch.arange(xt.numel(), device=dev), cnt, output_size=tot)
                k = torch.arange(tot, device=dev) - (torch.cumsum(cnt, 0) - cnt)[rep]
                nsr = sns[xs][rep]
                ca = tfs[xt][rep] + k // nsr
                cb = sfs[xs][rep] + k % nsr
                o = torch.sort(ca, stable=True)[1]
                pt, ps, pq = ca[o], cb[o], rank[rep][o]
            if int(status.item()):
                raise RuntimeError("defmm_dtt_build: a translation fell outside its level's key table")

            def cat(k, dt, shape=(0,)):
                return torch.cat(out[k]) if out[k] else torch.zeros(shape, dtype=dt, device=dev)

            ev_dense = cat("ev_dense", i64)
            trans_dense = torch.unique(ev_dense)
            blk_dense = cat("blk_dense", i64, (0, 27))
            bt = torch.searchsorted(trans_dense, blk_dense.clamp(min=0).reshape(-1)).reshape(-1, 27)
            row_cnt = cat("row_cnt", i64)
            nblk = cat("grp_nblk", i64)
            z = torch.zeros(1, dtype=i64, device=dev)
            a = {
                "ev_s": cat("ev_s", i32), "ev_trans": torch.searchsorted(trans_dense, ev_dense).to(i32),
                "row_ptr": torch.cat([z, torch.cumsum(row_cnt, 0)]), "row_t": cat("row_t", i32),
                "row_key": cat("row_key", i32), "row_lev": cat("row_lev", i32),
                "grp_rows": cat("grp_rows", i64, (0, 8)), "grp_p": cat("grp_p", i32), "grp_key": cat("grp_key", i32),
                "grp_lev": cat("grp_lev", i32), "grp_ptr": torch.cat([z, torch.cumsum(nblk, 0)]),
                "blk_src": cat("blk_src", i64, (0, 8)),
                "blk_trans": torch.where(blk_dense >= 0, bt, torch.full_like(bt, -1)).to(i32),
                "blk_mask": cat("blk_mask", i64), "p_t": cat("p_t", i32), "p_s": cat("p_s", i32),
                "trans_dense": trans_dense,
            }
            self._late = {k: a.pop(k) for k in self.LATE}
            # near-field pair count (counts["p2p_pairs"], traversal.py:303-317)
            tn, sn = up(tt.stop - tt.start), (None if same else up(st.stop - st.start))
            self.n_pairs = int((tn[a["p_t"].to(i64)] * (tn if same else sn)[a["p_s"].to(i64)]).sum().item())
            self.a = _to_host(a, dev)
            self._smarks = {lev: tuple(x.cpu().numpy() for x in v) for lev, v in smarks.items()}
            self._dev = {"ev_s": self._late["ev_s"], "row_lev": a["row_lev"], "row_key": a["row_key"],
                         "row_cnt": row_cnt}
        self.n_events = int(self._late["ev_s"].shape[0])

    # per-event and per-block lists: downloaded on first host access only
    LATE = ("ev_s", "ev_trans", "blk_src", "blk_trans")

    def __getitem__(self, k):
        if k not in self.a:
            self.a[k] = Deferred(self._late[k]).host()
        return self.a[k]

    def deferred(self, k) -> Deferred:
        """The list as a device-resident Deferred (no transfer)."""
        return Deferred(self._late[k])

    def entries(self, src_hat: torch.Tensor) -> Deferred:
        """The (n_events, 2) int32 M2L entry table {spectrum, translation id} in
        row order (plan.Plan.m2l_rows_entries), on the device."""
        return Deferred(torch.stack([src_hat.to(torch.int32), self._late["ev_trans"]], 1).contiguous())

    def source_hats(self, m_dense, base, nd, level_off, key_base, n_mult):
        """defmm_dtt_source_hats on the device lists: the spectrum index of every
        event's source expansion (a device tensor) and the used multipole slots,
        ascending (host)."""
        d = self._dev
        dev = d["ev_s"].device
        i64 = torch.int64
        with torch.cuda.device(dev):
            up = lambda x: torch.as_tensor(np.ascontiguousarray(x, np.int64)).to(dev)  # noqa: E731
            md, bs, ndl, lo, kb = up(m_dense), up(base), up(nd), up(level_off), up(key_base)
            ne = int(d["ev_s"].numel())
            rows = torch.repeat_interleave(torch.arange(d["row_cnt"].numel(), device=dev), d["row_cnt"],
                                           output_size=ne)
            lev = d["row_lev"].to(i64)[rows]
            key = d["row_key"].to(i64)[rows]
            loc = torch.where(key >= 0, key - kb[lev], torch.zeros_like(key))
            slot = md[bs[lev] + (d["ev_s"].to(i64) - lo[lev]) * ndl[lev] + loc]
            if ne and int(slot.min().item()) < 0:
                raise RuntimeError("missing source expansion: blank-pass bug")
            hat_slot = torch.unique(slot)
            src_hat = torch.searchsorted(hat_slot, slot).to(torch.int32)
            h = _to_host({"hat_slot": hat_slot}, dev)
        return src_hat, h["hat_slot"]

    def source_marks(self, lev: int):
        """(cells, global direction ids) of the distinct (source cell, key) pairs of
        the level's M2L events, in (cell, key) order (traversal.py:190-192's source
        marks); None for a level without events."""
        return self._smarks.get(int(lev))

    def close(self):
        self._dev = None
