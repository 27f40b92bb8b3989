"""CPU BASELINE -- TEST / MEASUREMENT INFRASTRUCTURE ONLY, never the product path.

The reference's matvec (helmfmm traversal.py:283-418, restated by
oracle/defmm_oracle.py) laid out so that ONE full-size matvec can be split
over all host cores: ``bench.py --impl reference`` (the reference arm) and the
b200 arm's ``cpu_baseline`` time it; nothing else imports this module.

Same algorithm and arithmetic as the oracle, per event like the reference
(one numpy Hadamard per M2L event, traversal.py:320-342; 1024-target
kernel-matrix blocks per P2P event, traversal.py:303-317; per-cell P2M / M2M /
M2F / F2L / L2L / L2P with the oracle's operator functions), complex128
throughout.  What is new is only the bookkeeping:

* the interaction lists are enumerated once (the plan, outside the timed
  matvec -- the reference's "blank" + "precompute" stages): the dual tree
  traversal's frontier below the top levels is dealt to worker processes;
* expansions live in flat arrays in shared memory (slot = (cell, key));
* a matvec runs as five phases: (A) upward on Morton chunks of subtrees below
  a cut level, in parallel; (A') the top levels; (B) M2L rows + P2P target
  leaves, parallel over target chunks (every output owned by one worker); (C')
  downward top levels; (C) downward subtrees in parallel.

Counts (cells, leaves, symbols, effective_expansions, p2p_pairs, m2l_events)
equal the oracle's (tests/test_cpu_matvec.py), and the potentials equal the
oracle's to rounding.
"""

from __future__ import annotations

import mmap
import os
import time

import numpy as np

from oracle import defmm_oracle as O

_P = None  # the plan, published before the worker pool forks


def _shared(shape, dtype):
    """Zeroed array in anonymous shared memory (visible to forked workers)."""
    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    buf = mmap.mmap(-1, max(n, 1))
    return np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)


def _chunks(weights, parts):
    """Contiguous [lo, hi) chunks of ``weights`` with about equal sums."""
    w = np.asarray(weights, float)
    if w.size == 0:
        return [(0, 0)] * parts
    cs = np.concatenate([[0.0], np.cumsum(w)])
    cuts = np.searchsorted(cs, cs[-1] * np.arange(1, parts) / parts)
    edges = np.concatenate([[0], np.clip(cuts, 0, w.size), [w.size]]).astype(np.int64)
    edges = np.maximum.accumulate(edges)
    return [(int(edges[k]), int(edges[k + 1])) for k in range(parts)]


# ----------------------------------------------------------------------------
# plan: tree, interaction lists, marks, slots, symbols


class _Traversal:
    """MAC / direction decisions of traversal.py:88-113, 187-190, cached per
    (level, gap^2) and (level, translation) -- the same expressions as the
    oracle, evaluated once per distinct argument."""

    def __init__(self, tr, kappa, eta, hf_max, dirs):
        self.tr, self.kappa, self.eta, self.hf_max, self.dirs = tr, kappa, eta, hf_max, dirs
        self.coords = np.asarray(tr.coords, np.int64)
        self.level = np.asarray(tr.level, np.int64)
        self.leaf = np.array([not s for s in tr.sons])
        self._mac, self._key = {}, {}

    def mac(self, t, s):
        ct, cs = self.coords[t], self.coords[s]
        g = [max(abs(int(a) - int(b)) - 1, 0) for a, b in zip(ct, cs)]
        g2 = g[0] * g[0] + g[1] * g[1] + g[2] * g[2]
        lev = int(self.level[t])
        k = (lev, g2)
        v = self._mac.get(k)
        if v is None:
            if lev > self.hf_max:
                v = float(g2) >= 1.0
            else:
                beta = self.tr.side / (1 << lev)
                w = O.SQRT3 * beta / 2.0
                v = bool(max(self.kappa * w * w, 2.0 * w) <= self.eta * (beta * np.sqrt(float(g2))))
            self._mac[k] = v
        return v

    def key(self, t, s):
        lev = int(self.level[t])
        tv = self.coords[t] - self.coords[s]
        k = (lev, int(tv[0]), int(tv[1]), int(tv[2]))
        v = self._key.get(k)
        if v is None:
            e = self.hf_max - lev
            v = (e, O.nearest(self.dirs[e], tv / np.linalg.norm(tv)))
            self._key[k] = v
        return v

    def walk(self, pairs):
        """Depth-first traversal (traversal.py:320-348) from the given pairs:
        (M2L events [t, s, e, i] with e = i = -1 at LF levels, P2P events [t, s])."""
        m2l, p2p = [], []
        sons = self.tr.sons
        stack = list(reversed(pairs))
        while stack:
            t, s = stack.pop()
            if self.mac(t, s):
                if self.level[t] <= self.hf_max:
                    e, i = self.key(t, s)
                else:
                    e = i = -1
                m2l.append((t, s, e, i))
            elif self.leaf[t] or self.leaf[s]:
                p2p.append((t, s))
            else:
                for a in reversed(sons[t]):
                    for b in reversed(sons[s]):
                        stack.append((a, b))
        return (np.asarray(m2l, np.int64).reshape(-1, 4), np.asarray(p2p, np.int64).reshape(-1, 2))


_TRAV = None


def _walk_job(pairs):
    return _TRAV.walk(pairs)


class CpuPlan:
    """Tree + lists + marks + slots + symbols of one single-tree problem."""

    def __init__(self, points, charges, order, ncrit, kappa, eta=1.0, hf_switch=2.0, cap=30, workers=0,
                 parts=1):
        global _TRAV
        t0 = time.perf_counter()
        L = self.L = order
        self.P = P = 2 * L - 1
        tr = self.tr = O.Tree(points, ncrit, cap)
        self.n = tr.points.shape[0]
        self.kappa = kappa
        self.tol = 1e-12 * tr.side  # traversal.py:465-467
        hf_max = -1
        if kappa > 0:  # traversal.py:145-160
            for lev in range(tr.depth + 1):
                if kappa * (np.sqrt(3.0) * (tr.side / (1 << lev)) / 2.0) >= hf_switch:
                    hf_max = lev
                else:
                    break
        self.hf_max = hf_max
        self.dirs, self.fathers = O.direction_levels(hf_max) if hf_max >= 0 else (None, None)
        trav = _TRAV = _Traversal(tr, kappa, eta, hf_max, self.dirs)
        # -- enumerate the interaction lists: breadth-first on the top levels,
        # the frontier dealt to the workers (depth-first below)
        frontier, m2l, p2p = [(0, 0)], [], []
        while frontier and len(frontier) < 256 * max(parts, 1):
            nxt = []
            for t, s in frontier:
                if trav.mac(t, s):
                    e, i = trav.key(t, s) if trav.level[t] <= hf_max else (-1, -1)
                    m2l.append(np.array([[t, s, e, i]], np.int64))
                elif trav.leaf[t] or trav.leaf[s]:
                    p2p.append(np.array([[t, s]], np.int64))
                else:
                    nxt.extend((a, b) for a in tr.sons[t] for b in tr.sons[s])
            frontier = nxt
        jobs = [frontier[a:b] for a, b in _chunks(np.ones(len(frontier)), max(4 * parts, 1)) if b > a]
        if workers and jobs:
            import multiprocessing as mp

            with mp.get_context("fork").Pool(workers) as pool:  # forked now: sees _TRAV
                res = pool.map(_walk_job, jobs)
        else:
            res = [_walk_job(j) for j in jobs]
        _TRAV = None
        m2l += [r[0] for r in res]
        p2p += [r[1] for r in res]
        ev = np.concatenate(m2l) if m2l else np.zeros((0, 4), np.int64)
        pp = np.concatenate(p2p) if p2p else np.zeros((0, 2), np.int64)
        self._slots(ev, pp)
        self.timings = {"plan": time.perf_counter() - t0}
        self.set_charges(charges)

    # ------------------------------------------------------------------
    def _slots(self, ev, pp):
        """Marks, expansion slots, symbols and per-row / per-leaf lists, with
        keys coded as ints: -1 = LF (None), else dir_off[e] + i."""
        tr, L, P, hf_max = self.tr, self.L, self.P, self.hf_max
        ncell = len(tr.level)
        level = np.asarray(tr.level, np.int64)
        coords = np.asarray(tr.coords, np.int64)
        nd = [0] if hf_max < 0 else [d.shape[0] for d in self.dirs]
        off = np.concatenate([[0], np.cumsum(nd)]).astype(np.int64)
        self.code_e = np.repeat(np.arange(len(nd)), nd)  # code -> (e, i)
        self.code_i = np.arange(int(off[-1])) - off[self.code_e]
        fcode = np.full(int(off[-1]), -1, np.int64)  # code -> father code (e >= 1)
        for e in range(1, len(nd)):
            fcode[off[e]:off[e + 1]] = off[e - 1] + np.asarray(self.fathers[e])
        code = np.where(ev[:, 2] >= 0, off[np.maximum(ev[:, 2], 0)] + ev[:, 3], -1)
        sons_ptr = np.zeros(ncell + 1, np.int64)
        sons_ptr[1:] = np.cumsum([len(x) for x in tr.sons])
        sons = np.array([x for xs in tr.sons for x in xs], np.int64)

        def push(cells, codes, hf_only):
            """(cell, code) pairs plus everything pushed to the sons, level by
            level (traversal.py:203-213 for marks, 355-391 for local keys)."""
            out_c, out_k = [cells], [codes]
            cur_c, cur_k = cells, codes
            for _ in range(int(level.max()) + 1):
                keep = np.ones(cur_c.shape[0], bool)
                if hf_only:
                    keep = (level[cur_c] <= hf_max) & (cur_k >= 0) & (self.code_e[np.maximum(cur_k, 0)] > 0)
                cc, kk = cur_c[keep], cur_k[keep]
                ns = sons_ptr[cc + 1] - sons_ptr[cc]
                rep_c = np.repeat(cc, ns)
                idx = np.repeat(sons_ptr[cc] - np.concatenate([[0], np.cumsum(ns)[:-1]]), ns) + np.arange(int(ns.sum()))
                sc = sons[idx]
                kk = np.repeat(kk, ns)
                if hf_only:
                    sk = fcode[kk]
                else:  # locals: HF son of an HF key -> father key, else LF
                    sk = np.where((kk >= 0) & (level[sc] <= hf_max), fcode[np.maximum(kk, 0)], -1)
                if sc.size == 0:
                    break
                u = np.unique(sc * (off[-1] + 1) + sk + 1)
                cur_c, cur_k = u // (off[-1] + 1), u % (off[-1] + 1) - 1
                out_c.append(cur_c)
                out_k.append(cur_k)
            u = np.unique(np.concatenate(out_c) * (off[-1] + 1) + np.concatenate(out_k) + 1)
            return u // (off[-1] + 1), u % (off[-1] + 1) - 1

        hf_ev = code >= 0
        mc, mk = push(np.concatenate([ev[hf_ev, 0], ev[hf_ev, 1]]), np.concatenate([code[hf_ev], code[hf_ev]]), True)
        # multipole slots (traversal.py:224-280): HF cells their sorted marks,
        # LF cells one (key None); sorted by (cell, code) = the oracle's order
        lf = np.nonzero(level > hf_max)[0]
        hf_sel = level[mc] <= hf_max
        mc = np.concatenate([mc[hf_sel], lf])
        mk = np.concatenate([mk[hf_sel], np.full(lf.shape[0], -1, np.int64)])
        o = np.lexsort((mk, mc))
        mc, mk = mc[o], mk[o]
        W = off[-1] + 2
        mkey = mc * W + mk + 1
        self.n_mult = mc.shape[0]
        self.m_slot = {(int(c), self._key(int(k))): j for j, (c, k) in enumerate(zip(mc.tolist(), mk.tolist()))}
        self.mkeys = [[] for _ in range(ncell)]
        for c, k in zip(mc.tolist(), mk.tolist()):
            self.mkeys[c].append(self._key(k))
        # symbols: one per distinct (level, translation), from its canonical one
        tv = coords[ev[:, 0]] - coords[ev[:, 1]]
        keyarr = np.concatenate([level[ev[:, 0]][:, None], tv], 1)
        uniq, inv = np.unique(keyarr, axis=0, return_inverse=True)
        canon, self.sym = {}, np.empty((uniq.shape[0], P**3), complex)
        for j, (lv, a, b, c) in enumerate(uniq.tolist()):
            cn, rid = O.canonicalize((a, b, c))
            base = canon.get((lv, cn))
            if base is None:
                base = canon[(lv, cn)] = O.symbol(self.kappa, self.tol, cn, tr.side / (1 << lv), L)
            self.sym[j] = base if cn == (a, b, c) else base[O.freq_perm(L, rid)]
        self.n_canon = len(canon)
        # M2L rows (target cell, key) -> entries (source multipole slot, symbol)
        src = np.searchsorted(mkey, ev[:, 1] * W + code + 1)
        rkey = ev[:, 0] * W + code + 1
        rows, row = np.unique(rkey, return_inverse=True)
        o = np.argsort(row, kind="stable")
        self.row_ptr = np.searchsorted(row[o], np.arange(rows.shape[0] + 1))
        self.ev_src, self.ev_sym = src[o], inv.reshape(-1)[o]
        self.row_cell = rows // W
        self.row_code = rows % W - 1
        self.l_slot = {(int(c), self._key(int(k))): r for r, (c, k) in enumerate(zip(self.row_cell.tolist(),
                                                                                     self.row_code.tolist()))}
        # local slots: rows' keys plus the keys pushed down by L2L (traversal.py:355-391)
        lc, lk = push(self.row_cell, self.row_code, False)
        korder = lambda k: (k is not None, k)  # noqa: E731  (oracle's downward order)
        self.lkeys = [[] for _ in range(ncell)]
        for c, k in zip(lc.tolist(), lk.tolist()):
            self.lkeys[c].append(self._key(k))
        self.lkeys = [sorted(ks, key=korder) for ks in self.lkeys]
        self.loc_slot = {}
        for c in range(ncell):
            for k in self.lkeys[c]:
                self.loc_slot[(c, k)] = len(self.loc_slot)
        # P2P: every event split into its target leaves (one owner per particle)
        start, stop = np.asarray(tr.start, np.int64), np.asarray(tr.stop, np.int64)
        self.p2p_pairs = int(((stop - start)[pp[:, 0]] * (stop - start)[pp[:, 1]]).sum()) if pp.size else 0
        leafs = np.nonzero(sons_ptr[1:] == sons_ptr[:-1])[0]  # Morton order = particle order
        lstart = start[leafs]
        p2p = {}
        for t, s in pp.tolist():
            a, b = np.searchsorted(lstart, start[t]), np.searchsorted(lstart, stop[t])
            for lf in leafs[a:b].tolist():
                p2p.setdefault(lf, []).append((int(start[s]), int(stop[s])))
        self.p2p = p2p
        self.counts = {
            "cells": ncell,
            "leaves": int(leafs.shape[0]),
            "symbols": self.n_canon,
            "effective_expansions": int(self.n_mult),
            "p2p_pairs": self.p2p_pairs,
            "m2l_events": int(ev.shape[0]),
        }
        # shared buffers
        self.mult = _shared((self.n_mult, L**3), complex)
        self.mhat = _shared((self.n_mult, P**3), complex)
        self.lhat = _shared((len(self.l_slot), P**3), complex)
        self.loc = _shared((len(self.loc_slot), L**3), complex)
        self.pot = _shared((self.n,), complex)
        self.q = _shared((self.n,), complex)

    def _key(self, code):
        return None if code < 0 else (int(self.code_e[code]), int(self.code_i[code]))

    def set_charges(self, charges):
        self.q[:] = np.asarray(charges, complex)[self.tr.perm]

    # ------------------------------------------------------------------
    def partition(self, parts):
        """Work split of one matvec into ``parts`` chunks (phases A, B, C)."""
        tr = self.tr
        level = np.asarray(tr.level, np.int64)
        ncell = level.shape[0]
        cnt = np.bincount(level)
        cut = next((lv for lv in range(len(cnt)) if cnt[lv] >= 8 * parts), len(cnt) - 1)
        self.cut = cut
        anc = np.full(ncell, -1, np.int64)  # cut-level ancestor
        parent = np.full(ncell, -1, np.int64)
        for c in range(ncell):
            for s in tr.sons[c]:
                parent[s] = c
        for c in range(ncell):
            if level[c] == cut:
                anc[c] = c
            elif level[c] > cut:
                anc[c] = anc[parent[c]]
        self.parent = parent
        cut_cells = np.nonzero(level == cut)[0]
        npart = np.asarray(tr.stop)[cut_cells] - np.asarray(tr.start)[cut_cells]
        owner = np.full(ncell, -1, np.int64)
        for k, (a, b) in enumerate(_chunks(npart, parts)):
            owner[cut_cells[a:b]] = k
        sub_owner = np.where(anc >= 0, owner[np.maximum(anc, 0)], -1)
        bottom_up = np.lexsort((np.arange(ncell), -level))
        top_down = np.lexsort((np.arange(ncell), level))
        self.up_cells = [bottom_up[sub_owner[bottom_up] == k] for k in range(parts)]
        self.down_cells = [top_down[sub_owner[top_down] == k] for k in range(parts)]
        self.up_top = bottom_up[sub_owner[bottom_up] < 0]
        self.down_top = top_down[sub_owner[top_down] < 0]
        # phase B: M2L rows + P2P leaves, cost-balanced contiguous target chunks
        P3 = self.P**3
        rows_of = {}
        for r, t in enumerate(self.row_cell.tolist()):
            rows_of.setdefault(t, []).append(r)
        cost = np.zeros(ncell)
        for t, rs in rows_of.items():
            cost[t] += sum(int(self.row_ptr[r + 1] - self.row_ptr[r]) for r in rs) * P3
        for lf, runs in self.p2p.items():
            cost[lf] += (tr.stop[lf] - tr.start[lf]) * sum(b - a for a, b in runs)
        self.b_parts = []
        for a, b in _chunks(cost, parts):
            cells = range(a, b)
            self.b_parts.append(([r for c in cells for r in rows_of.get(c, [])],
                                 [c for c in cells if c in self.p2p]))
        self.parts = parts

    # ------------------------------------------------------------------
    # matvec phases (each touches only the slots it owns)
    def _upward_cells(self, cells):
        tr, L, kappa = self.tr, self.L, self.kappa
        pos, q = tr.points, self.q
        for c in cells.tolist():
            lev = tr.level[c]
            hf = lev <= self.hf_max
            beta = tr.beta(lev)
            al = tr.alpha(c)
            keys = self.mkeys[c]
            if not keys:
                continue
            if not tr.sons[c]:  # traversal.py:224-236
                sl = slice(tr.start[c], tr.stop[c])
                for k in keys:
                    u = self.dirs[k[0]][k[1]] if hf else None
                    self.mult[self.m_slot[(c, k)]] = O.p2m(al, beta, L, pos[sl], q[sl], kappa, u) if hf else \
                        O.p2m(al, beta, L, pos[sl], q[sl])
            else:  # traversal.py:239-280
                fgrid = al + beta * O.ref_grid(L)
                acc = {k: np.zeros(L**3, complex) for k in keys}
                for s in tr.sons[c]:
                    fac = tuple(O.m2m_axis(L, int(o)) for o in np.asarray(tr.coords[s]) - 2 * np.asarray(tr.coords[c]))
                    if hf:
                        sgrid = tr.alpha(s) + tr.beta(lev + 1) * O.ref_grid(L)
                        for k in keys:
                            sk = (k[0] - 1, int(self.fathers[k[0]][k[1]])) if lev + 1 <= self.hf_max else None
                            u = self.dirs[k[0]][k[1]]
                            col = self.mult[self.m_slot[(s, sk)]] * np.conj(O.plane_wave(sgrid, kappa, u))
                            acc[k] += O.kron3(fac, col[:, None])[:, 0] * O.plane_wave(fgrid, kappa, u)
                    else:
                        acc[None] += O.kron3(fac, self.mult[self.m_slot[(s, None)]][:, None])[:, 0]
                for k in keys:
                    self.mult[self.m_slot[(c, k)]] = acc[k]
            for k in keys:  # traversal.py:293-296: every multipole is transformed
                j = self.m_slot[(c, k)]
                self.mhat[j] = O.m2f(self.mult[j], L)

    def _m2l_p2p(self, rows, leaves):
        sym, mhat, src, sid, ptr = self.sym, self.mhat, self.ev_src, self.ev_sym, self.row_ptr
        for r in rows:  # traversal.py:320-342, one Hadamard per event
            acc = self.lhat[r]
            acc[:] = 0.0
            for j in range(int(ptr[r]), int(ptr[r + 1])):
                acc += sym[sid[j]] * mhat[src[j]]
        tr, pos, q, pot = self.tr, self.tr.points, self.q, self.pot
        for lf in leaves:  # traversal.py:303-317 (1024-target blocks)
            t0, t1 = tr.start[lf], tr.stop[lf]
            for a, b in self.p2p[lf]:
                for lo in range(t0, t1, 1024):
                    hi = min(lo + 1024, t1)
                    pot[lo:hi] += O.kernel_matrix(pos[lo:hi], pos[a:b], self.kappa, self.tol) @ q[a:b]

    def _downward_cells(self, cells):
        tr, L, kappa = self.tr, self.L, self.kappa
        pos = tr.points
        for c in cells.tolist():
            lev = tr.level[c]
            beta = tr.beta(lev)
            keys = self.lkeys[c]
            for k in keys:  # traversal.py:405-414: F2L of every accumulated spectrum
                r = self.l_slot.get((c, k))
                if r is not None:
                    self.loc[self.loc_slot[(c, k)]] += O.f2l(self.lhat[r], L)
            if not keys:
                continue
            al = tr.alpha(c)
            if not tr.sons[c]:  # traversal.py:394-402
                sl = slice(tr.start[c], tr.stop[c])
                for k in keys:
                    u = self.dirs[k[0]][k[1]] if k is not None else None
                    loc = self.loc[self.loc_slot[(c, k)]]
                    self.pot[sl] += O.l2p(al, beta, L, pos[sl], loc, kappa, u) if u is not None else \
                        O.l2p(al, beta, L, pos[sl], loc)
                continue
            fgrid = al + beta * O.ref_grid(L)  # traversal.py:355-391
            for s in tr.sons[c]:
                fac = tuple(O.m2m_axis(L, int(o)).T for o in np.asarray(tr.coords[s]) - 2 * np.asarray(tr.coords[c]))
                sgrid = tr.alpha(s) + tr.beta(lev + 1) * O.ref_grid(L)
                for k in keys:
                    loc = self.loc[self.loc_slot[(c, k)]]
                    if k is None:
                        inc, sk = O.kron3(fac, loc[:, None])[:, 0], None
                    else:
                        u = self.dirs[k[0]][k[1]]
                        col = loc * np.conj(O.plane_wave(fgrid, kappa, u))
                        inc = O.kron3(fac, col[:, None])[:, 0] * O.plane_wave(sgrid, kappa, u)
                        sk = (k[0] - 1, int(self.fathers[k[0]][k[1]])) if lev + 1 <= self.hf_max else None
                    self.loc[self.loc_slot[(s, sk)]] += inc

    def matvec(self, pool=None, only=None):
        """One matvec with the loaded charges; returns potentials (caller order).
        ``only = k``: run just chunk k of phases A, B, C in this process (the
        one-core sample of bench.py's cpu_baseline) and return its phase times."""
        if only is not None:
            tm = {}
            t0 = time.perf_counter()
            self._upward_cells(self.up_cells[only])
            tm["upward"] = time.perf_counter() - t0
            t0 = time.perf_counter()
            self._m2l_p2p(*self.b_parts[only])
            tm["m2l_p2p"] = time.perf_counter() - t0
            t0 = time.perf_counter()
            self._downward_cells(self.down_cells[only])
            tm["downward"] = time.perf_counter() - t0
            return tm
        self.pot[:] = 0.0
        self.loc[:] = 0.0
        run = (lambda f, n: pool.map(f, range(n))) if pool is not None else (lambda f, n: [f(k) for k in range(n)])
        run(_phase_a, self.parts)
        self._upward_cells(self.up_top)
        run(_phase_b, self.parts)
        self._downward_cells(self.down_top)
        run(_phase_c, self.parts)
        out = np.empty(self.n, complex)
        out[self.tr.perm] = self.pot
        return out


def _phase_a(k):
    _P._upward_cells(_P.up_cells[k])


def _phase_b(k):
    _P._m2l_p2p(*_P.b_parts[k])


def _phase_c(k):
    _P._downward_cells(_P.down_cells[k])


def make(points, charges, order, ncrit, kappa, parts, workers=None):
    """(plan, pool): the plan built with a fork pool of ``workers`` processes
    (None: no pool), partitioned into ``parts`` chunks; the pool used for the
    matvec phases is forked after the plan so it sees the shared buffers."""
    import multiprocessing as mp

    from threadpoolctl import threadpool_limits

    global _P
    for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[var] = "1"
    threadpool_limits(limits=1)  # one BLAS thread per process (forked workers inherit it)
    ctx = mp.get_context("fork")
    plan = CpuPlan(points, charges, order, ncrit, kappa, workers=workers or 0, parts=parts)
    plan.partition(parts)
    _P = plan
    pool = ctx.Pool(workers) if workers else None
    return plan, pool


def _main():
    """``python -m oracle.cpu_matvec --workload cfg2 --parts 16 --sample``:
    the plan built with all cores, then ONE core runs chunk parts // 2 of
    the matvec's three parallel phases; prints the cpu_baseline JSON
    (particles/s extrapolated to the whole matvec on one core)."""
    import argparse
    import json
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2202_04894_b200.workloads import make_workload

    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--parts", type=int, default=16)
    ap.add_argument("--sample", action="store_true")
    a = ap.parse_args()
    pts, q, kappa, w = make_workload(a.workload)
    cores = max(1, min(os.cpu_count() or 1, 128))
    plan, pool = make(pts, q, w.order, w.ncrit, kappa, parts=a.parts, workers=cores)
    pool.close()
    k = a.parts // 2
    tm = plan.matvec(only=k)
    t_one = a.parts * sum(tm.values())
    print(json.dumps({"value": pts.shape[0] / t_one, "unit": "particles/s", "cores": 1, "kind": "port",
                      "sample": (f"1 core ran chunk {k} of {a.parts} work-balanced Morton chunks of one full "
                                 f"{w.name} matvec (N={pts.shape[0]}, complex128; upward {tm['upward']:.2f} s, "
                                 f"M2L+P2P {tm['m2l_p2p']:.2f} s, downward {tm['downward']:.2f} s), x{a.parts}; "
                                 f"plan built beforehand in {plan.timings['plan']:.1f} s on {cores} cores"),
                      "phase_s": tm}), flush=True)


if __name__ == "__main__":
    _main()
