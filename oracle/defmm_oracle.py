"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY, never the product path.

A numpy restatement of the reference's (helmfmm, /root/reference/pkg/src)
directional FFT-accelerated FMM matvec for G(r) = e^{i kappa r}/(4 pi r).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this module, and only as the checker or as
the timed CPU baseline.  The B200 product path (paper_2202_04894_b200) never
imports it and fails loudly when its CUDA library is missing.

Parity pinning: this restatement is checked bit-for-bit (discrete decisions:
tree, MAC, directions, interaction lists, counts) and to <= 1e-12 (floating
point) against golden vectors produced by the reference itself
(tests/golden/make_golden.py, make_golden_large.py -> tests/golden/*.npz; see
tests/test_oracle_golden.py).

Every function cites the reference file:line it restates.  The structure is
deliberately different from the reference (flat per-cell arrays, integer cell
ids, dict-of-slot expansions) -- only the arithmetic and the decisions follow it.
"""

from __future__ import annotations

import itertools
import time
from functools import lru_cache

import numpy as np

SQRT3 = float(np.sqrt(3.0))  # tree.py:33
FACES = ((0, 1), (0, -1), (1, 1), (1, -1), (2, 1), (2, -1))  # directions.py:24


# ----------------------------------------------------------------------------
# kernel (kernel.py)


def kernel_of_distance(r, kappa, tol):
    """kernel.py:37-43: e^{i kappa r}/(4 pi r), 0 where r < tol."""
    r = np.asarray(r, dtype=float)
    ok = r >= tol
    rs = np.where(ok, r, 1.0)
    return np.where(ok, np.exp(1j * kappa * rs) / (4.0 * np.pi * rs), 0.0)


def kernel_matrix(x, y, kappa, tol):
    """kernel.py:52-55."""
    d = x[:, None, :] - y[None, :, :]
    return kernel_of_distance(np.sqrt(np.einsum("ijk,ijk->ij", d, d)), kappa, tol)


def direct_sum(targets, sources, charges, kappa, tol, block=512):
    """kernel.py:58-75 (blocked O(M N) oracle)."""
    targets = np.atleast_2d(np.asarray(targets, float))
    sources = np.atleast_2d(np.asarray(sources, float))
    q = np.asarray(charges, complex)
    out = np.zeros(targets.shape[0], complex)
    for lo in range(0, targets.shape[0], block):
        hi = min(lo + block, targets.shape[0])
        out[lo:hi] = kernel_matrix(targets[lo:hi], sources, kappa, tol) @ q
    return out


def rel_l2(ref, app):
    """kernel.py:85-98 (rel_l2 member)."""
    return float(np.linalg.norm(app - ref) / np.linalg.norm(ref))


# ----------------------------------------------------------------------------
# equispaced interpolation (interpolation.py)


@lru_cache(maxsize=None)
def nodes(L):
    """interpolation.py:51-56."""
    return np.linspace(0.0, 1.0, L)


def lagrange_matrix(L, x):
    """(len(x), L) values S_k(x_j); interpolation.py:59-78."""
    x = np.asarray(x, float)
    nd = nodes(L)
    out = np.empty((x.shape[0], L))
    for k in range(L):
        v = np.ones_like(x)
        for j in range(L):
            if j != k:
                v = v * (x - nd[j]) / (nd[k] - nd[j])
        out[:, k] = v
    return out


def tensor_basis(L, unit):
    """(n, L^3) C-order tensor basis; interpolation.py:94-101."""
    ex, ey, ez = (lagrange_matrix(L, unit[:, a]) for a in range(3))
    return (ex[:, :, None, None] * ey[:, None, :, None] * ez[:, None, None, :]).reshape(unit.shape[0], -1)


@lru_cache(maxsize=None)
def ref_grid(L):
    """(L^3, 3) reference grid, axis 0 slowest; interpolation.py:81-86."""
    n = nodes(L)
    return np.stack(np.meshgrid(n, n, n, indexing="ij"), -1).reshape(-1, 3)


def plane_wave(x, kappa, u):
    """interpolation.py:104-106 (absolute coordinates)."""
    return np.exp(1j * kappa * (np.atleast_2d(x) @ np.asarray(u, float)))


def p2m(alpha, beta, L, pos, q, kappa=0.0, u=None):
    """interpolation.py:109-124."""
    b = tensor_basis(L, (pos - alpha) / beta)
    qq = np.asarray(q, complex)
    if u is not None:
        qq = qq * np.conj(plane_wave(pos, kappa, u))
    m = b.T @ qq
    if u is not None:
        m = m * plane_wave(alpha + beta * ref_grid(L), kappa, u)
    return m


def l2p(alpha, beta, L, pos, loc, kappa=0.0, u=None):
    """interpolation.py:127-137."""
    b = tensor_basis(L, (pos - alpha) / beta)
    c = np.asarray(loc, complex)
    if u is not None:
        c = c * np.conj(plane_wave(alpha + beta * ref_grid(L), kappa, u))
    v = b @ c
    if u is not None:
        v = v * plane_wave(pos, kappa, u).ravel()
    return v


@lru_cache(maxsize=None)
def m2m_axis(L, o):
    """A[l, r] = S_l((o + x_r)/2) for one axis; interpolation.py:140-148."""
    return lagrange_matrix(L, (o + nodes(L)) / 2.0).T.copy()


def kron3(f, x):
    """(f0 (x) f1 (x) f2) x for stacked columns x (L^3, m); interpolation.py:157-173."""
    L = f[0].shape[0]
    t = x.reshape(L, L, L, -1)
    t = np.einsum("ai,ijkm->ajkm", f[0], t)
    t = np.einsum("bj,ajkm->abkm", f[1], t)
    t = np.einsum("ck,abkm->abcm", f[2], t)
    return t.reshape(L**3, -1)


# ----------------------------------------------------------------------------
# Fourier-domain M2L (fourier.py)


def m2f(v, L):
    """Zero-pad into the P^3 corner + unitary fftn; fourier.py:67-72."""
    P = 2 * L - 1
    buf = np.zeros((P, P, P), complex)
    buf[:L, :L, :L] = np.asarray(v).reshape(L, L, L)
    return (np.fft.fftn(buf) / float(P) ** 1.5).ravel()


def f2l(w, L):
    """Unitary ifftn + crop; fourier.py:74-80."""
    P = 2 * L - 1
    out = np.fft.ifftn(np.asarray(w).reshape(P, P, P)) * float(P) ** 1.5
    return np.ascontiguousarray(out[:L, :L, :L]).ravel()


@lru_cache(maxsize=None)
def group48():
    """Signed permutation matrices in the reference's order; fourier.py:90-101."""
    mats = []
    for perm in itertools.permutations(range(3)):
        for sg in itertools.product((1, -1), repeat=3):
            m = np.zeros((3, 3), np.int64)
            for a in range(3):
                m[a, perm[a]] = sg[a]
            mats.append(m)
    return tuple(mats)


def canonicalize(t):
    """(|t| sorted descending, first rid with R canon = t); fourier.py:104-120."""
    t = np.asarray(t, np.int64)
    if not np.any(t):
        raise ValueError("zero translation cannot be canonicalized")
    c = np.sort(np.abs(t))[::-1].copy()
    for rid, r in enumerate(group48()):
        if np.array_equal(r @ c, t):
            return tuple(int(v) for v in c), rid
    raise AssertionError("unreachable")


@lru_cache(maxsize=None)
def freq_perm(L, rid):
    """fourier.py:123-143: D_t[j] = D_canon[perm[j]]."""
    P = 2 * L - 1
    f = np.stack(np.meshgrid(*([np.arange(P)] * 3), indexing="ij"), -1).reshape(-1, 3)
    mp = (f @ group48()[rid]) % P
    return (mp[:, 0] * P + mp[:, 1]) * P + mp[:, 2]


def symbol(kappa, tol, t, beta, L):
    """Unnormalised fftn of G(beta (t + z)) on the difference grid;
    fourier.py:156-183."""
    P = 2 * L - 1
    off = np.arange(P)
    off = np.where(off < L, off, off - P) * (1.0 / (L - 1))
    zx, zy, zz = np.meshgrid(t[0] + off, t[1] + off, t[2] + off, indexing="ij")
    r = beta * np.sqrt(zx**2 + zy**2 + zz**2)
    if np.min(r) < tol:
        raise ValueError("kernel singularity inside the M2L stencil: MAC violated")
    return np.fft.fftn(kernel_of_distance(r, kappa, tol)).ravel()


def dense_m2l(kappa, tol, t, beta, L):
    """fourier.py:199-208 (test oracle for the FFT path)."""
    g = ref_grid(L)
    d = (np.asarray(t, float) + g[:, None, :] - g[None, :, :]) * beta
    return kernel_of_distance(np.sqrt(np.einsum("ijk,ijk->ij", d, d)), kappa, tol)


# ----------------------------------------------------------------------------
# directions (directions.py)


def direction_levels(emax):
    """6*4^e unit directions + father indices; directions.py:52-75."""
    dirs, fathers = [], []
    for e in range(emax + 1):
        m = 1 << e
        d = np.empty((6 * m * m, 3))
        fa = np.full(6 * m * m, -1, np.int64)
        k = 0
        for f, (axis, sign) in enumerate(FACES):
            rest = [a for a in range(3) if a != axis]
            for i in range(m):
                for j in range(m):
                    p = np.empty(3)
                    p[axis] = float(sign)
                    p[rest[0]] = -1.0 + (2.0 * i + 1.0) / m
                    p[rest[1]] = -1.0 + (2.0 * j + 1.0) / m
                    d[k] = p / np.linalg.norm(p)
                    if e:
                        fa[k] = (f * (m // 2) + i // 2) * (m // 2) + j // 2
                    k += 1
        dirs.append(d)
        fathers.append(fa)
    return dirs, fathers


def nearest(dirs_e, v):
    """First argmin of squared distance; directions.py:78-89."""
    return int(np.argmin(np.sum((dirs_e - v) ** 2, axis=1)))


# ----------------------------------------------------------------------------
# octree (tree.py, geometry.py)


def root_box(points):
    """(lower, side) of geometry.py:82-97's centroid cube."""
    c = points.mean(axis=0)
    half = np.max(np.abs(points - c)) if points.shape[0] > 1 else 0.5
    if half == 0.0:
        half = 0.5
    half = half * (1.0 + 1e-6)
    return c - half, 2.0 * half


class Tree:
    """Flat cell arrays built by tree.py:132-213's recursive stable split."""

    def __init__(self, points, ncrit, cap=30, box=None):
        pts = np.atleast_2d(np.asarray(points, float))
        self.lower, self.side = root_box(pts) if box is None else box
        n = pts.shape[0]
        self.perm = np.arange(n)
        work = pts.copy()
        self.level, self.coords, self.start, self.stop, self.sons = [], [], [], [], []

        def new(lev, co, a, b):
            self.level.append(lev)
            self.coords.append(co)
            self.start.append(a)
            self.stop.append(b)
            self.sons.append([])
            return len(self.level) - 1

        def split(c):
            a, b, lev = self.start[c], self.stop[c], self.level[c]
            if b - a <= ncrit or lev >= cap:
                return
            beta = self.side / (1 << lev)
            ctr = (self.lower + self.coords[c] * beta) + 0.5 * beta
            p = work[a:b]
            oc = (p[:, 0] >= ctr[0]).astype(np.int64) * 4 + (p[:, 1] >= ctr[1]).astype(np.int64) * 2 + (p[:, 2] >= ctr[2]).astype(np.int64)
            o = np.argsort(oc, kind="stable")
            work[a:b] = p[o]
            self.perm[a:b] = self.perm[a:b][o]
            oc = oc[o]
            cuts = np.searchsorted(oc, np.arange(9))
            for k in range(8):
                if cuts[k] == cuts[k + 1]:
                    continue
                bit = np.array([(k >> 2) & 1, (k >> 1) & 1, k & 1], np.int64)
                s = new(lev + 1, self.coords[c] * 2 + bit, a + int(cuts[k]), a + int(cuts[k + 1]))
                self.sons[c].append(s)
                split(s)

        split(new(0, np.zeros(3, np.int64), 0, n))
        self.points = work
        self.depth = max(self.level)

    def beta(self, lev):
        return self.side / (1 << lev)

    def alpha(self, c):
        return self.lower + self.coords[c] * self.beta(self.level[c])

    def levels(self):
        """Cells per level in creation (= Morton) order."""
        out = [[] for _ in range(self.depth + 1)]
        for c, lev in enumerate(self.level):
            out[lev].append(c)
        return out


# ----------------------------------------------------------------------------
# the matvec driver (traversal.py)


def run(points, charges, order=5, ncrit=64, eta=1.0, kappa=0.0, hf_switch=2.0, cap=30, events=None):
    """Single-tree FMM (targets is sources); traversal.py:432-506.

    Returns (potentials in input order, counts, hf_max, timings).
    ``events`` (optional list) receives ("M2L"|"P2P", t, s, key) tuples.
    """
    L = order
    P = 2 * L - 1
    tm = {}
    t0 = time.perf_counter()
    tr = Tree(points, ncrit, cap)
    q = np.asarray(charges, complex)[tr.perm]
    pos = tr.points
    tm["tree"] = time.perf_counter() - t0
    tol = 1e-12 * tr.side  # traversal.py:465-467

    # hf_max scan; traversal.py:145-160
    hf_max = -1
    if kappa > 0:
        for lev in range(tr.depth + 1):
            w = np.sqrt(3.0) * (tr.side / (1 << lev)) / 2.0
            if kappa * w >= hf_switch:
                hf_max = lev
            else:
                break
    dirs, fathers = direction_levels(hf_max) if hf_max >= 0 else (None, None)

    def is_hf(lev):
        return lev <= hf_max

    def mac(t, s):  # traversal.py:88-113, 168-171
        g = np.maximum(np.abs(tr.coords[t] - tr.coords[s]) - 1, 0)
        g2 = float(g @ g)
        lev = tr.level[t]
        if not is_hf(lev):
            return g2 >= 1.0
        beta = tr.side / (1 << lev)
        w = SQRT3 * beta / 2.0
        return max(kappa * w * w, 2.0 * w) <= eta * (beta * np.sqrt(g2))

    def key_of(t, s):  # traversal.py:187-190
        tv = tr.coords[t] - tr.coords[s]
        e = hf_max - tr.level[t]
        return (e, nearest(dirs[e], tv / np.linalg.norm(tv)))

    ncell = len(tr.level)
    marks = [set() for _ in range(ncell)]
    canon_cache, deriv_cache = {}, {}

    def get_symbol(lev, tv):  # fourier.py:233-247
        k = (lev, tuple(int(v) for v in tv))
        d = deriv_cache.get(k)
        if d is None:
            c, rid = canonicalize(tv)
            base = canon_cache.get((lev, c))
            if base is None:
                base = symbol(kappa, tol, c, tr.side / (1 << lev), L)
                canon_cache[(lev, c)] = base
            d = base if c == k[1] else base[freq_perm(L, rid)]
            deriv_cache[k] = d
        return d

    # blank passes: traversal.py:182-213
    t0 = time.perf_counter()
    pre = 0.0

    def blank(t, s):
        nonlocal pre
        if not is_hf(tr.level[t]):
            return
        if mac(t, s):
            k = key_of(t, s)
            marks[t].add(k)
            marks[s].add(k)
            t1 = time.perf_counter()
            get_symbol(tr.level[t], tr.coords[t] - tr.coords[s])
            pre += time.perf_counter() - t1
            return
        for a in tr.sons[t]:
            for b in tr.sons[s]:
                blank(a, b)

    blank(0, 0)

    def push_marks(c):
        if not is_hf(tr.level[c]):
            return
        for e, i in sorted(marks[c]):
            if e > 0:
                for s in tr.sons[c]:
                    marks[s].add((e - 1, int(fathers[e][i])))
        for s in tr.sons[c]:
            push_marks(s)

    push_marks(0)
    tm["blank"] = time.perf_counter() - t0

    # upward: traversal.py:224-296
    t0 = time.perf_counter()
    mult = [dict() for _ in range(ncell)]
    levels = tr.levels()
    for lev in range(tr.depth, -1, -1):
        beta = tr.beta(lev)
        for c in levels[lev]:
            al = tr.alpha(c)
            if not tr.sons[c]:
                sl = slice(tr.start[c], tr.stop[c])
                if is_hf(lev):
                    for k in sorted(marks[c]):
                        mult[c][k] = p2m(al, beta, L, pos[sl], q[sl], kappa, dirs[k[0]][k[1]])
                else:
                    mult[c][None] = p2m(al, beta, L, pos[sl], q[sl])
                continue
            keys = sorted(marks[c]) if is_hf(lev) else [None]
            if is_hf(lev) and not keys:
                continue
            fgrid = al + beta * ref_grid(L)
            acc = {k: np.zeros(L**3, complex) for k in keys}
            for s in tr.sons[c]:
                oct_ = tuple(int(v) for v in tr.coords[s] - 2 * tr.coords[c])
                fac = tuple(m2m_axis(L, o) for o in oct_)
                if is_hf(lev):
                    sgrid = tr.alpha(s) + tr.beta(lev + 1) * ref_grid(L)
                    for k in keys:
                        sk = (k[0] - 1, int(fathers[k[0]][k[1]])) if is_hf(lev + 1) else None
                        if sk not in mult[s]:
                            raise RuntimeError("missing son expansion: blank-pass inconsistency")
                        u = dirs[k[0]][k[1]]
                        col = mult[s][sk] * np.conj(plane_wave(sgrid, kappa, u))
                        acc[k] += kron3(fac, col[:, None])[:, 0] * plane_wave(fgrid, kappa, u)
                else:
                    acc[None] += kron3(fac, mult[s][None][:, None])[:, 0]
            mult[c].update(acc)
    mhat = [{k: m2f(v, L) for k, v in mult[c].items()} for c in range(ncell)]
    tm["upward"] = time.perf_counter() - t0

    # DTT: traversal.py:303-348
    t0 = time.perf_counter()
    pre_dtt = pre
    pot = np.zeros(pos.shape[0], complex)
    lhat = [dict() for _ in range(ncell)]
    cnt = {"m2l": 0, "p2p": 0}

    def dtt(t, s):
        nonlocal pre
        lev = tr.level[t]
        if mac(t, s):
            tv = tr.coords[t] - tr.coords[s]
            t1 = time.perf_counter()
            D = get_symbol(lev, tv)
            pre += time.perf_counter() - t1
            k = key_of(t, s) if is_hf(lev) else None
            if k not in mhat[s]:
                raise RuntimeError("missing source expansion: blank-pass bug")
            a = lhat[t].get(k)
            if a is None:
                a = lhat[t][k] = np.zeros(P**3, complex)
            a += D * mhat[s][k]
            cnt["m2l"] += 1
            if events is not None:
                events.append(("M2L", t, s, k))
        elif not tr.sons[t] or not tr.sons[s]:
            ts, ss = slice(tr.start[t], tr.stop[t]), slice(tr.start[s], tr.stop[s])
            for lo in range(ts.start, ts.stop, 1024):
                hi = min(lo + 1024, ts.stop)
                pot[lo:hi] += kernel_matrix(pos[lo:hi], pos[ss], kappa, tol) @ q[ss]
            cnt["p2p"] += (ts.stop - ts.start) * (ss.stop - ss.start)
            if events is not None:
                events.append(("P2P", t, s, None))
        else:
            for a in tr.sons[t]:
                for b in tr.sons[s]:
                    dtt(a, b)

    dtt(0, 0)
    tm["m2l_p2p"] = time.perf_counter() - t0
    pre_in_dtt = pre - pre_dtt

    # downward: traversal.py:355-418
    t0 = time.perf_counter()
    loc = [dict() for _ in range(ncell)]

    def keyorder(k):
        return (k is not None, k)

    for lev in range(tr.depth + 1):
        beta = tr.beta(lev)
        for c in levels[lev]:
            for k in sorted(lhat[c], key=keyorder):
                v = f2l(lhat[c][k], L)
                loc[c][k] = loc[c][k] + v if k in loc[c] else v
            al = tr.alpha(c)
            if not tr.sons[c]:
                sl = slice(tr.start[c], tr.stop[c])
                for k in sorted(loc[c], key=keyorder):
                    u = dirs[k[0]][k[1]] if k is not None else None
                    pot[sl] += l2p(al, beta, L, pos[sl], loc[c][k], kappa, u)
                continue
            keys = sorted(loc[c], key=keyorder)
            if not keys:
                continue
            fgrid = al + beta * ref_grid(L)
            for s in tr.sons[c]:
                oct_ = tuple(int(v) for v in tr.coords[s] - 2 * tr.coords[c])
                fac = tuple(m2m_axis(L, o).T for o in oct_)
                sgrid = tr.alpha(s) + tr.beta(lev + 1) * ref_grid(L)
                for k in keys:
                    if k is None:
                        inc = kron3(fac, loc[c][None][:, None])[:, 0]
                        sk = None
                    else:
                        u = dirs[k[0]][k[1]]
                        col = loc[c][k] * np.conj(plane_wave(fgrid, kappa, u))
                        inc = kron3(fac, col[:, None])[:, 0] * plane_wave(sgrid, kappa, u)
                        sk = (k[0] - 1, int(fathers[k[0]][k[1]])) if is_hf(lev + 1) else None
                    loc[s][sk] = loc[s][sk] + inc if sk in loc[s] else inc.copy()
    tm["downward"] = time.perf_counter() - t0
    tm["precompute"] = pre
    tm["matvec"] = tm["upward"] + tm["m2l_p2p"] - pre_in_dtt + tm["downward"]

    out = np.empty_like(pot)
    out[tr.perm] = pot
    counts = {
        "cells": ncell,
        "leaves": sum(1 for c in range(ncell) if not tr.sons[c]),
        "symbols": len(canon_cache),
        "effective_expansions": sum(len(m) for m in mult),
        "p2p_pairs": cnt["p2p"],
        "m2l_events": cnt["m2l"],
        "translations": len(deriv_cache),
    }
    return out, counts, hf_max, tm, tr
