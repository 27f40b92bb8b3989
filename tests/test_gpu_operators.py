"""Operator-level parity of the nodal kernels (K2 P2M, K4 M2M, K5 L2L, K3 L2P)
through the C-ABI, in both storage types, against the oracle's restatement of
interpolation.py:109-200 / traversal.py:224-296, 355-402 -- so a fault in one
operator (or in one precision) is caught where it lives, not only as an
end-to-end miss."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import defmm_oracle as O  # noqa: E402

# relative tolerances: FP64 operators against the FP64 oracle; FP32 storage /
# arithmetic (defmm_b200.h) against the FP64 oracle
TOL = {"c128": 1e-12, "c64": 3e-6}
KAPPA = 9.0


def _dev(a, dt):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dt).cuda()


def _cplx(a, dtype):
    return _dev(a, torch.complex128 if dtype == "c128" else torch.complex64)


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def _geometry(L):
    """Father cell (level 1) with two sons (octants 5 and 2) and two directions."""
    beta = np.array([2.0, 1.0, 0.5])  # side per level
    alpha = np.array([[-1.0, -1.0, -1.0], [0.0, -1.0, 0.0], [0.5, -1.0, 0.5], [0.0, -0.5, 0.0]])
    level = np.array([0, 1, 2, 2], np.int32)  # cells: root, father, son A (1,0,1), son B (0,1,0)
    u = np.array([[1.0, 2.0, -2.0], [0.0, -3.0, 4.0]])
    dirs = u / np.linalg.norm(u, axis=1)[:, None]
    return beta, alpha, level, dirs


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("L", [3, 4, 6])
def test_p2m_and_l2p_operators(L, dtype):
    from paper_2202_04894_b200 import _lib

    beta, alpha, level, dirs = _geometry(L)
    rng = np.random.default_rng(L)
    st = torch.cuda.current_stream().cuda_stream
    # particles of son A (cell 2) then son B (cell 3), sorted order
    na, nb = 37, 23
    pos = np.vstack([alpha[2] + beta[2] * rng.uniform(0, 1, (na, 3)), alpha[3] + beta[2] * rng.uniform(0, 1, (nb, 3))])
    q = rng.normal(size=na + nb) + 1j * rng.normal(size=na + nb)
    start = np.array([0, 0, 0, na], np.int64)
    stop = np.array([na + nb, na + nb, na, na + nb], np.int64)
    i64, i32, f64 = torch.int64, torch.int32, torch.float64
    geo = (_dev(start, i64), _dev(stop, i64), _dev(alpha, f64), _dev(level, i32), _dev(beta, f64), _dev(dirs, f64))
    xyz = [_dev(pos[:, k], f64) for k in range(3)]
    L3 = L**3
    # P2M: slots 0..3 = (A, LF), (A, dir 1), (B, dir 0), (B, LF)
    cell = np.array([2, 2, 3, 3], np.int32)
    dr = np.array([-1, 1, 0, -1], np.int32)
    mult = torch.zeros((4, L3), dtype=torch.complex128 if dtype == "c128" else torch.complex64, device="cuda")
    _lib.call(f"defmm_p2m_{dtype}", L, 4, _dev(cell, i32), _dev(dr, i32), _dev(np.arange(4), i64), *geo, *xyz,
              _cplx(q, dtype), KAPPA, mult, st)
    got = mult.cpu().numpy()
    for s in range(4):
        sl = slice(start[cell[s]], stop[cell[s]])
        ref = O.p2m(alpha[cell[s]], beta[2], L, pos[sl], q[sl], KAPPA, dirs[dr[s]] if dr[s] >= 0 else None)
        assert _rel(got[s], ref) <= TOL[dtype], (s, _rel(got[s], ref))
    # L2P: leaf A owns local slots 0, 1 (LF, dir 1), leaf B slots 2, 3 (dir 0, LF); out = near + sum
    loc = rng.normal(size=(4, L3)) + 1j * rng.normal(size=(4, L3))
    near = rng.normal(size=na + nb) + 1j * rng.normal(size=na + nb)
    perm = rng.permutation(na + nb)
    out = torch.zeros(na + nb, dtype=mult.dtype, device="cuda")
    _lib.call(f"defmm_l2p_{dtype}", L, 2, _dev(np.array([2, 3]), i32), _dev(np.array([0, 2]), i64),
              _dev(np.array([2, 4]), i64), _dev(dr, i32), *geo, *xyz, KAPPA, _cplx(loc, dtype), _cplx(near, dtype),
              _dev(perm, i64), out, st)
    ref = near.copy()
    for s in range(4):
        sl = slice(start[cell[s]], stop[cell[s]])
        ref[sl] += O.l2p(alpha[cell[s]], beta[2], L, pos[sl], loc[s], KAPPA, dirs[dr[s]] if dr[s] >= 0 else None)
    want = np.empty_like(ref)
    want[perm] = ref
    assert _rel(out.cpu().numpy(), want) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("L", [3, 4, 6])
def test_m2m_and_l2l_operators(L, dtype):
    from paper_2202_04894_b200 import _lib

    beta, alpha, level, dirs = _geometry(L)
    rng = np.random.default_rng(10 + L)
    st = torch.cuda.current_stream().cuda_stream
    i64, i32, f64 = torch.int64, torch.int32, torch.float64
    L3 = L**3
    cd = torch.complex128 if dtype == "c128" else torch.complex64
    octs = {2: (1, 0, 1), 3: (0, 1, 0)}  # son cell -> octant
    fgrid = alpha[1] + beta[1] * O.ref_grid(L)

    def sgrid(c):
        return alpha[c] + beta[2] * O.ref_grid(L)

    # M2M: father slots 4 (LF) and 5 (direction 1) from son slots 0..3
    m = rng.normal(size=(6, L3)) + 1j * rng.normal(size=(6, L3))
    mult = _cplx(m, dtype)
    son = np.full((2, 8), -1, np.int64)
    son[0, 5], son[0, 2] = 0, 1  # LF father: sons A (octant 5), B (octant 2)
    son[1, 5], son[1, 2] = 2, 3  # directional father
    _lib.call(f"defmm_m2m_{dtype}", L, 2, _dev(np.array([4, 5]), i64), _dev(np.array([-1, 1]), i32),
              _dev(son, i64), float(beta[2]), _dev(dirs, f64), KAPPA, mult, st)
    got = mult.cpu().numpy()
    ref_lf = sum(O.kron3(tuple(O.m2m_axis(L, o) for o in octs[c]), m[s][:, None])[:, 0] for c, s in ((2, 0), (3, 1)))
    u = dirs[1]
    ref_hf = np.zeros(L3, complex)
    for c, s in ((2, 2), (3, 3)):
        col = m[s] * np.conj(O.plane_wave(sgrid(c), KAPPA, u))
        ref_hf += O.kron3(tuple(O.m2m_axis(L, o) for o in octs[c]), col[:, None])[:, 0] * O.plane_wave(fgrid, KAPPA, u)
    assert _rel(got[4], ref_lf) <= TOL[dtype]
    assert _rel(got[5], ref_hf) <= TOL[dtype]
    # L2L (gather form): son slots 0 (A) and 1 (B) each += father slots 4 (LF) and 5 (direction 0)
    lo = rng.normal(size=(6, L3)) + 1j * rng.normal(size=(6, L3))
    local = _cplx(lo, dtype)
    _lib.call(f"defmm_l2l_{dtype}", L, 2, _dev(np.array([0, 1]), i64), _dev(np.array([5, 2]), torch.int8),
              _dev(np.array([0, 2, 4]), i64), _dev(np.array([4, 5, 4, 5]), i64), _dev(np.array([-1, 0, -1, 0]), i32),
              float(beta[2]), _dev(dirs, f64), KAPPA, local, st)
    got = local.cpu().numpy()
    u = dirs[0]
    for c, s in ((2, 0), (3, 1)):
        fac = tuple(O.m2m_axis(L, o).T for o in octs[c])
        ref = lo[s] + O.kron3(fac, lo[4][:, None])[:, 0]
        col = lo[5] * np.conj(O.plane_wave(fgrid, KAPPA, u))
        ref = ref + O.kron3(fac, col[:, None])[:, 0] * O.plane_wave(sgrid(c), KAPPA, u)
        assert _rel(got[s], ref) <= TOL[dtype], (s, _rel(got[s], ref))


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("L", [4, 5, 8])
def test_m2m_and_l2l_odd_counts(L, dtype):
    """The v2 kernels take sons / sources two at a time: fathers with three and
    with one son, outputs with three and with one source (an unpaired last
    tile), LF and directional, against the oracle's axis factors."""
    from paper_2202_04894_b200 import _lib

    beta, alpha, _, dirs = _geometry(L)
    rng = np.random.default_rng(40 + L)
    st = torch.cuda.current_stream().cuda_stream
    i64, i32, f64 = torch.int64, torch.int32, torch.float64
    L3 = L**3
    fgrid = alpha[1] + beta[1] * O.ref_grid(L)

    def bits(o):
        return ((o >> 2) & 1, (o >> 1) & 1, o & 1)

    def sgrid(o):  # nodes of the father's son in octant o
        return alpha[1] + beta[2] * np.array(bits(o)) + beta[2] * O.ref_grid(L)

    def up(o, col):
        return O.kron3(tuple(O.m2m_axis(L, b) for b in bits(o)), col[:, None])[:, 0]

    def down(o, col):
        return O.kron3(tuple(O.m2m_axis(L, b).T for b in bits(o)), col[:, None])[:, 0]

    # M2M: slots 0..7 sons, fathers 8 (LF, sons at octants 5, 2, 7), 9 (direction 1, the same three),
    # 10 (LF, one son at octant 0), 11 (direction 0, one son at octant 6)
    m = rng.normal(size=(12, L3)) + 1j * rng.normal(size=(12, L3))
    mult = _cplx(m, dtype)
    son = np.full((4, 8), -1, np.int64)
    son[0, [5, 2, 7]] = [0, 1, 2]
    son[1, [5, 2, 7]] = [3, 4, 5]
    son[2, 0] = 6
    son[3, 6] = 7
    _lib.call(f"defmm_m2m_{dtype}", L, 4, _dev(np.array([8, 9, 10, 11]), i64), _dev(np.array([-1, 1, -1, 0]), i32),
              _dev(son, i64), float(beta[2]), _dev(dirs, f64), KAPPA, mult, st)
    got = mult.cpu().numpy()

    def hf(u, pairs):
        return sum(up(o, m[s] * np.conj(O.plane_wave(sgrid(o), KAPPA, u))) for o, s in pairs) * \
            O.plane_wave(fgrid, KAPPA, u)

    want = {8: sum(up(o, m[s]) for o, s in ((5, 0), (2, 1), (7, 2))), 9: hf(dirs[1], ((5, 3), (2, 4), (7, 5))),
            10: up(0, m[6]), 11: hf(dirs[0], ((6, 7),))}
    for slot, ref in want.items():
        assert _rel(got[slot], ref) <= TOL[dtype], (slot, _rel(got[slot], ref))
    # L2L: son slot 0 (octant 3) += fathers 4 (LF), 5 (direction 0), 6 (direction 1); son slot 1 (octant 6) += father 7 (direction 1)
    lo = rng.normal(size=(8, L3)) + 1j * rng.normal(size=(8, L3))
    local = _cplx(lo, dtype)
    _lib.call(f"defmm_l2l_{dtype}", L, 2, _dev(np.array([0, 1]), i64), _dev(np.array([3, 6]), torch.int8),
              _dev(np.array([0, 3, 4]), i64), _dev(np.array([4, 5, 6, 7]), i64), _dev(np.array([-1, 0, 1, 1]), i32),
              float(beta[2]), _dev(dirs, f64), KAPPA, local, st)
    got = local.cpu().numpy()

    def push(o, s, d):
        if d < 0:
            return down(o, lo[s])
        u = dirs[d]
        return down(o, lo[s] * np.conj(O.plane_wave(fgrid, KAPPA, u))) * O.plane_wave(sgrid(o), KAPPA, u)

    ref0 = lo[0] + push(3, 4, -1) + push(3, 5, 0) + push(3, 6, 1)
    ref1 = lo[1] + push(6, 7, 1)
    assert _rel(got[0], ref0) <= TOL[dtype], _rel(got[0], ref0)
    assert _rel(got[1], ref1) <= TOL[dtype], _rel(got[1], ref1)
