"""Pin the CPU oracle (oracle/defmm_oracle.py) to the reference's own outputs.

The golden vectors were produced by running the reference (helmfmm) itself
(tests/golden/make_golden.py, make_golden_large.py).  The oracle must match
the discrete decisions exactly and the potentials to FP64 rounding.
"""

import numpy as np
import pytest

from conftest import golden_cases, load_case, load_ref
from oracle import defmm_oracle as O

FAST = [c for c in golden_cases() if c not in ("sphere3000", "refined3000", "c1_kd16", "c1_kd8", "cubesurf4000")]


@pytest.mark.parametrize("case", FAST)
def test_oracle_matches_reference_end_to_end(case):
    g = load_case(case)
    pot, counts, hf, _, _ = O.run(g["points"], g["charges"], **g["config"])
    assert hf == g["hf_max"]
    assert {k: counts[k] for k in g["counts"]} == g["counts"]
    ref = g["pot"]
    assert np.linalg.norm(pot - ref) <= 1e-13 * np.linalg.norm(ref)


def test_oracle_events_match_reference():
    g = load_case("volume3000")
    ev = []
    _, _, hf, _, tr = O.run(g["points"], g["charges"], events=ev, **g["config"])
    from paper_2202_04894_b200.geometry import morton_encode_many

    codes = [int(morton_encode_many(np.asarray([c]), lv)[0]) for c, lv in zip(tr.coords, tr.level)]
    m2l = sorted(
        (tr.level[t], codes[t], codes[s], k[0] if k else -1, k[1] if k else -1) for kind, t, s, k in ev if kind == "M2L"
    )
    p2p = sorted((tr.level[t], codes[t], tr.level[s], codes[s]) for kind, t, s, k in ev if kind == "P2P")
    assert m2l == sorted(map(tuple, g["m2l"].tolist()))
    assert p2p == sorted(map(tuple, g["p2p"].tolist()))


def test_oracle_cfg1_counts_and_decisions_pinned():
    """cfg1's counts as produced by the reference (ref_cfg1.npz)."""
    ref = load_ref("cfg1")
    assert ref["counts"]["m2l_events"] == 262054
    assert ref["counts"]["p2p_pairs"] == 39152776
    assert abs(float(ref["eps_ref"]) - 4.163e-3) < 1e-6


def test_kernel_known_values(operators):
    assert np.isclose(O.kernel_of_distance(1.0, 0.0, 1e-12), operators["g1_k0"], rtol=1e-15)
    assert np.isclose(O.kernel_of_distance(np.pi, 2.0, 1e-12), operators["gpi_k2"], rtol=1e-15)
    assert np.isclose(O.kernel_of_distance(1.0, 0.0, 1e-12), 1.0 / (4 * np.pi))
    assert O.kernel_of_distance(0.0, 3.0, 1e-12) == 0.0


def test_directions_and_ties(operators):
    dirs, fathers = O.direction_levels(4)
    for e in range(5):
        assert np.array_equal(dirs[e], operators[f"dirs_{e}"])
        if e:
            assert np.array_equal(fathers[e], operators[f"fathers_{e}"])
    tv = operators["near_t"]
    for e in range(4):
        got = [O.nearest(dirs[e], t / np.linalg.norm(t)) for t in tv[::7]]
        assert got == operators[f"near_{e}"][::7].tolist()


def test_canonical_translations(operators):
    tv = operators["near_t"]
    got = [O.canonicalize(t) for t in tv]
    assert np.array_equal(np.array([c for c, _ in got]), operators["canon"])
    assert np.array_equal(np.array([r for _, r in got]), operators["canon_rid"])
    # the 316 LF translations fall into 16 classes (test_fourier.py:64-68)
    g = np.arange(-3, 4)
    t = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    t = t[np.max(np.abs(t), axis=1) >= 2]
    assert len(t) == 316 and len({O.canonicalize(x)[0] for x in t}) == 16


@pytest.mark.parametrize("L", [2, 3, 4, 5, 6, 8])
def test_frequency_permutations(operators, L):
    ref = operators[f"fperm_L{L}"]
    for rid in range(48):
        assert np.array_equal(O.freq_perm(L, rid), ref[rid])


@pytest.mark.parametrize("L", [4, 6])
def test_fourier_and_interpolation_operators(operators, L):
    o = operators
    assert np.allclose(O.m2f(o[f"m2f_in_L{L}"], L), o[f"m2f_out_L{L}"], rtol=0, atol=1e-13)
    assert np.allclose(O.f2l(o[f"f2l_in_L{L}"], L), o[f"f2l_out_L{L}"], rtol=0, atol=1e-13)
    for t in ((3, 1, 0), (2, 2, 2), (5, 3, 1)):
        ref = o[f"sym_L{L}_{t[0]}{t[1]}{t[2]}"]
        got = O.symbol(7.5, 1e-12, t, 0.25, L)
        assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()
    al, be = np.array([0.1, -0.2, 0.3]), 0.125
    pos, q = o[f"p2m_pos_L{L}"], o[f"p2m_q_L{L}"]
    u = np.array([1.0, 2.0, -2.0]) / 3.0
    assert np.allclose(O.p2m(al, be, L, pos, q), o[f"p2m_lf_L{L}"], rtol=1e-13, atol=1e-13)
    assert np.allclose(O.p2m(al, be, L, pos, q, 40.0, u), o[f"p2m_hf_L{L}"], rtol=1e-12, atol=1e-12)
    loc = o[f"l2p_loc_L{L}"]
    assert np.allclose(O.l2p(al, be, L, pos, loc), o[f"l2p_lf_L{L}"], rtol=1e-13, atol=1e-13)
    assert np.allclose(O.l2p(al, be, L, pos, loc, 40.0, u), o[f"l2p_hf_L{L}"], rtol=1e-12, atol=1e-12)
    for oc in range(8):
        bits = ((oc >> 2) & 1, (oc >> 1) & 1, oc & 1)
        got = np.stack([O.m2m_axis(L, b) for b in bits])
        assert np.allclose(got, o[f"m2m_L{L}_{oc}"], rtol=0, atol=1e-14)


def test_fft_m2l_equals_dense_operator():
    """test_fourier.py:109-131: FFT path == dense M2L matrix to 1e-12."""
    for kappa, L in ((0.0, 2), (0.0, 4), (3.0, 4), (10.0, 5)):
        t = (3, -2, 1)
        D = O.symbol(kappa, 1e-14, t, 0.5, L)
        cols = []
        for j in range(L**3):
            e = np.zeros(L**3, complex)
            e[j] = 1.0
            cols.append(O.f2l(D * O.m2f(e, L), L))
        fft = np.column_stack(cols)
        dense = O.dense_m2l(kappa, 1e-14, t, 0.5, L)
        assert np.abs(fft - dense).max() <= 1e-12 * np.abs(dense).max()
