"""B200 parity: the CUDA path (through the C-ABI) against the reference's
golden outputs and the CPU oracle.

Tolerances: the device computes in FP64 (complex128) like the reference, with
a different but deterministic summation order and cell-relative phases, so
potentials agree to ~1e-13 relative L2; the graded bar (north star) is
rel_L2(p_new, p_ref) <= 1e-2 * eps_ref with eps_ref the reference's own error
against direct summation.  Both are asserted.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import golden_cases, load_case, load_ref  # noqa: E402
from oracle import defmm_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-11  # relative L2, same-algorithm FP64 reassociation


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("case", golden_cases())
def test_run_fmm_matches_reference_golden(case):
    from paper_2202_04894_b200 import FmmConfig, run_fmm_full

    g = load_case(case)
    pts, q = g["points"], g["charges"]
    pot, info = run_fmm_full(pts, pts, q, FmmConfig(**g["config"]))
    assert info.hf_max_level == g["hf_max"]
    assert info.counts == g["counts"]
    assert pot.dtype == np.complex128 and pot.shape == q.shape
    assert _rel(pot, g["pot"]) <= FP64_TOL


# complex64 storage against the FP64 reference: the north-star bar 1e-2 eps_ref where FP32
# arithmetic can reach it, else the FP32 floor of these sums (measured <= 1.6e-6 on the small
# cases whose bar is below it; tools/gpu/c64_bar.py prints the table)
C64_FLOOR = 2e-6
C64_TOL = 5e-6  # bound used where eps_ref is not computed (kernel-variant tests)


def _c64_bar(g):
    """max(1e-2 eps_ref, C64_FLOOR), eps_ref = rel-L2 of the reference's potentials against
    the FP64 direct sum (kernel.py:58-75, evaluated by the GPU direct kernel)."""
    from paper_2202_04894_b200 import HelmholtzKernel, direct_sum
    from paper_2202_04894_b200.geometry import compute_root_box

    pts = g["points"]
    kern = HelmholtzKernel(kappa=g["config"].get("kappa", 0.0), singularity_tol=1e-12 * compute_root_box(pts).side)
    d = direct_sum(kern, pts, pts, g["charges"])
    return max(1e-2 * _rel(g["pot"], d), C64_FLOOR)


@pytest.mark.parametrize("case", ["cubesurf4000", "c1_kd8", "c1_kd16", "ellipsoid3000", "volume3000", "sphere3000",
                                  "refined3000"])
def test_run_fmm_c64_matches_reference_golden(case):
    """complex64 storage (BASELINE cfg2/3/4 dtype): same lists, FP32 streams; orders 4, 5
    (ellipsoid3000) and 6."""
    from paper_2202_04894_b200 import FmmConfig, run_fmm_full

    g = load_case(case)
    pts, q = g["points"], g["charges"]
    pot, info = run_fmm_full(pts, pts, q, FmmConfig(dtype="c64", **g["config"]))
    assert info.counts == g["counts"]
    assert pot.dtype == np.complex128
    assert _rel(pot, g["pot"]) <= _c64_bar(g)


def test_flat_tree_is_exact_p2p():
    """test_traversal.py:163-170: one leaf -> pure P2P equals direct sum."""
    from paper_2202_04894_b200 import FmmConfig, run_fmm_full

    g = load_case("flat50")
    pot, info = run_fmm_full(g["points"], g["points"], g["charges"], FmmConfig(**g["config"]))
    assert info.counts["m2l_events"] == 0
    box_side = 2 * np.max(np.abs(g["points"] - g["points"].mean(0))) * (1 + 1e-6)
    ref = O.direct_sum(g["points"], g["points"], g["charges"], g["config"]["kappa"], 1e-12 * box_side)
    assert np.allclose(pot, ref, rtol=0, atol=1e-12 * np.abs(ref).max())


def test_single_particle_is_zero():
    from paper_2202_04894_b200 import FmmConfig, run_fmm

    pts = np.array([[0.5, 0.5, 0.5]])
    assert run_fmm(pts, pts, np.array([1.0 + 0j]), FmmConfig(order=3))[0] == 0.0


def test_bitwise_deterministic_rerun():
    from paper_2202_04894_b200 import FmmConfig, FmmPlan

    g = load_case("cubesurf4000")
    plan = FmmPlan(g["points"], None, FmmConfig(**g["config"]), charges=g["charges"])
    a = plan.apply().clone()
    b = plan.apply().clone()
    assert torch.equal(a, b)


def test_gpu_direct_sum_matches_oracle():
    from paper_2202_04894_b200 import HelmholtzKernel, direct_sum

    rng = np.random.default_rng(11)
    src = rng.uniform(-1, 1, (3000, 3))
    tgt = np.vstack([src[:50], rng.uniform(-1, 1, (77, 3))])
    q = rng.normal(size=3000) + 1j * rng.normal(size=3000)
    got = direct_sum(HelmholtzKernel(kappa=17.0, singularity_tol=1e-12), tgt, src, q)
    ref = O.direct_sum(tgt, src, q, 17.0, 1e-12)
    assert _rel(got, ref) <= 1e-13


@pytest.mark.parametrize("L", [2, 4, 5, 6, 8])
def test_symbol_and_m2f_kernels(L):
    from paper_2202_04894_b200 import _lib
    from paper_2202_04894_b200.fmm import spectral_layout

    dev = torch.device("cuda")
    st = torch.cuda.current_stream().cuda_stream
    tv = np.array([[3, 1, 0], [2, 2, 2], [5, 3, 1], [2, 0, 0]], np.int32)
    beta = np.array([0.25, 0.5, 0.125, 1.0])
    P3 = (2 * L - 1) ** 3
    sym = torch.empty((4, P3), dtype=torch.complex128, device=dev)
    _lib.call("defmm_symbols_c128", L, 4, torch.as_tensor(tv.reshape(-1)).to(dev), torch.as_tensor(beta).to(dev),
              7.5, sym, st)
    forder, _ = spectral_layout(L)  # device spectra are stored in orbit order
    got = np.empty((4, P3), complex)
    got[:, forder] = sym.cpu().numpy()
    for i in range(4):
        ref = O.symbol(7.5, 1e-12, tuple(tv[i]), beta[i], L)
        assert np.abs(got[i] - ref).max() <= 1e-12 * np.abs(ref).max()
    rng = np.random.default_rng(L)
    m = rng.normal(size=(5, L**3)) + 1j * rng.normal(size=(5, L**3))
    mult = torch.as_tensor(m).to(dev)
    hat = torch.empty((3, P3), dtype=torch.complex128, device=dev)
    src = torch.as_tensor(np.array([4, 0, 2], np.int64)).to(dev)
    _lib.call("defmm_m2f_c128", L, 3, src, mult, hat, st)
    h = np.empty((3, P3), complex)
    h[:, forder] = hat.cpu().numpy()
    for k, j in enumerate((4, 0, 2)):
        assert np.abs(h[k] - O.m2f(m[j], L)).max() <= 1e-13 * np.abs(m[j]).sum()


@pytest.mark.parametrize("case", ["cubesurf4000", "c1_kd8", "volume3000"])
def test_m2l_canonical_gather_and_derived_symbols_agree(case):
    """The canonical-gather M2L (in-loop rotation), the row-wise derived-symbol
    M2L and the parent-pair blocked M2L (product path) agree."""
    from paper_2202_04894_b200 import FmmConfig, FmmPlan

    g = load_case(case)
    plan = FmmPlan(g["points"], None, FmmConfig(**g["config"]), charges=g["charges"])
    plan.m2l_variant = "canonical"
    a = plan.apply().cpu().numpy()
    plan.m2l_variant = "derived"
    b = plan.apply().cpu().numpy()
    assert _rel(b, a) <= 1e-13
    plan.m2l_variant = "hybrid"
    c = plan.apply().cpu().numpy()
    assert _rel(c, a) <= 1e-13
    for mode in ("blocked_all", "rows", "hybrid_rows", "pairs_all", "triples_all", "quartets_all", "staged_all",
                 "staged"):
        p2 = FmmPlan(g["points"], None, FmmConfig(**g["config"]), charges=g["charges"], reuse=plan, m2l=mode)
        assert _rel(p2.apply().cpu().numpy(), a) <= 1e-13, mode
    # every kernel on some level at once (per-level overrides)
    levels = sorted(plan.level_kinds)
    mix = {lv: ("staged", "rows", "blocked", "pair", "triple", "quartet")[i % 6] for i, lv in enumerate(levels)}
    p2 = FmmPlan(g["points"], None, FmmConfig(**g["config"]), charges=g["charges"], reuse=plan, m2l_levels=mix)
    assert p2.level_kinds == mix
    assert _rel(p2.apply().cpu().numpy(), a) <= 1e-13
    assert _rel(b, g["pot"]) <= FP64_TOL


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("case", ["cubesurf4000", "volume3000"])
def test_group_m2l_kernels_match_reference(case, dtype):
    """Pairs, triples and quartets (m2l_group) reproduce the reference's
    potentials and rerun bitwise identically (no atomics)."""
    from paper_2202_04894_b200 import FmmConfig, FmmPlan

    g = load_case(case)
    cfg = FmmConfig(**{**g["config"], "dtype": dtype})
    base = FmmPlan(g["points"], None, cfg, charges=g["charges"])
    for mode in ("pairs_all", "triples_all", "quartets_all", "staged_all"):
        p2 = FmmPlan(g["points"], None, cfg, charges=g["charges"], reuse=base, m2l=mode)
        a = p2.apply().cpu().numpy().astype(np.complex128)
        assert _rel(a, g["pot"]) <= (FP64_TOL if dtype == "c128" else C64_TOL)
        assert np.array_equal(p2.apply().cpu().numpy().astype(np.complex128), a)


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("case", ["cubesurf4000", "volume3000", "refined3000", "flat50"])
def test_mutual_p2p_matches_reference(case, dtype, monkeypatch):
    """K1 v2 (every near-field pair evaluated once for both directions, column sums gathered
    in fixed order) against the reference potentials and the one-directional K1; reruns are
    bitwise identical."""
    from paper_2202_04894_b200 import FmmConfig, FmmPlan

    g = load_case(case)
    cfg = FmmConfig(**{**g["config"], "dtype": dtype})
    monkeypatch.setenv("DEFMM_P2P_MUTUAL", "1")
    pm = FmmPlan(g["points"], None, cfg, charges=g["charges"])
    assert pm.p2p_mut is not None
    a = pm.apply().cpu().numpy().astype(np.complex128)
    assert np.array_equal(pm.apply().cpu().numpy().astype(np.complex128), a)
    monkeypatch.setenv("DEFMM_P2P_MUTUAL", "0")
    po = FmmPlan(g["points"], None, cfg, charges=g["charges"], reuse=pm)
    assert po.p2p_mut is None
    b = po.apply().cpu().numpy().astype(np.complex128)
    tol = FP64_TOL if dtype == "c128" else C64_TOL
    assert _rel(a, g["pot"]) <= tol and _rel(b, g["pot"]) <= tol
    assert _rel(pm.near.cpu().numpy(), po.near.cpu().numpy()) <= (1e-13 if dtype == "c128" else 2e-6)


def test_linearity_in_the_charges():
    from paper_2202_04894_b200 import FmmConfig, FmmPlan

    g = load_case("ellipsoid3000")
    plan = FmmPlan(g["points"], None, FmmConfig(**g["config"]), charges=g["charges"])
    rng = np.random.default_rng(3)
    q1 = g["charges"]
    q2 = rng.normal(size=q1.shape) + 1j * rng.normal(size=q1.shape)
    plan.set_charges(q1)
    p1 = plan.apply().cpu().numpy()
    plan.set_charges(q2)
    p2 = plan.apply().cpu().numpy()
    plan.set_charges((2 - 1j) * q1 + 0.5 * q2)
    p3 = plan.apply().cpu().numpy()
    assert _rel(p3, (2 - 1j) * p1 + 0.5 * p2) <= 1e-13


def test_cfg1_full_size_parity():
    """BASELINE cfg1 (N=20k sphere, kappa*D=32, L=4) against the reference run."""
    from paper_2202_04894_b200 import FmmConfig, run_fmm_full
    from paper_2202_04894_b200.workloads import make_workload

    ref = load_ref("cfg1")
    pts, q, k, w = make_workload("cfg1")
    pot, info = run_fmm_full(pts, pts, q, FmmConfig(order=w.order, ncrit=w.ncrit, kappa=k))
    assert {kk: info.counts[kk] for kk in info.counts} == {kk: ref["counts"][kk] for kk in info.counts}
    eps_ref = float(ref["eps_ref"])
    r = _rel(pot, ref["pot"])
    assert r <= 1e-2 * eps_ref and r <= FP64_TOL
    eps_new = _rel(pot[ref["sample"]], ref["direct_sample"])
    assert eps_new <= (1 + 1e-2) * eps_ref


# (golden file, workload, dtype): every BASELINE config at its BASELINE dtype
# (cfg2: c64 and c128; cfg3: c64, plus c128; cfg5: c128) and every order
FULL_SIZE = [("cfg2", "cfg2", "c64"), ("cfg2", "cfg2", "c128"), ("cfg2_L6", "cfg2", "c64"),
             ("cfg2_L6", "cfg2", "c128"), ("cfg3", "cfg3", "c64"), ("cfg3", "cfg3", "c128"),
             ("cfg5", "cfg5", "c128"), ("cfg5_L6", "cfg5", "c128"), ("cfg5_L8", "cfg5", "c128")]


@pytest.mark.parametrize("name,workload,dtype", FULL_SIZE)
def test_full_size_sampled_parity(name, workload, dtype):
    """BASELINE cfg2/cfg3/cfg5 at full size (1M / 4M / 2M points), each order
    the survey runs: counts equal the reference's run_fmm_full
    (traversal.py:495-505) exactly; on the 1,000 sampled targets
    (harness.py:151-165) rel-L2(p_new, p_ref) <= 1e-2 eps_ref (the north-star
    bar) and eps_new <= (1 + 1e-2) eps_ref against FP64 direct sums
    (tests/golden/ref_*.npz, written by make_golden_large.py from the
    reference itself)."""
    from paper_2202_04894_b200 import FmmConfig, HelmholtzKernel, direct_sum, run_fmm_full
    from paper_2202_04894_b200.workloads import make_workload

    ref = load_ref(name)
    pts, q, k, w = make_workload(workload)
    assert abs(k - float(ref["kappa"])) == 0.0
    pot, info = run_fmm_full(pts, pts, q, FmmConfig(order=int(ref["order"]), ncrit=w.ncrit, kappa=k, dtype=dtype))
    assert {kk: info.counts[kk] for kk in info.counts} == {kk: ref["counts"][kk] for kk in info.counts}
    assert info.hf_max_level == int(ref["hf_max"])
    s = ref["sample"]
    eps_ref = float(ref["eps_ref"])
    r = _rel(pot[s], ref["pot_sample"])
    assert r <= 1e-2 * eps_ref  # the north-star parity bar
    if dtype == "c128":
        assert r <= FP64_TOL
    side = 2 * np.max(np.abs(pts - pts.mean(0))) * (1 + 1e-6)
    d = direct_sum(HelmholtzKernel(kappa=k, singularity_tol=1e-12 * side), pts[s], pts, q)
    assert _rel(d, ref["direct_sample"]) <= 1e-12  # the GPU direct sum = the reference's
    assert _rel(pot[s], d) <= (1 + 1e-2) * eps_ref


def test_cfg4_counts_and_accuracy():
    """BASELINE cfg4 (N=16M refined cube, kappa*D=512, L=6, ncrit=128) on one
    GPU.  The reference's full matvec does not fit this container (spectra
    alone > 62 GB), so tests/golden/ref_cfg4_counts.npz holds the reference's
    own counts (its tree, blank passes and dual tree traversal run with the
    arithmetic stubbed, make_golden_counts.py) and FP64 direct sums on the
    1,000 sampled targets: counts must be equal; the complex128 path (the
    reference's arithmetic) sets eps, and complex64 storage must stay within
    1% of it."""
    from paper_2202_04894_b200 import FmmConfig, FmmPlan
    from paper_2202_04894_b200.workloads import make_workload

    ref = load_ref("cfg4_counts")
    pts, q, k, w = make_workload("cfg4")
    assert abs(k - float(ref["kappa"])) == 0.0
    s = ref["sample"]
    eps = {}
    base = None
    for dtype in ("c128", "c64"):
        cfg = FmmConfig(order=w.order, ncrit=w.ncrit, kappa=k, dtype=dtype)
        plan = FmmPlan(pts, None, cfg, charges=q, reuse=base)
        if base is None:
            base = plan
            counts = {kk: v for kk, v in plan.plan.counts.items() if kk != "translations"}
            assert counts == {kk: ref["counts"][kk] for kk in counts}
            assert plan.plan.hf_max == int(ref["hf_max"])
        pot = plan.apply().cpu().numpy().astype(np.complex128)
        eps[dtype] = _rel(pot[s], ref["direct_sample"])
        del pot
    assert eps["c128"] < 1e-3
    assert eps["c64"] <= (1 + 1e-2) * eps["c128"]


@pytest.mark.parametrize("dtype", ["c128", "c64"])
@pytest.mark.parametrize("case", __import__("conftest").two_tree_cases())
def test_two_tree_run_fmm_matches_reference(case, dtype):
    """test_traversal.py:173-181 analogue against the reference's own output."""
    from conftest import load_two_tree
    from paper_2202_04894_b200 import FmmConfig, run_fmm_full

    g = load_two_tree(case)
    pot, info = run_fmm_full(g["targets"], g["sources"], g["charges"], FmmConfig(dtype=dtype, **g["config"]))
    assert info.counts == g["counts"]
    assert pot.shape == (len(g["targets"]),)
    assert _rel(pot, g["pot"]) <= (FP64_TOL if dtype == "c128" else C64_TOL)


def test_event_log_partitions_all_pairs():
    """test_traversal.py:190-201: events= receives every M2L/P2P event; their
    particle blocks cover every (target, source) pair exactly once."""
    from paper_2202_04894_b200 import FmmConfig, run_fmm_full

    g = load_case("volume3000")
    events = []
    pot, info = run_fmm_full(g["points"], g["points"], g["charges"], FmmConfig(**g["config"]), events=events)
    n = len(g["points"])
    cov = np.zeros((n, n), np.int8)
    for ev in events:
        cov[ev.target.start : ev.target.stop, ev.source.start : ev.source.stop] += 1
    assert np.all(cov == 1)
    assert info.counts["m2l_events"] == sum(1 for e in events if e.kind == "M2L")
    ref = sorted(map(tuple, g["m2l"].tolist()))
    mine = sorted((e.target.level, e.target.key.code, e.source.key.code, *(e.direction or (-1, -1)))
                  for e in events if e.kind == "M2L")
    assert mine == ref


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", ["cubesurf4000", "sphere3000"])
def test_virtual_ranks_match_single_gpu(case, world):
    """§8(e): the Morton-sharded path, emulated as `world` virtual ranks on one
    GPU (phase 1 on every rank, the multipole all-reduce as a device sum,
    phase 2 on every rank), reproduces the single-plan potentials."""
    from paper_2202_04894_b200 import FmmConfig, FmmPlan

    g = load_case(case)
    cfg = FmmConfig(**g["config"])
    base = FmmPlan(g["points"], None, cfg, charges=g["charges"])
    ref = base.apply().clone()
    ranks = [FmmPlan(g["points"], None, cfg, charges=g["charges"], reuse=base, shard=(r, world),
                     allreduce=lambda t: None) for r in range(world)]
    for r in ranks:
        r.apply_upward()
    total = sum(r.mult for r in ranks)
    for r in ranks:
        r.mult.copy_(total)
    out = sum(r.apply_rest().clone() for r in ranks)
    assert _rel(out.cpu().numpy(), ref.cpu().numpy()) <= 1e-13
    assert _rel(out.cpu().numpy(), g["pot"]) <= FP64_TOL


@pytest.mark.parametrize("case,world", [("cubesurf4000", 2), ("volume3000", 3)])
def test_virtual_ranks_halo_exchange_matches_single_gpu(case, world):
    """The halo exchange of the N > 1 path (parallel.make_halo: span all-reduce
    + owner -> reader copies of complete multipoles), emulated between virtual
    ranks on one GPU with the same index sets: every rank's potentials, summed,
    reproduce the single-plan matvec -- only the halo is exchanged."""
    from paper_2202_04894_b200 import FmmConfig, FmmPlan
    from paper_2202_04894_b200.parallel import make_halo

    g = load_case(case)
    cfg = FmmConfig(**g["config"])
    base = FmmPlan(g["points"], None, cfg, charges=g["charges"])
    ref = base.apply().clone()
    ranks = [FmmPlan(g["points"], None, cfg, charges=g["charges"], reuse=base, shard=(r, world),
                     allreduce=lambda t: None) for r in range(world)]
    halos = [make_halo(base.plan, base.tt, r.shard.cuts, k, world) for k, r in enumerate(ranks)]
    for r in ranks:
        r.apply_upward()
    dev = ranks[0].mult.device
    idx = lambda a: torch.as_tensor(a, dtype=torch.int64, device=dev)  # noqa: E731
    span = idx(halos[0].span)
    tot = sum(r.mult.index_select(0, span) for r in ranks)
    sent = {}
    for k, h in enumerate(halos):  # owner k -> reader j, in rank order
        off = 0
        for j, c in enumerate(h.send_counts):
            sent[(k, j)] = ranks[k].mult.index_select(0, idx(h.send[off:off + c]))
            off += c
    for j, (r, h) in enumerate(zip(ranks, halos)):
        r.mult.index_copy_(0, span, tot)
        off = 0
        for k, c in enumerate(h.recv_counts):
            if c:
                r.mult.index_copy_(0, idx(h.recv[off:off + c]), sent[(k, j)])
            off += c
    out = sum(r.apply_rest().clone() for r in ranks)
    assert _rel(out.cpu().numpy(), ref.cpu().numpy()) <= 1e-13
    assert _rel(out.cpu().numpy(), g["pot"]) <= FP64_TOL


def test_cuda_graph_replay_matches_eager():
    from paper_2202_04894_b200 import FmmConfig, FmmPlan

    g = load_case("cubesurf4000")
    plan = FmmPlan(g["points"], None, FmmConfig(**g["config"]), charges=g["charges"])
    a = plan.apply().clone()
    plan.capture_graph()
    b = plan.replay().clone()
    assert torch.equal(a, b)
    plan.set_charges(2 * g["charges"])  # replay picks up new charges
    c = plan.replay().clone()
    assert _rel(c.cpu().numpy(), 2 * a.cpu().numpy()) <= 1e-14
    # after capture, the public apply() replays the graph (same buffers, same sums)
    d = plan.apply().clone()
    assert torch.equal(c, d)
    plan.set_charges(g["charges"])
    assert torch.equal(plan.apply(), a)
    # stage timers (or an explicit out=) take the eager path
    e = plan.apply(stage_events=[]).clone()
    assert torch.equal(e, a)
