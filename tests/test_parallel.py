"""Multi-rank (Morton-sharded) plan logic on CPU with world_size-2 gloo groups.

The device kernels are not run here; what is checked is the host-side
bookkeeping the N>1 path depends on (parallel.py): leaf chunks tile the
particles on leaf boundaries, every P2P leaf / P2M leaf / M2L row is owned by
some rank, and the partial upward pass + one all-reduce reconstructs every
multipole -- emulated with an exactly-additive quantity (the particle count
below each multipole slot) reduced over a real gloo process group.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import load_case
from paper_2202_04894_b200.config import TreeConfig
from paper_2202_04894_b200.parallel import make_shard, partition_leaves
from paper_2202_04894_b200.plan import build_plan
from paper_2202_04894_b200.tree import build_tree


def _plan(case):
    g = load_case(case)
    kw = g["config"]
    tr, ps = build_tree(g["points"], g["charges"], TreeConfig(ncrit=kw["ncrit"]))
    return tr, build_plan(tr, tr, kw["order"], kw["kappa"], 1.0, 2.0)


def _partial_counts(tr, pl, sh):
    """Particles of this rank's chunk below every multipole slot (0 elsewhere),
    propagated like the upward pass: leaf slots from particles, fathers as sums
    over son slots -- only on active slots."""
    cnt = np.zeros(pl.n_mult, np.int64)
    for s in sh.p2m_idx:
        c = pl.m_cell[s]
        cnt[s] = max(0, min(tr.stop[c], sh.hi) - max(tr.start[c], sh.lo))
    for k, (lev, slots, son_slot) in enumerate(pl.m2m_levels):
        keep = sh.m2m_keep[k]
        for s, sons in zip(slots[keep], son_slot[keep]):
            cnt[s] = sum(cnt[x] for x in sons if x >= 0)
    return cnt


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr, pl = _plan(case)
        sh = make_shard(pl, tr, tr, rank, world)
        part = torch.from_numpy(_partial_counts(tr, pl, sh))
        dist.all_reduce(part)  # the multipole all-reduce of the device path
        full = np.array([tr.stop[c] - tr.start[c] for c in pl.m_cell])
        # every multipole that is computed at all (plan.m_used: read by an M2L or by a needed father)
        ok_counts = bool(np.array_equal(part.numpy()[pl.m_used], full[pl.m_used]))
        cover = {}
        for name, mask in (("leaves", sh.leaf_keep), ("rows", sh.row_keep)):
            t = torch.from_numpy(mask.astype(np.int64))
            dist.all_reduce(t)
            cover[name] = t.numpy()
        p2m = np.zeros(pl.n_mult, np.int64)
        p2m[sh.p2m_idx] = 1
        t = torch.from_numpy(p2m)
        dist.all_reduce(t)
        q.put((rank, ok_counts, cover["leaves"].tolist(), int(cover["rows"].min()), t.numpy()[pl.p2m_idx].tolist()))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case", ["cubesurf4000", "volume3000"])
def test_sharded_upward_allreduce_reconstructs_multipoles_gloo(case):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_counts, leaves, rows_min, p2m in res:
        assert ok_counts, f"rank {rank}: partial multipoles + all-reduce != full"
        assert all(v == 1 for v in leaves)  # every target leaf owned by exactly one rank
        assert rows_min >= 1  # every M2L row computed by at least one rank
        assert all(v == 1 for v in p2m)  # every leaf multipole produced exactly once


@pytest.mark.parametrize("world", [2, 3, 8])
def test_partition_cuts_on_leaf_boundaries_and_balanced(world):
    tr, pl = _plan("volume3000")
    cuts = partition_leaves(pl, tr, world)
    assert cuts[0] == 0 and cuts[-1] == tr.stop[0] and np.all(np.diff(cuts) >= 0)
    leaf_bounds = set(tr.stop[pl.leaf_cells].tolist()) | {0}
    assert all(int(c) in leaf_bounds for c in cuts)
    from paper_2202_04894_b200.parallel import leaf_costs

    cost = leaf_costs(pl, tr)
    lstart = tr.start[pl.leaf_cells]
    per = [cost[(lstart >= a) & (lstart < b)].sum() for a, b in zip(cuts[:-1], cuts[1:])]
    assert max(per) <= 1.6 * (sum(per) / world)


def test_sharding_rejects_two_tree_plans():
    g = load_case("laplace500")
    tr, ps = build_tree(g["points"], g["charges"], TreeConfig(ncrit=32))
    tr2, ps2 = build_tree(g["points"] * 0.5, g["charges"], TreeConfig(ncrit=32), root_box=tr.root_box)
    pl = build_plan(tr2, tr, 5, 0.0, 1.0, 2.0)
    with pytest.raises(ValueError):
        make_shard(pl, tr2, tr, 0, 2)


def _halo_worker(rank, world, port, case, q):
    """Halo exchange (span all-reduce + all_to_all of owned complete multipoles)
    over a real gloo group, on the exactly-additive emulation: afterwards every
    multipole this rank's M2F reads equals the full particle count below it."""
    from paper_2202_04894_b200.parallel import _needed, halo_exchange, make_halo

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tr, pl = _plan(case)
        sh = make_shard(pl, tr, tr, rank, world)
        h = make_halo(pl, tr, sh.cuts, rank, world)
        cnt = _partial_counts(tr, pl, sh).astype(np.float64)
        mult = torch.from_numpy(np.stack([cnt, 2.0 * cnt], 1)).to(torch.complex128)
        mult[:, 1] *= 1j
        idx = lambda a: torch.as_tensor(a, dtype=torch.int64)  # noqa: E731
        halo_exchange(mult, (idx(h.span), idx(h.send), h.send_counts, idx(h.recv), h.recv_counts, h.active))
        need = _needed(pl, tr, sh.cuts, rank)
        full = np.array([tr.stop[c] - tr.start[c] for c in pl.m_cell], np.float64)
        got = mult.numpy()
        ok = bool(np.array_equal(got[need, 0].real, full[need]) and np.array_equal(got[need, 1].imag, 2 * full[need]))
        # the exchange moves far fewer multipoles than an all-reduce of all of them
        q.put((rank, ok, int(h.span.shape[0]), int(h.send.shape[0]), int(h.recv.shape[0]), pl.n_mult))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("cubesurf4000", 2), ("cubesurf4000", 3), ("volume3000", 4)])
def test_halo_exchange_completes_every_needed_multipole(case, world):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = [q.get() for _ in range(world)]
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok, n_span, n_send, n_recv, n_mult in res:
        assert ok, rank
        assert n_span + n_recv < n_mult  # a halo, not the whole multipole array


def _charge_worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_04894_b200.parallel import _p2p_sources, charge_exchange, make_charge_halo

        tr, pl = _plan(case)
        sh = make_shard(pl, tr, tr, rank, world)
        h = make_charge_halo(pl, tr, sh.cuts, rank, world)
        n = int(tr.stop[0])
        full = torch.arange(n, dtype=torch.float64) + 1j * torch.arange(n, dtype=torch.float64) / 7
        mine = full.clone()
        mine[: sh.lo] = 0
        mine[sh.hi:] = 0
        dev = (torch.as_tensor(h.send), list(h.send_counts), torch.as_tensor(h.recv), list(h.recv_counts), h.active)
        charge_exchange(mine, dev)
        need = _p2p_sources(pl, tr, sh.cuts, rank)
        own = torch.arange(sh.lo, sh.hi)
        ok = bool(torch.equal(mine[need], full[need])) and bool(torch.equal(mine[own], full[own]))
        # every source a kept P2P run reads is now present
        leaves = pl.leaf_cells[sh.leaf_keep]
        sel = np.repeat(sh.leaf_keep, np.diff(pl.p2p_ptr))
        runs_ok = all(bool(torch.equal(mine[a:b], full[a:b])) for a, b in zip(pl.p2p_lo[sel], pl.p2p_hi[sel]))
        q.put((rank, ok and runs_ok and leaves.size > 0, int(h.send.size), int(h.recv.size)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", ["cubesurf4000", "volume3000"])
def test_gloo_near_field_charge_halo(case, world):
    """Each rank starts from its own chunk's charges only; one all_to_all
    (parallel.charge_exchange) brings every source charge its P2P runs read."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_charge_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] for r in res), res
    assert sum(r[2] for r in res) == sum(r[3] for r in res) > 0
