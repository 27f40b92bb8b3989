"""Morton-order sharding of one FMM plan over the ranks of one node.

SURVEY.md §8(e): the target leaves, already in Morton (= particle) order, are
cut into ``world`` contiguous chunks balanced by an estimate of their work
(24 flop per P2P pair + 8 P^3 flop per M2L event, weighted by the measured
per-unit costs), with cuts on leaf boundaries so no leaf straddles two ranks.

Rank r then owns the particle range [cut[r], cut[r+1]) and works only on the
cells whose particle range intersects it ("active" cells):

* upward: P2M on its own leaves, M2M on its active cells.  A cell spanning
  several chunks gets a PARTIAL multipole on each rank (its other sons are
  zero there); a cell inside one chunk is complete on its owner only;
* halo exchange (the only data-path communication): one
  ``all_reduce(sum)`` over the few spanning (top-of-tree) multipoles -- M2M is
  linear, so the partial sums complete them -- and one ``all_to_all`` that
  sends each rank exactly the complete nodal multipoles (L^3 each, 5-7x fewer
  bytes than spectra) its M2L rows read from other ranks' chunks.  Index sets
  are static per plan (``Halo``); ``allreduce=`` (sum of the whole multipole
  array) remains for the virtual-rank tests;
* M2F only for the spectra its own M2L rows read;
* M2L rows, L2L slots and L2P/P2P leaves of its active target cells (shared
  top cells are computed redundantly by every rank that needs them), so the
  far field needs no halo exchange of locals;
* near-field halo: a rank is given only the charges of its own chunk; one
  ``all_to_all`` per matvec (``ChargeHalo``, ``charge_exchange``) brings in
  exactly the source charges its P2P leaves read from other chunks (the
  near-field source leaves next to its boundary).  Positions are geometry,
  static per plan.

Single-tree mode (targets is sources) only; the two-tree mode runs replicas.
Everything here is host-side index bookkeeping (numpy); it is exercised with
world_size-2 gloo process groups on CPU in tests/test_parallel.py.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["Shard", "Halo", "ChargeHalo", "leaf_costs", "partition_leaves", "make_shard", "make_halo",
           "halo_exchange", "make_charge_halo", "charge_exchange"]

# relative unit costs measured on the B200 (profiles/r01_summary_v2.md, c64):
# M2L ~2.9 ms / 10.8 M events; P2P ~0.77 ms / 3.83e8 pairs
_COST_M2L_EVENT = 2.9e-3 / 10.84e6
_COST_P2P_PAIR = 0.77e-3 / 3.83e8


def leaf_costs(plan, tt) -> np.ndarray:
    """Estimated work per target leaf (in plan.leaf_cells order)."""
    leaves = plan.leaf_cells
    n_t = (tt.stop[leaves] - tt.start[leaves]).astype(np.float64)
    n_src = np.zeros(leaves.shape[0], np.float64)
    run_len = (plan.p2p_hi - plan.p2p_lo).astype(np.float64)
    cs = np.concatenate([[0.0], np.cumsum(run_len)])
    n_src = cs[plan.p2p_ptr[1:]] - cs[plan.p2p_ptr[:-1]]
    cost = n_t * n_src * _COST_P2P_PAIR
    # M2L events of every row whose target cell contains the leaf, spread over
    # the leaves by particle count
    rows = plan.m2l_row_slot
    rc = plan.l_cell[rows]
    ev = np.diff(plan.m2l_row_ptr).astype(np.float64)
    lstart = tt.start[leaves]
    a = np.searchsorted(lstart, tt.start[rc])
    b = np.searchsorted(lstart, tt.stop[rc])
    per_particle = ev * _COST_M2L_EVENT / (tt.stop[rc] - tt.start[rc])
    # difference array over leaf indices, weighted by the leaf's particle count
    acc = np.zeros(leaves.shape[0] + 1, np.float64)
    np.add.at(acc, a, per_particle)
    np.add.at(acc, b, -per_particle)
    cost += np.cumsum(acc)[:-1] * n_t
    return cost


def partition_leaves(plan, tt, world: int) -> np.ndarray:
    """Particle-index cuts (world+1) on leaf boundaries, balanced by cost."""
    leaves = plan.leaf_cells
    if world <= 1 or leaves.shape[0] < world:
        return np.array([0, int(tt.stop[0])] if world <= 1 else [0] + [int(tt.stop[0])] * world, np.int64)
    c = np.cumsum(leaf_costs(plan, tt))
    targets = c[-1] * np.arange(1, world) / world
    k = np.searchsorted(c, targets)  # leaf index where each chunk ends
    k = np.clip(k, 0, leaves.shape[0] - 1)
    cuts = [0] + [int(tt.stop[leaves[i]]) for i in k] + [int(tt.stop[0])]
    return np.maximum.accumulate(np.array(cuts, np.int64))


@dataclass
class Shard:
    rank: int
    world: int
    lo: int  # owned particle range [lo, hi)
    hi: int
    p2m_idx: np.ndarray  # subset of plan.p2m_idx
    m2m_keep: list  # per plan.m2m_levels entry: row mask
    hat_keep: np.ndarray  # spectra this rank transforms
    row_keep: np.ndarray  # M2L rows this rank computes
    l2l_keep: list  # per plan.l2l_levels entry: out mask
    leaf_keep: np.ndarray  # target leaves (plan.leaf_cells order)
    cuts: np.ndarray = None  # particle cuts of all ranks (world + 1)


def make_shard(plan, tt, st, rank: int, world: int, cuts=None) -> Shard:
    if tt is not st:
        raise ValueError("sharding is implemented for single-tree plans (targets is sources)")
    cuts = partition_leaves(plan, tt, world) if cuts is None else np.asarray(cuts)
    lo, hi = int(cuts[rank]), int(cuts[rank + 1])

    def active(cells):
        return (tt.start[cells] < hi) & (tt.stop[cells] > lo)

    p2m_idx = plan.p2m_idx[active(plan.m_cell[plan.p2m_idx])]
    m2m_keep = [active(plan.m_cell[slots]) for _, slots, _ in plan.m2m_levels]
    rows = plan.m2l_row_slot
    row_keep = active(plan.l_cell[rows])
    # spectra read by the kept rows
    e = np.repeat(row_keep, np.diff(plan.m2l_row_ptr))
    hat_keep = np.zeros(plan.n_hat, bool)
    hat_keep[plan.m2l_rows_entries[e, 0]] = True
    l2l_keep = [active(plan.l_cell[outs]) for _, outs, *_ in plan.l2l_levels]
    leaf_keep = active(plan.leaf_cells)
    return Shard(rank, world, lo, hi, p2m_idx, m2m_keep, hat_keep, row_keep, l2l_keep, leaf_keep, np.asarray(cuts))


@dataclass
class Halo:
    """Static index sets of one rank's multipole exchange (slots into the
    plan's multipole array; counts per peer rank, in rank order)."""
    span: np.ndarray  # spanning multipoles (same list on every rank), all-reduced
    send: np.ndarray  # complete multipoles this rank owns and others read, by destination
    send_counts: list
    recv: np.ndarray  # multipoles this rank reads from others, by source
    recv_counts: list
    active: bool = True  # any rank exchanges anything (the all_to_all is collective: same on every rank)


def _rank_span(plan, tt, cuts):
    """First and last rank whose chunk intersects each multipole's cell."""
    cells = plan.m_cell
    a = np.searchsorted(cuts, tt.start[cells], side="right") - 1
    b = np.searchsorted(cuts, tt.stop[cells] - 1, side="right") - 1
    return a, b


def _needed(plan, tt, cuts, r) -> np.ndarray:
    """Multipole slots whose spectra rank r's M2L rows read (sorted)."""
    lo, hi = int(cuts[r]), int(cuts[r + 1])
    rc = plan.l_cell[plan.m2l_row_slot]
    keep = (tt.start[rc] < hi) & (tt.stop[rc] > lo)
    e = np.repeat(keep, np.diff(plan.m2l_row_ptr))
    hats = np.unique(plan.m2l_rows_entries[e, 0])
    return np.unique(plan.hat_slot[hats])


def make_halo(plan, tt, cuts, rank: int, world: int) -> Halo:
    cuts = np.asarray(cuts)
    a, b = _rank_span(plan, tt, cuts)
    span = np.nonzero(a != b)[0]
    owner = np.where(a == b, a, -1)
    need = [_needed(plan, tt, cuts, r) for r in range(world)]
    # does any rank read a multipole owned by another one? (identical on every rank)
    active = any(bool(np.any((owner[nd] >= 0) & (owner[nd] != r))) for r, nd in enumerate(need))
    send, send_counts, recv, recv_counts = [], [], [], []
    for r in range(world):
        if r == rank:
            send_counts.append(0)
            recv_counts.append(0)
            continue
        s_r = need[r][owner[need[r]] == rank]  # mine, read by r
        v_r = need[rank][owner[need[rank]] == r]  # r's, read by me
        send.append(s_r)
        recv.append(v_r)
        send_counts.append(int(s_r.shape[0]))
        recv_counts.append(int(v_r.shape[0]))
    cat = lambda xs: np.concatenate(xs).astype(np.int64) if xs else np.zeros(0, np.int64)  # noqa: E731
    return Halo(span.astype(np.int64), cat(send), send_counts, cat(recv), recv_counts, active)


def halo_exchange(mult, halo_dev, group=None):
    """Complete the multipoles this rank's M2F reads.  ``mult``: (n_mult, L^3)
    complex tensor; ``halo_dev`` = (span, send, send_counts, recv, recv_counts,
    active) with the index tensors on mult's device.  Complex data travels as its real
    view (NCCL / gloo have no complex types)."""
    import torch
    import torch.distributed as dist

    span, send, send_counts, recv, recv_counts, active = halo_dev
    if span.numel():  # the same list on every rank
        buf = mult.index_select(0, span)
        dist.all_reduce(torch.view_as_real(buf), group=group)
        mult.index_copy_(0, span, buf)
    if active:  # collective: decided identically on every rank (Halo.active)
        per = 2 * mult.shape[1]  # reals per multipole
        sbuf = torch.view_as_real(mult.index_select(0, send)).contiguous()
        rbuf = torch.empty((recv.shape[0], mult.shape[1], 2), dtype=sbuf.dtype, device=mult.device)
        dist.all_to_all_single(rbuf.view(-1), sbuf.view(-1), [c * per for c in recv_counts],
                               [c * per for c in send_counts], group=group)
        mult.index_copy_(0, recv, torch.view_as_complex(rbuf))


@dataclass
class ChargeHalo:
    """Static particle index sets of one rank's near-field charge exchange
    (sorted particle order; counts per peer rank, in rank order)."""
    send: np.ndarray  # own particles other ranks' P2P reads, by destination
    send_counts: list
    recv: np.ndarray  # other ranks' particles this rank's P2P reads, by source
    recv_counts: list
    active: bool = True  # identical on every rank (the all_to_all is collective)


def _p2p_sources(plan, tt, cuts, r) -> np.ndarray:
    """Sorted particle indices the P2P leaves of rank r read, outside its chunk."""
    lo, hi = int(cuts[r]), int(cuts[r + 1])
    leaves = plan.leaf_cells
    keep = (tt.start[leaves] < hi) & (tt.stop[leaves] > lo)
    e = np.repeat(keep, np.diff(plan.p2p_ptr))
    a, b = plan.p2p_lo[e], plan.p2p_hi[e]
    if a.size == 0:
        return np.zeros(0, np.int64)
    # union of the runs, then drop the own chunk
    o = np.argsort(a, kind="stable")
    a, b = a[o], b[o]
    cover = np.zeros(int(tt.stop[0]) + 1, np.int64)
    np.add.at(cover, a, 1)
    np.add.at(cover, b, -1)
    idx = np.nonzero(np.cumsum(cover)[:-1] > 0)[0]
    return idx[(idx < lo) | (idx >= hi)].astype(np.int64)


def make_charge_halo(plan, tt, cuts, rank: int, world: int) -> ChargeHalo:
    cuts = np.asarray(cuts)
    need = [_p2p_sources(plan, tt, cuts, r) for r in range(world)]
    active = any(x.size for x in need)
    send, send_counts, recv, recv_counts = [], [], [], []
    for r in range(world):
        if r == rank:
            send_counts.append(0)
            recv_counts.append(0)
            continue
        lo, hi = int(cuts[rank]), int(cuts[rank + 1])
        s_r = need[r][(need[r] >= lo) & (need[r] < hi)]  # mine, read by r
        rlo, rhi = int(cuts[r]), int(cuts[r + 1])
        v_r = need[rank][(need[rank] >= rlo) & (need[rank] < rhi)]  # r's, read by me
        send.append(s_r)
        recv.append(v_r)
        send_counts.append(int(s_r.shape[0]))
        recv_counts.append(int(v_r.shape[0]))
    cat = lambda xs: np.concatenate(xs).astype(np.int64) if xs else np.zeros(0, np.int64)  # noqa: E731
    return ChargeHalo(cat(send), send_counts, cat(recv), recv_counts, bool(active))


def charge_exchange(q, halo_dev, group=None):
    """Fill the other-chunk source charges this rank's P2P reads: ``q`` is
    the (n,) complex charge vector in sorted order holding this rank's chunk;
    ``halo_dev`` = (send, send_counts, recv, recv_counts, active) with index
    tensors on q's device."""
    import torch
    import torch.distributed as dist

    send, send_counts, recv, recv_counts, active = halo_dev
    if not active:
        return
    sbuf = torch.view_as_real(q.index_select(0, send)).contiguous()
    rbuf = torch.empty((recv.shape[0], 2), dtype=sbuf.dtype, device=q.device)
    dist.all_to_all_single(rbuf.view(-1), sbuf.view(-1), [2 * c for c in recv_counts],
                           [2 * c for c in send_counts], group=group)
    q.index_copy_(0, recv, torch.view_as_complex(rbuf))
