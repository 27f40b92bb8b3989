"""Octree (drop-in for helmfmm.tree), built natively by libdefmm_b200.

``build_tree`` keeps the reference signature (tree.py:132-137) and its exact
decisions: the C++ builder (csrc/tree_build.cpp) performs the same recursive
stable octant partition with the same FP64 comparisons.  The tree is stored
as flat arrays in level-major Morton order -- the layout the device plan
consumes; ``Cell`` objects (tree.py:62-99) are materialised lazily for callers
that walk ``tree.levels`` or ``cell.sons``.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .config import TreeConfig
from .geometry import BoundingBox, CellFrame, MortonKey, compute_root_box

__all__ = [
    "TreeConfig",
    "ParticleSet",
    "Cell",
    "ClusterTree",
    "build_tree",
    "level_radius",
    "accumulate_potentials",
    "SQRT3",
]

SQRT3 = float(np.sqrt(3.0))  # tree.py:33


@dataclass
class ParticleSet:
    """Permuted SoA particles (tree.py:48-59)."""

    positions: np.ndarray
    charges: np.ndarray
    potentials: np.ndarray
    original_index: np.ndarray

    @property
    def n(self) -> int:
        return self.positions.shape[0]


@dataclass(eq=False)
class Cell:
    """Read-only view of one cell (tree.py:62-99)."""

    key: MortonKey
    level: int
    coords: np.ndarray
    start: int
    stop: int
    frame: CellFrame
    index: int = -1
    sons: list = field(default_factory=list)

    @property
    def is_leaf(self) -> bool:
        return not self.sons

    @property
    def n_particles(self) -> int:
        return self.stop - self.start

    @property
    def center(self) -> np.ndarray:
        return self.frame.center

    @property
    def side(self) -> float:
        return self.frame.beta

    @property
    def radius(self) -> float:
        return SQRT3 * self.frame.beta / 2.0


class ClusterTree:
    """Array octree.  Cells are indexed level-major, Morton order inside a level.

    Arrays: ``level, coords (m,3), start, stop, parent, first_son, n_sons,
    alpha (m,3)``; ``level_offsets[l]:level_offsets[l+1]`` spans level l.
    """

    def __init__(self, root_box, config, level, coords, start, stop, parent):
        self.root_box = root_box
        self.config = config
        self.level = level
        self.coords = coords
        self.start = start
        self.stop = stop
        self.parent = parent
        m = level.shape[0]
        self.depth = int(level.max())
        self.level_offsets = np.searchsorted(level, np.arange(self.depth + 2)).astype(np.int64)
        self.n_sons = np.bincount(parent[parent >= 0], minlength=m).astype(np.int64)
        first = np.full(m, -1, np.int64)
        kids = np.nonzero(parent >= 0)[0]
        # sons of a cell are contiguous in the next level (Morton order)
        fathers, idx = np.unique(parent[kids], return_index=True)
        first[fathers] = kids[idx]
        self.first_son = first
        self.is_leaf = self.n_sons == 0
        # frames: alpha = root.lower + coords * beta  (tree.py:165-166)
        self.level_beta = np.array([root_box.side / (1 << l) for l in range(self.depth + 1)])
        self.alpha = root_box.lower + coords * self.level_beta[level][:, None]
        self._levels = None

    # -- reference-compatible views -------------------------------------
    @property
    def n_cells(self) -> int:
        return int(self.level.shape[0])

    def side_at(self, level: int) -> float:
        return self.root_box.side / (1 << level)

    def morton_code(self, idx) -> np.ndarray:
        """Morton codes (tree.py:195 ``(father << 3) | octant``) of cells."""
        from .geometry import morton_encode_many

        idx = np.atleast_1d(idx)
        out = np.empty(idx.shape[0], np.uint64)
        for lev in np.unique(self.level[idx]):
            sel = self.level[idx] == lev
            out[sel] = morton_encode_many(self.coords[idx[sel]], int(lev))
        return out

    @property
    def levels(self) -> list:
        if self._levels is None:
            codes = self.morton_code(np.arange(self.n_cells))
            cells = [
                Cell(
                    key=MortonKey(int(codes[c]), int(self.level[c])),
                    level=int(self.level[c]),
                    coords=self.coords[c].copy(),
                    start=int(self.start[c]),
                    stop=int(self.stop[c]),
                    frame=CellFrame(alpha=self.alpha[c], beta=self.level_beta[self.level[c]]),
                    index=c,
                )
                for c in range(self.n_cells)
            ]
            for c in range(1, self.n_cells):
                cells[self.parent[c]].sons.append(cells[c])
            self._levels = [
                cells[self.level_offsets[l] : self.level_offsets[l + 1]] for l in range(self.depth + 1)
            ]
        return self._levels

    @property
    def root(self) -> Cell:
        return self.levels[0][0]

    @property
    def leaves(self) -> list:
        return [c for lv in self.levels for c in lv if c.is_leaf]

    @property
    def n_leaves(self) -> int:
        return int(self.is_leaf.sum())


def level_radius(tree: ClusterTree, level: int) -> float:
    if level < 0 or level > tree.depth:
        raise ValueError("level out of range")
    return SQRT3 * tree.side_at(level) / 2.0


def build_tree(points, charges, config: TreeConfig = TreeConfig(), root_box: BoundingBox | None = None):
    """Ncrit octree + permuted particles; same decisions as tree.py:132-213."""
    points = np.atleast_2d(np.asarray(points, dtype=float))
    charges = np.asarray(charges, dtype=complex)
    if points.shape[0] == 0:
        raise ValueError("at least one particle is required")
    if points.shape[0] != charges.shape[0]:
        raise ValueError("points and charges length mismatch")
    if not np.all(np.isfinite(points)):
        raise ValueError("particle coordinates must be finite")
    if root_box is None:
        root_box = compute_root_box(points)
    lib = _lib.load()
    pts = np.ascontiguousarray(points, dtype=np.float64)
    n = pts.shape[0]
    lower = np.ascontiguousarray(root_box.lower, dtype=np.float64)
    handle = C.c_void_p()
    _lib.check(
        lib.defmm_tree_build(pts.ctypes.data, n, lower.ctypes.data, float(root_box.side), int(config.ncrit),
                             int(config.hard_depth_cap), C.byref(handle)),
        "defmm_tree_build",
    )
    try:
        m = int(lib.defmm_tree_ncells(handle))
        perm = np.empty(n, np.int64)
        spts = np.empty((n, 3), np.float64)
        level = np.empty(m, np.int32)
        coords = np.empty((m, 3), np.int64)
        start = np.empty(m, np.int64)
        stop = np.empty(m, np.int64)
        parent = np.empty(m, np.int64)
        _lib.check(
            lib.defmm_tree_fetch(handle, perm.ctypes.data, spts.ctypes.data, level.ctypes.data, coords.ctypes.data,
                                 start.ctypes.data, stop.ctypes.data, parent.ctypes.data),
            "defmm_tree_fetch",
        )
    finally:
        lib.defmm_tree_free(handle)
    # DFS creation order -> level-major; inside a level DFS order is Morton
    # order, i.e. increasing start (tree.py:168-170 appends per level in DFS order)
    order = np.lexsort((np.arange(m), level))
    inv = np.empty(m, np.int64)
    inv[order] = np.arange(m)
    par = parent[order]
    par = np.where(par >= 0, inv[np.maximum(par, 0)], -1)
    tree = ClusterTree(root_box, config, level[order].astype(np.int64), coords[order], start[order], stop[order], par)
    pset = ParticleSet(
        positions=spts,
        charges=charges[perm].copy(),
        potentials=np.zeros(n, dtype=complex),
        original_index=perm,
    )
    return tree, pset


def accumulate_potentials(pset: ParticleSet) -> np.ndarray:
    """Un-permute (tree.py:224-228)."""
    out = np.empty_like(pset.potentials)
    out[pset.original_index] = pset.potentials
    return out
