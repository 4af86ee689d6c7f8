"""Slab decomposition of the implicit MPM Newton step along grid axis 0
(SURVEY.md §8(e)).

Axis 0 is the slowest index of Grid::flat (grid.hpp:30-34) and DofMap::build
numbers DOFs in ascending node order (grid.hpp:76-85), so a slab of owned
nodes [a, b) along axis 0 is a contiguous node range, a contiguous range of
global DOFs and a contiguous block of Jacobian rows. Each rank keeps:

  - owned nodes [a, b): their residual and Jacobian rows are computed here;
  - particles whose support (first node f, <= 3 nodes) meets [a, b):
    f in [a - 2, b), the owned bins plus two ghost bin layers below;
  - a local grid [a - 2, b + 2) (clamped), which holds every support node of
    the kept particles and the 2-node x-halo that the +-2 Jacobian coupling
    (jacobian.hpp:38) reads.

The collectives per Newton iteration are the ones the north star names: the
2-layer halo of vectors before each SpMV / residual, fp64 allreduces for the
Krylov dots and the Newton norm, and an allgather of owned free-DOF counts
once per load step (global numbering = exclusive scan, bit-exact with the
single-GPU DofMap). Particles migrate between slabs at the end of each load step.
"""
from dataclasses import dataclass

import numpy as np

from .particles import GridSpec, ParticleArray


def support_first(grid: GridSpec, parts: np.ndarray, axis: int = 0, use_X: bool = False):
    """First support node along `axis` (src/gimp.cpp:46-53, same fp64 ops)."""
    pa = ParticleArray(parts, grid.dim)
    x = (pa.X if use_X else pa.x)[:, axis]
    lp = pa.lp[:, axis]
    lo = (x - grid.origin[axis] - (grid.h + lp)) / grid.h
    return np.floor(lo).astype(np.int64) + 1


@dataclass
class Slab:
    rank: int
    nranks: int
    own_lo: int      # owned nodes [own_lo, own_hi) along axis 0 (global index)
    own_hi: int
    loc_lo: int      # local grid [loc_lo, loc_hi) along axis 0 (global index)
    loc_hi: int
    grid: GridSpec   # local grid (origin shifted)
    particle_ids: np.ndarray  # global particle indices kept (owned first, then ghosts)
    n_owned_particles: int

    @property
    def own_local(self):
        return self.own_lo - self.loc_lo, self.own_hi - self.loc_lo


def partition_nodes(n0: int, nranks: int, weights=None):
    """Contiguous axis-0 node ranges; balanced by per-plane weight (e.g. the
    particle count of each bin plane) or by node count."""
    w = np.ones(n0) if weights is None else np.asarray(weights, dtype=float) + 1e-9
    c = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for r in range(1, nranks):
        cuts.append(int(np.searchsorted(c, c[-1] * r / nranks)))
    cuts.append(n0)
    for r in range(1, nranks + 1):  # keep every slab non-empty
        cuts[r] = max(cuts[r], cuts[r - 1] + 1)
    cuts[-1] = n0
    return [(cuts[r], cuts[r + 1]) for r in range(nranks)]


def make_slab(grid: GridSpec, parts: np.ndarray, rank: int, nranks: int, ranges=None, use_X=False):
    n0 = int(grid.nodes[0])
    first = support_first(grid, parts, 0, use_X)
    if ranges is None:
        ranges = partition_nodes(n0, nranks, np.bincount(np.clip(first, 0, n0 - 1), minlength=n0))
    a, b = ranges[rank]
    lo, hi = max(0, a - 2), min(n0, b + 2)
    owned = np.nonzero((first >= a) & (first < b))[0]
    ghost = np.nonzero((first >= a - 2) & (first < a))[0]
    origin = list(grid.origin)
    origin[0] = grid.origin[0] + lo * grid.h
    nodes = list(grid.nodes)
    nodes[0] = hi - lo
    lg = GridSpec(grid.dim, tuple(origin), grid.h, tuple(nodes))
    return Slab(rank, nranks, a, b, lo, hi, lg, np.concatenate([owned, ghost]), len(owned))


def local_node_map(grid: GridSpec, slab: Slab):
    """global flat node index of every local node (local flat order)."""
    inner = int(np.prod(grid.nodes[1:grid.dim])) if grid.dim > 1 else 1
    loc_n0 = slab.loc_hi - slab.loc_lo
    return (np.arange(loc_n0)[:, None] + slab.loc_lo) * inner + np.arange(inner)[None, :]


def owned_node_mask(slab: Slab, grid: GridSpec):
    inner = int(np.prod(grid.nodes[1:grid.dim])) if grid.dim > 1 else 1
    i0 = np.repeat(np.arange(slab.loc_lo, slab.loc_hi), inner)
    return (i0 >= slab.own_lo) & (i0 < slab.own_hi)


def global_dof_offsets(owned_counts):
    """exclusive scan of the allgathered owned free-DOF counts."""
    return np.concatenate([[0], np.cumsum(owned_counts)])[:-1]


def halo_plan(slab: Slab, grid: GridSpec):
    """(send, recv) local-node index ranges per neighbour for the 2-layer
    x-halo along axis 0: send my first / last two owned planes, receive the
    neighbour's into my halo planes."""
    inner = int(np.prod(grid.nodes[1:grid.dim])) if grid.dim > 1 else 1
    a, b = slab.own_local
    nloc = slab.loc_hi - slab.loc_lo
    plan = {}
    if slab.rank > 0:
        plan[slab.rank - 1] = ((a * inner, min(a + 2, b) * inner), (0, a * inner))
    if slab.rank < slab.nranks - 1:
        plan[slab.rank + 1] = ((max(b - 2, a) * inner, b * inner), (b * inner, nloc * inner))
    return plan


def migrate(grid: GridSpec, parts_global_ids, parts: np.ndarray, ranges, use_X=False):
    """owner rank of every particle after a step (bin of its first support node)."""
    first = support_first(grid, parts, 0, use_X)
    bounds = np.array([r[0] for r in ranges] + [ranges[-1][1]])
    return np.clip(np.searchsorted(bounds, first, side="right") - 1, 0, len(ranges) - 1)
