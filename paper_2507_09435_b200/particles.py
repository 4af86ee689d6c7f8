"""Particle records in the reference's AoS layout and the box seeder.

impm::Particle<D> (/root/reference/proj/include/impm/particle.hpp:10-29) is a
struct of doubles; a particle set is held here as a float64 array of shape
(P, 6D+22+D*D) with the same field order, so it can be handed to the C ABI
(and to a C++ caller's std::vector<Particle<D>>) without conversion.
"""
from dataclasses import dataclass

import numpy as np


def particle_fields(D):
    """(name, offset, width) of every field of Particle<D>, in layout order."""
    spec = [("X", D), ("x", D), ("m", 1), ("V0", 1), ("V", 1), ("F", D * D), ("sigma", 9), ("lp0", D),
            ("lp", D), ("B_e", 9), ("alpha", 1), ("traction_force", D), ("point_load", D)]
    out, off = [], 0
    for name, w in spec:
        out.append((name, off, w))
        off += w
    return out


def particle_doubles(D):
    return 6 * D + 22 + D * D


class ParticleArray:
    """Named views into a (P, ND) float64 particle array (no copies)."""

    def __init__(self, data, D):
        self.D = D
        self.data = np.ascontiguousarray(data, dtype=np.float64)
        assert self.data.ndim == 2 and self.data.shape[1] == particle_doubles(D)
        self._fields = {name: (off, w) for name, off, w in particle_fields(D)}

    def __len__(self):
        return self.data.shape[0]

    def field(self, name):
        off, w = self._fields[name]
        return self.data[:, off:off + w]

    def __getattr__(self, name):
        if name.startswith("_") or name not in self.__dict__.get("_fields", {}):
            raise AttributeError(name)
        return self.field(name)

    def offset(self, name):
        return self._fields[name][0]


@dataclass
class GridSpec:
    """impm::Grid<D> (grid.hpp:18-58)."""
    dim: int
    origin: tuple
    h: float
    nodes: tuple

    def node_count(self):
        n = 1
        for a in range(self.dim):
            n *= int(self.nodes[a])
        return n

    def node_positions(self):
        """(N, D) node coordinates in flat order (axis 0 slowest, grid.hpp:30-34)."""
        idx = np.indices([int(n) for n in self.nodes[: self.dim]]).reshape(self.dim, -1).T
        return np.asarray(self.origin[: self.dim], dtype=np.float64) + idx * self.h


def seed_box_rows(grid: GridSpec, lo, hi, ppc, density, rows):
    """The particles of seed_box(grid, lo, hi, ppc, density) whose axis-0
    lattice index is in `rows` (ascending), with their global ids (row index in
    the full seed_box array), generated without the full array: axis 0 is the
    slowest lattice index, so each row is a contiguous id range."""
    D = grid.dim
    cells = [int(np.floor((hi[a] - lo[a]) / grid.h + 0.5)) for a in range(D)]
    spacing = grid.h / ppc
    vol = 1.0
    for _ in range(D):
        vol *= spacing
    sub = [c * ppc for c in cells]
    rows = np.asarray(rows, dtype=np.int64)
    inner = int(np.prod(sub[1:])) if D > 1 else 1
    total = rows.size * inner
    out = np.zeros((total, particle_doubles(D)), dtype=np.float64)
    ids = (rows[:, None] * inner + np.arange(inner, dtype=np.int64)[None, :]).reshape(-1)
    if total == 0:
        return out, ids
    pa = ParticleArray(out, D)
    idx = [np.repeat(rows, inner)]
    if D > 1:
        rest = np.indices(sub[1:]).reshape(D - 1, -1)
        for a in range(D - 1):
            idx.append(np.tile(rest[a], rows.size))
    for a in range(D):
        X = lo[a] + (idx[a].astype(np.float64) + 0.5) * spacing
        pa.X[:, a] = X
        pa.x[:, a] = X
        pa.lp0[:, a] = 0.5 * spacing
        pa.lp[:, a] = 0.5 * spacing
    pa.V0[:, 0] = vol
    pa.V[:, 0] = vol
    pa.m[:, 0] = density * vol
    F = pa.F
    for a in range(D):
        F[:, a * D + a] = 1.0
    pa.B_e[:, 0] = pa.B_e[:, 4] = pa.B_e[:, 8] = 1.0
    return out, ids


def seed_box(grid: GridSpec, lo, hi, ppc, density):
    """ppc^D equally spaced particles per cell in [lo, hi] (particle.hpp:33-69)."""
    D = grid.dim
    cells = [int(np.floor((hi[a] - lo[a]) / grid.h + 0.5)) for a in range(D)]  # std::round, positive
    spacing = grid.h / ppc
    vol = 1.0
    for _ in range(D):
        vol *= spacing
    sub = [c * ppc for c in cells]
    total = int(np.prod(sub)) if sub else 0
    out = np.zeros((total, particle_doubles(D)), dtype=np.float64)
    pa = ParticleArray(out, D)
    if total == 0:
        return out
    idx = np.indices(sub).reshape(D, -1)  # C order: last axis fastest, as the reference's k loop
    for a in range(D):
        X = lo[a] + (idx[a].astype(np.float64) + 0.5) * spacing
        pa.X[:, a] = X
        pa.x[:, a] = X
        pa.lp0[:, a] = 0.5 * spacing
        pa.lp[:, a] = 0.5 * spacing
    pa.V0[:, 0] = vol
    pa.V[:, 0] = vol
    pa.m[:, 0] = density * vol
    F = pa.F
    for a in range(D):
        F[:, a * D + a] = 1.0
    pa.B_e[:, 0] = pa.B_e[:, 4] = pa.B_e[:, 8] = 1.0
    return out
