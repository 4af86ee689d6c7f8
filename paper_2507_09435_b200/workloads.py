"""Synthetic problems of BASELINE.json's configs.

All use seed_box (particle.hpp:33-69) on the scenario grid convention of the
reference (origin -h, cells+3 nodes per axis, src/scenarios.cpp:96-98),
fp64, fixed seeds. Where a config names a model the reference does not have
(Drucker-Prager, modified Cam-Clay) the pinned substitute of SURVEY.md §8(d)
is used and the substitution is named in `Problem.note`.
"""
from dataclasses import dataclass, field

import numpy as np

from .particles import GridSpec, ParticleArray, seed_box
from .sim import ElasticParams, MaterialSpec, SolverOptions


@dataclass
class Problem:
    name: str
    grid: GridSpec
    particles: np.ndarray
    material: MaterialSpec
    options: SolverOptions
    fixed: np.ndarray
    gravity: np.ndarray
    load_steps: int
    note: str = ""
    meta: dict = field(default_factory=dict)


def _column_fixed(grid: GridSpec, extent):
    """base fixed, lateral rollers (src/inverse.cpp:33-36 pattern, D-dimensional)."""
    D = grid.dim
    pos = grid.node_positions()
    fixed = np.zeros((pos.shape[0], D), dtype=np.uint8)
    fixed[pos[:, D - 1] <= 1e-12, :] = 1
    for a in range(D - 1):
        side = (pos[:, a] <= 1e-12) | (pos[:, a] >= extent[a] - 1e-12)
        fixed[side, a] = 1
    return fixed.reshape(-1)


def _strip_traction(parts, D, extent, frac, t_hat, axes=None):
    """traction on the top particle layer under a centred strip/patch
    (src/inverse.cpp:45-61 pattern); axes = lateral axes the strip is narrow in."""
    pa = ParticleArray(parts, D)
    X = pa.X
    top = X[:, D - 1].max()
    sel = X[:, D - 1] >= top - 1e-9
    axes = list(range(D - 1)) if axes is None else axes
    area = 1.0
    for a in range(D - 1):
        if a in axes:
            lo, hi = 0.5 * extent[a] * (1 - frac), 0.5 * extent[a] * (1 + frac)
            sel &= (X[:, a] >= lo) & (X[:, a] <= hi)
            area *= extent[a] * frac
        else:
            area *= extent[a]
    n = int(sel.sum())
    pa.traction_force[sel, D - 1] = -t_hat * area / max(n, 1)
    return n


def column2d_nh(cells=64, ppc=2, h=1.0, steps=10):
    """cfg 1: 2D neo-Hookean column under self-weight, 64x64 cells, ~16K particles."""
    grid = GridSpec(2, (-h, -h), h, (cells + 3, cells + 3))
    W = cells * h
    parts = seed_box(grid, (0.0, 0.0), (W, W), ppc, 2000.0)
    mat = MaterialSpec("neo_hookean", ElasticParams(10e6, 0.3))
    return Problem("cfg1_column2d_nh", grid, parts, mat, SolverOptions(tol=1e-10), _column_fixed(grid, (W, W)),
                   np.array([0.0, -9.81]), steps, note="GIMP transfer (pinned); B-spline variant unpinned")


def slope2d(cells=(256, 128), ppc=4, h=0.5, steps=20, friction_deg=30.0, E=10e6, nu=0.3, material="drucker_prager",
            slope_deg=45.0, kappa=400e3, cohesion=120e3):
    """cfg 2: 2D slope under a gravity ramp, 256x128 cells, ppc 4 (401,216
    particles after the slope cut). Drucker-Prager is an extension (parity
    unpinned); the pinned substitute of SURVEY.md §8(d) is hencky_j2 (pass
    material="hencky_j2"). Body = seed_box filtered by y <= (x - x_toe)
    tan(beta) up to the crest, base fixed, lateral rollers, gravity ramped over
    `steps` increments.

    The reference is quasi-static (no inertia, mpm_solver.hpp:248-355): past
    the limit load no equilibrium exists and Newton cannot follow a collapse.
    The default strengths put the 64 m, 45 deg slope near its limit state
    (J2: kappa 400 kPa, i.e. c_u = 283 kPa against Taylor's ~230 kPa; DP:
    30 deg with 120 kPa cohesion), so a plastic zone forms at full gravity."""
    W, H = cells[0] * h, cells[1] * h
    grid = GridSpec(2, (-h, -h), h, (cells[0] + 3, cells[1] + 3))
    parts = seed_box(grid, (0.0, 0.0), (W, H), ppc, 2000.0)
    pa = ParticleArray(parts, 2)
    x_toe = W - H / np.tan(np.radians(slope_deg))
    keep = pa.X[:, 1] <= np.maximum(0.25 * H, (W - pa.X[:, 0]) * np.tan(np.radians(slope_deg)) + 0.0 * x_toe)
    parts = np.ascontiguousarray(parts[keep])
    mat = MaterialSpec(material, ElasticParams(E, nu), kappa if material == "hencky_j2" else 0.0, friction_deg,
                       cohesion)
    return Problem("cfg2_slope2d_" + material, grid, parts, mat, SolverOptions(tol=1e-10),
                   _column_fixed(grid, (W, H)), np.array([0.0, -9.81]), steps,
                   note=("Drucker-Prager (extension, parity unpinned)" if material == "drucker_prager"
                         else "hencky_j2 pinned substitute for Drucker-Prager"))


# cfg 4 clay (modified Cam-Clay, extension): critical-state angle 30 deg
# (M = 1.2), preconsolidation 600 kPa (lightly overconsolidated over the 32 m
# depth: mean overburden reaches ~400 kPa), theta = (1 + e0)/(lambda - kappa)
# = 10, tensile intercept 5 kPa
CAM_CLAY = {"friction_deg": 30.0, "cohesion": 5e3, "pc0": 600e3, "hardening": 10.0}

# north_star's target material (extension, parity unpinned): Drucker-Prager on
# Hencky strain, 30 deg friction, 20 kPa cohesion. Under the 100 kPa strip the
# shallow soil beside the footing edges yields (the plastic zone of a
# bearing-capacity problem); the deeper soil stays elastic.
DRUCKER_PRAGER = {"friction_deg": 30.0, "cohesion": 20e3}


def _footing_material(material, E, nu):
    """(MaterialSpec, tag, note) of the cfg 4 / cfg 5 soil."""
    if material == "cam_clay":
        return (MaterialSpec("cam_clay", ElasticParams(E, nu), **CAM_CLAY), "mcc",
                "modified Cam-Clay (extension, parity unpinned); strip traction footing")
    if material == "drucker_prager":
        return (MaterialSpec("drucker_prager", ElasticParams(E, nu), **DRUCKER_PRAGER), "dp",
                "Drucker-Prager (north_star target material; extension, parity unpinned); strip traction footing")
    tag = "nh" if material == "neo_hookean" else material
    return (MaterialSpec(material, ElasticParams(E, nu)), tag,
            "neo-Hookean substitute for modified Cam-Clay (pinned in 3D); strip traction footing")


def footing3d(cells=(128, 128, 64), ppc=2, h=0.5, steps=20, t_hat=100e3, frac=0.125, E=10e6, nu=0.3,
              material="neo_hookean"):
    """cfg 4 / cfg 5 slab: 3D strip footing, 128x128x64 cells, ppc 2 (8,388,608
    particles). Modified Cam-Clay is absent from the reference: the pinned
    substitute is neo-Hookean; material="cam_clay" runs the
    (unpinned) modified Cam-Clay extension. The rigid footing is a strip
    traction on the top layer (the reference has no contact)."""
    D = 3
    grid = GridSpec(3, (-h, -h, -h), h, tuple(c + 3 for c in cells))
    ext = tuple(c * h for c in cells)
    parts = seed_box(grid, (0.0, 0.0, 0.0), ext, ppc, 2000.0)
    n_strip = _strip_traction(parts, D, ext, frac, t_hat, axes=[0])
    mat, tag, note = _footing_material(material, E, nu)
    name = f"cfg4_footing3d_{tag}"
    return Problem(name, grid, parts, mat, SolverOptions(tol=1e-10), _column_fixed(grid, ext),
                   np.array([0.0, 0.0, -9.81]), steps, note=note, meta={"strip_particles": n_strip})


def footing3d_slab(nranks, rank, cells=(128, 128, 64), ppc=2, h=0.5, steps=20, t_hat=100e3, frac=0.125, E=10e6,
                   nu=0.3, density=2000.0, material="neo_hookean"):
    """cfg 5 (weak scaling): cfg 4 per GPU stacked along axis 0, i.e. the
    footing3d problem on (cells[0] * nranks) x cells[1] x cells[2] cells, of
    which only rank `rank`'s slab (owned + ghost particles) is generated. The
    strip-traction magnitude uses the GLOBAL strip particle count (computed
    from the lattice), so nranks = 1 reproduces footing3d() exactly. Returns a
    Problem whose meta holds the global ids, cuts and global grid."""
    from .distributed import keep_mask, slab_cuts_from_weights, seed_box_slab

    D = 3
    gcells = (cells[0] * nranks, cells[1], cells[2])
    grid = GridSpec(3, (-h, -h, -h), h, tuple(c + 3 for c in gcells))
    ext = tuple(c * h for c in gcells)
    spacing = h / ppc
    sub = [c * ppc for c in gcells]
    x0 = 0.0 + (np.arange(sub[0], dtype=np.float64) + 0.5) * spacing
    lp = np.full(sub[0], 0.5 * spacing)
    first = np.floor((x0 - grid.origin[0] - (grid.h + lp)) / grid.h).astype(np.int64) + 1
    n0 = int(grid.nodes[0])
    w = np.bincount(np.clip(first, 0, n0 - 1), minlength=n0).astype(float) * (sub[1] * sub[2])
    cuts = slab_cuts_from_weights(n0, nranks, w)
    parts, ids = seed_box_slab(grid, (0.0, 0.0, 0.0), ext, ppc, density, cuts, rank)
    # strip traction on the top layer under the centred strip (as _strip_traction)
    lo, hi = 0.5 * ext[0] * (1 - frac), 0.5 * ext[0] * (1 + frac)
    n_strip = int(((x0 >= lo) & (x0 <= hi)).sum()) * sub[1]
    area = ext[0] * frac * ext[1]
    pa = ParticleArray(parts, D)
    top = 0.0 + (sub[2] - 1 + 0.5) * spacing
    sel = (pa.X[:, 2] >= top - 1e-9) & (pa.X[:, 0] >= lo) & (pa.X[:, 0] <= hi)
    pa.traction_force[sel, 2] = -t_hat * area / max(n_strip, 1)
    mat, tag, note = _footing_material(material, E, nu)
    return Problem(f"cfg5_footing3d_{tag}_slab{rank}of{nranks}", grid, parts, mat, SolverOptions(tol=1e-10),
                   _column_fixed(grid, ext), np.array([0.0, 0.0, -9.81]), steps,
                   note="cfg4 per GPU stacked along axis 0; " + note,
                   meta={"ids": ids, "cuts": cuts, "strip_particles": n_strip, "rank": rank, "nranks": nranks,
                         "global_particles": int(np.prod(sub))})


def terzaghi2d(cells=(512, 512), ppc=2, height=10.0, t_hat=1e3, tol=1e-10):
    """cfg 3: 2D Terzaghi consolidation with coupled u-p (CoupledSim, 3x3 BSR
    blocks), 512x512 cells, ppc 2 (1,048,576 particles). The reference's
    consolidation scenario (configs/consolidation.cfg, src/scenarios.cpp:387-418:
    lambda = mu = 600 kPa, k = 1e-12 m^2, mu_f = 0.1 Pa s, drained top, base
    fixed, lateral rollers, 1 kPa surface traction) widened from one column to
    a square block. Returns a ready CoupledSim and its parameters."""
    return terzaghi(cells, ppc, height, t_hat, tol)


def terzaghi3d(cells=(8, 8, 64), ppc=2, height=10.0, t_hat=1e3, tol=1e-10):
    """cfg 3, 3D variant (4x4 u-p node blocks; extension, parity unpinned):
    the same column with rollers on all four lateral faces."""
    return terzaghi(cells, ppc, height, t_hat, tol)


def terzaghi(cells, ppc=2, height=10.0, t_hat=1e3, tol=1e-10):
    from .sim import CoupledSim, PoroParams

    D = len(cells)
    h = height / cells[-1]
    grid = GridSpec(D, (-h,) * D, h, tuple(c + 3 for c in cells))
    ext = tuple(c * h for c in cells[:-1]) + (height,)
    parts = seed_box(grid, (0.0,) * D, ext, ppc, 2000.0)
    pa = ParticleArray(parts, D)
    top = pa.X[:, D - 1] >= pa.X[:, D - 1].max() - 1e-9
    area = float(np.prod(ext[:-1]))
    pa.traction_force[top, D - 1] = -t_hat * area / top.sum()
    pp = PoroParams(600e3, 600e3, 1e-12, 0.1, 1000.0)
    sim = CoupledSim(grid, parts, pp, SolverOptions(tol=tol))
    for a in range(D - 1):
        w = ext[a]
        sim.fix_displacement(lambda x, a=a, w=w: (x[:, a] <= 1e-12) | (x[:, a] >= w - 1e-9), a)
    sim.fix_displacement(lambda x: x[:, D - 1] <= 1e-12)
    sim.fix_pressure(lambda x: x[:, D - 1] >= height - 1e-9)
    sim.initialize()
    return sim, {"height": height, "t_hat": t_hat, "c_v": 1e-12 * (600e3 + 2 * 600e3) / 0.1, "h": h,
                 "particles": parts.shape[0]}


def by_name(name, **kw):
    table = {"cfg1": column2d_nh, "cfg2": slope2d, "cfg4": footing3d, "cfg5": footing3d}
    return table[name](**kw)
