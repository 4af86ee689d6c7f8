"""paper_2507_09435_b200 — B200-native implicit MPM Newton step (GeoWarp,
arXiv 2507.09435), drop-in for the reference `impm` solver surface.

Python mirror of the reference's `impm` module
(/root/reference/proj/bindings/py_module.cpp:68-198) for the hot path:
MpmSim (mpm_solver.hpp), seed_box (particle.hpp), gimp_weight_1d /
block_size (gimp.hpp), the exception classes (errors.hpp). All simulation
work runs in libimpm_gpu.so (CUDA, sm_100a) through the C ABI in
include/impm_gpu.h.
"""
from .errors import (ConfigError, CudaError, DomainError, Error, LinearSolverError, NonConvergenceError,
                     OutOfDomainError, SeedingFault, UnsupportedOperation)
from .particles import GridSpec, ParticleArray, particle_doubles, particle_fields, seed_box
from .sparse import CsrMatrix, sparse_lu_solve
from .sim import CoupledSim, DofMap, ElasticParams, MaterialSpec, MpmSim, PoroParams, SolverOptions, StepRecord

__all__ = [
    "ConfigError", "CudaError", "DomainError", "Error", "LinearSolverError", "NonConvergenceError",
    "OutOfDomainError", "SeedingFault", "UnsupportedOperation", "GridSpec", "ParticleArray", "particle_doubles",
    "particle_fields", "seed_box", "DofMap", "ElasticParams", "MaterialSpec", "MpmSim", "SolverOptions",
    "StepRecord", "gimp_weight_1d", "block_size", "CoupledSim", "PoroParams", "Config", "run_scenario",
    "run_scenario_text", "bench_scenario", "CsrMatrix", "sparse_lu_solve",
]


def gimp_weight_1d(xi, lp, h):
    """(w, dw) of the 1D cpGIMP weight (src/gimp.cpp:27-44); host-side utility."""
    if not (lp > 0.0) or lp >= 0.5 * h:
        raise ConfigError(f"GIMP requires 0 < lp < h/2 (lp = {lp:f}, h = {h:f})")
    ax = abs(xi)
    sgn = 1.0 if xi >= 0.0 else -1.0
    if ax < lp:
        return 1.0 - (xi * xi + lp * lp) / (2.0 * h * lp), -xi / (h * lp)
    if ax < h - lp:
        return 1.0 - ax / h, -sgn / h
    if ax < h + lp:
        t = h + lp - ax
        return t * t / (4.0 * h * lp), -sgn * t / (2.0 * h * lp)
    return 0.0, 0.0


_BLOCK = {"linear": 3, "gimp": 5, "quadratic-bspline": 5, "cubic-bspline": 7}


def block_size(kind):
    """Seeding block size per axis (src/gimp.cpp:7-15)."""
    if kind not in _BLOCK:
        raise ConfigError("unknown shape function kind: " + kind)
    return _BLOCK[kind]


from .config import Config  # noqa: E402
from .scenarios import bench_scenario, run_scenario, run_scenario_text  # noqa: E402
