"""Host mirror of impm::MpmSim<D> over the C ABI (include/impm_gpu.h).

Same members and method names as the reference class
(/root/reference/proj/include/impm/mpm_solver.hpp:51-478); every method is a
thin call into libimpm_gpu.so, which runs the step on the GPU. There is no
CPU path: a missing library raises ExtensionMissing.
"""
import ctypes
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _abi
from .errors import raise_for
from .particles import GridSpec, ParticleArray, particle_doubles

MATERIAL_KINDS = {"hencky": 0, "hencky_j2": 1, "neo_hookean": 2, "drucker_prager": 3, "cam_clay": 4}
SHAPES = {"gimp": 1, "quadratic-bspline": 2, "quadratic_bspline": 2}
KRYLOV = {"auto": 0, "cg": 1, "bicgstab": 2, "gmres": 3, "iterative": 4}
PRECOND = {"mg": 0, "multigrid": 0, "block_jacobi": 1, "jacobi": 1}
STRATEGIES = {"sparse": 0, "dense": 1}
INTERFERENCE = {"off": 0, "sampled": 1, "always": 2}


@dataclass
class ElasticParams:
    """materials.hpp:12-23"""
    E: float
    nu: float

    def lam(self):
        return self.E * self.nu / ((1.0 + self.nu) * (1.0 - 2.0 * self.nu))

    def mu(self):
        return self.E / (2.0 * (1.0 + self.nu))


@dataclass
class MaterialSpec:
    """mpm_solver.hpp:21-25"""
    kind: str = "hencky"
    elastic: ElasticParams = field(default_factory=lambda: ElasticParams(1.0, 0.0))
    kappa: float = 0.0
    friction_deg: float = 30.0  # Drucker-Prager friction / Cam-Clay critical-state angle (extensions)
    cohesion: float = 0.0  # Drucker-Prager cohesion / Cam-Clay tensile intercept p_t
    pc0: float = 0.0  # Cam-Clay initial preconsolidation pressure
    hardening: float = 0.0  # Cam-Clay theta = (1 + e0) / (lambda - kappa)


@dataclass
class SolverOptions:
    """mpm_solver.hpp:27-36 + the GPU linear-solver knobs"""
    tol: float = 1e-11
    abs_floor: float = 1e-14
    max_iterations: int = 20
    total_lagrangian: bool = False
    shape: str = "gimp"
    krylov: str = "auto"
    krylov_rtol: float = 1e-12
    krylov_max_iter: int = 0
    profile: bool = False
    precond: str = "mg"
    mg_smooth: int = 1
    strategy: str = "sparse"  # JacobianStrategy (jacobian.hpp:18)
    interference: str = "off"  # InterferenceCheck (jacobian.hpp:20)

    def to_c(self):
        return _abi.Options(self.tol, self.abs_floor, int(self.max_iterations), int(bool(self.total_lagrangian)),
                            SHAPES[self.shape], KRYLOV[self.krylov], self.krylov_rtol, int(self.krylov_max_iter),
                            int(bool(self.profile)), PRECOND[self.precond], int(self.mg_smooth),
                            STRATEGIES[self.strategy], INTERFERENCE[self.interference])


@dataclass
class StepRecord:
    """mpm_solver.hpp:38-46 + GPU counters"""
    step: int = 0
    iterations: int = 0
    rel_residuals: List[float] = field(default_factory=list)
    r0_norm: float = 0.0
    seconds: float = 0.0
    diff_seconds: float = 0.0
    backward_passes: int = 0
    krylov_iterations: int = 0
    solve_seconds: float = 0.0
    residual_seconds: float = 0.0
    nnz_assembled: int = 0


@dataclass
class DofMap:
    """grid.hpp:66-93"""
    n_fields: int
    n_dofs: int
    dof_of: np.ndarray
    node_of: np.ndarray
    field_of: np.ndarray

    def dof(self, node, fld):
        return int(self.dof_of[node * self.n_fields + fld])


class _Handle:
    """Owns one impm_sim* and turns statuses into impm exceptions."""

    def __init__(self, grid: GridSpec, material: MaterialSpec, options: SolverOptions, device=0):
        L = _abi.lib()
        self._L = L
        g = _abi.Grid()
        g.dim = grid.dim
        for a in range(3):
            g.nodes[a] = int(grid.nodes[a]) if a < grid.dim else 1
            g.origin[a] = float(grid.origin[a]) if a < grid.dim else 0.0
        g.h = float(grid.h)
        m = _abi.Material(MATERIAL_KINDS[material.kind], 0, material.elastic.E, material.elastic.nu, material.kappa,
                          material.friction_deg, material.cohesion, material.pc0, material.hardening)
        o = options.to_c()
        h = ctypes.c_void_p()
        st = L.impm_sim_create(ctypes.byref(g), ctypes.byref(m), ctypes.byref(o), device, ctypes.byref(h))
        if st != _abi.OK:
            raise_for(st, L.impm_create_error().decode())
        self.h = h

    def call(self, name, *args):
        st = getattr(self._L, name)(self.h, *args)
        if st != _abi.OK:
            buf = ctypes.create_string_buffer(4096)
            n = ctypes.c_int32(256)
            hist = np.zeros(256)
            self._L.impm_sim_last_error(self.h, buf, 4096, _abi.ptr(hist), ctypes.byref(n))
            raise_for(st, buf.value.decode(), hist[: min(n.value, 256)].tolist())

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self._L.impm_sim_destroy(self.h)
                self.h = None
        except Exception:
            pass


class MpmSim:
    """Implicit quasi-static MPM over a structured grid with cpGIMP transfers
    (mpm_solver.hpp:48-52), stepped on the GPU."""

    def __init__(self, grid: GridSpec, particles, material: MaterialSpec, options: Optional[SolverOptions] = None,
                 device: int = 0):
        self.grid = grid
        self.D = grid.dim
        self.material = material
        self.options = options or SolverOptions()
        self._h = _Handle(grid, material, self.options, device)
        self._N = grid.node_count()
        self.fixed = np.zeros(self._N * self.D, dtype=np.uint8)  # [node*D + comp]
        self._fixed_sent = None
        self._gravity = np.zeros(self.D)
        self.set_particles(particles)
        self._push_gravity()

    # ------------------------------------------------------------ members
    @property
    def particles(self) -> ParticleArray:
        """Downloads the particle state (reference AoS layout, original order)."""
        P = self.n_particles
        out = np.zeros((P, particle_doubles(self.D)), dtype=np.float64)
        self._h.call("impm_sim_get_particles", _abi.ptr(out), P, out.strides[0])
        return ParticleArray(out, self.D)

    @particles.setter
    def particles(self, value):
        self.set_particles(value)

    def set_particles(self, particles):
        data = particles.data if isinstance(particles, ParticleArray) else np.asarray(particles, dtype=np.float64)
        data = np.ascontiguousarray(data, dtype=np.float64)
        if data.ndim != 2 or data.shape[1] != particle_doubles(self.D):
            raise ValueError(f"particles must be (P, {particle_doubles(self.D)}) float64")
        self._h.call("impm_sim_set_particles", _abi.ptr(data), data.shape[0], data.strides[0])
        self._n_particles = data.shape[0]

    def set_particle_field(self, name, values):
        """Overwrites one scalar column (e.g. 'traction_force', component c) by original index."""
        raise NotImplementedError

    @property
    def n_particles(self):
        return self._n_particles

    @property
    def gravity(self):
        return self._gravity.copy()

    @gravity.setter
    def gravity(self, g):
        self._gravity = np.asarray(g, dtype=np.float64).reshape(self.D).copy()
        self._push_gravity()

    def _push_gravity(self):
        g3 = np.zeros(3)
        g3[: self.D] = self._gravity
        self._h.call("impm_sim_set_gravity", _abi.ptr(g3))

    def set_options(self, options: SolverOptions):
        self.options = options
        o = options.to_c()
        self._h.call("impm_sim_set_options", ctypes.byref(o))

    def fix_nodes(self, predicate, component=-1):
        """mpm_solver.hpp:70-78; predicate gets an (N, D) array of node positions
        and returns a boolean mask (or is applied per node if it is not vectorised)."""
        pos = self.grid.node_positions()
        try:
            mask = np.asarray(predicate(pos), dtype=bool).reshape(-1)
            if mask.shape[0] != pos.shape[0]:
                raise ValueError
        except Exception:
            mask = np.array([bool(predicate(p)) for p in pos])
        for c in range(self.D):
            if component < 0 or component == c:
                self.fixed[np.nonzero(mask)[0] * self.D + c] = 1

    def _sync_fixed(self):
        if self._fixed_sent is None or not np.array_equal(self._fixed_sent, self.fixed):
            f = np.ascontiguousarray(self.fixed, dtype=np.uint8)
            self._h.call("impm_sim_set_fixed", _abi.ptr(f))
            self._fixed_sent = f.copy()

    # ------------------------------------------------------------ stages
    def begin_step(self):
        self._sync_fixed()
        self._h.call("impm_sim_begin_step")

    def n_dofs(self):
        n = ctypes.c_int32()
        self._h.call("impm_sim_n_dofs", ctypes.byref(n))
        return n.value

    def dofs(self) -> DofMap:
        n = self.n_dofs()
        dof_of = np.zeros(self._N * self.D, dtype=np.int32)
        node_of = np.zeros(max(n, 1), dtype=np.int32)
        field_of = np.zeros(max(n, 1), dtype=np.int32)
        self._h.call("impm_sim_dof_map", _abi.ptr(dof_of), _abi.ptr(node_of), _abi.ptr(field_of))
        return DofMap(self.D, n, dof_of, node_of[:n], field_of[:n])

    def colour_groups(self):
        n = self.n_dofs()
        out = np.zeros(max(n, 1), dtype=np.int32)
        ng = ctypes.c_int32()
        self._h.call("impm_sim_colour_groups", _abi.ptr(out), ctypes.byref(ng))
        return out[:n], ng.value

    def support_stats(self):
        """Support-size statistics of the current step (impm_sim_support_stats)."""
        out = np.zeros(34, dtype=np.int64)
        self._h.call("impm_sim_support_stats", _abi.ptr(out))
        P = max(int(out[0]), 1)
        return {"particles": int(out[0]), "mean_s": out[1] / P, "mean_s2": out[2] / P,
                "mean_bin_box": out[3] / P, "mean_bin_box2": out[4] / P, "bins": int(out[5]),
                "s_hist": {int(k): int(out[6 + k]) for k in range(1, 28) if out[6 + k]}}

    def node_mass(self):
        out = np.zeros(self._N)
        self._h.call("impm_sim_node_mass", _abi.ptr(out))
        return out

    def total_node_mass(self):
        return float(np.sum(self.node_mass()))

    def p2g_map(self, per_particle):
        f = _abi.f64(per_particle)
        out = np.zeros(self._N)
        self._h.call("impm_sim_p2g_map", _abi.ptr(f), _abi.ptr(out))
        return out

    def residual(self, u, load_scale):
        u = _abi.f64(u)
        r = np.zeros(max(self.n_dofs(), 1))
        self._h.call("impm_sim_residual", _abi.ptr(u), float(load_scale), _abi.ptr(r))
        return r[: self.n_dofs()]

    def jacobian_csr(self, u, load_scale=1.0):
        """J(u) in the reference's CSR pattern: (row_ptr int64, cols int32, vals f64)."""
        u = _abi.f64(u)
        n = self.n_dofs()
        nnz = ctypes.c_int64()
        self._h.call("impm_sim_jacobian_csr", None, float(load_scale), ctypes.byref(nnz), None, None, None)
        rp = np.zeros(n + 1, dtype=np.int64)
        cols = np.zeros(max(nnz.value, 1), dtype=np.int32)
        vals = np.zeros(max(nnz.value, 1))
        self._h.call("impm_sim_jacobian_csr", _abi.ptr(u), float(load_scale), ctypes.byref(nnz), _abi.ptr(rp),
                     _abi.ptr(cols), _abi.ptr(vals))
        return rp, cols[: nnz.value], vals[: nnz.value]

    def linear_solve(self, u, load_scale, rhs):
        u, rhs = _abi.f64(u), _abi.f64(rhs)
        out = np.zeros(max(self.n_dofs(), 1))
        it = ctypes.c_int32()
        self._h.call("impm_sim_linear_solve", _abi.ptr(u), float(load_scale), _abi.ptr(rhs), _abi.ptr(out),
                     ctypes.byref(it))
        return out[: self.n_dofs()], it.value

    def apply_jacobian(self, u, load_scale, x_grid):
        """y = J(u) x for a grid-layout vector x [N * D] (u = free-DOF vector);
        on a slab the owned rows are valid and halo columns come from the
        neighbours."""
        u = _abi.f64(u)
        x = np.ascontiguousarray(x_grid, dtype=np.float64).reshape(-1)
        if x.size != self._N * self.D:
            raise ValueError("x must be a grid vector [N_local * D]")
        y = np.zeros_like(x)
        self._h.call("impm_sim_apply_jacobian", _abi.ptr(u), float(load_scale), _abi.ptr(x), _abi.ptr(y))
        return y

    def _record(self):
        buf = np.zeros(256)
        rec = _abi.StepRecordC()
        rec.rel_residuals = buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        rec.rel_capacity = 256
        return rec, buf

    @staticmethod
    def _to_record(rec, buf):
        return StepRecord(rec.step, rec.iterations, buf[: rec.n_rel].tolist(), rec.r0_norm, rec.seconds,
                          rec.diff_seconds, rec.backward_passes, rec.krylov_iterations, rec.solve_seconds,
                          rec.residual_seconds, rec.nnz_assembled)

    def newton_solve(self, load_scale) -> StepRecord:
        rec, buf = self._record()
        self._h.call("impm_sim_newton_solve", float(load_scale), ctypes.byref(rec))
        return self._to_record(rec, buf)

    def commit_step(self):
        self._h.call("impm_sim_commit_step")

    def step(self, load_scale) -> StepRecord:
        self._sync_fixed()
        rec, buf = self._record()
        self._h.call("impm_sim_step", float(load_scale), ctypes.byref(rec))
        return self._to_record(rec, buf)

    def nodal_solution(self):
        out = np.zeros(max(self.n_dofs(), 1))
        self._h.call("impm_sim_nodal_solution", _abi.ptr(out))
        return out[: self.n_dofs()]

    def set_nodal_solution(self, u):
        u = _abi.f64(u)
        self._h.call("impm_sim_set_nodal_solution", _abi.ptr(u))

    def kernel_times(self, reset=False):
        names = (ctypes.c_char_p * 32)()
        ms = np.zeros(32)
        launches = np.zeros(32, dtype=np.int64)
        n = ctypes.c_int32()
        self._h.call("impm_sim_kernel_times", names, _abi.ptr(ms), _abi.ptr(launches), ctypes.byref(n), int(reset))
        return {names[i].decode(): (float(ms[i]), int(launches[i])) for i in range(n.value)}

    def matrix_info(self):
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        self._h.call("impm_sim_matrix_info", ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
        return {"rows": a.value, "row_values": b.value, "ref_nnz": c.value}

    def set_stream(self, stream_ptr):
        self._h.call("impm_sim_set_stream", ctypes.c_void_p(stream_ptr))


@dataclass
class PoroParams:
    """impm::PoroParams (porous.hpp:22-38)."""
    lambda_: float
    mu: float
    k: float
    mu_f: float
    rho_f: float = 1000.0

    def mobility(self):
        return self.k / self.mu_f

    def consolidation_coefficient(self):
        return self.k * (self.lambda_ + 2.0 * self.mu) / self.mu_f


class CoupledSim:
    """impm::CoupledSim (porous.hpp:48-125): small-strain u-p on reference-
    configuration weights, fields (u_0 .. u_{D-1}, p) per node, stepped on the
    GPU. D = 2 is the reference; D = 3 (4x4 node blocks) is an extension
    (parity unpinned)."""

    def __init__(self, grid: GridSpec, particles, poro: PoroParams, options: Optional[SolverOptions] = None,
                 device: int = 0):
        if grid.dim not in (2, 3):
            from .errors import ConfigError
            raise ConfigError("coupled u-p requires a 2D or 3D grid")
        self.grid = grid
        self.D = D = grid.dim
        self.F = D + 1
        self.poro = poro
        self.options = options or SolverOptions()
        L = _abi.lib()
        g = _abi.Grid()
        g.dim = D
        for a in range(3):
            g.nodes[a] = int(grid.nodes[a]) if a < D else 1
            g.origin[a] = float(grid.origin[a]) if a < D else 0.0
        g.h = float(grid.h)
        pc = _abi.Poro(poro.lambda_, poro.mu, poro.k, poro.mu_f, poro.rho_f)
        o = self.options.to_c()
        h = ctypes.c_void_p()
        st = L.impm_coupled_create(ctypes.byref(g), ctypes.byref(pc), ctypes.byref(o), device, ctypes.byref(h))
        if st != _abi.OK:
            raise_for(st, L.impm_create_error().decode())
        self._h = _Handle.__new__(_Handle)
        self._h._L = L
        self._h.h = h
        self._N = grid.node_count()
        self.fixed_u = np.zeros(self._N * D, dtype=np.uint8)  # [node*D + comp]
        self.fixed_p = np.zeros(self._N, dtype=np.uint8)
        self._gravity = np.zeros(D)
        data = np.ascontiguousarray(particles.data if isinstance(particles, ParticleArray) else particles,
                                    dtype=np.float64)
        self._h.call("impm_sim_set_particles", _abi.ptr(data), data.shape[0], data.strides[0])
        self._n_particles = data.shape[0]
        self._X1 = data[:, D - 1].copy()  # reference vertical coordinate (Particle<D>::X[D-1])
        self._initialized = False
        self.gravity = np.zeros(D)

    @property
    def gravity(self):
        return self._gravity.copy()

    @gravity.setter
    def gravity(self, gv):
        self._gravity = np.asarray(gv, dtype=np.float64).reshape(self.D).copy()
        g3 = np.zeros(3)
        g3[: self.D] = self._gravity
        self._h.call("impm_sim_set_gravity", _abi.ptr(g3))

    @property
    def particles(self) -> ParticleArray:
        out = np.zeros((self._n_particles, particle_doubles(self.D)))
        self._h.call("impm_sim_get_particles", _abi.ptr(out), self._n_particles, out.strides[0])
        return ParticleArray(out, self.D)

    def fix_displacement(self, predicate, component=-1):
        pos = self.grid.node_positions()
        mask = np.asarray(predicate(pos), dtype=bool).reshape(-1)
        for c in range(self.D):
            if component < 0 or component == c:
                self.fixed_u[np.nonzero(mask)[0] * self.D + c] = 1

    def fix_pressure(self, predicate):
        pos = self.grid.node_positions()
        mask = np.asarray(predicate(pos), dtype=bool).reshape(-1)
        self.fixed_p[mask] = 1

    def initialize(self):
        """src/porous.cpp:25-72"""
        D, F = self.D, self.F
        fixed3 = np.zeros(self._N * F, dtype=np.uint8)
        for c in range(D):
            fixed3[c::F] = self.fixed_u[c::D]
        fixed3[D::F] = self.fixed_p
        self._h.call("impm_sim_set_fixed", _abi.ptr(fixed3))
        self._h.call("impm_coupled_initialize")
        self._initialized = True

    def n_dofs(self):
        n = ctypes.c_int32()
        self._h.call("impm_sim_n_dofs", ctypes.byref(n))
        return n.value

    def dofs(self) -> DofMap:
        n = self.n_dofs()
        dof_of = np.zeros(self._N * self.F, dtype=np.int32)
        node_of = np.zeros(max(n, 1), dtype=np.int32)
        field_of = np.zeros(max(n, 1), dtype=np.int32)
        self._h.call("impm_sim_dof_map", _abi.ptr(dof_of), _abi.ptr(node_of), _abi.ptr(field_of))
        return DofMap(self.F, n, dof_of, node_of[:n], field_of[:n])

    def residual(self, x, dt):
        x = _abi.f64(x)
        r = np.zeros(max(self.n_dofs(), 1))
        self._h.call("impm_sim_residual", _abi.ptr(x), float(dt), _abi.ptr(r))
        return r[: self.n_dofs()]

    def jacobian_csr(self, x, dt):
        return MpmSim.jacobian_csr(self, x, dt)

    def step(self, dt) -> StepRecord:
        if not self._initialized:
            self.initialize()
        rec, buf = MpmSim._record(self)
        self._h.call("impm_coupled_step", float(dt), ctypes.byref(rec))
        return MpmSim._to_record(rec, buf)

    def nodal_pressure(self):
        out = np.zeros(self._N)
        self._h.call("impm_coupled_nodal_pressure", _abi.ptr(out))
        return out

    def _settlement(self):
        out = np.zeros(max(self._n_particles, 1))
        t = ctypes.c_double()
        self._h.call("impm_coupled_settlement", _abi.ptr(out), ctypes.byref(t))
        return out[: self._n_particles], t.value

    def time(self):
        return self._settlement()[1]

    def top_settlement(self):
        """mean downward displacement of the top particle row (src/porous.cpp:170-183)"""
        uty, _ = self._settlement()
        top = self._X1 >= self._X1.max() - 1e-9
        return float(-uty[top].sum() / top.sum()) if top.any() else 0.0

    def pressure_profile(self, x_index, surface_y):
        """nodal pressures on one vertical grid column by depth (src/porous.cpp:185-199);
        x_index: the column's index along axis 0 (2D) or its (i, j) pair (3D)"""
        mass = np.zeros(self._N)
        self._h.call("impm_sim_node_mass", _abi.ptr(mass))
        pm = self.particles.m[:, 0].max() if self._n_particles else 0.0
        active = mass > 1e-12 * pm
        pos = self.grid.node_positions()
        p = self.nodal_pressure()
        D = self.D
        nv = int(self.grid.nodes[D - 1])
        col = x_index if D == 2 else int(x_index[0]) * int(self.grid.nodes[1]) + int(x_index[1])
        nodes = col * nv + np.arange(nv)
        out = []
        for n in nodes:
            if not active[n]:
                continue
            y = pos[n, D - 1]
            if y < -1e-9 or y > surface_y + 1e-9:
                continue
            out.append((surface_y - y, 0.0 if self.fixed_p[n] else p[n]))
        return sorted(out)
