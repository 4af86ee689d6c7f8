"""Inverse stiffness identification on the GPU path (drop-in for
impm::InverseProblem, /root/reference/proj/include/impm/inverse.hpp:45-80,
src/inverse.cpp:14-195).

Forward model: total-Lagrangian strip-loaded column, one warm-started GPU
Newton solve per load level (inverse.cpp:40-87). Gradient: per-level
implicit-function adjoint (inverse.cpp:147-173). J^T lambda = dL/du is solved
on the device (J is symmetric for Hencky, so J^T = J), and dr/d(ln E) is the
internal force f_int(u) = r(u, load_scale=0): Hencky stress is linear in E.
That replaces the reference's extra tape input plus one seeded backward pass.
"""
import math
import os

import numpy as np

from . import gimp_weight_1d
from .errors import ConfigError, NonConvergenceError
from .particles import GridSpec, ParticleArray, seed_box
from .sim import ElasticParams, MaterialSpec, MpmSim, SolverOptions


class InverseOptions:  # inverse.hpp:18-33
    def __init__(self, **kw):
        self.E_true, self.nu, self.width, self.height, self.h, self.ppc = 1.0e6, 0.2, 4.0, 4.0, 0.5, 2
        self.strip_fraction, self.t_hat, self.levels = 0.5, 40.0e3, 10
        self.lr, self.loss_threshold, self.max_gd_iterations = 0.2, 1.0e-10, 20
        for k, v in kw.items():
            setattr(self, k, v)


def fd_slope(x, y):  # inverse.cpp:88-108
    x, y = np.asarray(x, float), np.asarray(y, float)
    xb, yb = x.mean(), y.mean()
    return float(((x - xb) * (y - yb)).sum() / ((x - xb) ** 2).sum())


class InverseProblem:
    def __init__(self, opt: InverseOptions):
        if not opt.E_true > 0.0:
            raise ConfigError("inverse: E_true must be positive")
        if not opt.lr > 0.0:
            raise ConfigError("inverse: learning rate must be positive")
        self.opt = opt
        self.reference = None
        self.sim = None

    def _build(self, E):  # inverse.cpp:14-38
        o = self.opt
        h = o.h
        grid = GridSpec(2, (-h, -h), h, (int(round(o.width / h)) + 3, int(round(o.height / h)) + 3))
        parts = seed_box(grid, (0.0, 0.0), (o.width, o.height), o.ppc, 1000.0)
        sim = MpmSim(grid, parts, MaterialSpec("hencky", ElasticParams(E, o.nu)),
                     SolverOptions(tol=1e-11, max_iterations=30, total_lagrangian=True))
        sim.fix_nodes(lambda x: x[:, 1] <= 1e-12)
        w = o.width
        sim.fix_nodes(lambda x: (x[:, 0] <= 1e-12) | (x[:, 0] >= w - 1e-12), 0)
        return sim, parts

    def _gauge(self, sim, parts, strip):
        """add_interpolation_weights(pi, 1, 1/n) over the strip (mpm_solver.hpp:427-434)."""
        g = sim.grid
        dofs = sim.dofs()
        out = np.zeros(dofs.n_dofs)
        pa = ParticleArray(parts, 2)
        for pi in strip:
            axes = []
            for a in range(2):
                x, lp = pa.x[pi, a], pa.lp[pi, a]
                lo = (x - g.origin[a] - (g.h + lp)) / g.h
                hi = (x - g.origin[a] + (g.h + lp)) / g.h
                first = int(math.floor(lo)) + 1
                last = int(math.ceil(hi)) - 1
                axes.append([(i, gimp_weight_1d(x - (g.origin[a] + i * g.h), lp, g.h)[0])
                             for i in range(first, last + 1)])
            for i, wi in axes[0]:
                for j, wj in axes[1]:
                    d = dofs.dof(i * g.nodes[1] + j, 1)
                    if d >= 0:
                        out[d] += (1.0 / len(strip)) * (wi * wj)
        return out

    def simulate(self, log_E):  # inverse.cpp:40-87
        o = self.opt
        sim, parts = self._build(math.exp(log_E))
        pa = ParticleArray(parts, 2)
        top = pa.X[:, 1].max()
        x_lo, x_hi = 0.5 * o.width * (1 - o.strip_fraction), 0.5 * o.width * (1 + o.strip_fraction)
        strip = np.nonzero((pa.X[:, 1] >= top - 1e-9) & (pa.X[:, 0] >= x_lo) & (pa.X[:, 0] <= x_hi))[0]
        if len(strip) == 0:
            raise ConfigError("inverse: empty strip-load particle set")
        strip_width = o.width * o.strip_fraction
        pa.traction_force[strip, 1] = -o.t_hat * (strip_width / len(strip))
        sim.set_particles(parts)
        sim.begin_step()
        self.gauge = self._gauge(sim, parts, strip)
        disp, force, self.u_levels, self.s_levels = [], [], [], []
        for level in range(1, o.levels + 1):
            s = level / o.levels
            sim.newton_solve(s)
            u = sim.nodal_solution()
            self.u_levels.append(u)
            self.s_levels.append(s)
            disp.append(-float(self.gauge @ u))
            force.append(o.t_hat * s * strip_width)
        sim.commit_step()
        self.sim = sim
        return {"displacement": disp, "force": force}

    def generate_reference(self):
        self.reference = self.simulate(math.log(self.opt.E_true))

    def loss(self, run):  # inverse.cpp:110-121
        s, s_ref = fd_slope(run["displacement"], run["force"]), fd_slope(self.reference["displacement"],
                                                                        self.reference["force"])
        if not (s > 0.0 and s_ref > 0.0):
            raise NonConvergenceError("inverse: non-positive force-displacement slope", [])
        return math.log(s / s_ref) ** 2

    def _dL_ddelta(self, run):  # inverse.cpp:123-145
        d, f = np.asarray(run["displacement"]), np.asarray(run["force"])
        s_ref = fd_slope(self.reference["displacement"], self.reference["force"])
        s = fd_slope(d, f)
        D, G = d - d.mean(), f - f.mean()
        sxx = (D ** 2).sum()
        pref = 2.0 * math.log(s / s_ref) / s
        return pref * (G - 2.0 * s * D) / sxx

    def gradient(self, log_E, run):  # inverse.cpp:147-173
        sim = self.sim
        if sim is None:
            raise ConfigError("inverse: no retained forward run")
        g = self._dL_ddelta(run)
        dL = 0.0
        for lvl, (u, s) in enumerate(zip(self.u_levels, self.s_levels)):
            rhs = -g[lvl] * self.gauge
            lam, _ = sim.linear_solve(u, s, rhs)   # J^T lambda = dL/du (J symmetric)
            dr_dtheta = sim.residual(u, 0.0)       # d r / d ln E = f_int(u)
            dL -= float(lam @ dr_dtheta)
        return dL

    def gradient_descent(self, E0):  # inverse.cpp:175-195
        if self.reference is None:
            self.generate_reference()
        theta = math.log(E0)
        traj, initial = [], -1.0
        for it in range(self.opt.max_gd_iterations):
            run = self.simulate(theta)
            L = self.loss(run)
            if it == 0:
                initial = max(L, 1e-300)
            if L > 1e6 * initial:
                raise NonConvergenceError("inverse gradient descent diverged; reduce the learning rate", [])
            gr = self.gradient(theta, run)
            traj.append((it, math.exp(theta), L, gr))
            if L <= self.opt.loss_threshold:
                break
            theta -= self.opt.lr * gr
        return traj


def run_inverse(cfg, with_checks, rep):  # scenarios.cpp:545-607
    from .scenarios import _Csv, _out_dir

    d = _out_dir(cfg, "inverse")
    o = InverseOptions()
    o.E_true = cfg.get_double("material", "E_true", o.E_true)
    o.nu = cfg.get_double("material", "nu", o.nu)
    o.width = cfg.get_double("geometry", "width", o.width)
    o.height = cfg.get_double("geometry", "height", o.height)
    o.h = cfg.get_double("geometry", "h", o.h)
    o.ppc = cfg.get_int("geometry", "particles_per_cell", o.ppc)
    o.strip_fraction = cfg.get_double("schedule", "strip_fraction", o.strip_fraction)
    o.t_hat = cfg.get_double("schedule", "t_hat", o.t_hat)
    o.levels = cfg.get_int("schedule", "levels", o.levels)
    o.lr = cfg.get_double("optimizer", "learning_rate", o.lr)
    o.loss_threshold = cfg.get_double("optimizer", "loss_threshold", o.loss_threshold)
    o.max_gd_iterations = cfg.get_int("optimizer", "max_iterations", o.max_gd_iterations)
    prob = InverseProblem(o)
    if cfg.has("reference", "csv"):
        path = cfg.get_string("reference", "csv")
        if not os.path.exists(path):
            raise ConfigError("cannot open reference csv")
        a = np.loadtxt(path, delimiter=",", skiprows=1, ndmin=2)
        prob.reference = {"displacement": a[:, 0].tolist(), "force": a[:, 1].tolist()}
    else:
        prob.generate_reference()
        c = _Csv(d + "/reference.csv", "displacement,force", rep)
        for dd, ff in zip(prob.reference["displacement"], prob.reference["force"]):
            c.row(dd, ff)
        c.close()
    traj = prob.gradient_descent(cfg.get_double("optimizer", "E0", 0.1 * o.E_true))
    rep.steps = len(traj)
    c = _Csv(d + "/optimization.csv", "iteration,theta,E,loss,gradient", rep)
    for it, E, L, gr in traj:
        c.row(str(it), math.log(E), E, L, gr)
    c.close()
    if not with_checks:
        return
    rep.check_near("inverse.recovered_E", traj[-1][1], o.E_true, 0.01)
    rep.check_le("inverse.gd_iterations", float(len(traj)), 20.0)
    for probe in range(min(2, len(traj))):
        theta = math.log(traj[probe][1])
        run = prob.simulate(theta)
        g_adj = prob.gradient(theta, run)
        hh = 1e-5
        Lp = prob.loss(prob.simulate(theta + hh))
        Lm = prob.loss(prob.simulate(theta - hh))
        rep.check_near(f"inverse.adjoint_vs_fd_iter{probe}", g_adj, (Lp - Lm) / (2 * hh), 1e-4)
