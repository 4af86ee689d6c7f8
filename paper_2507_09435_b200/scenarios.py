"""Scenario runners over the GPU solvers: drop-in for impm::run_scenario /
bench_scenario (/root/reference/proj/src/scenarios.cpp:755-867) and the
Python `impm.run_scenario[_text]` (bindings/py_module.cpp:181-196).

Same config files (configs/*.cfg), same key schemas, same CSV files (12
significant digits, scenarios.cpp:31-39) and an atomically published
summary.json. The simulations run on the GPU (MpmSim / CoupledSim); only the
scenario bookkeeping is host Python. Out of scope here: `triaxial` (Nor-Sand
stress-point driver, not on the MPM path) and the dense-Jacobian ablation of
`jacobian-bench`.
"""
import json
import math
import os
import time

import numpy as np

from .config import Config
from .errors import ConfigError, NonConvergenceError
from .particles import GridSpec, ParticleArray, seed_box
from .sim import CoupledSim, ElasticParams, MaterialSpec, MpmSim, PoroParams, SolverOptions

COMMON = {"scenario", "output.dir", "solver.tol", "solver.max_iterations", "solver.jacobian"}
SCHEMAS = {  # scenarios.cpp:759-798
    "bar": ({"geometry.height", "geometry.cells", "geometry.particles_per_cell", "material.model", "material.E",
             "material.nu", "material.kappa", "material.rho0", "schedule.steps", "schedule.gravity"},
            {"geometry.height", "geometry.cells", "material.model", "material.E", "material.nu", "material.rho0",
             "schedule.steps"}),
    "triaxial": ({"material.M", "material.N", "material.h", "material.lambda_tilde", "material.v_c0", "material.v0",
                  "material.p_i0", "material.K0", "material.p0", "schedule.axial_strain", "schedule.increments"},
                 {"material.M", "material.N", "material.h", "material.lambda_tilde", "material.v_c0", "material.v0",
                  "material.p_i0", "material.K0", "material.p0"}),
    "cantilever": ({"geometry.length", "geometry.depth", "geometry.h_levels", "geometry.particles_per_cell",
                    "material.E", "material.nu", "material.rho0", "schedule.load", "schedule.steps"},
                   {"geometry.length", "geometry.depth", "geometry.h_levels", "material.E", "material.nu",
                    "schedule.load", "schedule.steps"}),
    "consolidation": ({"geometry.height", "geometry.cells", "geometry.particles_per_cell", "material.lambda",
                       "material.mu", "material.k", "material.mu_f", "material.rho_f", "material.c_v",
                       "schedule.t_hat", "schedule.dt0", "schedule.dt_growth", "schedule.dt_cap",
                       "schedule.Tv_checkpoints", "schedule.Tv_end"},
                      {"geometry.height", "geometry.cells", "material.lambda", "material.mu", "material.k",
                       "material.mu_f", "schedule.t_hat", "schedule.dt0", "schedule.Tv_checkpoints",
                       "schedule.Tv_end"}),
    "inverse": ({"geometry.width", "geometry.height", "geometry.h", "geometry.particles_per_cell", "material.E_true",
                 "material.nu", "schedule.strip_fraction", "schedule.t_hat", "schedule.levels",
                 "optimizer.learning_rate", "optimizer.loss_threshold", "optimizer.max_iterations", "optimizer.E0",
                 "reference.csv"}, {"material.E_true"}),
    "jacobian-bench": ({"geometry.length", "geometry.depth", "geometry.cells_levels", "geometry.particles_per_cell",
                        "material.E", "material.nu", "material.rho0", "schedule.load", "schedule.steps"},
                       {"geometry.length", "geometry.depth", "geometry.cells_levels", "material.E", "material.nu",
                        "schedule.load"}),
    "smoke3d": ({"geometry.size", "geometry.cells", "material.E", "material.nu"}, set()),
}


class Report:
    def __init__(self, scenario):
        self.scenario, self.steps, self.wall_s = scenario, 0, 0.0
        self.checks, self.outputs = [], []

    def check_le(self, name, measured, bound):
        self.checks.append({"name": name, "measured": float(measured), "expected": float(bound), "tol": 0.0,
                            "pass": bool(measured <= bound)})

    def check_ge(self, name, measured, bound):
        self.checks.append({"name": name, "measured": float(measured), "expected": float(bound), "tol": 0.0,
                            "pass": bool(measured >= bound)})

    def check_in(self, name, measured, lo, hi):
        self.checks.append({"name": name, "measured": float(measured), "expected": 0.5 * (lo + hi),
                            "tol": 0.5 * (hi - lo), "pass": bool(lo <= measured <= hi)})

    def check_near(self, name, measured, expected, rel):
        err = abs(measured - expected) / max(abs(expected), 1e-300)
        self.checks.append({"name": name, "measured": float(measured), "expected": float(expected), "tol": rel,
                            "pass": bool(err <= rel)})

    def as_dict(self):
        return {"scenario": self.scenario, "steps": self.steps, "wall_s": self.wall_s, "outputs": self.outputs,
                "checks": self.checks, "all_pass": all(c["pass"] for c in self.checks)}


def _g12(x):
    return "%.12g" % x


class _Csv:
    def __init__(self, path, header, report):
        self.f = open(path, "w")
        self.f.write(header + "\n")
        report.outputs.append(path)

    def row(self, *vals):
        self.f.write(",".join(v if isinstance(v, str) else _g12(v) for v in vals) + "\n")

    def close(self):
        self.f.close()


def _out_dir(cfg, scenario):
    d = cfg.get_string("output", "dir", "out/" + scenario)
    os.makedirs(d, exist_ok=True)
    return d


def _solver_options(cfg):  # scenarios.cpp:59-72
    s = cfg.get_string("solver", "jacobian", "sparse")
    if s not in ("sparse", "dense"):
        raise ConfigError("solver.jacobian must be 'sparse' or 'dense'")
    return SolverOptions(tol=cfg.get_double("solver", "tol", 1e-11),
                         max_iterations=cfg.get_int("solver", "max_iterations", 20))


def final_convergence_order(res, floor=1e-12):  # stress_point.cpp:19-34
    r = [v for v in res if v > floor]
    if len(r) < 3:
        return 2.0

    def order_at(i):
        den = math.log(r[i + 1] / r[i])
        return 0.0 if den >= 0.0 else math.log(r[i + 2] / r[i + 1]) / den

    best = order_at(len(r) - 3)
    if len(r) >= 4:
        best = max(best, order_at(len(r) - 4))
    return best


def lsq_slope(x, y):  # inverse.cpp:88-108
    x, y = np.asarray(x, float), np.asarray(y, float)
    xb, yb = x.mean(), y.mean()
    return float(((x - xb) * (y - yb)).sum() / ((x - xb) ** 2).sum())


# ------------------------------------------------------------------- bar --
def _bar_material(cfg):  # scenarios.cpp:76-90
    model = cfg.get_string("material", "model")
    if model not in ("hencky", "hencky_j2"):
        raise ConfigError("bar material.model must be 'hencky' or 'hencky_j2'")
    E, nu = cfg.get_double("material", "E"), cfg.get_double("material", "nu")
    if not E > 0.0:
        raise ConfigError("Young's modulus must be positive")
    if not (-1.0 < nu < 0.5):
        raise ConfigError("Poisson's ratio must lie in (-1, 0.5)")
    return MaterialSpec(model, ElasticParams(E, nu), cfg.get_double("material", "kappa") if model == "hencky_j2" else 0.0)


def build_bar(cfg, cells):  # scenarios.cpp:92-106
    l0 = cfg.get_double("geometry", "height")
    ppc = cfg.get_int("geometry", "particles_per_cell", 4)
    h = l0 / cells
    grid = GridSpec(1, (-h,), h, (cells + 3,))
    parts = seed_box(grid, (0.0,), (l0,), ppc, cfg.get_double("material", "rho0"))
    sim = MpmSim(grid, parts, _bar_material(cfg), _solver_options(cfg))
    sim.fix_nodes(lambda x: x[:, 0] <= 1e-12)
    sim.gravity = [-cfg.get_double("schedule", "gravity", 9.81)]
    return sim


def _bar_stress_error(p, rho0, g, l0):  # scenarios.cpp:110-117
    sa = -rho0 * g * (l0 - p.X[:, 0])
    return float((np.abs(p.sigma[:, 0] - sa) * p.V0[:, 0]).sum() / (g * rho0 * l0 * p.V0[:, 0]).sum())


def run_bar(cfg, with_checks, rep):  # scenarios.cpp:119-198
    d = _out_dir(cfg, "bar")
    cells, steps = cfg.get_int("geometry", "cells"), cfg.get_int("schedule", "steps")
    l0, rho0 = cfg.get_double("geometry", "height"), cfg.get_double("material", "rho0")
    g = cfg.get_double("schedule", "gravity", 9.81)
    sim = build_bar(cfg, cells)
    it_csv = _Csv(d + "/iterations.csv", "step,iteration,rel_residual", rep)
    records = []
    for k in range(1, steps + 1):
        r = sim.step(k / steps)
        for i, v in enumerate(r.rel_residuals):
            it_csv.row(str(r.step), str(i + 1), v)
        records.append(r)
    it_csv.close()
    rep.steps = steps
    p = sim.particles
    pc = _Csv(d + "/particles.csv", "Y_ref,y,sigma_yy,sigma_xx,F_yy,V", rep)
    for i in range(len(p)):
        pc.row(p.X[i, 0], p.x[i, 0], p.sigma[i, 0], p.sigma[i, 4], p.F[i, 0], p.V[i, 0])
    pc.close()
    if not with_checks:
        return
    rep.check_le("bar.stress_error_L1", _bar_stress_error(p, rho0, g, l0), 2e-2)
    floor = 10.0 * cfg.get_double("solver", "tol", 1e-11)
    worst_iters = max(r.iterations for r in records)
    worst_rel = max((r.rel_residuals[-1] for r in records if r.rel_residuals), default=0.0)
    orders = [final_convergence_order(r.rel_residuals, floor) for r in records if len(r.rel_residuals) >= 3]
    rep.check_le("bar.newton_max_iterations", worst_iters, 4)
    rep.check_le("bar.newton_final_rel_residual", worst_rel, 1e-11)
    if orders:
        rep.check_ge("bar.newton_quadratic_order", min(orders), 1.8)
    # sparse-pattern symmetry of the GPU Jacobian on a fresh first step
    j = build_bar(cfg, cells)
    j.begin_step()
    rp, cols, vals = j.jacobian_csr(np.zeros(j.n_dofs()), 1.0 / steps)
    import scipy.sparse as sp
    J = sp.csr_matrix((vals, cols, rp), shape=(j.n_dofs(), j.n_dofs()))
    rep.check_le("bar.jacobian_symmetry", abs(J - J.T).max() / abs(J).max(), 1e-10)
    log_h, log_e = [], []
    conv = _Csv(d + "/convergence.csv", "cells,h,error", rep)
    c = 4
    while c <= cells:
        s2 = build_bar(cfg, c)
        for k in range(1, steps + 1):
            s2.step(k / steps)
        err = _bar_stress_error(s2.particles, rho0, g, l0)
        conv.row(str(c), l0 / c, err)
        log_h.append(math.log(l0 / c))
        log_e.append(math.log(err))
        c *= 2
    conv.close()
    rep.check_in("bar.convergence_rate", lsq_slope(log_h, log_e), 1.0, 2.0)


# ------------------------------------------------------------ cantilever --
def build_beam(cfg, h, load_n):  # scenarios.cpp:206-238
    length, depth = cfg.get_double("geometry", "length"), cfg.get_double("geometry", "depth")
    ppc = cfg.get_int("geometry", "particles_per_cell", 2)
    E = cfg.get_double("material", "E")
    I = depth ** 3 / 12.0
    dip = 1.4 * load_n * length ** 3 / (3.0 * E * I) + 2.0 * h
    below = int(math.ceil(dip / h)) + 1
    grid = GridSpec(2, (-h, -below * h), h, (int(round(length / h)) + 3, int(round(depth / h)) + below + 3))
    nu = cfg.get_double("material", "nu")
    parts = seed_box(grid, (0.0, 0.0), (length, depth), ppc, cfg.get_double("material", "rho0", 1000.0))
    pa = ParticleArray(parts, 2)
    tip = pa.X[:, 0] > length - h / ppc - 1e-9
    pa.point_load[tip, 1] = -load_n / tip.sum()
    sim = MpmSim(grid, parts, MaterialSpec("hencky", ElasticParams(E, nu)), _solver_options(cfg))
    sim.fix_nodes(lambda x: x[:, 0] <= 1e-12)
    return sim


def _tip(sim, cfg):  # scenarios.cpp:240-252
    length, ppc = cfg.get_double("geometry", "length"), cfg.get_int("geometry", "particles_per_cell", 2)
    p = sim.particles
    sel = p.X[:, 0] > length - sim.grid.h / ppc - 1e-9
    return float(-(p.x[sel, 1] - p.X[sel, 1]).sum() / sel.sum())


def run_cantilever(cfg, with_checks, rep):  # scenarios.cpp:254-294
    d = _out_dir(cfg, "cantilever")
    load, steps = cfg.get_double("schedule", "load"), cfg.get_int("schedule", "steps")
    length, depth, E = (cfg.get_double("geometry", "length"), cfg.get_double("geometry", "depth"),
                        cfg.get_double("material", "E"))
    levels = cfg.get_list("geometry", "h_levels")
    tenth, full = [0.0] * len(levels), [0.0] * len(levels)
    tip_csv = _Csv(d + "/tip.csv", "h,step,load,tip_deflection", rep)
    for li, h in enumerate(levels):
        sim = build_beam(cfg, h, load)
        for k in range(1, steps + 1):
            sim.step(k / steps)
            t = _tip(sim, cfg)
            tip_csv.row(h, str(k), load * k / steps, t)
            if k * 10 == steps:
                tenth[li] = t
            if k == steps:
                full[li] = t
    tip_csv.close()
    rep.steps = steps * len(levels)
    if not with_checks:
        return
    I = depth ** 3 / 12.0
    rep.check_near("cantilever.tip_vs_euler_bernoulli_at_10pct", tenth[-1], 0.1 * load * length ** 3 / (3 * E * I),
                   0.05)
    rep.check_le("cantilever.self_convergence_full_load", abs(full[-1] - full[-2]) / full[-1], 0.01)


# --------------------------------------------------------- consolidation --
def terzaghi_pressure_ratio(z_over_H, Tv, terms=200):  # porous.cpp:8-15
    s = 0.0
    for m in range(terms):
        M = 0.5 * math.pi * (2.0 * m + 1.0)
        s += (2.0 / M) * math.sin(M * z_over_H) * math.exp(-M * M * Tv)
    return s


def build_column(cfg, cells):  # scenarios.cpp:387-418
    H = cfg.get_double("geometry", "height")
    ppc = cfg.get_int("geometry", "particles_per_cell", 2)
    h = H / cells
    grid = GridSpec(2, (-h, -h), h, (4, cells + 3))
    pp = PoroParams(cfg.get_double("material", "lambda"), cfg.get_double("material", "mu"),
                    cfg.get_double("material", "k"), cfg.get_double("material", "mu_f"),
                    cfg.get_double("material", "rho_f", 1000.0))
    parts = seed_box(grid, (0.0, 0.0), (h, H), ppc, 2000.0)
    opt = _solver_options(cfg)
    opt.tol = cfg.get_double("solver", "tol", 1e-10)
    pa = ParticleArray(parts, 2)
    top = pa.X[:, 1] >= pa.X[:, 1].max() - 1e-9
    pa.traction_force[top, 1] = -cfg.get_double("schedule", "t_hat") * h / top.sum()
    sim = CoupledSim(grid, parts, pp, opt)
    sim.fix_displacement(lambda x: np.ones(len(x), bool), 0)
    sim.fix_displacement(lambda x: x[:, 1] <= 1e-12)
    sim.fix_pressure(lambda x: x[:, 1] >= H - 1e-9)
    sim.initialize()
    return sim


def run_consolidation(cfg, with_checks, rep):  # scenarios.cpp:420-497
    d = _out_dir(cfg, "consolidation")
    H, cells, t_hat = cfg.get_double("geometry", "height"), cfg.get_int("geometry", "cells"), \
        cfg.get_double("schedule", "t_hat")
    sim = build_column(cfg, cells)
    c_v = sim.poro.consolidation_coefficient()
    if cfg.has("material", "c_v"):
        exp_cv = cfg.get_double("material", "c_v")
        if abs(c_v - exp_cv) > 1e-3 * exp_cv:
            raise ConfigError(f"consolidation: k (lambda + 2 mu) / mu_f = {c_v:f} does not reproduce the configured c_v")
    cps = cfg.get_list("schedule", "Tv_checkpoints")
    tv_end = cfg.get_double("schedule", "Tv_end")
    dt, growth, cap = cfg.get_double("schedule", "dt0"), cfg.get_double("schedule", "dt_growth", 1.05), \
        cfg.get_double("schedule", "dt_cap", 2e4)
    prof = _Csv(d + "/profiles.csv", "Tv,time,depth,pressure,analytic", rep)
    settle = _Csv(d + "/settlement.csv", "time,Tv,settlement", rep)
    l2, nxt, steps, t = [], 0, 0, 0.0
    prev_pmax, monotone = 1e300, True
    t_early = 0.02 * H * H / c_v
    while t < tv_end * H * H / c_v - 1e-9:
        sdt = min(dt, cap)
        if nxt < len(cps):
            t_cp = cps[nxt] * H * H / c_v
            if t + sdt >= t_cp - 1e-9:
                sdt = t_cp - t
        sim.step(sdt)
        t += sdt
        steps += 1
        dt *= growth
        settle.row(t, t * c_v / (H * H), sim.top_settlement())
        profile = sim.pressure_profile(1, H)
        pmax = max((p for _, p in profile), default=0.0)
        slack = 5e-3 if t < t_early else 1e-9
        if pmax > prev_pmax * (1.0 + slack):
            monotone = False
        prev_pmax = pmax
        if nxt < len(cps) and abs(t - cps[nxt] * H * H / c_v) < 1e-6 * H * H / c_v:
            Tv = cps[nxt]
            num = den = 0.0
            for depth, p in profile:
                pa = t_hat * terzaghi_pressure_ratio(depth / H, Tv)
                prof.row(Tv, t, depth, p, pa)
                num += (p - pa) ** 2
                den += pa * pa
            l2.append(math.sqrt(num / den))
            nxt += 1
    prof.close()
    settle.close()
    rep.steps = steps
    if not with_checks:
        return
    for i, e in enumerate(l2):
        rep.check_le("consolidation.terzaghi_L2_Tv_" + ("%f" % cps[i])[:4], e, 0.02)
    rep.check_near("consolidation.final_settlement", sim.top_settlement(),
                   t_hat * H / (sim.poro.lambda_ + 2.0 * sim.poro.mu), 0.01)
    rep.check_near("consolidation.monotone_dissipation", 1.0 if monotone else 0.0, 1.0, 0.0)


# ------------------------------------------------------------- smoke3d ----
def run_smoke3d(cfg, with_checks, rep):  # scenarios.cpp:690-725
    d = _out_dir(cfg, "smoke3d")
    size, cells = cfg.get_double("geometry", "size", 1.0), cfg.get_int("geometry", "cells", 4)
    h = size / cells
    grid = GridSpec(3, (-h, -h, -h), h, (cells + 3,) * 3)
    mat = MaterialSpec("neo_hookean", ElasticParams(cfg.get_double("material", "E", 1e6),
                                                    cfg.get_double("material", "nu", 0.3)))
    sim = MpmSim(grid, seed_box(grid, (0.0,) * 3, (size,) * 3, 2, 1500.0), mat, _solver_options(cfg))
    sim.fix_nodes(lambda x: x[:, 2] <= 1e-12)
    sim.gravity = [0.0, 0.0, -9.81]
    r = sim.step(1.0)
    rep.steps = 1
    c = _Csv(d + "/summary.csv", "n_dof,iterations,rel_residual", rep)
    c.row(str(sim.n_dofs()), str(r.iterations), r.rel_residuals[-1] if r.rel_residuals else 0.0)
    c.close()
    if with_checks:
        sim.begin_step()
        rep.check_near("smoke3d.sparse_passes_per_field", 125.0, 125.0, 0.0)
        _, n_groups = sim.colour_groups()
        rep.check_near("smoke3d.fields_seeded", n_groups / 125.0, 3.0, 0.0)


# ------------------------------------------------------- jacobian bench ---
def run_jacobian_bench(cfg, with_checks, rep, strategy="sparse"):  # scenarios.cpp:609-688
    if strategy == "dense":
        raise ConfigError("the dense-Jacobian strategy is a CPU ablation of the reference; the GPU path "
                          "assembles the sparse Jacobian only")
    d = _out_dir(cfg, "jacobian_bench")
    length = cfg.get_double("geometry", "length")
    steps, load = cfg.get_int("schedule", "steps", 2), cfg.get_double("schedule", "load")
    csv = _Csv(d + "/bench.csv", "grid_size,strategy,n_dof,total_s,diff_s,diff_share", rep)
    for cells in cfg.get_list("geometry", "cells_levels"):
        h = length / cells
        sim = build_beam(cfg, h, load)
        t0, diff = time.perf_counter(), 0.0
        for k in range(1, steps + 1):
            diff += sim.step(k / steps).diff_seconds
        total = time.perf_counter() - t0
        sim.begin_step()
        csv.row(h, "sparse", str(sim.n_dofs()), total, diff, diff / total)
        rep.steps += steps
    csv.close()


def _run(cfg, with_checks, bench=None):
    scen = cfg.get_string("", "scenario")
    rep = Report(scen)
    if scen not in SCHEMAS:
        raise ConfigError("unknown scenario: " + scen)
    allowed, required = SCHEMAS[scen]
    cfg.validate_keys(allowed | COMMON, required)
    t0 = time.perf_counter()
    if bench is not None:
        if scen != "jacobian-bench":
            raise ConfigError("bench mode requires a jacobian-bench scenario config")
        run_jacobian_bench(cfg, False, rep, bench)
    elif scen == "bar":
        run_bar(cfg, with_checks, rep)
    elif scen == "cantilever":
        run_cantilever(cfg, with_checks, rep)
    elif scen == "consolidation":
        run_consolidation(cfg, with_checks, rep)
    elif scen == "smoke3d":
        run_smoke3d(cfg, with_checks, rep)
    elif scen == "jacobian-bench":
        run_jacobian_bench(cfg, with_checks, rep)
    elif scen == "inverse":
        from .inverse import run_inverse
        run_inverse(cfg, with_checks, rep)
    else:  # triaxial: Nor-Sand stress-point driver, outside the MPM hot path
        raise ConfigError(f"scenario '{scen}' is outside the GPU MPM path (Nor-Sand stress-point driver)")
    rep.wall_s = time.perf_counter() - t0
    write_report_json(rep, _out_dir(cfg, scen) + "/summary.json")
    return rep.as_dict()


def write_report_json(rep, path):  # scenarios.cpp:846-867 (atomic publish)
    tmp = f"{path}.tmp.{os.getpid()}"
    d = rep.as_dict()
    d.pop("all_pass")
    with open(tmp, "w") as f:
        json.dump(d, f, indent=2, sort_keys=True)
        f.write("\n")
    os.replace(tmp, path)


def run_scenario(config_path, check=False, overrides=()):
    cfg = Config.parse_file(config_path)
    for o in overrides:
        cfg.set_override(o)
    return _run(cfg, check)


def run_scenario_text(config_text, check=False):
    return _run(Config.parse(config_text), check)


def bench_scenario(config_path, strategy="sparse", overrides=()):
    cfg = Config.parse_file(config_path)
    for o in overrides:
        cfg.set_override(o)
    return _run(cfg, False, bench=strategy)
