"""Linear solves and Newton on the jittered fixtures (3-node supports from
step 0, fringe nodes at ~1e-14 of the bulk stiffness) against the reference's
LU solve / Newton trace. GPU only:  python scripts/jitter_probe.py"""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import golden_util as gu  # noqa: E402


def make(name, **kw):
    import paper_2507_09435_b200 as impm

    fx = gu.load(name)
    dim, grid, mat, opts, parts, fixed, grav, spec = gu.problem(fx)
    g = impm.GridSpec(dim, grid["origin"], grid["h"], grid["nodes"])
    m = impm.MaterialSpec(mat["kind"], impm.ElasticParams(mat["E"], mat["nu"]), mat["kappa"])
    o = impm.SolverOptions(tol=opts["tol"], max_iterations=opts["max_iterations"],
                           total_lagrangian=opts["total_lagrangian"], **kw)
    sim = impm.MpmSim(g, parts, m, o)
    sim.fixed[:] = fixed
    sim.gravity = grav
    return sim, fx, spec


for name in ["cant2d_hencky", "cube3d_nh", "col2d_nh", "col2d_nh_newton"]:
    for kw in [{}, {"krylov": "gmres"}, {"precond": "block_jacobi", "krylov": "gmres"}]:
        try:
            sim, fx, spec = make(name, **kw)
            s0 = float(spec.get("probe_scale", 0.5))
            sim.begin_step()
            d, its = sim.linear_solve(fx["u1"], s0, -fx["r1"])
            err = gu.rel_err(d, fx["delta1"])
            # scaled residual of the reference solution and ours under our J
            print(f"{name} {kw}: solve its={its} rel_err={err:.3e}", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"{name} {kw}: solve FAILED {type(e).__name__}: {str(e)[:120]}", flush=True)
    if "newton_iters" in gu.load(name):
        for env in [None, "1"]:
            if env:
                os.environ["IMPM_EXACT_NEWTON"] = env
            try:
                sim, fx, spec = make(name)
                steps = int(spec.get("steps", 1))
                its = [sim.step(k / steps).iterations for k in range(1, steps + 1)]
                print(f"{name} newton exact={env}: {its} ref {fx['newton_iters'].tolist()}", flush=True)
            except Exception as e:  # noqa: BLE001
                print(f"{name} newton exact={env}: FAILED {type(e).__name__}: {str(e)[:160]}", flush=True)
            os.environ.pop("IMPM_EXACT_NEWTON", None)
