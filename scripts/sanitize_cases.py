"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck, one tool per run): every kernel family of the product
path at tiny sizes. GPU only:
    compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize_cases.py"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import golden_util as gu  # noqa: E402
import paper_2507_09435_b200 as impm  # noqa: E402
from paper_2507_09435_b200 import workloads  # noqa: E402


def fixture_steps(name, krylov, steps=2):
    fx = gu.load(name)
    dim, grid, mat, opts, parts, fixed, grav, spec = gu.problem(fx)
    g = impm.GridSpec(dim, grid["origin"], grid["h"], grid["nodes"])
    m = impm.MaterialSpec(mat["kind"], impm.ElasticParams(mat["E"], mat["nu"]), mat["kappa"])
    sim = impm.MpmSim(g, parts, m, impm.SolverOptions(tol=opts["tol"], krylov=krylov))
    sim.fixed[:] = fixed
    sim.gravity = grav
    n = int(spec.get("steps", 2)) or 2
    for k in range(1, min(steps, n) + 1):
        sim.step(k / n)
    sim.begin_step()
    sim.jacobian_csr(np.zeros(sim.n_dofs()))
    print(name, krylov, "ok", flush=True)


for name, kry in [("cube3d_nh_newton", "iterative"), ("cube3d_nh_newton", "auto"), ("col2d_j2", "iterative"),
                  ("bar1d_j2", "iterative"), ("tl2d_hencky", "iterative"), ("cant2d_hencky_newton", "gmres")]:
    fixture_steps(name, kry)
for mat in ["drucker_prager", "cam_clay", "hencky_j2"]:
    prob = workloads.footing3d(cells=(6, 6, 4), steps=10, t_hat=300e3, material=mat)
    if mat == "hencky_j2":
        prob.material.kappa = 40e3
    sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options)
    sim.fixed[:] = prob.fixed
    sim.gravity = prob.gravity
    for k in range(1, 3):
        sim.step(k / prob.load_steps)
    print(mat, "ok", flush=True)
sim, _ = workloads.terzaghi((4, 16), ppc=2)
for _ in range(2):
    sim.step(100.0)
print("coupled ok", flush=True)
from paper_2507_09435_b200.sparse import CsrMatrix, sparse_lu_solve  # noqa: E402

A = CsrMatrix(2, [0, 2, 4], [0, 1, 0, 1], [2.0, 1.0, 1.0, 2.0])
print("csr ok", sparse_lu_solve(A, np.array([3.0, 3.0])), flush=True)
from paper_2507_09435_b200 import _abi  # noqa: E402

oob = _abi.lib().impm_debug_oob_count()
print("out-of-range scattered accesses counted:", oob, "(-1: not a checked build)", flush=True)
if oob > 0:
    sys.exit(1)
