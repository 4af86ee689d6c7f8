import sys
sys.path.insert(0, ".")
import numpy as np, scipy.sparse as sp
import paper_2507_09435_b200 as impm
from paper_2507_09435_b200 import workloads
mat = sys.argv[1]
prob = workloads.slope2d(cells=(24, 12), ppc=2, h=0.5, steps=10, material=mat, friction_deg=40.0, slope_deg=30.0, cohesion=2e3)
prob.options.precond = sys.argv[2]
prob.options.krylov = sys.argv[3]
sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options)
sim.fixed[:] = prob.fixed
sim.gravity = prob.gravity
for k in range(1, 11):
    try:
        rec = sim.step(k / 10)
        print(k, rec.iterations, rec.krylov_iterations, ["%.1e" % x for x in rec.rel_residuals], flush=True)
    except Exception as e:
        print(k, "ERR", e)
        sim.begin_step()
        n = sim.n_dofs()
        rp, cols, vals = sim.jacobian_csr(np.zeros(n), k / 10)
        J = sp.csr_matrix((vals, cols, rp), shape=(n, n)).toarray()
        d = np.diag(J)
        print("n", n, "zero diag", (np.abs(d) < 1e-12 * np.abs(d).max()).sum(), "cond", np.linalg.cond(J),
              "asym", np.abs(J - J.T).max() / np.abs(J).max())
        break
