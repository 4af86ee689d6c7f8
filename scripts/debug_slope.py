import sys
sys.path.insert(0, ".")
import numpy as np, scipy.sparse as sp
import paper_2507_09435_b200 as impm
from paper_2507_09435_b200 import workloads
mat = sys.argv[1] if len(sys.argv) > 1 else "drucker_prager"
prob = workloads.slope2d(cells=(24, 12), ppc=2, h=0.5, steps=10, material=mat)
sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options)
sim.fixed[:] = prob.fixed
sim.gravity = prob.gravity
print("particles", prob.particles.shape)
sim.begin_step()
n = sim.n_dofs()
u = np.zeros(n)
r = sim.residual(u, 0.1)
rp, cols, vals = sim.jacobian_csr(u, 0.1)
J = sp.csr_matrix((vals, cols, rp), shape=(n, n)).toarray()
print("n", n, "nan", np.isnan(J).any(), "asym", np.abs(J - J.T).max() / np.abs(J).max())
d = np.diag(J); print("diag min/max", d.min(), d.max(), "zero diag", (d == 0).sum())
ev = np.linalg.eigvalsh(0.5 * (J + J.T)); print("eig min/max", ev.min(), ev.max(), "neg", (ev < 0).sum())
print("rowmax min", np.abs(J).max(1).min())
for pc in ["block_jacobi", "mg"]:
    o = prob.options; o.precond = pc; o.krylov = "gmres"; sim.set_options(o)
    try:
        x, it = sim.linear_solve(u, 0.1, -r)
        print(pc, "its", it, "res", np.linalg.norm(J @ x + r) / np.linalg.norm(r))
    except Exception as e:
        print(pc, "ERR", e)
x = np.linalg.lstsq(J, -r, rcond=None)[0]; print("lstsq res", np.linalg.norm(J @ x + r) / np.linalg.norm(r))
