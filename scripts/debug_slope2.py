import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2507_09435_b200 as impm
from paper_2507_09435_b200 import workloads
for mat in ["hencky", "hencky_j2", "drucker_prager", "neo_hookean"]:
    for shape in ["gimp", "quadratic-bspline"]:
        prob = workloads.slope2d(cells=(24, 12), ppc=2, h=0.5, steps=10, material=mat)
        prob.options.shape = shape
        sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options)
        sim.fixed[:] = prob.fixed
        sim.gravity = prob.gravity
        sim.begin_step()
        n = sim.n_dofs()
        rp, cols, vals = sim.jacobian_csr(np.zeros(n), 0.1)
        r = sim.residual(np.zeros(n), 0.1)
        print(mat, shape, n, "J", np.abs(vals).max(), "r", np.abs(r).max(), "mass", sim.node_mass().sum(), flush=True)
