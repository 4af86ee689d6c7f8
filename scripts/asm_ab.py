"""A/B of the 3D Jacobian assembly: the owner-computes z-sweep
(impm_asm_sweep.cuh) against the colour-batched kernel (IMPM_ASM_SWEEP=0) on
the same state. Prints the row-scaled max difference of J and the per-class
timing of one profiled load step for both. GPU only:
    python scripts/asm_ab.py [cells_x cells_y cells_z] [material]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")


def build(env, cells, material):
    os.environ["IMPM_ASM_SWEEP"] = env
    import paper_2507_09435_b200 as impm
    from paper_2507_09435_b200 import workloads

    prob = workloads.footing3d(cells=cells, steps=10, material=material)
    if material == "cam_clay":
        prob.material.pc0 = 40e3
    sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options)
    sim.fixed[:] = prob.fixed
    sim.gravity = prob.gravity
    return sim, prob


cells = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (32, 32, 16)
material = sys.argv[4] if len(sys.argv) > 4 else "neo_hookean"
res = {}
for env in ["1", "0"]:
    sim, prob = build(env, cells, material)
    its = [sim.step(k / prob.load_steps).iterations for k in range(1, 4)]
    sim.begin_step()
    u = sim.nodal_solution() if sim.n_dofs() else np.zeros(0)
    u = np.random.default_rng(1).standard_normal(sim.n_dofs()) * 1e-4 * prob.grid.h
    rp, cols, vals = sim.jacobian_csr(u, 0.4)
    res[env] = (rp, cols, vals, its)
    print(f"IMPM_ASM_SWEEP={env}: newton {its}, nnz {len(vals)}", flush=True)
import golden_util as gu  # noqa: E402

rp1, c1, v1, i1 = res["1"]
rp0, c0, v0, i0 = res["0"]
assert np.array_equal(rp1, rp0) and np.array_equal(c1, c0)
print("row-scaled max |J_sweep - J_colour| =", gu.csr_row_scaled_err(rp0, v1, v0), "newton", i1, i0, flush=True)
