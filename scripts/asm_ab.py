"""A/B of the 3D Jacobian (tangent + assembly) under two environment settings
on the same state: prints the row-scaled max difference of J and the Newton
counts of both. GPU only:
    python scripts/asm_ab.py "IMPM_ASM_RMW=0" "" [cells_x cells_y cells_z] [material]
Each setting runs in its own process (the switches are read at sim creation)."""
import os
import subprocess
import sys
import tempfile

import numpy as np

CHILD = r'''
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2507_09435_b200 as impm
from paper_2507_09435_b200 import workloads
cells = tuple(int(v) for v in sys.argv[1:4]); material = sys.argv[4]; out = sys.argv[5]
prob = workloads.footing3d(cells=cells, steps=10, material=material)
if material == "cam_clay":
    prob.material.pc0 = 40e3
sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options)
sim.fixed[:] = prob.fixed
sim.gravity = prob.gravity
its = [sim.step(k / prob.load_steps).iterations for k in range(1, 4)]
sim.begin_step()
u = np.random.default_rng(1).standard_normal(sim.n_dofs()) * 1e-4 * prob.grid.h
rp, cols, vals = sim.jacobian_csr(u, 0.4)
np.savez(out, rp=rp, cols=cols, vals=vals, its=np.array(its))
'''


def run(env_str, cells, material, out):
    env = dict(os.environ)
    for kv in env_str.split():
        k, v = kv.split("=", 1)
        env[k] = v
    subprocess.run([sys.executable, "-c", CHILD, *map(str, cells), material, out], env=env, check=True)
    return np.load(out)


def main():
    a_env, b_env = sys.argv[1], sys.argv[2]
    cells = tuple(int(v) for v in sys.argv[3:6]) if len(sys.argv) > 5 else (32, 32, 16)
    material = sys.argv[6] if len(sys.argv) > 6 else "neo_hookean"
    sys.path.insert(0, "tests")
    import golden_util as gu

    with tempfile.TemporaryDirectory() as tmp:
        a = run(a_env, cells, material, os.path.join(tmp, "a.npz"))
        b = run(b_env, cells, material, os.path.join(tmp, "b.npz"))
        assert np.array_equal(a["rp"], b["rp"]) and np.array_equal(a["cols"], b["cols"])
        err = gu.csr_row_scaled_err(a["rp"], a["vals"], b["vals"])
        print(f"[{a_env}] vs [{b_env}] {material} {cells}: row-scaled max |dJ| = {err:.3e}, "
              f"newton {a['its'].tolist()} {b['its'].tolist()}, bitwise {np.array_equal(a['vals'], b['vals'])}")


if __name__ == "__main__":
    main()
