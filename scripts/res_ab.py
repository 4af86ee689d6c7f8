"""Residual A/B under two environment settings on the same state (3D footing):
prints max |dr| and whether the two are bitwise equal. GPU only:
    python scripts/res_ab.py "IMPM_RES_PIPE=0" "" [cells_x cells_y cells_z]
Each setting runs in its own process (switches are read at sim creation)."""
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
cells = tuple(int(v) for v in sys.argv[1:4]); out = sys.argv[4]
prob = workloads.footing3d(cells=cells, steps=10)
sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options)
sim.fixed[:] = prob.fixed
sim.gravity = prob.gravity
its = [sim.step(k / prob.load_steps).iterations for k in range(1, 3)]
sim.begin_step()
u = np.random.default_rng(1).standard_normal(sim.n_dofs()) * 1e-4 * prob.grid.h
np.savez(out, r=sim.residual(u, 0.3), its=np.array(its))
'''


def run(env_str, cells, out):
    env = dict(os.environ)
    for kv in env_str.split():
        k, v = kv.split("=", 1)
        env[k] = v
    subprocess.run([sys.executable, "-c", CHILD, *map(str, cells), out], env=env, check=True)
    return np.load(out)


def main():
    a_env, b_env = sys.argv[1], sys.argv[2]
    cells = tuple(int(v) for v in sys.argv[3:6]) if len(sys.argv) > 5 else (32, 32, 16)
    with tempfile.TemporaryDirectory() as tmp:
        a = run(a_env, cells, os.path.join(tmp, "a.npz"))
        b = run(b_env, cells, os.path.join(tmp, "b.npz"))
        d = np.abs(a["r"] - b["r"]).max()
        print(f"[{a_env}] vs [{b_env}] {cells}: max |dr| = {d:.3e} (|r| max {np.abs(a['r']).max():.3e}), "
              f"newton {a['its'].tolist()} {b['its'].tolist()}, bitwise {np.array_equal(a['r'], b['r'])}")


if __name__ == "__main__":
    main()
