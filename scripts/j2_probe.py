"""Newton counts on the J2 fixtures and the bar_elastoplastic scenario under
linear-solver settings (A/B for the count-preserving forcing term). GPU only:
    python scripts/j2_probe.py"""
import os
import subprocess
import sys
import tempfile

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import golden_util as gu  # noqa: E402

SETTINGS = [
    {"IMPM_EXACT_NEWTON": "0"},
    {"IMPM_EXACT_NEWTON": "1", "IMPM_EXACT_RTOL": "1e-12"},
    {"IMPM_EXACT_NEWTON": "1", "IMPM_EXACT_RTOL": "1e-13"},
    {"IMPM_EXACT_NEWTON": "1", "IMPM_EXACT_RTOL": "1e-14"},
]
CHILD = r'''
import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import golden_util as gu, paper_2507_09435_b200 as impm
name, kry = sys.argv[1], sys.argv[2]
fx = gu.load(name)
dim, grid, mat, opts, parts, fixed, grav, spec = gu.problem(fx)
g = impm.GridSpec(dim, grid["origin"], grid["h"], grid["nodes"])
m = impm.MaterialSpec(mat["kind"], impm.ElasticParams(mat["E"], mat["nu"]), mat["kappa"])
o = impm.SolverOptions(tol=opts["tol"], max_iterations=opts["max_iterations"], krylov=kry)
sim = impm.MpmSim(g, parts, m, o); sim.fixed[:] = fixed; sim.gravity = grav
steps = int(spec.get("steps", 1))
its = np.array([sim.step(k / steps).iterations for k in range(1, steps + 1)])
ref = fx["newton_iters"]
print(name, kry, "diff steps", int((its != ref).sum()), "of", steps, "its", its.tolist(), "ref", ref.tolist())
'''
for st in SETTINGS:
    env = dict(os.environ, **st)
    for name in ["bar1d_j2", "col2d_j2"]:
        for kry in ["auto", "gmres"]:
            r = subprocess.run([sys.executable, "-c", CHILD, name, kry], env=env, capture_output=True, text=True)
            print(st, (r.stdout.strip() or r.stderr.strip()[-300:]), flush=True)
    with tempfile.TemporaryDirectory() as tmp:
        code = ("import sys; sys.path.insert(0,'.'); import paper_2507_09435_b200 as impm, numpy as np;"
                f"impm.run_scenario('tests/golden/configs/bar_elastoplastic.cfg', False, ['output.dir={tmp}']);"
                f"g=np.loadtxt('{tmp}/iterations.csv',delimiter=',',skiprows=1,ndmin=2);"
                "r=np.load('tests/golden/reference_out.npz')['bar_elastoplastic__iterations'];"
                "a=np.bincount(g[:,0].astype(int));b=np.bincount(r[:,0].astype(int));"
                "print('bar_elastoplastic diff steps', int((a!=b).sum()), 'of', len(b)-1)")
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        print(st, (r.stdout.strip() or r.stderr.strip()[-300:]), flush=True)
