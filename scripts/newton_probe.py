"""Newton counts and relative residuals on one fixture under the current
environment (A/B of forcing terms). GPU only:
    python scripts/newton_probe.py footing3d_16 [krylov]"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import golden_util as gu  # noqa: E402
import paper_2507_09435_b200 as impm  # noqa: E402

name = sys.argv[1]
kry = sys.argv[2] if len(sys.argv) > 2 else "auto"
fx = gu.load(name)
dim, grid, mat, opts, parts, fixed, grav, spec = gu.problem(fx)
g = impm.GridSpec(dim, grid["origin"], grid["h"], grid["nodes"])
m = impm.MaterialSpec(mat["kind"], impm.ElasticParams(mat["E"], mat["nu"]), mat["kappa"])
o = impm.SolverOptions(tol=opts["tol"], max_iterations=opts["max_iterations"], krylov=kry)
sim = impm.MpmSim(g, parts, m, o)
sim.fixed[:] = fixed
sim.gravity = grav
steps = int(spec.get("steps", 1))
ref_it, ref_rel = fx["newton_iters"], fx["newton_rel"]
o_ = 0
bad = 0
for k in range(1, steps + 1):
    rec = sim.step(k / steps)
    n = int(ref_it[k - 1])
    mine = ["%.4e" % r for r in rec.rel_residuals]
    ref = ["%.4e" % r for r in ref_rel[o_:o_ + n]]
    o_ += n
    flag = "" if rec.iterations == n else "  <-- differs"
    bad += rec.iterations != n
    print(k, rec.iterations, n, mine, ref, rec.krylov_iterations, flag, flush=True)
print(name, kry, "steps differing:", bad)
