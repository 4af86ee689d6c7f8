"""Prints per-step Newton histories of the GPU path next to the reference's."""
import sys
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import golden_util as gu
from test_gpu_parity import make_sim

name = sys.argv[1]
rtol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-12
import paper_2507_09435_b200 as impm
sim, fx, spec = make_sim(name)
o = sim.options
o.krylov_rtol = rtol
sim.set_options(o)
it = fx["newton_iters"]; rel = fx["newton_rel"]; off = np.concatenate([[0], np.cumsum(it)])
steps = int(spec.get("steps", 2))
for k in range(1, steps + 1):
    rec = sim.step(k / steps)
    ref = rel[off[k - 1]:off[k]]
    print(k, rec.iterations, it[k - 1], "kry", rec.krylov_iterations)
    print("   gpu", " ".join("%.3e" % x for x in rec.rel_residuals))
    print("   ref", " ".join("%.3e" % x for x in ref))
