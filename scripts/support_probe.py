"""Support-size statistics along the cfg 4 load ramp (sizes the Jacobian
work: sum_p s_p^2 block contributions, bin boxes). GPU only."""
import json
import sys

sys.path.insert(0, ".")
import paper_2507_09435_b200 as impm  # noqa: E402
from paper_2507_09435_b200 import workloads  # noqa: E402

material = sys.argv[1] if len(sys.argv) > 1 else "neo_hookean"
prob = workloads.footing3d(material=material, steps=20)
sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options)
sim.fixed[:] = prob.fixed
sim.gravity = prob.gravity
for k in range(1, 21):
    sim.begin_step()
    st = sim.support_stats()
    info = sim.matrix_info() if k > 1 else {}
    rec = sim.step(k / 20)
    if k in (1, 2, 5, 10, 15, 20):
        print(json.dumps({"step": k, "iters": rec.iterations, "kry": rec.krylov_iterations, **st,
                          "stored_blocks_per_row": info.get("row_values", 0) / max(info.get("rows", 1), 1) / 9}),
              flush=True)
