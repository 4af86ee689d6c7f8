"""One cfg4 (or cfg1) load step on the GPU for ncu captures: python scripts/profile_step.py [cfg4|cfg1] [steps]"""
import sys
sys.path.insert(0, ".")
from paper_2507_09435_b200 import workloads
import paper_2507_09435_b200 as impm

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
prob = workloads.footing3d() if cfg == "cfg4" else workloads.column2d_nh()
sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options)
sim.fixed[:] = prob.fixed
sim.gravity = prob.gravity
for k in range(1, steps + 1):
    rec = sim.step(k / prob.load_steps)
    print(k, rec.iterations, rec.krylov_iterations, f"{rec.seconds:.3f}s", flush=True)
