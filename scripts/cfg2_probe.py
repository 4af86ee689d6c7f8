"""cfg 2 (2D slope, 256x128 cells, ppc 4, ~0.5M particles) on the GPU: time the
gravity-ramp load steps for a material."""
import sys
import time

sys.path.insert(0, ".")
import paper_2507_09435_b200 as impm  # noqa: E402
from paper_2507_09435_b200 import workloads  # noqa: E402

material = sys.argv[1] if len(sys.argv) > 1 else "drucker_prager"
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
kw = {}
if material == "drucker_prager":
    kw = {"cohesion": float(sys.argv[3]) if len(sys.argv) > 3 else 0.0}
elif material == "hencky_j2" and len(sys.argv) > 3:
    kw = {"kappa": float(sys.argv[3])}
prob = workloads.slope2d(material=material, **kw)
sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options)
sim.fixed[:] = prob.fixed
sim.gravity = prob.gravity
print("particles", prob.particles.shape[0], flush=True)
for k in range(1, nsteps + 1):
    t = time.time()
    try:
        rec = sim.step(k / prob.load_steps)
    except Exception as e:  # noqa: BLE001
        print("step", k, "FAILED", type(e).__name__, str(e)[:200], flush=True)
        break
    print(f"step {k} its {rec.iterations} krylov {rec.krylov_iterations} rel {rec.rel_residuals[-1] if rec.rel_residuals else 0:.2e} {time.time() - t:.3f}s", flush=True)
p = sim.particles
print("plastic particles", int((p.alpha[:, 0] > 0).sum()))
