"""cfg 3 (2D Terzaghi u-p, 512x512 cells, 1M particles) on the GPU: time a few
steps and compare the pressure profile with the series solution."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2507_09435_b200 import workloads  # noqa: E402
from paper_2507_09435_b200.scenarios import terzaghi_pressure_ratio  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 512
nsteps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
Tv_end = float(sys.argv[3]) if len(sys.argv) > 3 else 0.05
t0 = time.time()
sim, prm = workloads.terzaghi2d(cells=(cells, cells))
print("setup", time.time() - t0, prm, flush=True)
H, cv = prm["height"], prm["c_v"]
t_end = Tv_end * H * H / cv
dt = t_end / nsteps
for k in range(nsteps):
    t1 = time.time()
    rec = sim.step(dt)
    print(f"step {k} its {rec.iterations} krylov {rec.krylov_iterations} {time.time() - t1:.3f}s", flush=True)
prof = sim.pressure_profile(cells // 2, H)
num = den = 0.0
for depth, p in prof:
    pa = prm["t_hat"] * terzaghi_pressure_ratio(depth / H, Tv_end)
    num += (p - pa) ** 2
    den += pa * pa
print("L2", np.sqrt(num / den), "settlement", sim.top_settlement())
