"""cfg 4 load steps 4-8 split into begin_step / newton_solve / commit_step by
host timers (synchronised), to see where the time outside the Newton solve
goes. GPU only:
    python scripts/phase_probe.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2507_09435_b200 as impm  # noqa: E402
from paper_2507_09435_b200 import workloads  # noqa: E402

prob = workloads.footing3d(steps=20)
sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options, device=0)
sim.fixed[:] = prob.fixed
sim.gravity = prob.gravity
for k in range(1, 4):
    sim.step(k / 20)
torch.cuda.synchronize()
for k in range(4, 9):
    t0 = time.perf_counter()
    sim.begin_step()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    rec = sim.newton_solve(k / 20)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    sim.commit_step()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"step {k}: begin {1e3 * (t1 - t0):.1f} ms, newton {1e3 * (t2 - t1):.1f} ms ({rec.iterations} it), "
          f"commit {1e3 * (t3 - t2):.1f} ms", flush=True)
