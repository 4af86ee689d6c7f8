"""cfg 4 load steps 4-6 timed with CUDA events, the sim on its own
non-blocking stream vs on torch's current (legacy default) stream. GPU only:
    python scripts/stream_probe.py [own|torch]"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2507_09435_b200 as impm  # noqa: E402
from paper_2507_09435_b200 import workloads  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "own"
prob = workloads.footing3d(steps=20)
sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options, device=0)
sim.fixed[:] = prob.fixed
sim.gravity = prob.gravity
stream = torch.cuda.current_stream(0)
if mode == "torch":
    sim.set_stream(stream.cuda_stream)
elif mode == "side":
    side = torch.cuda.Stream(0)
    sim.set_stream(side.cuda_stream)
    stream = side
for k in range(1, 4):
    sim.step(k / 20)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
ev0.record(stream)
secs = []
for k in range(4, 7):
    secs.append(sim.step(k / 20).seconds)
ev1.record(stream)
torch.cuda.synchronize()
print(f"{mode}: {ev0.elapsed_time(ev1) / 3:.1f} ms/step (events on the {'sim' if mode != 'own' else 'torch'} "
      f"stream), host {1e3 * (time.perf_counter() - t0) / 3:.1f} ms/step, step records {[round(s * 1e3) for s in secs]}")
