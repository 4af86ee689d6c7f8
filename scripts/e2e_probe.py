"""Where the end-to-end (host buffers) step time goes: upload / step / download
per iteration, the StepRecord split and per-kernel-class device time.
python scripts/e2e_probe.py [reps]"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_09435_b200 as impm  # noqa: E402
from paper_2507_09435_b200 import _abi, workloads  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
prob = workloads.footing3d()
opts = prob.options
opts.profile = True
sim = impm.MpmSim(prob.grid, prob.particles, prob.material, opts)
sim.fixed[:] = prob.fixed
sim.gravity = prob.gravity
host = torch.empty(prob.particles.shape, dtype=torch.float64, pin_memory=True).numpy()
host[:] = prob.particles
back = torch.empty(prob.particles.shape, dtype=torch.float64, pin_memory=True).numpy()
for r in range(reps):
    sim.kernel_times(reset=True)
    t0 = time.perf_counter()
    sim.set_particles(host)
    t1 = time.perf_counter()
    rec = sim.step(1.0 / prob.load_steps)
    t2 = time.perf_counter()
    sim._h.call("impm_sim_get_particles", _abi.ptr(back), back.shape[0], back.strides[0])
    t3 = time.perf_counter()
    kt = sim.kernel_times()
    print(json.dumps({"rep": r, "upload_s": round(t1 - t0, 4), "step_s": round(t2 - t1, 4),
                      "download_s": round(t3 - t2, 4), "iters": rec.iterations, "krylov": rec.krylov_iterations,
                      "rec_seconds": round(rec.seconds, 4), "diff_s": round(rec.diff_seconds, 4),
                      "solve_s": round(rec.solve_seconds, 4), "resid_s": round(rec.residual_seconds, 4),
                      "kernel_ms": {k: round(v[0], 1) for k, v in kt.items() if v[0] > 0.5}}), flush=True)
