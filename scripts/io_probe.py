"""Particle state I/O through the C ABI on cfg 4 (8.39 M particles, 3.3 GB AoS):
impm_sim_set_particles / impm_sim_get_particles against a plain pinned
torch copy of the same size, to split the e2e upload/download phases into
transfer and layout work. GPU only:
    python scripts/io_probe.py
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_09435_b200 as impm  # noqa: E402
from paper_2507_09435_b200 import _abi, workloads  # noqa: E402


def best(fn, reps=3):
    t = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        t = min(t, time.perf_counter() - t0)
    return t


def main():
    prob = workloads.footing3d(cells=(128, 128, 64), steps=20)
    sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options)
    sim.fixed[:] = prob.fixed
    sim.gravity = prob.gravity
    n, w = prob.particles.shape
    host = torch.empty((n, w), dtype=torch.float64, pin_memory=True).numpy()
    host[:] = prob.particles
    nbytes = host.nbytes
    dev = torch.empty(n * w, dtype=torch.float64, device="cuda")
    th = torch.from_numpy(host).view(-1)
    t_h2d = best(lambda: dev.copy_(th, non_blocking=True))
    t_d2h = best(lambda: th.copy_(dev, non_blocking=True))
    t_set = best(lambda: sim.set_particles(host))
    # round trip: a download right after an upload returns the upload, bit for bit
    back = np.zeros_like(host)
    sim._h.call("impm_sim_get_particles", _abi.ptr(back), n, back.strides[0])
    assert np.array_equal(back, prob.particles), "particle round trip differs"
    sim.step(1 / prob.load_steps)
    # after a step (sorted particles): the chunked download equals the one-copy path
    a = np.zeros_like(host)
    sim._h.call("impm_sim_get_particles", _abi.ptr(a), n, a.strides[0])
    print("round trip ok; chunks", os.environ.get("IMPM_IO_CHUNKS", "default"), float(np.abs(a).sum()), flush=True)
    t_get = best(lambda: sim._h.call("impm_sim_get_particles", _abi.ptr(host), n, host.strides[0]))
    print(f"{nbytes / 1e9:.2f} GB: torch H2D {t_h2d * 1e3:.1f} ms, set_particles {t_set * 1e3:.1f} ms; "
          f"torch D2H {t_d2h * 1e3:.1f} ms, get_particles {t_get * 1e3:.1f} ms", flush=True)


if __name__ == "__main__":
    main()
