"""Compares MG smoothing counts on cfg4: python scripts/mg_sweep.py"""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_2507_09435_b200 import workloads
import paper_2507_09435_b200 as impm

prob = workloads.footing3d()
for nu in [int(a) for a in (sys.argv[1:] or ["1", "2", "3"])]:
    opts = prob.options
    opts.mg_smooth = nu
    opts.profile = False
    sim = impm.MpmSim(prob.grid, prob.particles, prob.material, opts)
    sim.fixed[:] = prob.fixed
    sim.gravity = prob.gravity
    sim.step(1 / 20)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    its = kry = 0
    for k in range(2, 5):
        r = sim.step(k / 20)
        its += r.iterations
        kry += r.krylov_iterations
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"nu={nu}: {dt/3*1e3:.1f} ms/step, newton {its}, cg {kry}, {its/dt:.3f} newton/s", flush=True)
    del sim
