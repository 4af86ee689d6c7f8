"""Krylov iterations of the slab decomposition (ranks as in-process threads on
one GPU) against the single-GPU solve of the same cfg 5 mini problem: the
MG preconditioner is rank-local, so the CG count can grow with the rank count.
GPU only:  python scripts/slab_kry_probe.py [nranks] [cx cy cz per rank] [steps]"""
import sys

sys.path.insert(0, ".")
import paper_2507_09435_b200 as impm  # noqa: E402
from paper_2507_09435_b200 import workloads  # noqa: E402
from paper_2507_09435_b200.distributed import SlabSim, run_local_ranks  # noqa: E402

nr = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cells = tuple(int(v) for v in sys.argv[2:5]) if len(sys.argv) > 4 else (16, 16, 8)
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
whole = workloads.footing3d(cells=(cells[0] * nr, cells[1], cells[2]), steps=10)
o = whole.options
o.krylov = "iterative"
single = impm.MpmSim(whole.grid, whole.particles, whole.material, o)
single.fixed[:] = whole.fixed
single.gravity = whole.gravity
ref = [single.step(k / 10) for k in range(1, steps + 1)]
print("single", [r.iterations for r in ref], "krylov", [r.krylov_iterations for r in ref], flush=True)


def body(rank, comm):
    p = workloads.footing3d_slab(nr, rank, cells=cells, steps=10)
    po = p.options
    po.krylov = "iterative"
    sim = SlabSim(p.grid, comm, p.meta["cuts"], p.particles, p.meta["ids"], p.material, po)
    sim.set_fixed_global(p.fixed)
    sim.gravity = p.gravity
    recs = [sim.step(k / 10) for k in range(1, steps + 1)]
    return [r.iterations for r in recs], [r.krylov_iterations for r in recs]


res = run_local_ranks(nr, body)
print(f"{nr} ranks", res[0][0], "krylov", res[0][1], flush=True)
tot_s, tot_r = sum(r.krylov_iterations for r in ref), sum(res[0][1])
print(f"krylov ratio slabs/single = {tot_r / max(tot_s, 1):.3f}")
