"""Slab decomposition on the GPU, through the C ABI.

Ranks run as host threads of one process on the one GPU of the box, over the
in-process transport of csrc/impm_comm.cuh (host-ordered collectives: stream
sync + barrier + device copies, no kernel waits on another rank); the NCCL
transport drives the same code path and is exercised at nranks = 1.

Checks, against the reference fixtures and the single-GPU path:
  * the distributed DofMap (local owned numbering + allgathered offsets) is the
    reference's global DofMap bit for bit (grid.hpp:69-86);
  * owned residual rows and J x rows (halo columns from the neighbours) are
    BITWISE those of the single-GPU run: same particle order per bin, same
    colour-batch order, weights relative to the global origin;
  * full load steps: per-step Newton counts equal the reference's on every rank
    and the gathered owned particles match the final state to 1e-7, with
    particles migrating across slab boundaries (bar1d_j2 moves ~9 cells).
"""
import numpy as np
import pytest

import golden_util as gu

pytestmark = pytest.mark.gpu

STATE_TOL = 1e-7


def _setup(name):
    import paper_2507_09435_b200 as impm

    fx = gu.load(name)
    dim, grid, mat, opts, parts, fixed, grav, spec = gu.problem(fx)
    g = impm.GridSpec(dim, grid["origin"], grid["h"], grid["nodes"])
    m = impm.MaterialSpec(mat["kind"], impm.ElasticParams(mat["E"], mat["nu"]), mat["kappa"])
    o = impm.SolverOptions(tol=opts["tol"], max_iterations=opts["max_iterations"],
                           total_lagrangian=opts["total_lagrangian"])
    return impm, fx, g, m, o, parts, fixed, grav, spec


def _slab(comm, cuts, g, m, o, parts, fixed, grav):
    from paper_2507_09435_b200.distributed import SlabSim

    sim = SlabSim.from_global(g, comm, cuts, parts, m, o)
    sim.set_fixed_global(fixed)
    sim.gravity = grav
    return sim


def _cuts(g, parts, nranks, o):
    from paper_2507_09435_b200.distributed import slab_cuts

    return slab_cuts(g, nranks, parts, bool(o.total_lagrangian))


STAGE_CASES = [("cube3d_nh_newton", 2), ("footing3d_nh", 2), ("cant2d_hencky", 2), ("cant2d_hencky_newton", 3),
               ("cfg1_nh", 3), ("bar1d_j2", 3)]


@pytest.mark.parametrize("name,nranks", STAGE_CASES)
def test_slab_dofmap_residual_and_jacobian_rows_bitwise(name, nranks):
    from paper_2507_09435_b200.distributed import run_local_ranks

    impm, fx, g, m, o, parts, fixed, grav, spec = _setup(name)
    D = g.dim
    s0 = float(spec.get("probe_scale", 0.5))
    single = impm.MpmSim(g, parts, m, o)
    single.fixed[:] = fixed
    single.gravity = grav
    single.begin_step()
    r_single = single.residual(fx["u1"], s0)
    dof_glob = fx["dof_of"].reshape(-1, D)
    rng = np.random.default_rng(7)
    x_glob = np.where(dof_glob >= 0, rng.standard_normal(dof_glob.shape), 0.0).reshape(-1)
    y_single = single.apply_jacobian(fx["u1"], s0, x_glob).reshape(-1, D)
    cuts = _cuts(g, parts, nranks, o)

    def body(rank, comm):
        sim = _slab(comm, cuts, g, m, o, parts, fixed, grav)
        sim.begin_step()
        nodes, gd = sim.global_dofs()
        info = sim.slab_info()
        dm = sim.dofs()
        ld = dm.dof_of.reshape(-1, D)
        own = sim.owned_node_mask()
        u_loc = np.zeros(dm.n_dofs)
        sel = ld[own] >= 0
        u_loc[ld[own][sel]] = fx["u1"][gd[sel]]
        r_loc = sim.residual(u_loc, s0)
        r_rows = {int(gi): float(r_loc[li]) for gi, li in zip(gd[sel], ld[own][sel])}
        gnode = sim.global_node_ids()
        y = sim.apply_jacobian(u_loc, s0, x_glob.reshape(-1, D)[gnode].reshape(-1)).reshape(-1, D)
        return nodes, gd, info, r_rows, y[own]

    res = run_local_ranks(nranks, body)
    all_nodes = np.concatenate([r[0] for r in res])
    np.testing.assert_array_equal(np.sort(all_nodes), np.arange(dof_glob.shape[0]))  # each node owned once
    for nodes, gd, info, _, _ in res:
        np.testing.assert_array_equal(gd, dof_glob[nodes])  # global DofMap, bit for bit
        assert info["n_dofs_global"] == len(fx["node_of"])
    r = np.zeros(len(fx["node_of"]))
    seen = np.zeros(len(r), dtype=bool)
    for _, _, _, rows, _ in res:
        for k, v in rows.items():
            r[k] = v
            seen[k] = True
    assert seen.all()
    np.testing.assert_array_equal(r, r_single)  # bitwise the single-GPU residual
    assert gu.rel_err(r, fx["r1"]) <= 1e-9
    for nodes, gd, _, _, y_own in res:
        np.testing.assert_array_equal(y_own, y_single[nodes])  # J rows incl. halo columns, bitwise


NEWTON_CASES = [("cube3d_nh_newton", 2), ("footing3d_nh", 2), ("cant2d_hencky_newton", 3), ("cfg1_nh", 4),
                ("bar1d_j2", 2), ("bar1d_j2", 3), ("tl2d_hencky", 2)]


def _assert_state_close(got, ref, D, h, tol=STATE_TOL):
    from paper_2507_09435_b200 import particle_fields

    for fname, off, w in particle_fields(D):
        gv, rv = got[:, off:off + w], ref[:, off:off + w]
        scale = max(np.abs(rv).max(initial=0.0), 1e-300)
        if fname in ("X", "x"):
            scale = max(scale, h)
        err = float(np.abs(gv - rv).max(initial=0.0)) / scale
        assert err <= tol, (fname, err)


@pytest.mark.parametrize("name,nranks", NEWTON_CASES)
def test_slab_newton_steps_match_reference(name, nranks):
    from paper_2507_09435_b200.distributed import gather_owned, run_local_ranks, slab_member_ids

    impm, fx, g, m, o, parts, fixed, grav, spec = _setup(name)
    steps = int(spec.get("steps", 2))
    cuts = _cuts(g, parts, nranks, o)

    def body(rank, comm):
        sim = _slab(comm, cuts, g, m, o, parts, fixed, grav)
        iters, held = [], []
        for k in range(1, steps + 1):
            rec = sim.step(k / steps)
            iters.append(rec.iterations)
        pa, ids = sim.local_particles()
        return iters, sim.owned_particles(), (pa.data, ids)

    res = run_local_ranks(nranks, body)
    iters = [np.array(r[0]) for r in res]
    for it in iters[1:]:
        np.testing.assert_array_equal(it, iters[0])  # every rank took the same Newton path
    ref_iters = fx["newton_iters"]
    # identical counts on every case, J2 included (exact-equivalent solves on
    # return-map materials, see test_gpu_parity.test_newton_counts_and_final_state)
    np.testing.assert_array_equal(iters[0], ref_iters)
    owned, ids = gather_owned([r[1] for r in res], g.dim)
    np.testing.assert_array_equal(ids, np.arange(len(parts)))  # every particle owned exactly once
    _assert_state_close(owned.data, fx["particles_final"], g.dim, g.h)
    # after the last migration each rank holds exactly its owned + ghost set
    for rank, r in enumerate(res):
        data, held = r[2]
        want = slab_member_ids(g, owned.data, cuts, rank, bool(o.total_lagrangian))
        np.testing.assert_array_equal(np.sort(held), want)


def test_slab_migration_crosses_boundaries():
    """bar1d_j2 particles travel ~9 cells along axis 0: the owned sets must
    change between the first and the last step."""
    from paper_2507_09435_b200.distributed import run_local_ranks

    impm, fx, g, m, o, parts, fixed, grav, spec = _setup("bar1d_j2")
    cuts = _cuts(g, parts, 2, o)

    def body(rank, comm):
        sim = _slab(comm, cuts, g, m, o, parts, fixed, grav)
        first = set(sim.owned_particles()[1].tolist())
        for k in range(1, 21):
            sim.step(k / 20)
        return first, set(sim.owned_particles()[1].tolist())

    res = run_local_ranks(2, body)
    moved = sum(len(a ^ b) for a, b in res)
    assert moved > 0


def test_nccl_transport_single_rank():
    """The NCCL transport (one process per GPU) at nranks = 1: communicator
    creation and a full slab run through the same entry points."""
    from paper_2507_09435_b200.distributed import Communicator, SlabSim

    impm, fx, g, m, o, parts, fixed, grav, spec = _setup("cube3d_nh_newton")
    comm = Communicator.nccl(0, 1, 0)
    assert comm.kind == "nccl" and comm.nranks == 1
    sim = SlabSim.from_global(g, comm, [0, g.nodes[0]], parts, m, o)
    sim.set_fixed_global(fixed)
    sim.gravity = grav
    steps = int(spec.get("steps", 2))
    iters = [sim.step(k / steps).iterations for k in range(1, steps + 1)]
    np.testing.assert_array_equal(iters, fx["newton_iters"])
    pa, ids = sim.local_particles()
    order = np.argsort(ids)
    _assert_state_close(pa.data[order], fx["particles_final"], g.dim, g.h)


def test_slab_rejects_bad_geometry():
    from paper_2507_09435_b200.distributed import Communicator, SlabSim
    from paper_2507_09435_b200.errors import ConfigError

    impm, fx, g, m, o, parts, fixed, grav, spec = _setup("cube3d_nh_newton")
    comms = Communicator.local_group(3)
    with pytest.raises(ConfigError):  # 8 planes cannot give 3 slabs of >= 4
        SlabSim.from_global(g, comms[0], [0, 3, 5, 8], parts, m, o)


def test_cfg5_slab_workload_matches_single_gpu():
    """The bench's multi-GPU workload (workloads.footing3d_slab: cfg 4 per GPU
    stacked along axis 0, generated per rank) on 2 in-process ranks vs the same
    problem on one GPU: identical Newton counts, particle state within 1e-7."""
    from paper_2507_09435_b200 import workloads
    from paper_2507_09435_b200.distributed import SlabSim, gather_owned, run_local_ranks
    import paper_2507_09435_b200 as impm

    cells = (12, 8, 6)
    whole = workloads.footing3d(cells=(24, 8, 6), steps=3)
    single = impm.MpmSim(whole.grid, whole.particles, whole.material, whole.options)
    single.fixed[:] = whole.fixed
    single.gravity = whole.gravity
    ref_iters = [single.step(k / 3).iterations for k in range(1, 4)]
    ref = single.particles.data

    def body(rank, comm):
        p = workloads.footing3d_slab(2, rank, cells=cells, steps=3)
        assert np.array_equal(p.particles, whole.particles[p.meta["ids"]])
        sim = SlabSim(p.grid, comm, p.meta["cuts"], p.particles, p.meta["ids"], p.material, p.options)
        sim.set_fixed_global(p.fixed)
        sim.gravity = p.gravity
        its = [sim.step(k / 3).iterations for k in range(1, 4)]
        return its, sim.owned_particles()

    res = run_local_ranks(2, body)
    assert res[0][0] == ref_iters and res[1][0] == ref_iters
    owned, ids = gather_owned([r[1] for r in res], 3)
    np.testing.assert_array_equal(ids, np.arange(len(ref)))
    _assert_state_close(owned.data, ref, 3, whole.grid.h)
