"""Multi-rank (world_size 2, gloo, CPU) validation of the slab decomposition
(paper_2507_09435_b200/slabs.py) with the CPU oracle as the
per-rank compute. It checks that:

  * per-slab node activity + the allgathered owned free-DOF counts give the
    reference's global DofMap bit for bit (grid.hpp:69-86);
  * owned residual rows computed from owned + ghost particles equal the
    reference's global residual (mpm_solver.hpp:156-211);
  * a distributed Jacobi-PCG with the 2-layer halo exchange before every SpMV
    and allreduced dots reproduces the reference's linear solve.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import golden_util as gu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "oracle"))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allgather_obj(obj):
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def _worker(rank, world, port, case, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        _run(rank, world, case)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # report to the parent
        import traceback

        errq.put(f"rank {rank}: {e}\n{traceback.format_exc()}")
        raise


def _run(rank, world, case):
    import oracle
    from paper_2507_09435_b200 import slabs
    from paper_2507_09435_b200.particles import GridSpec

    fx = gu.load(case)
    dim, grid, mat, opts, parts, fixed, grav, spec = gu.problem(fx)
    G = GridSpec(dim, grid["origin"], grid["h"], grid["nodes"])
    D = dim
    slab = slabs.make_slab(G, parts, rank, world)
    lg = slab.grid
    gnode = slabs.local_node_map(G, slab).reshape(-1)
    own = slabs.owned_node_mask(slab, G)

    # local problem: owned + ghost particles, sliced fixed mask
    o = oracle.OracleSim(dim, lg.nodes, lg.origin, lg.h, mat["kind"], mat["E"], mat["nu"], mat["kappa"],
                         opts["tol"], opts["max_iterations"], opts["total_lagrangian"])
    o.set_particles(parts[slab.particle_ids])
    fixed_g = fixed.reshape(-1, D)
    o.set_fixed(np.ascontiguousarray(fixed_g[gnode].reshape(-1)))
    o.set_gravity(grav)
    o.begin_step()
    ldof_of, lnode_of, lfield_of, _ = o.dof_map()

    # --- global DOF numbering: owned counts -> allgather -> exclusive scan
    ld = ldof_of.reshape(-1, D)
    owned_ldofs = np.sort(ld[own][ld[own] >= 0])
    counts = _allgather_obj(int(owned_ldofs.size))
    offset = int(slabs.global_dof_offsets(counts)[rank])
    gdof_local = -np.ones_like(ld)
    gdof_local[own] = np.where(ld[own] >= 0, 0, -1)
    rank_in_owned = {int(d): i for i, d in enumerate(owned_ldofs)}
    for n in np.nonzero(own)[0]:
        for f in range(D):
            if ld[n, f] >= 0:
                gdof_local[n, f] = offset + rank_in_owned[int(ld[n, f])]
    ref_dof = fx["dof_of"].reshape(-1, D)
    assert np.array_equal(gdof_local[own], ref_dof[gnode[own]]), "distributed DofMap != reference"
    # Halo nodes see only the kept particles, so their local mass is partial:
    # activity and DOF ids of halo nodes come from their owners (halo
    # exchange of ints once per load step). Invariants that make this exact:
    # a locally active halo DOF is globally active, and a globally active
    # halo node that is locally inactive has zero local mass (no kept
    # particle touches it, so it cannot influence an owned row).
    halo = ~own
    loc_act, glob_act = ld[halo] >= 0, ref_dof[gnode[halo]] >= 0
    assert not np.any(loc_act & ~glob_act), "locally active halo DOF that is globally inactive"
    _, _, _, lmass = o.dof_map()
    missing_nodes = np.nonzero(halo)[0][np.any(glob_act & ~loc_act, axis=1)]
    assert np.all(lmass[missing_nodes] == 0.0), "partial-mass halo node dropped by the local cutoff"
    gdof_local[halo] = np.where(loc_act, ref_dof[gnode[halo]], -1)

    # --- residual: owned rows from owned + ghost particles
    u_local = np.zeros(o.n_dofs())
    for n in range(len(gnode)):
        for f in range(D):
            if ld[n, f] >= 0:
                u_local[ld[n, f]] = fx["u1"][gdof_local[n, f]]
    s0 = float(spec.get("probe_scale", 0.5))
    r_local = o.residual(u_local, s0)
    mine = {int(gdof_local[n, f]): float(r_local[ld[n, f]]) for n in np.nonzero(own)[0] for f in range(D)
            if ld[n, f] >= 0}
    merged = {}
    for part in _allgather_obj(mine):
        merged.update(part)
    r = np.array([merged[i] for i in range(len(fx["r1"]))])
    assert gu.rel_err(r, fx["r1"]) <= 1e-12

    # --- distributed Jacobi-PCG on owned rows with a halo exchange per SpMV
    vals = o.jacobian(u_local, s0)
    rp, cols = o.pattern()
    loc2g = np.full(o.n_dofs(), -1)
    for n in range(len(gnode)):
        for f in range(D):
            if ld[n, f] >= 0:
                loc2g[ld[n, f]] = gdof_local[n, f]
    rows = [int(ld[n, f]) for n in np.nonzero(own)[0] for f in range(D) if ld[n, f] >= 0]
    g_rows = loc2g[rows]
    A = {}
    for lr, gr in zip(rows, g_rows):
        A[int(gr)] = (loc2g[cols[rp[lr]:rp[lr + 1]]], vals[rp[lr]:rp[lr + 1]])
    owned_g = np.array(sorted(A))
    diag = np.array([A[g][1][A[g][0] == g][0] for g in owned_g])
    b = -np.array([merged[int(g)] for g in owned_g])

    # halo plan: which of my owned DOFs each neighbour needs (its halo columns)
    need = sorted({int(c) for g in owned_g for c in A[g][0]} - set(owned_g.tolist()))
    requests = _allgather_obj(need)

    def exchange(xo):
        xmap = dict(zip(owned_g.tolist(), xo.tolist()))
        send = {r2: {c: xmap[c] for c in requests[r2] if c in xmap} for r2 in range(world) if r2 != rank}
        got = _allgather_obj(send)
        full = dict(xmap)
        for r2, msg in enumerate(got):
            if r2 != rank:
                full.update(msg.get(rank, {}))
        return full

    def spmv(xo):
        full = exchange(xo)
        return np.array([np.dot(A[g][1], [full[int(c)] for c in A[g][0]]) for g in owned_g])

    def dot(a, c):
        t = torch.tensor([float(np.dot(a, c))], dtype=torch.float64)
        dist.all_reduce(t)
        return float(t.item())

    x = np.zeros_like(b)
    rr = b.copy()
    z = rr / diag
    p = z.copy()
    rz = dot(rr, z)
    bb = dot(b, b)
    for _ in range(5000):
        q = spmv(p)
        alpha = rz / dot(p, q)
        x += alpha * p
        rr -= alpha * q
        if dot(rr, rr) <= 1e-24 * bb:
            break
        z = rr / diag
        rz_new = dot(rr, z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    sol = {}
    for part in _allgather_obj(dict(zip(owned_g.tolist(), x.tolist()))):
        sol.update(part)
    delta = np.array([sol[i] for i in range(len(fx["delta1"]))])
    assert gu.rel_err(delta, fx["delta1"]) <= 1e-8


@pytest.mark.parametrize("case", ["cube3d_nh_newton", "footing3d_nh", "col2d_j2"])
def test_two_slab_decomposition_matches_single_process(case):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert all(p.exitcode == 0 for p in procs), "\n".join(errs)


# ---------------------------------------------------------------- GPU-slab host logic
def test_seed_box_rows_and_slab_seeding_match_global_seed_box():
    """seed_box_rows / seed_box_slab generate exactly the rows (and global ids)
    of seed_box that each rank holds, without the global array."""
    from paper_2507_09435_b200 import distributed as dd
    from paper_2507_09435_b200.particles import GridSpec, seed_box, seed_box_rows

    for D, nodes, hi in [(1, (19,), (16.0,)), (2, (19, 7), (16.0, 4.0)), (3, (11, 11, 7), (8.0, 8.0, 4.0))]:
        g = GridSpec(D, tuple([-1.0] * D), 1.0, nodes)
        full = seed_box(g, (0.0,) * D, hi, 2, 2000.0)
        p, ids = seed_box_rows(g, (0.0,) * D, hi, 2, 2000.0, np.arange(int(round(hi[0])) * 2))
        assert np.array_equal(p, full) and np.array_equal(ids, np.arange(len(full)))
        cuts = dd.slab_cuts(g, 2, full)
        held = []
        for r in range(2):
            ps, ids = dd.seed_box_slab(g, (0.0,) * D, hi, 2, 2000.0, cuts, r)
            assert np.array_equal(ids, dd.slab_member_ids(g, full, cuts, r))
            assert np.array_equal(ps, full[ids])
            held.append(ids)
        from paper_2507_09435_b200 import slabs

        first = slabs.support_first(g, full)
        owned = np.concatenate([np.nonzero(dd.owned_mask(first, cuts, r))[0] for r in range(2)])
        assert np.array_equal(np.sort(owned), np.arange(len(full)))  # every particle owned once


def test_slab_cuts_respect_minimum_width_and_balance():
    from paper_2507_09435_b200 import distributed as dd
    from paper_2507_09435_b200.errors import ConfigError
    from paper_2507_09435_b200.particles import GridSpec, seed_box

    g = GridSpec(3, (-0.5, -0.5, -0.5), 0.5, (67, 11, 7))
    parts = seed_box(g, (0.0, 0.0, 0.0), (32.0, 4.0, 2.0), 2, 2000.0)
    for nr in (1, 2, 3, 4, 8):
        cuts = dd.slab_cuts(g, nr, parts)
        assert cuts[0] == 0 and cuts[-1] == 67 and len(cuts) == nr + 1
        if nr > 1:
            assert min(np.diff(cuts)) >= dd.MIN_PLANES
    with pytest.raises(ConfigError):
        dd.slab_cuts(GridSpec(2, (-1.0, -1.0), 1.0, (7, 7)), 2)
