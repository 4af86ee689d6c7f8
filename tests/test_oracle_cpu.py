"""Pins the CPU restatement oracle (oracle/impm_oracle.cpp) against fixtures
produced by the unmodified reference core (oracle/_ref, make_golden.py) and
against the reference's committed golden outputs. No GPU needed."""
import os
import sys

import numpy as np
import pytest

import golden_util as gu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "oracle"))

import oracle  # noqa: E402

FAST = ["bar1d_j2", "cant2d_hencky", "cant2d_hencky_newton", "col2d_j2", "col2d_nh", "cube3d_nh_newton",
        "tl2d_hencky", "footing3d_nh", "cube3d_nh"]


def make(name):
    fx = gu.load(name)
    dim, grid, mat, opts, parts, fixed, grav, spec = gu.problem(fx)
    o = oracle.OracleSim(dim, grid["nodes"], grid["origin"], grid["h"], mat["kind"], mat["E"], mat["nu"],
                         mat["kappa"], opts["tol"], opts["max_iterations"], opts["total_lagrangian"])
    o.set_particles(parts)
    o.set_fixed(fixed)
    o.set_gravity(grav)
    return o, fx, spec


@pytest.mark.parametrize("name", FAST + ["cfg1_nh"])
def test_oracle_integer_stages_bit_exact(name):
    o, fx, _ = make(name)
    o.begin_step()
    dof_of, node_of, field_of, mass = o.dof_map()
    np.testing.assert_array_equal(dof_of, fx["dof_of"])
    np.testing.assert_array_equal(node_of, fx["node_of"])
    np.testing.assert_array_equal(field_of, fx["field_of"])
    rp, cols = o.pattern()
    np.testing.assert_array_equal(rp, fx["row_ptr"])
    np.testing.assert_array_equal(cols, fx["cols"])
    assert gu.rel_err(mass, fx["node_mass"]) <= 1e-14


@pytest.mark.parametrize("name", FAST + ["cfg1_nh"])
def test_oracle_residual(name):
    o, fx, spec = make(name)
    s0 = float(spec.get("probe_scale", 0.5))
    o.begin_step()
    assert gu.rel_err(o.residual(np.zeros(o.n_dofs()), s0), fx["r0"]) <= 1e-13
    assert gu.rel_err(o.residual(fx["u1"], s0), fx["r1"]) <= 1e-13


@pytest.mark.parametrize("name", FAST)
def test_oracle_jacobian_colour_seeded(name):
    o, fx, spec = make(name)
    o.begin_step()
    vals = o.jacobian(fx["u1"], float(spec.get("probe_scale", 0.5)))
    assert gu.csr_row_scaled_err(fx["row_ptr"], vals, fx["J1_vals"]) <= 1e-11


@pytest.mark.parametrize("name", ["col2d_nh", "cube3d_nh_newton", "col2d_j2", "footing3d_nh"])
def test_oracle_linear_solve(name):
    o, fx, spec = make(name)
    o.begin_step()
    x = o.solve(fx["J1_vals"], -fx["r1"])
    assert gu.rel_err(x, fx["delta1"]) <= 1e-9


@pytest.mark.parametrize("name", ["bar1d_j2", "col2d_j2", "cant2d_hencky", "cube3d_nh"])
def test_oracle_commit(name):
    o, fx, _ = make(name)
    o.begin_step()
    o.set_nodal_solution(fx["u1"])
    o.commit_step()
    got, ref = o.particles(), fx["particles_commit1"]
    assert np.abs(got - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("name", ["bar1d_j2", "cant2d_hencky_newton", "tl2d_hencky", "cube3d_nh_newton"])
def test_oracle_newton_trace(name):
    o, fx, spec = make(name)
    steps = int(spec.get("steps", 2))
    its = [o.step(k / steps)[0] for k in range(1, steps + 1)]
    np.testing.assert_array_equal(its, fx["newton_iters"])
    got, ref = o.particles(), fx["particles_final"]
    scale = np.maximum(np.abs(ref).max(axis=0), 1e-300)
    assert (np.abs(got - ref).max(axis=0) / scale)[np.abs(ref).max(axis=0) > 1e-9].max() <= 1e-9


def test_reference_bar_elastic_golden_csv_reproduced():
    """The oracle re-runs configs/bar_elastic.cfg (scenarios.cpp:92-126) and
    matches the reference's committed out/bar_elastic/particles.csv."""
    ref = np.load(os.path.join(gu.GOLDEN, "reference_out.npz"))
    golden = ref["bar_elastic__particles"]
    H, cells, ppc = 50.0, 64, 4
    h = H / cells
    import paper_2507_09435_b200.particles as pp

    grid = pp.GridSpec(1, (-h,), h, (cells + 3,))
    parts = pp.seed_box(grid, (0.0,), (H,), ppc, 80.0)
    o = oracle.OracleSim(1, (cells + 3,), (-h,), h, "hencky", 10e3, 0.0, tol=1e-11)
    o.set_particles(parts)
    fixed = (grid.node_positions()[:, 0] <= 1e-12).astype(np.uint8)
    o.set_fixed(fixed)
    o.set_gravity([-9.81])
    for k in range(1, 41):
        o.step(k / 40)
    p = pp.ParticleArray(o.particles(), 1)
    got = np.stack([p.X[:, 0], p.x[:, 0], p.sigma[:, 0], p.sigma[:, 4], p.F[:, 0], p.V[:, 0]], axis=1)
    err = np.abs(got - golden).max(axis=0) / np.maximum(np.abs(golden).max(axis=0), 1e-300)
    assert err.max() <= 1e-10, err
