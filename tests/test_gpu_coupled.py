"""GPU parity of the coupled u-p path (CoupledSim, porous.hpp:48-186,
src/porous.cpp:25-168) against the reference-generated `upcol` fixture
(10-cell consolidation column, scenarios.cpp:387-418)."""
import numpy as np
import pytest

import golden_util as gu

pytestmark = pytest.mark.gpu


def make():
    import paper_2507_09435_b200 as impm

    fx = gu.load("upcol")
    g = fx["grid"]
    grid = impm.GridSpec(2, tuple(g[0:2]), float(g[3]), (int(g[4]), int(g[5])))
    lam, mu, k, mu_f, rho_f, tol = fx["poro"]
    sim = impm.CoupledSim(grid, fx["particles0"], impm.PoroParams(lam, mu, k, mu_f, rho_f),
                          impm.SolverOptions(tol=tol))
    sim.fixed_u[:] = fx["fixed_u"]
    sim.fixed_p[:] = fx["fixed_p"]
    sim.gravity = fx["gravity"]
    return sim, fx


def test_coupled_dofs_pattern_bit_exact():
    sim, fx = make()
    sim.initialize()
    np.testing.assert_array_equal(sim.dofs().dof_of, fx["dof_of"])
    rp, cols, _ = sim.jacobian_csr(np.zeros(sim.n_dofs()), 100.0)
    np.testing.assert_array_equal(rp, fx["row_ptr"])
    np.testing.assert_array_equal(cols, fx["cols"])


def test_coupled_residual_and_jacobian():
    sim, fx = make()
    sim.initialize()
    r = sim.residual(fx["x1"], 100.0)
    assert gu.rel_err(r, fx["r1"]) <= 1e-9
    rp, cols, vals = sim.jacobian_csr(fx["x1"], 100.0)
    assert gu.csr_row_scaled_err(rp, vals, fx["J1_vals"]) <= 1e-9


def test_coupled_steps_counts_settlement_pressure():
    sim, fx = make()
    its, settle = [], []
    for _ in range(len(fx["newton_iters"])):
        rec = sim.step(100.0)
        its.append(rec.iterations)
        settle.append(sim.top_settlement())
    np.testing.assert_array_equal(its, fx["newton_iters"])
    assert gu.rel_err(settle, fx["settlement"]) <= 1e-7
    assert gu.rel_err(sim.nodal_pressure(), fx["p_nodes"]) <= 1e-7
    got, ref = sim.particles.data, fx["particles_final"]
    scale = np.maximum(np.abs(ref).max(axis=0), 1e-300)
    err = np.abs(got - ref).max(axis=0) / scale
    assert err[np.abs(ref).max(axis=0) > 1e-12].max() <= 1e-7


def test_cfg3_terzaghi_full_size_matches_series_solution():
    """BASELINE cfg 3 at full size: 2D Terzaghi consolidation, 512x512 cells,
    1,048,576 particles, coupled u-p (3x3 blocks, ~790k DOFs). Size-independent
    check: the pressure profile against the series solution (porous.cpp:8-15)
    within the reference's own acceptance bound (L2 <= 0.02,
    src/scenarios.cpp consolidation.terzaghi_L2_Tv_*), drained-top
    dissipation monotone, and the Newton count the reference needs on the
    column (2 per step)."""
    from paper_2507_09435_b200 import workloads
    from paper_2507_09435_b200.scenarios import terzaghi_pressure_ratio

    sim, prm = workloads.terzaghi2d(cells=(512, 512))
    assert prm["particles"] == 1_048_576
    H, cv, t_hat = prm["height"], prm["c_v"], prm["t_hat"]
    Tv = 0.05
    n = 10
    dt = Tv * H * H / cv / n
    pmax_prev = np.inf
    for _ in range(n):
        rec = sim.step(dt)
        assert rec.iterations <= 3
        prof = sim.pressure_profile(256, H)
        pmax = max(p for _, p in prof)
        assert pmax <= pmax_prev * (1 + 1e-9)
        pmax_prev = pmax
    num = den = 0.0
    for depth, p in prof:
        pa = t_hat * terzaghi_pressure_ratio(depth / H, Tv)
        num += (p - pa) ** 2
        den += pa * pa
    assert np.sqrt(num / den) <= 0.02


def test_3d_up_terzaghi_column_matches_series_solution():
    """3D u-p (4x4 node blocks; extension, parity unpinned): a 3D column with
    rollers on the four lateral faces consolidates like the 1D series solution
    (the reference's acceptance bound L2 <= 0.02), and the 2-Newton-iteration
    behaviour of the 2D column is kept."""
    from paper_2507_09435_b200 import workloads
    from paper_2507_09435_b200.scenarios import terzaghi_pressure_ratio

    sim, prm = workloads.terzaghi3d(cells=(4, 4, 64))
    H, cv, t_hat = prm["height"], prm["c_v"], prm["t_hat"]
    Tv, n = 0.05, 10
    dt = Tv * H * H / cv / n
    for _ in range(n):
        rec = sim.step(dt)
        assert rec.iterations <= 3
    prof = sim.pressure_profile((2, 2), H)
    num = den = 0.0
    for depth, p in prof:
        pa = t_hat * terzaghi_pressure_ratio(depth / H, Tv)
        num += (p - pa) ** 2
        den += pa * pa
    assert np.sqrt(num / den) <= 0.02
    assert sim.dofs().n_fields == 4


def test_3d_up_jacobian_matches_finite_differences():
    import scipy.sparse as sp
    from paper_2507_09435_b200 import workloads

    sim, prm = workloads.terzaghi3d(cells=(3, 3, 8))
    dt = 1e4
    sim.step(dt)
    n = sim.n_dofs()
    x = 1e-6 * np.random.default_rng(4).standard_normal(n)
    rp, cols, vals = sim.jacobian_csr(x, dt)
    J = sp.csr_matrix((vals, cols, rp), shape=(n, n))
    v = np.random.default_rng(5).standard_normal(n)
    eps = 1e-7
    fd = (sim.residual(x + eps * v, dt) - sim.residual(x - eps * v, dt)) / (2 * eps)
    assert np.linalg.norm(J @ v - fd) <= 1e-6 * np.linalg.norm(J @ v)
