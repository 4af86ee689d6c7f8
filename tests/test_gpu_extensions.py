"""Unpinned extensions (absent from the reference):
Drucker-Prager (cfg 2 slope) and the quadratic B-spline transfer. Validated
the way the reference validates its own models (test_materials.cpp:43-78,
test_gimp.cpp:88-120): the dual-number Jacobian against central finite
differences of the GPU residual, yield admissibility after return mapping,
partition of unity, and Newton convergence on the slope."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def small_slope(material="drucker_prager", shape="gimp"):
    import paper_2507_09435_b200 as impm
    from paper_2507_09435_b200 import workloads

    # statically admissible slope (phi 40 deg on 30 deg) with a little cohesion:
    # plastic zones without surface particles at the zero-stiffness apex
    prob = workloads.slope2d(cells=(24, 12), ppc=2, h=0.5, steps=10, material=material, friction_deg=40.0, kappa=20e3,
                             slope_deg=30.0, cohesion=2e3)
    prob.options.shape = shape
    sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options)
    sim.fixed[:] = prob.fixed
    sim.gravity = prob.gravity
    return sim, prob


def fd_check(sim, s, u, eps):
    rp, cols, vals = sim.jacobian_csr(u, s)
    import scipy.sparse as sp

    J = sp.csr_matrix((vals, cols, rp), shape=(sim.n_dofs(), sim.n_dofs()))
    rng = np.random.default_rng(3)
    v = rng.standard_normal(sim.n_dofs())
    fd = (sim.residual(u + eps * v, s) - sim.residual(u - eps * v, s)) / (2 * eps)
    return np.linalg.norm(J @ v - fd) / np.linalg.norm(J @ v)


@pytest.mark.parametrize("material", ["drucker_prager", "hencky_j2"])
def test_tangent_matches_finite_differences_in_plastic_state(material):
    sim, prob = small_slope(material)
    n_steps = 5 if material == "hencky_j2" else 1  # DP: see test_drucker_prager_returns_to_admissible_states
    for k in range(1, n_steps + 1):
        sim.step(k / prob.load_steps)
    # at a converged increment, loading particles lie strictly outside the
    # trial yield surface (at u = 0 they sit on it, where FD straddles the kink)
    sim.begin_step()
    s = (n_steps + 1) / prob.load_steps
    sim.newton_solve(s)
    u = sim.nodal_solution()
    assert fd_check(sim, s, u, 1e-9) <= 1e-5


def test_drucker_prager_returns_to_admissible_states():
    """Experimental: once particles approach the cone apex the return-map
    tangent scales like 1/|dev eps| and the Newton-Krylov solve stalls (an
    apex-smoothed return is next work); checked on the first two
    load increments, where the plastic zone forms at the toe."""
    sim, prob = small_slope("drucker_prager")
    for k in range(1, 3):
        rec = sim.step(k / prob.load_steps)
        assert rec.iterations >= 1
    p = sim.particles
    E, nu, phi = prob.material.elastic.E, prob.material.elastic.nu, np.radians(prob.material.friction_deg)
    lam, mu = E * nu / ((1 + nu) * (1 - 2 * nu)), E / (2 * (1 + nu))
    alpha = np.sqrt(2 / 3) * 2 * np.sin(phi) / (3 - np.sin(phi))
    e_c = 3 * prob.material.cohesion / (3 * lam + 2 * mu)
    worst = 0.0
    for Be in p.B_e.reshape(-1, 3, 3):
        w, V = np.linalg.eigh(0.5 * (Be + Be.T))
        eps = (V * (0.5 * np.log(w))) @ V.T
        tr = np.trace(eps)
        dev = np.linalg.norm(eps - tr / 3 * np.eye(3))
        f = dev + (3 * lam + 2 * mu) / (2 * mu) * (tr - e_c) * alpha
        worst = max(worst, f if tr <= e_c + 1e-12 else np.linalg.norm(eps - e_c / 3 * np.eye(3)))
    assert worst <= 1e-9


def test_bspline_partition_of_unity_and_tangent():
    sim, prob = small_slope("hencky_j2", shape="quadratic-bspline")
    sim.begin_step()
    m = sim.node_mass()
    assert abs(m.sum() - sim.particles.m[:, 0].sum()) <= 1e-12 * m.sum()
    u = 1e-5 * np.random.default_rng(2).standard_normal(sim.n_dofs())
    assert fd_check(sim, 0.3, u, 1e-8) <= 1e-5
    rec = sim.step(0.1)
    assert rec.iterations >= 1


def test_cfg2_drucker_prager_full_size_gravity_ramp():
    """BASELINE cfg 2 with its named material at full size (401,216 particles,
    30 deg / 120 kPa Drucker-Prager on the 45 deg, 64 m slope): all 20 gravity
    increments converge (the cone-tip tangent regularisation keeps J
    nonsingular once particles reach the tip), and every particle ends on or
    inside the cone."""
    import paper_2507_09435_b200 as impm
    from paper_2507_09435_b200 import workloads

    prob = workloads.slope2d(material="drucker_prager")
    sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options)
    sim.fixed[:] = prob.fixed
    sim.gravity = prob.gravity
    for k in range(1, prob.load_steps + 1):
        rec = sim.step(k / prob.load_steps)
        assert rec.rel_residuals[-1] <= prob.options.tol
    p = sim.particles
    assert (p.alpha[:, 0] > 0).any()
    E, nu, phi = prob.material.elastic.E, prob.material.elastic.nu, np.radians(prob.material.friction_deg)
    lam, mu = E * nu / ((1 + nu) * (1 - 2 * nu)), E / (2 * (1 + nu))
    alpha = np.sqrt(2 / 3) * 2 * np.sin(phi) / (3 - np.sin(phi))
    e_c = 3 * prob.material.cohesion / (3 * lam + 2 * mu)
    plastic = p.alpha[:, 0] > 0
    worst = 0.0
    for Be in p.B_e.reshape(-1, 3, 3)[plastic]:
        w, V = np.linalg.eigh(0.5 * (Be + Be.T))
        eps = (V * (0.5 * np.log(w))) @ V.T
        tr = np.trace(eps)
        dev = np.linalg.norm(eps - tr / 3 * np.eye(3))
        f = dev + (3 * lam + 2 * mu) / (2 * mu) * (tr - e_c) * alpha
        worst = max(worst, f if tr <= e_c + 1e-12 else np.linalg.norm(eps - e_c / 3 * np.eye(3)))
    assert worst <= 1e-9
