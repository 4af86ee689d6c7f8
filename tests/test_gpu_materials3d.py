"""3D constitutive extensions on the GPU (parity unpinned: the reference has
Hencky / J2 only for D <= 2, mpm_solver.hpp:448-453, and no Drucker-Prager or
Cam-Clay): the cfg 4 strip footing at reduced size with
modified Cam-Clay (the material BASELINE.json names), 3D J2 and 3D Hencky.

Checked as the reference checks its own models (test_materials.cpp:43-78):
the assembled dual-number Jacobian against central finite differences of the
GPU residual at a converged plastic increment, Newton convergence, yield
admissibility of every particle after commit, and the elastic limit (a 3D
Hencky / Cam-Clay run under a load far inside the yield surface matches the
Hencky run)."""
import numpy as np
import pytest
import scipy.linalg as sla

pytestmark = pytest.mark.gpu


def footing(material, cells=(16, 16, 8), steps=10, t_hat=100e3, **mat_over):
    import paper_2507_09435_b200 as impm
    from paper_2507_09435_b200 import workloads

    prob = workloads.footing3d(cells=cells, ppc=2, h=0.5, steps=steps, t_hat=t_hat, material=material)
    for k, v in mat_over.items():
        setattr(prob.material, k, v)
    sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options)
    sim.fixed[:] = prob.fixed
    sim.gravity = prob.gravity
    return sim, prob


def fd_check(sim, s, u, eps):
    import scipy.sparse as sp

    rp, cols, vals = sim.jacobian_csr(u, s)
    J = sp.csr_matrix((vals, cols, rp), shape=(sim.n_dofs(), sim.n_dofs()))
    v = np.random.default_rng(3).standard_normal(sim.n_dofs())
    fd = (sim.residual(u + eps * v, s) - sim.residual(u - eps * v, s)) / (2 * eps)
    return np.linalg.norm(J @ v - fd) / np.linalg.norm(J @ v), J


def test_cam_clay_footing_converges_and_is_admissible():
    sim, prob = footing("cam_clay", t_hat=400e3, pc0=40e3)
    its = []
    for k in range(1, 5):
        rec = sim.step(k / prob.load_steps)
        its.append(rec.iterations)
        assert rec.rel_residuals[-1] <= prob.options.tol or rec.iterations == 0
    assert max(its) <= 12, its
    p = sim.particles
    m = prob.material
    E, nu = m.elastic.E, m.elastic.nu
    lam, mu = E * nu / ((1 + nu) * (1 - 2 * nu)), E / (2 * (1 + nu))
    K = lam + 2 * mu / 3
    sphi = np.sin(np.radians(m.friction_deg))
    M = 6 * sphi / (3 - sphi)
    alpha = p.alpha[:, 0]
    assert (alpha != 0).any(), "the load must drive part of the clay plastic"
    worst, worst_el = 0.0, 0.0
    for Be, a in zip(p.B_e.reshape(-1, 3, 3), alpha):
        eps = 0.5 * sla.logm(0.5 * (Be + Be.T)).real
        P = -K * np.trace(eps)
        q = np.sqrt(6) * mu * np.linalg.norm(eps - np.trace(eps) / 3 * np.eye(3))
        pc = m.pc0 * np.exp(m.hardening * a)
        f = (q * q / M ** 2 + (P + m.cohesion) * (P - pc)) / (pc * pc)
        worst = max(worst, f)
    assert worst <= 1e-9, worst


def test_cam_clay_tangent_matches_fd_in_plastic_state():
    sim, prob = footing("cam_clay", t_hat=400e3, pc0=40e3)
    for k in range(1, 3):
        sim.step(k / prob.load_steps)
    sim.begin_step()
    s = 3 / prob.load_steps
    sim.newton_solve(s)
    u = sim.nodal_solution()
    err, J = fd_check(sim, s, u, 1e-9)
    assert err <= 1e-5, err
    # nonsymmetric: assembled in full (no mirrored blocks)
    asym = abs(J - J.T).max() / abs(J).max()
    assert asym > 1e-8


@pytest.mark.parametrize("material", ["hencky_j2", "hencky"])
def test_3d_hencky_family_tangent_and_convergence(material):
    sim, prob = footing(material, kappa=4e4)
    for k in range(1, 4):
        rec = sim.step(k / prob.load_steps)
        assert rec.iterations <= 8
    sim.begin_step()
    s = 4 / prob.load_steps
    sim.newton_solve(s)
    u = sim.nodal_solution()
    err, J = fd_check(sim, s, u, 1e-9)
    assert err <= 1e-5, err
    # associative J2 / hyperelastic Hencky: J symmetric (mirrored assembly)
    assert abs(J - J.T).max() <= 1e-10 * abs(J).max()


def test_cam_clay_elastic_limit_matches_hencky():
    """Far inside the yield surface (huge p_c, tiny load) Cam-Clay is the Hencky
    model with the same K, G: identical Newton counts and states to 1e-9."""
    a, prob = footing("cam_clay", t_hat=1e3, pc0=1e12, cohesion=1e11)
    b, _ = footing("hencky", t_hat=1e3)
    for k in range(1, 3):
        ra, rb = a.step(0.05 * k), b.step(0.05 * k)
        assert ra.iterations == rb.iterations
    pa, pb = a.particles, b.particles
    assert (pa.alpha == 0).all()
    for f in ("x", "sigma"):
        x, y = getattr(pa, f), getattr(pb, f)
        assert np.abs(x - y).max() <= 1e-9 * np.abs(y).max()


@pytest.mark.parametrize("material", ["hencky", "cam_clay", "neo_hookean"])
@pytest.mark.parametrize("ppc", [2, 3])
def test_3d_assembly_resident_and_restaged_bins(ppc, material):
    """The staged assembly keeps a bin of <= 8 particles resident across its
    task rounds (ppc 2: 8 per cell) and restages larger bins per round and
    chunk (ppc 3: 27 per cell, 4 chunks). Both paths must give the FD Jacobian
    of the GPU residual, symmetric for hyperelastic Hencky."""
    import paper_2507_09435_b200 as impm
    from paper_2507_09435_b200 import workloads

    prob = workloads.footing3d(cells=(8, 8, 4), ppc=ppc, h=0.5, steps=10,
                               t_hat=400e3 if material == "cam_clay" else 100e3, material=material)
    if material == "cam_clay":
        prob.material.pc0 = 40e3  # plastic from the first increments (non-symmetric tangent)
    sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options)
    sim.fixed[:] = prob.fixed
    sim.gravity = prob.gravity
    assert sim.step(1 / prob.load_steps).iterations <= 8
    sim.begin_step()
    s = 2 / prob.load_steps
    sim.newton_solve(s)
    u = sim.nodal_solution()
    err, J = fd_check(sim, s, u, 1e-9)
    assert err <= 1e-5, err
    if material in ("hencky", "neo_hookean"):
        assert abs(J - J.T).max() <= 1e-10 * abs(J).max()


@pytest.mark.parametrize("tl", [False, True])
@pytest.mark.parametrize("ppc", [2, 3])
def test_factored_neo_hookean_assembly_matches_tangent_path(ppc, tl, monkeypatch):
    """3D neo-Hookean J from the factored tangent (k_tangent_nh3q +
    k_assemble_nh3f, the default) equals the J assembled from the 81-entry
    dP/dG (IMPM_ASM_NHF=0: k_tangent_nh3 + k_assemble_bins_staged) to rounding,
    updated and total Lagrangian, resident and restaged bins, at a deformed
    state."""
    import paper_2507_09435_b200 as impm
    import golden_util as gu
    from paper_2507_09435_b200 import workloads

    prob = workloads.footing3d(cells=(8, 8, 4), ppc=ppc, h=0.5, steps=10, material="neo_hookean")
    prob.options.total_lagrangian = tl
    out = {}
    for nhf in ("0", "1"):
        monkeypatch.setenv("IMPM_ASM_NHF", nhf)  # read at sim creation
        sim = impm.MpmSim(prob.grid, prob.particles, prob.material, prob.options)
        sim.fixed[:] = prob.fixed
        sim.gravity = prob.gravity
        assert sim.step(1 / prob.load_steps).iterations <= 8
        sim.begin_step()
        u = np.random.default_rng(5).standard_normal(sim.n_dofs()) * 1e-3 * prob.grid.h
        out[nhf] = sim.jacobian_csr(u, 2 / prob.load_steps)
    (rp0, c0, v0), (rp1, c1, v1) = out["0"], out["1"]
    assert np.array_equal(rp0, rp1) and np.array_equal(c0, c1)
    assert gu.csr_row_scaled_err(rp0, v0, v1) <= 1e-13


def dp_yield(prob, p):
    """Drucker-Prager yield function of every particle's committed elastic
    Hencky strain eps = log(B_e) / 2 (impm_math.cuh dp_update): ||dev eps|| +
    (3 lam + 2 mu) / (2 mu) (tr eps - e_c) alpha, normalised by the apex
    strain scale, and the tension cut-off tr eps - e_c."""
    m = prob.material
    E, nu = m.elastic.E, m.elastic.nu
    lam, mu = E * nu / ((1 + nu) * (1 - 2 * nu)), E / (2 * (1 + nu))
    sphi = np.sin(np.radians(m.friction_deg))
    alpha = np.sqrt(2.0 / 3.0) * 2.0 * sphi / (3.0 - sphi)
    e_c = 3.0 * m.cohesion / (3.0 * lam + 2.0 * mu)
    f, tcut, scale = [], [], 0.0
    for Be in p.B_e.reshape(-1, 3, 3):
        eps = 0.5 * sla.logm(0.5 * (Be + Be.T)).real
        tr = np.trace(eps)
        dev = eps - tr / 3 * np.eye(3)
        f.append(np.linalg.norm(dev) + (3 * lam + 2 * mu) / (2 * mu) * (tr - e_c) * alpha)
        tcut.append(tr - e_c)
        scale = max(scale, np.linalg.norm(eps))
    return np.array(f), np.array(tcut), scale


def test_drucker_prager_3d_footing_converges_and_is_admissible():
    """north_star's target material in 3D (extension, parity unpinned; the
    hook is update_stress, mpm_solver.hpp:445-454): the cfg 4 strip footing at
    16x16x8 cells (16,384 particles) with Drucker-Prager (30 deg, 20 kPa)
    converges over all 10 increments of a 300 kPa strip load, a plastic zone
    forms, and every particle's committed state lies on or inside the cone
    (yield function <= 1e-9 of the strain scale)."""
    sim, prob = footing("drucker_prager", t_hat=300e3)
    for k in range(1, prob.load_steps + 1):
        rec = sim.step(k / prob.load_steps)
        assert rec.iterations == 0 or rec.rel_residuals[-1] <= prob.options.tol
        assert rec.iterations <= 15, (k, rec.iterations)
    p = sim.particles
    assert (p.alpha[:, 0] > 0).sum() > 10, "the strip load must drive part of the soil plastic"
    f, tcut, scale = dp_yield(prob, p)
    assert f.max() <= 1e-9 * scale, f.max() / scale
    assert tcut.max() <= 1e-9 * scale


def test_drucker_prager_3d_tangent_matches_fd_in_plastic_state():
    """The dual-number consistent tangent of 3D Drucker-Prager (spectral
    log/exp + cone return) against central differences of the GPU residual
    at a converged plastic increment; non-associative flow makes J
    nonsymmetric (assembled in full)."""
    sim, prob = footing("drucker_prager", t_hat=300e3)
    for k in range(1, 6):
        sim.step(k / prob.load_steps)
    assert (sim.particles.alpha[:, 0] > 0).any()
    sim.begin_step()
    s = 6 / prob.load_steps
    sim.newton_solve(s)
    u = sim.nodal_solution()
    err, J = fd_check(sim, s, u, 1e-9)
    assert err <= 1e-5, err
    asym = abs(J - J.T).max() / abs(J).max()
    assert asym > 1e-8
