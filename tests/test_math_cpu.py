"""The device constitutive code (csrc/impm_math.cuh) compiled for the host
(tests/cpp/math_probe.cu): the 3x3 spectral log/exp that extends the
reference's D <= 2 closed forms (materials.hpp:61-105) to 3D, and the return
maps built on it (J2, Drucker-Prager, modified Cam-Clay; parity unpinned).

Checked the way the reference checks its own models (test_materials.cpp:43-78):
values against an independent implementation (scipy.linalg.logm / expm),
dual-number tangents against central finite differences, yield admissibility,
objectivity, and -- the transitive pin -- the 3D spectral path against the 2D
closed-form path (itself pinned to the reference) on plane-strain states."""
import numpy as np
import pytest
import scipy.linalg as sla

import math_probe as mp


def spd(rng, spread=1.0):
    A = rng.standard_normal((3, 3))
    Q, _ = np.linalg.qr(A)
    lam = np.exp(spread * rng.uniform(-0.7, 0.7, 3))
    return (Q * lam) @ Q.T


def sym_dirs(rng):
    d = rng.standard_normal((3, 3, 3))
    return d + d.transpose(0, 2, 1)


CASES = ["random", "identity", "double", "near_double", "diag"]


def make_B(case, rng):
    if case == "random":
        return spd(rng)
    if case == "identity":
        return np.eye(3)
    Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    lam = {"double": [1.3, 1.3, 0.8], "near_double": [1.3, 1.3 + 1e-9, 0.8], "diag": [1.1, 0.9, 1.2]}[case]
    B = (Q * lam) @ Q.T if case != "diag" else np.diag(lam)
    return 0.5 * (B + B.T)


@pytest.mark.parametrize("case", CASES)
def test_spectral_log_exp_values(case):
    rng = np.random.default_rng(1)
    B = make_B(case, rng)
    L, _ = mp.sym_fun3(B, np.zeros((3, 3, 3)), 0)
    assert np.all(np.isfinite(L))  # dual value path == double path (else NaN)
    assert np.abs(L - sla.logm(B).real).max() <= 1e-14 * max(1.0, np.abs(L).max()) + 1e-15
    E, _ = mp.sym_fun3(L, np.zeros((3, 3, 3)), 1)
    assert np.abs(E - sla.expm(L)).max() <= 1e-14 * np.abs(E).max()
    assert np.abs(E - B).max() <= 1e-14 * np.abs(B).max()


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("fn", [0, 1])
def test_spectral_tangent_matches_fd(case, fn):
    rng = np.random.default_rng(2)
    B = make_B(case, rng) if fn == 0 else 0.3 * sla.logm(make_B(case, rng)).real
    dirs = sym_dirs(rng)
    _, d = mp.sym_fun3(B, dirs, fn)
    f = (lambda X: sla.logm(X).real) if fn == 0 else sla.expm
    for k in range(3):
        h = 1e-6
        fd = (f(B + h * dirs[k]) - f(B - h * dirs[k])) / (2 * h)
        assert np.abs(d[k] - fd).max() <= 1e-7 * max(1.0, np.abs(fd).max())


def test_eigen_decomposition_orthogonal():
    rng = np.random.default_rng(3)
    for _ in range(50):
        B = spd(rng, 2.0)
        lam, Q = mp.eig3(B)
        assert np.abs(Q.T @ Q - np.eye(3)).max() <= 4e-16 * 8
        assert np.abs((Q * lam) @ Q.T - B).max() <= 1e-15 * 8 * np.abs(B).max()


def rot(rng):
    Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    return Q if np.linalg.det(Q) > 0 else -Q


def load_increment(kind):
    """A compressive-shear increment: elastic for 'small', plastic for 'large'."""
    return {
        "small": np.eye(3) + np.array([[-2e-4, 1e-4, 0], [0, -1e-4, 0], [0, 5e-5, -3e-4]]),
        "large": np.eye(3) + np.array([[-2e-2, 3e-2, 0], [0, -1e-2, 1e-2], [0, 5e-3, -4e-2]]),
    }[kind]


PLASTIC = ["hencky_j2", "drucker_prager", "cam_clay"]


@pytest.mark.parametrize("kind", ["hencky", "neo_hookean"] + PLASTIC)
@pytest.mark.parametrize("inc", ["small", "large"])
def test_stress_tangent_matches_fd(kind, inc):
    """dsigma/df_inc by duals (the tangent kernel's arithmetic) vs central FD."""
    f = load_increment(inc)
    Fn = np.eye(3) + np.array([[-1e-3, 0, 2e-3], [0, -2e-3, 0], [1e-3, 0, -1e-3]])
    Be_n = Fn @ Fn.T
    r = mp.stress3(kind, f, Fn, Be_n)
    h = 1e-7
    fd = np.zeros((9, 9))
    for k in range(9):
        e = np.zeros(9)
        e[k] = h
        sp = mp.stress3(kind, f + e.reshape(3, 3), Fn, Be_n)["sigma"].reshape(9)
        sm = mp.stress3(kind, f - e.reshape(3, 3), Fn, Be_n)["sigma"].reshape(9)
        fd[:, k] = (sp - sm) / (2 * h)
    scale = np.abs(fd).max()
    assert np.abs(r["dsig"] - fd).max() <= 2e-6 * scale


@pytest.mark.parametrize("kind", ["hencky"] + PLASTIC)
def test_objectivity(kind):
    rng = np.random.default_rng(5)
    R = rot(rng)
    f = load_increment("large")
    a = mp.stress3(kind, f)
    b = mp.stress3(kind, R @ f)
    assert np.abs(b["sigma"] - R @ a["sigma"] @ R.T).max() <= 1e-9 * np.abs(a["sigma"]).max()
    if kind in PLASTIC:
        assert abs(a["dg"] - b["dg"]) <= 1e-12 + 1e-9 * abs(a["dg"])


@pytest.mark.parametrize("kind", ["hencky", "hencky_j2", "drucker_prager"])
def test_3d_spectral_path_equals_2d_closed_form_on_plane_strain(kind):
    """The 2D closed forms are pinned to the reference (tests/test_gpu_parity.py);
    on plane-strain states the 3D spectral path must reproduce them."""
    rng = np.random.default_rng(6)
    for _ in range(10):
        f2 = np.eye(2) + 0.02 * rng.standard_normal((2, 2))
        F2 = np.eye(2) + 0.01 * rng.standard_normal((2, 2))
        f3, F3 = np.eye(3), np.eye(3)
        f3[:2, :2], F3[:2, :2] = f2, F2
        Be = np.eye(3)
        Be[:2, :2] = F2 @ F2.T
        a = mp.stress2(kind, f2, F2, Be)
        b = mp.stress3(kind, f3, F3, Be)
        s = np.abs(a["sigma"]).max()
        assert np.abs(a["sigma"] - b["sigma"]).max() <= 1e-12 * s
        if kind != "hencky":
            assert np.abs(a["Be"] - b["Be"]).max() <= 1e-13
            assert abs(a["dg"] - b["dg"]) <= 1e-13


def mcc_invariants(sig, J, prm):
    tau = sig * J
    P = -np.trace(tau) / 3
    s = tau + P * np.eye(3)
    q = np.sqrt(1.5) * np.linalg.norm(s)
    return P, q


def test_cam_clay_rest_state_is_elastic_and_stress_free():
    r = mp.stress3("cam_clay", np.eye(3))
    assert np.abs(r["sigma"]).max() == 0.0 and r["dg"] == 0.0
    assert np.abs(r["Be"] - np.eye(3)).max() <= 1e-15


@pytest.mark.parametrize("alpha", [0.0, 0.01])
@pytest.mark.parametrize("scale", [1.0, 3.0, -1.0])
def test_cam_clay_return_is_admissible(alpha, scale):
    """After the return: f(P, q, p_c) = 0 on the updated surface, p_c hardened by
    the returned compaction, and B_e carries the returned elastic strain."""
    f = np.eye(3) + scale * np.array([[-2e-2, 3e-2, 0], [0, -1e-2, 1e-2], [0, 5e-3, -4e-2]])
    r = mp.stress3("cam_clay", f, alpha=alpha)
    lam, mu, M, pc0, theta, pt = r["prm"][0], r["prm"][1], r["prm"][5], r["prm"][6], r["prm"][7], r["prm"][8]
    K = lam + 2 * mu / 3
    P, q = mcc_invariants(r["sigma"], r["J"], r["prm"])
    pc = pc0 * np.exp(theta * (alpha + r["dg"]))
    fy = q * q / M ** 2 + (P + pt) * (P - pc)
    assert r["dg"] != 0.0
    assert abs(fy) <= 1e-9 * pc * pc
    eps_e = 0.5 * sla.logm(r["Be"]).real
    assert abs(-K * np.trace(eps_e) - P) <= 1e-9 * pc
    dev = eps_e - np.trace(eps_e) / 3 * np.eye(3)
    assert abs(np.sqrt(6) * mu * np.linalg.norm(dev) - q) <= 1e-9 * pc
