"""The C++ facade (include/impm_gpu.hpp) used as a drop-in for impm::MpmSim<3>
on the smoke3d scenario: n_dof 300 and 3 Newton iterations, as the reference's
committed out/smoke3d/summary.csv."""
import subprocess

import numpy as np
import pytest

import golden_util as gu
from test_abi_cpu import build_facade_smoke

pytestmark = pytest.mark.gpu


def test_cpp_facade_smoke3d_matches_reference(tmp_path):
    exe = build_facade_smoke(str(tmp_path / "facade_smoke"))
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    ref = np.load(gu.GOLDEN + "/reference_out.npz")["smoke3d__summary"]
    assert int(out[0]) == int(ref[0, 0]) == 300
    assert int(out[1]) == int(ref[0, 1]) == 3
    # sparse_lu_solve seam through the C++ facade (test_linear_solver.cpp:60-65, :92-97)
    assert abs(float(out[2]) - 1.0) <= 1e-14 and abs(float(out[3]) - 1.0) <= 1e-14
    assert int(out[4]) == 1


def test_reference_bar_scenario_by_type_swap():
    """The reference's own bar scenario (src/scenarios.cpp:92-142, built on
    impm::Grid / seed_box / MaterialSpec / SolverOptions) with only MpmSim
    swapped for impm_gpu::MpmSim (tests/cpp/bar_swap.cpp) reproduces the
    reference's committed out/bar_elastic: identical Newton iteration counts
    per step and particles.csv to 1e-7 (column-max scaled)."""
    import os

    from paper_2507_09435_b200 import build

    exe = build.build_bar_swap()
    if exe is None:
        pytest.skip("bar_swap not built (needs the reference headers at build time)")
    # configs/bar_elastic.cfg: height 50, 64 cells, ppc 4, E 10 kPa, nu 0, rho0 80, 40 steps, g 9.81, tol 1e-11
    out = subprocess.run([exe, "50", "64", "4", "1e4", "0", "80", "40", "9.81", "1e-11", "20"], capture_output=True,
                         text=True, check=True).stdout.splitlines()
    its = np.array([[int(v) for v in l.split()[1:]] for l in out if l.startswith("it ")])
    parts = np.array([[float(v) for v in l.split()[1:]] for l in out if l.startswith("p ")])
    ref = np.load(gu.GOLDEN + "/reference_out.npz")
    ref_it = ref["bar_elastic__iterations"]  # step, iteration, rel_residual
    ref_counts = np.array([int(ref_it[ref_it[:, 0] == k, 1].max()) for k in range(1, 41)])
    np.testing.assert_array_equal(its[:, 1], ref_counts)
    rp = ref["bar_elastic__particles"]  # Y_ref, y, sigma_yy, sigma_xx, F_yy, V
    assert parts.shape == rp.shape
    err = np.abs(parts - rp).max(axis=0) / np.maximum(np.abs(rp).max(axis=0), 1e-300)
    assert err.max() <= 1e-7, err
