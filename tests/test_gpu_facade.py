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
