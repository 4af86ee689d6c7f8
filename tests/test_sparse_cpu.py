"""Host side of the CSR seam (paper_2507_09435_b200/sparse.py) without a GPU:
the impm::CsrMatrix surface (sparse.hpp:11-31, src/sparse.cpp:9-42) and the
workload generators of BASELINE.json's configs (shapes only)."""
import numpy as np
import pytest


def test_csr_from_pattern_and_accessors():
    from paper_2507_09435_b200 import CsrMatrix, Error

    A = CsrMatrix.from_pattern(3, [[0, 2], [1], [0, 1, 2]])  # src/sparse.cpp:9-22
    np.testing.assert_array_equal(A.row_ptr, [0, 2, 3, 6])
    np.testing.assert_array_equal(A.cols, [0, 2, 1, 0, 1, 2])
    assert A.nnz == 6 and (A.vals == 0).all()
    A.set(2, 1, 4.5)
    assert A.get(2, 1) == 4.5 and A.get(1, 0) == 0.0  # get: 0 outside the pattern
    with pytest.raises(Error, match="outside the pattern"):  # at: existing entries only
        A.at(1, 2)
    A.vals[:] = [1, -7, 2, 3, 4.5, 5]
    assert A.max_abs() == 7.0
    D = A.to_dense()
    B = CsrMatrix.from_dense(D)
    np.testing.assert_array_equal(B.to_dense(), D)
    A.zero_values()
    assert A.max_abs() == 0.0


def test_cfg2_slope_shape():
    from paper_2507_09435_b200 import workloads

    prob = workloads.slope2d(material="hencky_j2")
    assert prob.particles.shape == (401_216, 6 * 2 + 22 + 4)
    assert prob.material.kappa == 400e3 and prob.load_steps == 20


def test_cfg4_cam_clay_material():
    from paper_2507_09435_b200 import workloads

    prob = workloads.footing3d(cells=(8, 8, 4), material="cam_clay")
    m = prob.material
    assert m.kind == "cam_clay" and m.pc0 == 600e3 and m.hardening == 10.0
    assert prob.particles.shape[0] == 8 * 8 * 4 * 8
