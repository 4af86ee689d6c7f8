"""General CSR matrices on the device: the reference's link-level seam.

Mirrors impm::CsrMatrix (/root/reference/proj/include/impm/sparse.hpp:11-31,
src/sparse.cpp) and impm::sparse_lu_solve (sparse.hpp:43,
src/linear_solver.cpp:11-88). The host object keeps the reference's fields
(n, row_ptr int64, cols int32, vals float64); multiply / transposed /
sparse_lu_solve run in libimpm_gpu.so (impm_csr_multiply,
impm_csr_transposed, impm_sparse_lu_solve). No CPU fallback.
"""
import numpy as np

from . import _abi
from .errors import Error, raise_for


class CsrMatrix:
    """impm::CsrMatrix: square n x n, column indices sorted and unique per row."""

    def __init__(self, n=0, row_ptr=None, cols=None, vals=None):
        self.n = int(n)
        self.row_ptr = np.zeros(self.n + 1, np.int64) if row_ptr is None else np.ascontiguousarray(row_ptr, np.int64)
        self.cols = np.zeros(0, np.int32) if cols is None else np.ascontiguousarray(cols, np.int32)
        self.vals = np.zeros(len(self.cols), np.float64) if vals is None else np.ascontiguousarray(vals, np.float64)

    @staticmethod
    def from_pattern(n, pattern):  # src/sparse.cpp:9-22
        rp = np.zeros(n + 1, np.int64)
        rp[1:] = np.cumsum([len(p) for p in pattern])
        cols = np.concatenate([np.asarray(p, np.int32) for p in pattern]) if n else np.zeros(0, np.int32)
        return CsrMatrix(n, rp, cols, np.zeros(len(cols)))

    @staticmethod
    def from_dense(A):
        A = np.asarray(A, np.float64)
        n = A.shape[0]
        pattern = [np.nonzero(A[i])[0] for i in range(n)]
        m = CsrMatrix.from_pattern(n, pattern)
        m.vals[:] = np.concatenate([A[i, p] for i, p in enumerate(pattern)]) if n else []
        return m

    @property
    def nnz(self):
        return int(self.row_ptr[-1])

    def _find(self, row, col):
        a, b = int(self.row_ptr[row]), int(self.row_ptr[row + 1])
        k = a + int(np.searchsorted(self.cols[a:b], col))
        return k if k < b and self.cols[k] == col else -1

    def at(self, row, col):  # src/sparse.cpp:24-31 (index of an existing entry)
        k = self._find(row, col)
        if k < 0:
            raise Error(f"CSR entry ({row}, {col}) is outside the pattern")
        return k

    def get(self, row, col):  # src/sparse.cpp:33-39
        k = self._find(row, col)
        return 0.0 if k < 0 else float(self.vals[k])

    def set(self, row, col, value):
        self.vals[self.at(row, col)] = value

    def zero_values(self):
        self.vals[:] = 0.0

    def max_abs(self):  # src/sparse.cpp:72-76
        return float(np.abs(self.vals).max()) if len(self.vals) else 0.0

    def to_dense(self):
        A = np.zeros((self.n, self.n))
        for i in range(self.n):
            a, b = self.row_ptr[i], self.row_ptr[i + 1]
            A[i, self.cols[a:b]] = self.vals[a:b]
        return A

    def multiply(self, x, device=0):  # src/sparse.cpp:44-53, on the device
        x = _abi.f64(x)
        if len(x) != self.n:
            raise Error("vector size does not match the matrix dimension")
        y = np.zeros(self.n)
        st = _abi.lib().impm_csr_multiply(self.n, _abi.ptr(self.row_ptr), _abi.ptr(self.cols), _abi.ptr(self.vals),
                                          _abi.ptr(x), _abi.ptr(y), device)
        _check(st)
        return y

    def transposed(self, device=0):  # src/sparse.cpp:55-70, on the device
        t = CsrMatrix(self.n, np.zeros(self.n + 1, np.int64), np.zeros(self.nnz, np.int32), np.zeros(self.nnz))
        st = _abi.lib().impm_csr_transposed(self.n, _abi.ptr(self.row_ptr), _abi.ptr(self.cols), _abi.ptr(self.vals),
                                            _abi.ptr(t.row_ptr), _abi.ptr(t.cols), _abi.ptr(t.vals), device)
        _check(st)
        return t


def _check(st):
    if st != _abi.OK:
        raise_for(st, _abi.lib().impm_csr_last_error().decode())


def sparse_lu_solve(A: CsrMatrix, b, device=0, return_iterations=False):
    """impm::sparse_lu_solve (src/linear_solver.cpp:11-88) on the device.
    Raises LinearSolverError with the reference's messages."""
    b = _abi.f64(b)
    x = np.zeros(A.n)
    its = _abi.c_int32(0)
    st = _abi.lib().impm_sparse_lu_solve(A.n, _abi.ptr(A.row_ptr), _abi.ptr(A.cols), _abi.ptr(A.vals), _abi.ptr(b),
                                         len(b), _abi.ptr(x), device, _abi.ctypes.byref(its))
    _check(st)
    return (x, its.value) if return_iterations else x
