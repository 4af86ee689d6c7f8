"""ctypes wrapper of oracle/liboracle.so — the CPU restatement oracle.

TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and the
cpu_baseline leg of bench.py as the checker. The product never imports it.
"""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
KINDS = {"hencky": 0, "hencky_j2": 1, "neo_hookean": 2}

_c = ctypes
_lib = None


def build():
    subprocess.run(["make", "-C", HERE, "oracle"], check=True, stdout=subprocess.DEVNULL)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        L = _c.CDLL(LIB)
        vp, ip, dp = _c.c_void_p, _c.c_void_p, _c.c_void_p
        L.oracle_create.restype = vp
        L.oracle_create.argtypes = [_c.c_int, ip, dp, _c.c_double, _c.c_int, _c.c_double, _c.c_double,
                                    _c.c_double, _c.c_double, _c.c_int, _c.c_int]
        L.oracle_destroy.argtypes = [vp]
        L.oracle_error.restype = _c.c_char_p
        L.oracle_error.argtypes = [vp]
        L.oracle_set_particles.argtypes = [vp, dp, _c.c_int]
        L.oracle_get_particles.argtypes = [vp, dp]
        L.oracle_set_fixed.argtypes = [vp, vp]
        L.oracle_set_gravity.argtypes = [vp, dp]
        L.oracle_n_dofs.argtypes = [vp]
        L.oracle_nnz.restype = _c.c_int64
        L.oracle_nnz.argtypes = [vp]
        L.oracle_dof_map.argtypes = [vp, ip, ip, ip, dp]
        L.oracle_pattern.argtypes = [vp, ip, ip]
        for name in ("oracle_begin_step", "oracle_commit"):
            getattr(L, name).argtypes = [vp]
        L.oracle_residual.argtypes = [vp, dp, _c.c_double, dp]
        L.oracle_jacobian.argtypes = [vp, dp, _c.c_double, dp]
        L.oracle_solve.argtypes = [vp, dp, dp, dp]
        L.oracle_set_u.argtypes = [vp, dp]
        L.oracle_step.argtypes = [vp, _c.c_double, _c.POINTER(_c.c_int), dp, _c.c_int]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_c.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class OracleSim:
    """Reference-faithful CPU MpmSim<D> (restated); same fixtures as the GPU sim."""

    def __init__(self, dim, nodes, origin, h, kind, E, nu, kappa=0.0, tol=1e-11, max_iterations=20,
                 total_lagrangian=False):
        L = lib()
        self.L = L
        self.D = dim
        self.N = int(np.prod(nodes[:dim]))
        self.ND = 6 * dim + 22 + dim * dim
        n = np.array(list(nodes) + [1] * (3 - len(nodes)), dtype=np.int32)
        o = np.array(list(origin) + [0.0] * (3 - len(origin)), dtype=np.float64)
        self.h = L.oracle_create(dim, _p(n), _p(o), float(h), KINDS[kind] if isinstance(kind, str) else int(kind),
                                 float(E), float(nu), float(kappa), float(tol), int(max_iterations),
                                 int(total_lagrangian))

    def __del__(self):
        if getattr(self, "h", None):
            self.L.oracle_destroy(self.h)
            self.h = None

    def _chk(self, code):
        if code != 0:
            raise OracleError(code, self.L.oracle_error(self.h).decode())

    def set_particles(self, parts):
        a = np.ascontiguousarray(parts, dtype=np.float64)
        self.P = a.shape[0]
        self.L.oracle_set_particles(self.h, _p(a), self.P)

    def particles(self):
        out = np.zeros((self.P, self.ND))
        self.L.oracle_get_particles(self.h, _p(out))
        return out

    def set_fixed(self, fixed):
        f = np.ascontiguousarray(fixed, dtype=np.uint8)
        self.L.oracle_set_fixed(self.h, _p(f))

    def set_gravity(self, g):
        g = np.ascontiguousarray(g, dtype=np.float64)
        self.L.oracle_set_gravity(self.h, _p(g))

    def begin_step(self):
        self._chk(self.L.oracle_begin_step(self.h))

    def n_dofs(self):
        return self.L.oracle_n_dofs(self.h)

    def dof_map(self):
        n = self.n_dofs()
        dof_of = np.zeros(self.N * self.D, dtype=np.int32)
        node_of = np.zeros(max(n, 1), dtype=np.int32)
        field_of = np.zeros(max(n, 1), dtype=np.int32)
        mass = np.zeros(self.N)
        self.L.oracle_dof_map(self.h, _p(dof_of), _p(node_of), _p(field_of), _p(mass))
        return dof_of, node_of[:n], field_of[:n], mass

    def pattern(self):
        n = self.n_dofs()
        rp = np.zeros(n + 1, dtype=np.int64)
        cols = np.zeros(max(self.L.oracle_nnz(self.h), 1), dtype=np.int32)
        self.L.oracle_pattern(self.h, _p(rp), _p(cols))
        return rp, cols[: rp[-1]]

    def residual(self, u, s):
        u = np.ascontiguousarray(u, dtype=np.float64)
        r = np.zeros(max(self.n_dofs(), 1))
        self._chk(self.L.oracle_residual(self.h, _p(u), float(s), _p(r)))
        return r[: self.n_dofs()]

    def jacobian(self, u, s=1.0):
        u = np.ascontiguousarray(u, dtype=np.float64)
        v = np.zeros(max(self.L.oracle_nnz(self.h), 1))
        self._chk(self.L.oracle_jacobian(self.h, _p(u), float(s), _p(v)))
        return v[: self.L.oracle_nnz(self.h)]

    def solve(self, vals, b):
        vals = np.ascontiguousarray(vals, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(max(self.n_dofs(), 1))
        self._chk(self.L.oracle_solve(self.h, _p(vals), _p(b), _p(x)))
        return x[: self.n_dofs()]

    def set_nodal_solution(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        self.L.oracle_set_u(self.h, _p(u))

    def commit_step(self):
        self._chk(self.L.oracle_commit(self.h))

    def step(self, s):
        it = _c.c_int(0)
        rel = np.zeros(64)
        self._chk(self.L.oracle_step(self.h, float(s), _c.byref(it), _p(rel), 64))
        return it.value, rel[: it.value].tolist()
