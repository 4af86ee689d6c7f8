"""Builds and binds tests/cpp/math_probe.cu (host-compiled device math, test harness only)."""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cpp", "math_probe.cu")
OUT = os.path.join(HERE, "_build", "libmath_probe.so")
DEPS = [SRC, os.path.join(os.path.dirname(HERE), "paper_2507_09435_b200", "csrc", "impm_math.cuh")]
_lib = None


def lib():
    global _lib
    if _lib is None:
        os.makedirs(os.path.dirname(OUT), exist_ok=True)
        if not os.path.exists(OUT) or any(os.path.getmtime(d) > os.path.getmtime(OUT) for d in DEPS):
            subprocess.run(["nvcc", "-std=c++20", "-O2", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC", "-shared", "-o", OUT, SRC], check=True)
        _lib = ctypes.CDLL(OUT)
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def sym_fun3(B, dB, fn):
    B = np.ascontiguousarray(B, np.float64).reshape(9)
    dB = np.ascontiguousarray(dB, np.float64).reshape(27)
    out, dout = np.zeros(9), np.zeros(27)
    lib().probe_sym_fun3(_p(B), _p(dB), ctypes.c_int(fn), _p(out), _p(dout))
    return out.reshape(3, 3), dout.reshape(3, 3, 3)


def eig3(B):
    B = np.ascontiguousarray(B, np.float64).reshape(9)
    l, Q = np.zeros(3), np.zeros(9)
    lib().probe_eig3(_p(B), _p(l), _p(Q))
    return l, Q.reshape(3, 3)


KINDS = {"hencky": 0, "hencky_j2": 1, "neo_hookean": 2, "drucker_prager": 3, "cam_clay": 4}


def stress3(kind, f_inc, F_n=None, Be_n=None, alpha=0.0, lam=5.77e6, mu=3.85e6, kappa=2e4, friction_deg=30.0,
            cohesion=5e3, pc0=6e5, theta=10.0):
    f_inc = np.ascontiguousarray(f_inc, np.float64).reshape(9)
    F_n = np.eye(3).reshape(9) if F_n is None else np.ascontiguousarray(F_n, np.float64).reshape(9)
    Be = np.zeros(10)
    Be[:9] = np.eye(3).reshape(9) if Be_n is None else np.asarray(Be_n, np.float64).reshape(9)
    Be[9] = alpha
    sphi = np.sin(np.radians(friction_deg))
    prm = np.array([lam, mu, kappa, np.sqrt(2 / 3) * 2 * sphi / (3 - sphi), 3 * cohesion / (3 * lam + 2 * mu),
                    6 * sphi / (3 - sphi), pc0, theta, cohesion])
    sig, J, Bo, dg, dsig = np.zeros(9), np.zeros(1), np.zeros(9), np.zeros(1), np.zeros(81)
    lib().probe_stress3(ctypes.c_int(KINDS[kind]), _p(f_inc), _p(F_n), _p(Be), _p(prm), _p(sig), _p(J), _p(Bo),
                        _p(dg), _p(dsig))
    return {"sigma": sig.reshape(3, 3), "J": J[0], "Be": Bo.reshape(3, 3), "dg": dg[0], "dsig": dsig.reshape(9, 9),
            "prm": prm}


def stress2(kind, f_inc, F_n=None, Be_n=None, alpha=0.0, **kw):
    """The D = 2 (plane strain, closed-form log) path; same parameters as stress3."""
    f_inc = np.ascontiguousarray(f_inc, np.float64).reshape(4)
    F_n = np.eye(2).reshape(4) if F_n is None else np.ascontiguousarray(F_n, np.float64).reshape(4)
    Be = np.zeros(10)
    Be[:9] = np.eye(3).reshape(9) if Be_n is None else np.asarray(Be_n, np.float64).reshape(9)
    Be[9] = alpha
    prm = stress3("neo_hookean", np.eye(3), **kw)["prm"]
    sig, J, Bo, dg = np.zeros(9), np.zeros(1), np.zeros(9), np.zeros(1)
    lib().probe_stress2(ctypes.c_int(KINDS[kind]), _p(f_inc), _p(F_n), _p(Be), _p(prm), _p(sig), _p(J), _p(Bo),
                        _p(dg))
    return {"sigma": sig.reshape(3, 3), "J": J[0], "Be": Bo.reshape(3, 3), "dg": dg[0]}
