"""Loads the reference-generated fixtures (tests/golden/*.npz, written by
tests/golden/make_golden.py from the unmodified reference core) into problem
descriptions the product and the oracle can both consume."""
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
MATERIAL_NAMES = {0: "hencky", 1: "hencky_j2", 2: "neo_hookean"}

MPM_CASES = ["bar1d_j2", "cant2d_hencky", "cant2d_hencky_newton", "col2d_j2", "col2d_nh", "col2d_nh_newton",
             "cube3d_nh", "cube3d_nh_newton", "footing3d_nh", "footing3d_16", "bench_sample3d", "tl2d_hencky",
             "cfg1_nh"]


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return {k: z[k] for k in z.files}


def spec_of(fx):
    text = bytes(fx["spec"]).decode()
    out = {}
    for line in text.splitlines():
        line = line.split("#")[0]
        if "=" in line:
            k, v = line.split("=", 1)
            out[k.strip()] = v.strip()
    return out


def problem(fx):
    """(dim, grid dict, material dict, options dict, particles0, fixed, gravity)."""
    g = fx["grid"]
    spec = spec_of(fx)
    dim = int(spec.get("dim", 2))
    grid = {"dim": dim, "origin": tuple(g[0:3][:dim]), "h": float(g[3]),
            "nodes": tuple(int(v) for v in g[4:7][:dim])}
    m = fx["material"]
    mat = {"kind": MATERIAL_NAMES[int(m[0])], "E": float(m[1]), "nu": float(m[2]), "kappa": float(m[3])}
    opts = {"tol": float(m[4]), "max_iterations": int(m[5]), "total_lagrangian": bool(m[6])}
    return dim, grid, mat, opts, fx["particles0"], fx["fixed"], fx["gravity"], spec


def rel_err(a, b, scale=None):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    s = scale if scale is not None else max(np.abs(b).max(initial=0.0), 1e-300)
    return float(np.abs(a - b).max(initial=0.0) / s)


def csr_row_scaled_err(rp, vals_a, vals_b):
    """max over rows of max|a-b| / max|b| in that row (test_jacobian.cpp:41-49 style)."""
    worst = 0.0
    for i in range(len(rp) - 1):
        s, e = rp[i], rp[i + 1]
        if e == s:
            continue
        sc = np.abs(vals_b[s:e]).max()
        if sc == 0:
            sc = 1.0
        worst = max(worst, float(np.abs(vals_a[s:e] - vals_b[s:e]).max() / sc))
    return worst
