"""ctypes binding of include/impm_gpu.h (the C ABI of libimpm_gpu.so).

The product path loads ONLY the in-tree CUDA library; there is no CPU
fallback. If libimpm_gpu.so is missing the import of any simulation class
fails loudly with ExtensionMissing.
"""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IMPM_LIB") or os.path.join(HERE, "libimpm_gpu.so")  # IMPM_LIB: A/B builds only

c_int32, c_int64, c_double, c_void_p = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p


class ExtensionMissing(ImportError):
    pass


class Grid(ctypes.Structure):
    _fields_ = [("dim", c_int32), ("nodes", c_int32 * 3), ("origin", c_double * 3), ("h", c_double)]


class Material(ctypes.Structure):
    _fields_ = [("kind", c_int32), ("pad_", c_int32), ("E", c_double), ("nu", c_double), ("kappa", c_double),
                ("friction_deg", c_double), ("cohesion", c_double), ("pc0", c_double), ("hardening", c_double)]


class Options(ctypes.Structure):
    _fields_ = [
        ("tol", c_double),
        ("abs_floor", c_double),
        ("max_iterations", c_int32),
        ("total_lagrangian", c_int32),
        ("shape", c_int32),
        ("krylov", c_int32),
        ("krylov_rtol", c_double),
        ("krylov_max_iter", c_int32),
        ("profile", c_int32),
        ("precond", c_int32),
        ("mg_smooth", c_int32),
        ("strategy", c_int32),
        ("interference", c_int32),
    ]


class Poro(ctypes.Structure):
    _fields_ = [("lambda_", c_double), ("mu", c_double), ("k", c_double), ("mu_f", c_double), ("rho_f", c_double)]


class StepRecordC(ctypes.Structure):
    _fields_ = [
        ("step", c_int32),
        ("iterations", c_int32),
        ("r0_norm", c_double),
        ("seconds", c_double),
        ("diff_seconds", c_double),
        ("backward_passes", c_int32),
        ("n_rel", c_int32),
        ("rel_residuals", ctypes.POINTER(c_double)),
        ("rel_capacity", c_int32),
        ("krylov_iterations", c_int32),
        ("solve_seconds", c_double),
        ("residual_seconds", c_double),
        ("nnz_assembled", c_int64),
    ]


# status codes (impm_status)
OK, ERR_CONFIG, ERR_DOMAIN, ERR_OUT_OF_DOMAIN, ERR_NONCONVERGENCE, ERR_LINEAR_SOLVER, ERR_CUDA, ERR_NCCL, \
    ERR_SEEDING, ERR_UNSUPPORTED = range(10)

_P = ctypes.POINTER
_SIGNATURES = {
    "impm_version": (ctypes.c_char_p, []),
    "impm_particle_doubles": (c_int32, [c_int32]),
    "impm_create_error": (ctypes.c_char_p, []),
    "impm_launch_count": (c_int64, []),
    "impm_sim_create": (c_int32, [_P(Grid), _P(Material), _P(Options), c_int32, _P(c_void_p)]),
    "impm_sim_destroy": (c_int32, [c_void_p]),
    "impm_coupled_create": (c_int32, [_P(Grid), _P(Poro), _P(Options), c_int32, _P(c_void_p)]),
    "impm_coupled_initialize": (c_int32, [c_void_p]),
    "impm_coupled_step": (c_int32, [c_void_p, c_double, _P(StepRecordC)]),
    "impm_coupled_nodal_pressure": (c_int32, [c_void_p, c_void_p]),
    "impm_coupled_settlement": (c_int32, [c_void_p, c_void_p, _P(c_double)]),
    "impm_sim_set_stream": (c_int32, [c_void_p, c_void_p]),
    "impm_sim_set_particles": (c_int32, [c_void_p, c_void_p, c_int64, c_int64]),
    "impm_sim_get_particles": (c_int32, [c_void_p, c_void_p, c_int64, c_int64]),
    "impm_sim_set_particle_field": (c_int32, [c_void_p, c_int32, c_void_p]),
    "impm_sim_n_particles": (c_int32, [c_void_p, _P(c_int64)]),
    "impm_sim_set_fixed": (c_int32, [c_void_p, c_void_p]),
    "impm_sim_set_gravity": (c_int32, [c_void_p, c_void_p]),
    "impm_sim_set_options": (c_int32, [c_void_p, _P(Options)]),
    "impm_sim_begin_step": (c_int32, [c_void_p]),
    "impm_sim_n_dofs": (c_int32, [c_void_p, _P(c_int32)]),
    "impm_sim_dof_map": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "impm_sim_node_mass": (c_int32, [c_void_p, c_void_p]),
    "impm_sim_colour_groups": (c_int32, [c_void_p, c_void_p, _P(c_int32)]),
    "impm_sim_support_stats": (c_int32, [c_void_p, c_void_p]),
    "impm_debug_oob_count": (c_int64, []),
    "impm_sim_p2g_map": (c_int32, [c_void_p, c_void_p, c_void_p]),
    "impm_sim_residual": (c_int32, [c_void_p, c_void_p, c_double, c_void_p]),
    "impm_sim_jacobian_csr": (c_int32, [c_void_p, c_void_p, c_double, _P(c_int64), c_void_p, c_void_p, c_void_p]),
    "impm_sim_linear_solve": (c_int32, [c_void_p, c_void_p, c_double, c_void_p, c_void_p, _P(c_int32)]),
    "impm_sim_newton_solve": (c_int32, [c_void_p, c_double, _P(StepRecordC)]),
    "impm_sim_commit_step": (c_int32, [c_void_p]),
    "impm_sim_step": (c_int32, [c_void_p, c_double, _P(StepRecordC)]),
    "impm_sim_nodal_solution": (c_int32, [c_void_p, c_void_p]),
    "impm_sim_set_nodal_solution": (c_int32, [c_void_p, c_void_p]),
    "impm_sim_last_error": (c_int32, [c_void_p, ctypes.c_char_p, ctypes.c_size_t, c_void_p, _P(c_int32)]),
    "impm_sim_kernel_times": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, _P(c_int32), c_int32]),
    "impm_sim_matrix_info": (c_int32, [c_void_p, _P(c_int64), _P(c_int64), _P(c_int64)]),
    # slab decomposition
    "impm_comm_nccl_id": (c_int32, [c_void_p, c_int32]),
    "impm_comm_nccl_create": (c_int32, [c_void_p, c_int32, c_int32, c_int32, _P(c_void_p)]),
    "impm_comm_local_group": (c_int32, [c_int32, c_int32, c_void_p]),
    "impm_comm_destroy": (c_int32, [c_void_p]),
    "impm_comm_info": (c_int32, [c_void_p, _P(c_int32), _P(c_int32), _P(ctypes.c_char_p)]),
    "impm_sim_set_slab": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p]),
    "impm_sim_set_particles_ids": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_int64]),
    "impm_sim_get_particles_ids": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_int64]),
    "impm_sim_migrate": (c_int32, [c_void_p]),
    "impm_sim_slab_info": (c_int32, [c_void_p, _P(c_int64), _P(c_int64), _P(c_int32)]),
    "impm_sim_apply_jacobian": (c_int32, [c_void_p, c_void_p, c_double, c_void_p, c_void_p]),
    # link-level seam: general CSR (sparse.hpp:11-43)
    "impm_sparse_lu_solve": (c_int32, [c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_int32,
                                       _P(c_int32)]),
    "impm_csr_multiply": (c_int32, [c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int32]),
    "impm_csr_transposed": (c_int32, [c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int32]),
    "impm_csr_last_error": (ctypes.c_char_p, []),
}

# every symbol include/impm_gpu.h declares (checked by tests without a GPU)
EXPORTED = sorted(_SIGNATURES)

_lib = None


def lib():
    """Loads the in-tree CUDA library (fails loudly if it is not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ExtensionMissing(
                f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`; "
                "the CUDA path has no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def ptr(a):
    """Raw pointer of a contiguous numpy array (or None)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data_as(c_void_p)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)
