/* impm_gpu.h — C ABI of the B200-native implicit MPM Newton step.
 *
 * Drop-in boundary for the reference's hot path. The
 * reference has no FFI; its seams are the C++ class `impm::MpmSim<D>`
 * (/root/reference/proj/include/impm/mpm_solver.hpp:51-478), the coupled
 * `impm::CoupledSim` (include/impm/porous.hpp:48-125) and the link-level
 * `impm::sparse_lu_solve` (include/impm/sparse.hpp:43). Each entry point below
 * names the reference member it replaces. Plain pointers and sizes only; every
 * call returns an impm_status and is synchronous to the host (stream-ordered
 * inside). Errors keep the reference's exception classes (errors.hpp:9-50) as
 * status codes; the message and a NonConvergenceError's residual history are
 * read back with impm_sim_last_error. The C++ facade in include/impm_gpu.hpp
 * rethrows them as impm:: exceptions.
 *
 * Particle records are exchanged in the reference's own AoS layout
 * `impm::Particle<D>` (include/impm/particle.hpp:10-29): all doubles, in order
 *   X[D] x[D] m V0 V F[D*D] sigma[9] lp0[D] lp[D] B_e[9] alpha traction_force[D] point_load[D]
 * i.e. 6D+22+D*D doubles (232/304/392 bytes for D = 1/2/3).
 */
#ifndef IMPM_GPU_H
#define IMPM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum impm_status {
  IMPM_OK = 0,
  IMPM_ERR_CONFIG = 1,          /* impm::ConfigError */
  IMPM_ERR_DOMAIN = 2,          /* impm::DomainError */
  IMPM_ERR_OUT_OF_DOMAIN = 3,   /* impm::OutOfDomainError */
  IMPM_ERR_NONCONVERGENCE = 4,  /* impm::NonConvergenceError */
  IMPM_ERR_LINEAR_SOLVER = 5,   /* impm::LinearSolverError */
  IMPM_ERR_CUDA = 6,
  IMPM_ERR_NCCL = 7,
  IMPM_ERR_SEEDING = 8,         /* impm::SeedingFault */
  IMPM_ERR_UNSUPPORTED = 9      /* impm::UnsupportedOperation */
} impm_status;

/* impm::Grid<D> (grid.hpp:18-58): nodes at origin + index*h, axis 0 slowest. */
typedef struct impm_grid {
  int32_t dim;        /* 1, 2 or 3 */
  int32_t nodes[3];   /* node count per axis (unused axes: 1) */
  double origin[3];
  double h;
} impm_grid;

/* impm::MaterialKind (materials.hpp:47) + extensions (parity unpinned). */
typedef enum impm_material_kind {
  IMPM_HENCKY = 0,
  IMPM_HENCKY_J2 = 1,
  IMPM_NEO_HOOKEAN = 2,
  IMPM_DRUCKER_PRAGER = 3, /* extension, parity unpinned */
  IMPM_CAM_CLAY = 4        /* modified Cam-Clay, extension, parity unpinned */
} impm_material_kind;

/* impm::MaterialSpec (mpm_solver.hpp:21-25) */
typedef struct impm_material {
  int32_t kind;       /* impm_material_kind */
  int32_t pad_;
  double E, nu;       /* ElasticParams (materials.hpp:12-23) */
  double kappa;       /* J2 yield strength */
  double friction_deg;  /* Drucker-Prager friction angle / Cam-Clay critical-state angle [deg] */
  double cohesion;      /* Drucker-Prager cohesion [Pa] (apex shift) / Cam-Clay tensile intercept p_t [Pa] */
  double pc0;           /* Cam-Clay initial preconsolidation pressure [Pa] */
  double hardening;     /* Cam-Clay hardening exponent theta = (1 + e0) / (lambda - kappa) */
} impm_material;

/* Transfer functions: impm::ShapeFunctionKind (gimp.hpp:11). */
typedef enum impm_shape_kind { IMPM_SHAPE_GIMP = 1, IMPM_SHAPE_BSPLINE2 = 2 } impm_shape_kind;

/* Linear solver behind the sparse_lu_solve seam (src/linear_solver.cpp:11-88).
 * AUTO: the reference's own equilibrated pivoted LU on the device below 2048
 * free DOFs (one GPU), else ITERATIVE. ITERATIVE: MG-CG for a symmetric J
 * (GMRES on CG breakdown), MG-GMRES for a nonsymmetric one. CG / BICGSTAB /
 * GMRES force one method. */
typedef enum impm_krylov_kind {
  IMPM_KRYLOV_AUTO = 0, IMPM_KRYLOV_CG = 1, IMPM_KRYLOV_BICGSTAB = 2, IMPM_KRYLOV_GMRES = 3,
  IMPM_KRYLOV_ITERATIVE = 4
} impm_krylov_kind;

/* Preconditioner of the Krylov solve. */
typedef enum impm_precond_kind { IMPM_PRECOND_MG = 0, IMPM_PRECOND_BLOCK_JACOBI = 1 } impm_precond_kind;

/* impm::JacobianStrategy (jacobian.hpp:18). Both produce the same values (the
 * reference's dense == sparse tests); the GPU always assembles by bins, and the
 * strategy sets the reference-equivalent StepRecord::backward_passes: n_dofs
 * per Jacobian (Algorithm 1) or fields*b^D (Algorithm 2). Zero = the reference
 * default (sparse). */
typedef enum impm_jacobian_strategy { IMPM_STRATEGY_SPARSE = 0, IMPM_STRATEGY_DENSE = 1 } impm_jacobian_strategy;

/* impm::InterferenceCheck (jacobian.hpp:20, verify_no_interference :167-182).
 * On the GPU the seeding hazard is a particle whose support reaches beyond
 * the (b-1)/2 = 2-node stencil of the pattern (it would write outside every
 * seeded pattern of its group): the check verifies every particle support on
 * the device (always: every Jacobian; sampled: 1 Jacobian in 8) and fails with
 * IMPM_ERR_SEEDING (impm::SeedingFault) and the reference's message text. */
typedef enum impm_interference_check {
  IMPM_INTERFERENCE_OFF = 0, IMPM_INTERFERENCE_SAMPLED = 1, IMPM_INTERFERENCE_ALWAYS = 2
} impm_interference_check;

/* impm::SolverOptions (mpm_solver.hpp:27-36) + GPU linear-solver knobs. */
typedef struct impm_options {
  double tol;                 /* relative residual (1e-11) */
  double abs_floor;           /* 1e-14 */
  int32_t max_iterations;     /* 20 */
  int32_t total_lagrangian;   /* 0/1 */
  int32_t shape;              /* impm_shape_kind, GIMP default */
  int32_t krylov;             /* impm_krylov_kind */
  double krylov_rtol;         /* relative true-residual target (1e-12) */
  int32_t krylov_max_iter;    /* 0 => 10*n_dofs capped at 20000 */
  int32_t profile;            /* 1: per-kernel-class CUDA-event timing */
  int32_t precond;            /* impm_precond_kind */
  int32_t mg_smooth;          /* multigrid pre/post block-Jacobi sweeps (0 => 1) */
  int32_t strategy;           /* impm_jacobian_strategy value; SolverOptions::strategy, mpm_solver.hpp:30 */
  int32_t interference;       /* impm_interference_check value; SolverOptions::interference, mpm_solver.hpp:31 */
} impm_options;

/* impm::StepRecord (mpm_solver.hpp:38-46) + GPU counters. rel_residuals is
 * caller-owned storage of rel_capacity doubles. */
typedef struct impm_step_record {
  int32_t step;
  int32_t iterations;
  double r0_norm;
  double seconds;
  double diff_seconds;          /* Jacobian assembly time (JacobianStats::seconds) */
  int32_t backward_passes;      /* reference-equivalent pass count fields*b^D per iteration */
  int32_t n_rel;
  double* rel_residuals;
  int32_t rel_capacity;
  int32_t krylov_iterations;    /* total over the step */
  double solve_seconds;
  double residual_seconds;
  int64_t nnz_assembled;        /* reference-pattern scalar nnz x iterations */
} impm_step_record;

/* impm::PoroParams (porous.hpp:22-38) */
typedef struct impm_poro {
  double lambda, mu;  /* Lame constants [Pa] */
  double k;           /* intrinsic permeability [m^2] */
  double mu_f;        /* fluid viscosity [Pa s] */
  double rho_f;       /* fluid density [kg/m^3] */
} impm_poro;

typedef struct impm_sim impm_sim; /* opaque: one MpmSim<D> (or CoupledSim) on one device */

/* version / capability */
const char* impm_version(void);
int32_t impm_particle_doubles(int32_t dim); /* 6D+22+D*D */
/* kernel launches this library has issued since load (all sims, all devices) */
int64_t impm_launch_count(void);
/* message of the last failed impm_sim_create on this thread */
const char* impm_create_error(void);

/* MpmSim(Grid, particles, MaterialSpec, SolverOptions) (mpm_solver.hpp:63-68) */
impm_status impm_sim_create(const impm_grid* grid, const impm_material* mat, const impm_options* opt,
                            int32_t device, impm_sim** out);
impm_status impm_sim_destroy(impm_sim* sim);
/* Runs all work on this CUDA stream (cudaStream_t, NULL = the sim's own). */
impm_status impm_sim_set_stream(impm_sim* sim, void* stream);

/* public members particles / fixed / gravity (mpm_solver.hpp:56-61) */
impm_status impm_sim_set_particles(impm_sim* sim, const double* aos, int64_t n, int64_t stride_bytes);
impm_status impm_sim_get_particles(impm_sim* sim, double* aos, int64_t n, int64_t stride_bytes);
impm_status impm_sim_set_particle_field(impm_sim* sim, int32_t field, const double* vals /*[n]*/);
impm_status impm_sim_n_particles(impm_sim* sim, int64_t* n);
impm_status impm_sim_set_fixed(impm_sim* sim, const uint8_t* fixed /* [node*D + comp] */);
impm_status impm_sim_set_gravity(impm_sim* sim, const double* g /* [D] */);
impm_status impm_sim_set_options(impm_sim* sim, const impm_options* opt);

/* begin_step (mpm_solver.hpp:93-138): binning + counting sort, node mass,
 * active set, DofMap, BSR pattern. */
impm_status impm_sim_begin_step(impm_sim* sim);
/* n_dofs / dofs() / node_mass() / total_node_mass() (mpm_solver.hpp:80-88) */
impm_status impm_sim_n_dofs(impm_sim* sim, int32_t* n);
impm_status impm_sim_dof_map(impm_sim* sim, int32_t* dof_of /*[N*D]*/, int32_t* node_of /*[n]*/,
                             int32_t* field_of /*[n]*/);
impm_status impm_sim_node_mass(impm_sim* sim, double* mass /*[N]*/);
/* JacobianAssembler colouring (jacobian.hpp:101-110): group id per DOF. */
impm_status impm_sim_colour_groups(impm_sim* sim, int32_t* group_of_dof /*[n]*/, int32_t* n_groups);
/* Diagnostics of the current step's supports (sizing the Jacobian work):
 * out[34] = {P, sum s_p, sum s_p^2, sum_bins n_p*nk, sum_bins n_p*nk^2, bins,
 * histogram of s_p over 1..27 at out[7..33]} (s_p = support nodes of
 * particle p, nk = support box of its bin). */
impm_status impm_sim_support_stats(impm_sim* sim, int64_t* out);
/* Checked builds (-DIMPM_CHECKED): number of out-of-range scattered accesses
 * the device has counted so far; -1 in a regular build. */
int64_t impm_debug_oob_count(void);
/* p2g_map (mpm_solver.hpp:142-152) */
impm_status impm_sim_p2g_map(impm_sim* sim, const double* per_particle, double* out /*[N]*/);

/* residual (mpm_solver.hpp:213-218): r(u) over free DOFs. */
impm_status impm_sim_residual(impm_sim* sim, const double* u /*[n]*/, double load_scale, double* r /*[n]*/);
/* record_residual + JacobianAssembler::sparse (mpm_solver.hpp:223-242,
 * jacobian.hpp:95-137): J(u) exported in the reference CSR pattern
 * (jacobian.hpp:36-65). Call with row_ptr/cols/vals NULL to get nnz first. */
impm_status impm_sim_jacobian_csr(impm_sim* sim, const double* u, double load_scale, int64_t* nnz,
                                  int64_t* row_ptr /*[n+1]*/, int32_t* cols /*[nnz]*/, double* vals /*[nnz]*/);
/* the linear solve seam: delta = J(u)^-1 rhs on the device Krylov path */
impm_status impm_sim_linear_solve(impm_sim* sim, const double* u, double load_scale, const double* rhs,
                                  double* delta, int32_t* krylov_iterations);

/* newton_solve / newton_attempt (mpm_solver.hpp:248-355) */
impm_status impm_sim_newton_solve(impm_sim* sim, double load_scale, impm_step_record* rec);
/* commit_step (mpm_solver.hpp:359-400): G2P + particle update */
impm_status impm_sim_commit_step(impm_sim* sim);
/* step (mpm_solver.hpp:402-407) */
impm_status impm_sim_step(impm_sim* sim, double load_scale, impm_step_record* rec);

/* nodal_solution / set_nodal_solution (mpm_solver.hpp:409-410) */
impm_status impm_sim_nodal_solution(impm_sim* sim, double* u /*[n]*/);
impm_status impm_sim_set_nodal_solution(impm_sim* sim, const double* u /*[n]*/);

/* impm::CoupledSim (porous.hpp:48-125): u-p, fields (u_0 .. u_{D-1}, p) per
 * node. D = 2 is the reference; D = 3 (4x4 node blocks) is an extension, parity
 * unpinned. set_fixed takes [node*(D+1) + field] (fixed_u merged with fixed_p).
 * The shared impm_sim_residual / _jacobian_csr / _linear_solve take dt as
 * load_scale. */
impm_status impm_coupled_create(const impm_grid* grid, const impm_poro* poro, const impm_options* opt,
                                int32_t device, impm_sim** out);
/* CoupledSim::initialize (src/porous.cpp:25-72): weights at the reference configuration */
impm_status impm_coupled_initialize(impm_sim* sim);
/* CoupledSim::step (src/porous.cpp:91-168) */
impm_status impm_coupled_step(impm_sim* sim, double dt, impm_step_record* rec);
/* CoupledSim::nodal_pressure (porous.hpp:81) */
impm_status impm_coupled_nodal_pressure(impm_sim* sim, double* p /*[N]*/);
/* accumulated vertical displacement per particle (u_total_y_, porous.hpp:118) and time() */
impm_status impm_coupled_settlement(impm_sim* sim, double* u_total_y /*[P]*/, double* time);

/* Last error of this sim: message, and for NONCONVERGENCE the residual history. */
impm_status impm_sim_last_error(impm_sim* sim, char* msg, size_t cap, double* history, int32_t* hist_len);

/* Per-kernel-class device time accumulated since the last reset (profile=1):
 * names[i] (static strings), ms[i], launches[i]; returns count in *n. */
impm_status impm_sim_kernel_times(impm_sim* sim, const char** names, double* ms, int64_t* launches,
                                  int32_t* n, int32_t reset);
/* Bytes of the stored BSR (values) and algorithmic per-launch traffic figures. */
impm_status impm_sim_matrix_info(impm_sim* sim, int64_t* n_rows, int64_t* row_values, int64_t* ref_nnz);

/* ---------------------------------------------------------------------------
 * Slab decomposition along grid axis 0 (multi-GPU, one rank per GPU).
 *
 * Replaces nothing in the reference, which is single-process
 * (mpm_solver.hpp:56-477); this is the "multi-GPU create variant" of
 * SURVEY.md §8(b)/(e). Axis 0 is the slowest index of Grid::flat
 * (grid.hpp:30-34) and DofMap::build numbers nodes in ascending flat order
 * (grid.hpp:76-85), so rank r owns the node planes [cuts[r], cuts[r+1]), a
 * contiguous range of global DOFs and Jacobian rows. Its simulation is
 * created on the LOCAL grid {global origin, h, nodes[0] = hi - lo, other
 * axes global} with [lo, hi) = [max(0, cuts[r]-2), min(n0, cuts[r+1]+2)), and
 * holds its owned particles plus the ghost particles whose first support node
 * lies in [cuts[r]-2, cuts[r]). Per Newton iteration the ranks exchange a
 * 2-plane vector halo before each SpMV / residual and sum the reduction
 * partials of every dot product; the MG preconditioner is rank-local (block
 * Jacobi across slabs). All calls on a slab simulation are collective over
 * the communicator: every rank makes the same sequence of calls.
 * ------------------------------------------------------------------------- */
typedef struct impm_comm impm_comm; /* opaque communicator (NCCL or in-process) */

/* NCCL: rank 0 creates the unique id (cap >= 128 bytes), ships it to the
 * other ranks out of band (e.g. torch.distributed broadcast), then every
 * rank creates its communicator on its own device. */
impm_status impm_comm_nccl_id(uint8_t* id, int32_t cap);
impm_status impm_comm_nccl_create(const uint8_t* id, int32_t rank, int32_t nranks, int32_t device, impm_comm** out);
/* In-process group: `nranks` communicators for ranks driven by host threads
 * of one process on one device (host-ordered collectives; test transport). */
impm_status impm_comm_local_group(int32_t nranks, int32_t device, impm_comm** out /* [nranks] */);
impm_status impm_comm_destroy(impm_comm* comm);
impm_status impm_comm_info(impm_comm* comm, int32_t* rank, int32_t* nranks, const char** kind);

/* Attach the slab decomposition: global node count along axis 0 and the
 * ownership cuts [nranks + 1] (cuts[0] = 0, cuts[nranks] = n0, every slab
 * >= 4 planes when nranks > 1). Single-field MpmSim only. */
impm_status impm_sim_set_slab(impm_sim* sim, impm_comm* comm, int32_t global_n0, const int32_t* cuts);
/* Particles with their global ids (the single-GPU AoS index; < 2^29). */
impm_status impm_sim_set_particles_ids(impm_sim* sim, const double* aos, const int64_t* ids, int64_t n,
                                       int64_t stride_bytes);
/* Local particles (owned + ghost copies) in local order with their ids. */
impm_status impm_sim_get_particles_ids(impm_sim* sim, double* aos, int64_t* ids, int64_t n, int64_t stride_bytes);
/* After commit_step: send owned particles to the rank(s) that keep them for
 * the next step (impm_sim_step does this itself on a slab). */
impm_status impm_sim_migrate(impm_sim* sim);
/* Global free-DOF count, this rank's first global DOF (the local DofMap of
 * the owned nodes is the global one shifted by it), global axis-0 index of
 * local node 0. */
impm_status impm_sim_slab_info(impm_sim* sim, int64_t* n_dofs_global, int64_t* dof_offset, int32_t* base0);
/* Parity tap: assemble J(u) (u = local free-DOF vector) and y = J x in grid
 * layout [N*D] of the local grid (owned rows; halo columns from the
 * neighbours). */
impm_status impm_sim_apply_jacobian(impm_sim* sim, const double* u, double load_scale, const double* x, double* y);

/* ---------------------------------------------------------------------------
 * Link-level seam: general CSR matrices (impm::CsrMatrix, sparse.hpp:11-31;
 * n x n, int64 row_ptr[n+1], int32 column indices sorted and unique per row).
 * Host arrays in and out; the work runs on `device`.
 * ------------------------------------------------------------------------- */
/* impm::sparse_lu_solve (sparse.hpp:43, src/linear_solver.cpp:11-88): x = A^-1 b
 * with the reference's row equilibration, <= 2 refinement sweeps while the
 * normwise backward error exceeds 1e-14, and IMPM_ERR_LINEAR_SOLVER with the
 * reference's message texts ("empty matrix row i", "singular factorization: ...",
 * "solution backward error ... exceeds 1e-10; ...", "right-hand side size does
 * not match the matrix dimension"). Dense device LU for n <= 2048, Jacobi-
 * right-preconditioned GMRES above (*iterations = its Krylov count, may be NULL). */
impm_status impm_sparse_lu_solve(int32_t n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                                 const double* b, int64_t b_len, double* x /*[n]*/, int32_t device,
                                 int32_t* iterations);
/* CsrMatrix::multiply (src/sparse.cpp:44-53): y = A x, bitwise the reference's
 * in-order row sums. */
impm_status impm_csr_multiply(int32_t n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                              const double* x, double* y /*[n]*/, int32_t device);
/* CsrMatrix::transposed (src/sparse.cpp:55-70): same nnz, columns sorted. */
impm_status impm_csr_transposed(int32_t n, const int64_t* row_ptr, const int32_t* cols, const double* vals,
                                int64_t* t_row_ptr /*[n+1]*/, int32_t* t_cols /*[nnz]*/, double* t_vals /*[nnz]*/,
                                int32_t device);
/* message of the last failed impm_sparse_lu_solve / impm_csr_* call on this thread */
const char* impm_csr_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* IMPM_GPU_H */
