// impm_gpu.hpp — header-only C++ facade over the C ABI (impm_gpu.h).
//
// Source-compatible stand-in for the reference's `impm::MpmSim<D>`
// (/root/reference/proj/include/impm/mpm_solver.hpp:51-478) and
// `impm::CoupledSim` (porous.hpp:48-125): same public members (grid,
// particles, material, gravity, options, fixed) and method names, with the
// work done on the GPU by libimpm_gpu.so. Status codes are rethrown as the
// reference's exception classes (errors.hpp:9-50; own copies here unless
// IMPM_GPU_REFERENCE_TYPES is defined, in which case the reference's
// impm::Particle/Grid/exceptions are used directly).
//
// Ownership follows the reference: the caller mutates `particles` / `fixed`
// freely; they are uploaded at begin_step()/step() and downloaded after
// commit_step()/step().
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "impm_gpu.h"

#ifdef IMPM_GPU_REFERENCE_TYPES
// the reference's own value types (grid, particle, material, options, records)
#include "impm/mpm_solver.hpp"
#endif
#include <span>

namespace impm_gpu {

#ifdef IMPM_GPU_REFERENCE_TYPES
using impm::ConfigError;
using impm::DomainError;
using impm::Error;
using impm::LinearSolverError;
using impm::NonConvergenceError;
using impm::OutOfDomainError;
using impm::SeedingFault;
using impm::UnsupportedOperation;
using impm::CsrMatrix;
template <int D>
using Particle = impm::Particle<D>;
#else
struct Error : std::runtime_error {
  explicit Error(const std::string& w) : std::runtime_error(w) {}
};
struct ConfigError : Error {
  using Error::Error;
};
struct DomainError : Error {
  using Error::Error;
};
struct UnsupportedOperation : Error {
  using Error::Error;
};
struct NonConvergenceError : Error {
  NonConvergenceError(const std::string& w, std::vector<double> h) : Error(w), residual_history(std::move(h)) {}
  std::vector<double> residual_history;
};
struct LinearSolverError : Error {
  using Error::Error;
};
struct OutOfDomainError : Error {
  using Error::Error;
};
struct SeedingFault : Error {
  using Error::Error;
};

// impm::Particle<D> (particle.hpp:10-29), identical layout
template <int D>
struct Particle {
  std::array<double, D> X{}, x{};
  double m = 0.0, V0 = 0.0, V = 0.0;
  std::array<double, D * D> F{};
  std::array<double, 9> sigma{};
  std::array<double, D> lp0{}, lp{};
  std::array<double, 9> B_e{1, 0, 0, 0, 1, 0, 0, 0, 1};
  double alpha = 0.0;
  std::array<double, D> traction_force{}, point_load{};
  Particle() {
    for (int a = 0; a < D; ++a) F[a * D + a] = 1.0;
  }
};
static_assert(sizeof(Particle<1>) == 232 && sizeof(Particle<2>) == 304 && sizeof(Particle<3>) == 392,
              "layout of impm::Particle<D>");
#endif

// GPU-only solver knobs (no counterpart in impm::SolverOptions); passed as
// an optional extra constructor argument so that reference-typed callers keep
// the reference constructor MpmSim(Grid, particles, MaterialSpec, SolverOptions)
struct GpuOptions {
  impm_krylov_kind krylov = IMPM_KRYLOV_AUTO;
  impm_precond_kind precond = IMPM_PRECOND_MG;
  double krylov_rtol = 1e-12;
  int device = 0;
};

#ifdef IMPM_GPU_REFERENCE_TYPES
// grid.hpp:18-58, materials.hpp:12-47, mpm_solver.hpp:21-46, jacobian.hpp:18-20
template <int D>
using Grid = impm::Grid<D>;
using impm::DofMap;
using impm::ElasticParams;
using impm::InterferenceCheck;
using impm::JacobianStrategy;
using impm::MaterialKind;
using impm::MaterialSpec;
using impm::SolverOptions;
using impm::StepRecord;
template <int D>
using NodeVec = impm::Vec<double, D>;
#else
template <int D>
using NodeVec = std::array<double, D>;

// impm::Grid<D> (grid.hpp:18-58)
template <int D>
struct Grid {
  std::array<double, D> origin{};
  double h = 1.0;
  std::array<int, D> nodes{};
  int node_count() const {
    int n = 1;
    for (int a = 0; a < D; ++a) n *= nodes[a];
    return n;
  }
  std::array<double, D> node_pos(int f) const {
    std::array<double, D> x{};
    for (int a = D - 1; a >= 0; --a) {
      x[a] = origin[a] + (f % nodes[a]) * h;
      f /= nodes[a];
    }
    return x;
  }
};

enum class MaterialKind { hencky = IMPM_HENCKY, hencky_j2 = IMPM_HENCKY_J2, neo_hookean = IMPM_NEO_HOOKEAN };
enum class JacobianStrategy { dense, sparse };          // jacobian.hpp:18
enum class InterferenceCheck { off, sampled, always };  // jacobian.hpp:20

struct ElasticParams {
  double E = 1.0, nu = 0.0;
};

struct MaterialSpec {  // mpm_solver.hpp:21-25
  MaterialKind kind = MaterialKind::hencky;
  ElasticParams elastic{1.0, 0.0};
  double kappa = 0.0;
};

struct SolverOptions {  // mpm_solver.hpp:27-36
  double tol = 1e-11;
  double abs_floor = 1e-14;
  int max_iterations = 20;
  JacobianStrategy strategy = JacobianStrategy::sparse;
  InterferenceCheck interference = InterferenceCheck::off;
  bool total_lagrangian = false;
};

struct StepRecord {  // mpm_solver.hpp:38-46 (+ the Krylov count)
  int step = 0, iterations = 0;
  std::vector<double> rel_residuals;
  double r0_norm = 0.0, seconds = 0.0, diff_seconds = 0.0;
  int backward_passes = 0;
  int krylov_iterations = 0;
};

struct CsrMatrix {  // sparse.hpp:11-31 (fields only)
  int n = 0;
  std::vector<std::int64_t> row_ptr;
  std::vector<std::int32_t> cols;
  std::vector<double> vals;
};

struct DofMap {  // grid.hpp:66-93
  int n_fields = 0, n_dofs = 0;
  std::vector<std::int32_t> dof_of, node_of, field_of;
  std::int32_t dof(int node, int field) const { return dof_of[static_cast<std::size_t>(node) * n_fields + field]; }
};
#endif

namespace detail {
inline void check(impm_status st, impm_sim* h) {
  if (st == IMPM_OK) return;
  char msg[4096] = {0};
  std::vector<double> hist(256);
  std::int32_t n = 256;
  impm_sim_last_error(h, msg, sizeof msg, hist.data(), &n);
  if (!h) std::snprintf(msg, sizeof msg, "%s", impm_create_error());
  hist.resize(std::min<std::int32_t>(n, 256));
  switch (st) {
    case IMPM_ERR_CONFIG: throw ConfigError(msg);
    case IMPM_ERR_DOMAIN: throw DomainError(msg);
    case IMPM_ERR_OUT_OF_DOMAIN: throw OutOfDomainError(msg);
    case IMPM_ERR_NONCONVERGENCE: throw NonConvergenceError(msg, hist);
    case IMPM_ERR_LINEAR_SOLVER: throw LinearSolverError(msg);
    case IMPM_ERR_SEEDING: throw SeedingFault(msg);
    case IMPM_ERR_UNSUPPORTED: throw UnsupportedOperation(msg);
    default: throw Error(msg);
  }
}
inline impm_options to_c(const SolverOptions& o, const GpuOptions& gpu) {
  impm_options c{};
  c.tol = o.tol;
  c.abs_floor = o.abs_floor;
  c.max_iterations = o.max_iterations;
  c.total_lagrangian = o.total_lagrangian ? 1 : 0;
  c.shape = IMPM_SHAPE_GIMP;
  c.krylov = gpu.krylov;
  c.krylov_rtol = gpu.krylov_rtol;
  c.precond = gpu.precond;
  c.strategy = o.strategy == JacobianStrategy::dense ? IMPM_STRATEGY_DENSE : IMPM_STRATEGY_SPARSE;
  c.interference = o.interference == InterferenceCheck::always    ? IMPM_INTERFERENCE_ALWAYS
                   : o.interference == InterferenceCheck::sampled ? IMPM_INTERFERENCE_SAMPLED
                                                                  : IMPM_INTERFERENCE_OFF;
  return c;
}
inline impm_material to_c(const MaterialSpec& m) {
  impm_material c{};
  c.kind = static_cast<std::int32_t>(m.kind);  // same order as materials.hpp:47
  c.E = m.elastic.E;
  c.nu = m.elastic.nu;
  c.kappa = m.kappa;
  c.friction_deg = 30.0;
  return c;
}
template <class R>
inline void set_krylov(R& s, int v) {  // impm::StepRecord has no Krylov count
  if constexpr (requires { s.krylov_iterations; }) s.krylov_iterations = v;
}
inline StepRecord from_c(const impm_step_record& r, const std::vector<double>& rel) {
  StepRecord s;
  s.step = r.step;
  s.iterations = r.iterations;
  s.rel_residuals.assign(rel.begin(), rel.begin() + std::min<int>(r.n_rel, static_cast<int>(rel.size())));
  s.r0_norm = r.r0_norm;
  s.seconds = r.seconds;
  s.diff_seconds = r.diff_seconds;
  s.backward_passes = r.backward_passes;
  set_krylov(s, r.krylov_iterations);
  return s;
}
}  // namespace detail

// impm::MpmSim<D> (mpm_solver.hpp:51-478), stepped on the GPU.
template <int D>
class MpmSim {
 public:
  Grid<D> grid;
  std::vector<Particle<D>> particles;
  MaterialSpec material;
  NodeVec<D> gravity{};
  SolverOptions options;
  std::vector<std::uint8_t> fixed;  // [node * D + comp]

  // mpm_solver.hpp:63-68 (+ optional GPU knobs)
  MpmSim(Grid<D> g, std::vector<Particle<D>> parts, MaterialSpec mat, SolverOptions opt = {}, GpuOptions gpu = {})
      : grid(g), particles(std::move(parts)), material(mat), options(opt) {
    fixed.assign(static_cast<std::size_t>(grid.node_count()) * D, 0);
    if (options.total_lagrangian && mat.kind == MaterialKind::hencky_j2)  // mpm_solver.hpp:66-67
      throw ConfigError("total-Lagrangian stepping supports elastic materials only");
    impm_grid cg{};
    cg.dim = D;
    for (int a = 0; a < 3; ++a) {
      cg.nodes[a] = a < D ? grid.nodes[a] : 1;
      cg.origin[a] = a < D ? grid.origin[a] : 0.0;
    }
    cg.h = grid.h;
    const impm_material cm = detail::to_c(mat);
    const impm_options co = detail::to_c(options, gpu);
    detail::check(impm_sim_create(&cg, &cm, &co, gpu.device, &h_), nullptr);
  }
  ~MpmSim() {
    if (h_) impm_sim_destroy(h_);
  }
  MpmSim(const MpmSim&) = delete;
  MpmSim& operator=(const MpmSim&) = delete;
  // movable, so that builders return it by value (src/scenarios.cpp:92-106)
  MpmSim(MpmSim&& o) noexcept
      : grid(o.grid), particles(std::move(o.particles)), material(o.material), gravity(o.gravity),
        options(o.options), fixed(std::move(o.fixed)), h_(o.h_), shadow_(std::move(o.shadow_)) {
    o.h_ = nullptr;
  }
  MpmSim& operator=(MpmSim&& o) noexcept {
    if (this != &o) {
      if (h_) impm_sim_destroy(h_);
      grid = o.grid;
      particles = std::move(o.particles);
      material = o.material;
      gravity = o.gravity;
      options = o.options;
      fixed = std::move(o.fixed);
      h_ = o.h_;
      shadow_ = std::move(o.shadow_);
      o.h_ = nullptr;
    }
    return *this;
  }

  template <class Pred>
  void fix_nodes(Pred&& predicate, int component = -1) {  // mpm_solver.hpp:70-78
    for (int n = 0; n < grid.node_count(); ++n) {
      if (!predicate(grid.node_pos(n))) continue;
      for (int c = 0; c < D; ++c)
        if (component < 0 || component == c) fixed[static_cast<std::size_t>(n) * D + c] = 1;
    }
  }

  void begin_step() {
    upload();
    detail::check(impm_sim_begin_step(h_), h_);
  }
  int n_dofs() const {
    std::int32_t n = 0;
    detail::check(impm_sim_n_dofs(h_, &n), h_);
    return n;
  }
  DofMap dofs() const {
    DofMap d;
    d.n_fields = D;
    d.n_dofs = n_dofs();
    d.dof_of.resize(static_cast<std::size_t>(grid.node_count()) * D);
    d.node_of.resize(d.n_dofs);
    d.field_of.resize(d.n_dofs);
    detail::check(impm_sim_dof_map(h_, d.dof_of.data(), d.node_of.data(), d.field_of.data()), h_);
    return d;
  }
  std::vector<double> node_mass() const {
    std::vector<double> m(grid.node_count());
    detail::check(impm_sim_node_mass(h_, m.data()), h_);
    return m;
  }
  std::vector<double> residual(const std::vector<double>& u, double load_scale) const {
    std::vector<double> r(n_dofs());
    detail::check(impm_sim_residual(h_, u.data(), load_scale, r.data()), h_);
    return r;
  }
  StepRecord newton_solve(double load_scale) {
    std::vector<double> rel(256);
    impm_step_record r{};
    r.rel_residuals = rel.data();
    r.rel_capacity = 256;
    detail::check(impm_sim_newton_solve(h_, load_scale, &r), h_);
    return detail::from_c(r, rel);
  }
  void commit_step() {
    detail::check(impm_sim_commit_step(h_), h_);
    download();
  }
  StepRecord step(double load_scale) {  // mpm_solver.hpp:402-407
    upload();
    std::vector<double> rel(256);
    impm_step_record r{};
    r.rel_residuals = rel.data();
    r.rel_capacity = 256;
    detail::check(impm_sim_step(h_, load_scale, &r), h_);
    download();
    return detail::from_c(r, rel);
  }
  std::vector<double> nodal_solution() const {
    std::vector<double> u(n_dofs());
    detail::check(impm_sim_nodal_solution(h_, u.data()), h_);
    return u;
  }
  void set_nodal_solution(const std::vector<double>& u) { detail::check(impm_sim_set_nodal_solution(h_, u.data()), h_); }
  impm_sim* handle() const { return h_; }

 private:
  void upload() {
    // particles are re-sent only when the caller changed them (a re-upload
    // resets the device connectivity, which total-Lagrangian runs keep)
    const std::size_t bytes = particles.size() * sizeof(Particle<D>);
    if (shadow_.size() != bytes || std::memcmp(shadow_.data(), particles.data(), bytes) != 0) {
      detail::check(impm_sim_set_particles(h_, reinterpret_cast<const double*>(particles.data()),
                                           static_cast<std::int64_t>(particles.size()), sizeof(Particle<D>)),
                    h_);
      shadow_.assign(reinterpret_cast<const char*>(particles.data()),
                     reinterpret_cast<const char*>(particles.data()) + bytes);
    }
    detail::check(impm_sim_set_fixed(h_, fixed.data()), h_);
    double g3[3] = {0, 0, 0};
    for (int a = 0; a < D; ++a) g3[a] = gravity[a];
    detail::check(impm_sim_set_gravity(h_, g3), h_);
  }
  void download() {
    detail::check(impm_sim_get_particles(h_, reinterpret_cast<double*>(particles.data()),
                                         static_cast<std::int64_t>(particles.size()), sizeof(Particle<D>)),
                  h_);
    shadow_.assign(reinterpret_cast<const char*>(particles.data()),
                   reinterpret_cast<const char*>(particles.data()) + particles.size() * sizeof(Particle<D>));
  }
  impm_sim* h_ = nullptr;
  std::vector<char> shadow_;
};

// ---- link-level seam (sparse.hpp:43): drop-in for impm::sparse_lu_solve ----
namespace detail {
inline void check_csr(impm_status st) {
  if (st == IMPM_OK) return;
  const std::string msg = impm_csr_last_error();
  if (st == IMPM_ERR_LINEAR_SOLVER) throw LinearSolverError(msg);
  if (st == IMPM_ERR_CONFIG) throw ConfigError(msg);
  throw Error(msg);
}
}  // namespace detail

// impm::sparse_lu_solve (src/linear_solver.cpp:11-88) on the GPU.
inline std::vector<double> sparse_lu_solve(const CsrMatrix& A, std::span<const double> b, int device = 0) {
  std::vector<double> x(static_cast<std::size_t>(A.n));
  if (A.n == 0) return x;
  detail::check_csr(impm_sparse_lu_solve(A.n, A.row_ptr.data(), A.cols.data(), A.vals.data(), b.data(),
                                         static_cast<std::int64_t>(b.size()), x.data(), device, nullptr));
  return x;
}
// CsrMatrix::multiply (src/sparse.cpp:44-53) on the GPU, bitwise the reference's sums.
inline std::vector<double> csr_multiply(const CsrMatrix& A, std::span<const double> x, int device = 0) {
  std::vector<double> y(static_cast<std::size_t>(A.n));
  detail::check_csr(impm_csr_multiply(A.n, A.row_ptr.data(), A.cols.data(), A.vals.data(), x.data(), y.data(), device));
  return y;
}
// CsrMatrix::transposed (src/sparse.cpp:55-70) on the GPU.
inline CsrMatrix csr_transposed(const CsrMatrix& A, int device = 0) {
  CsrMatrix t;
  t.n = A.n;
  t.row_ptr.assign(static_cast<std::size_t>(A.n) + 1, 0);
  t.cols.resize(A.cols.size());
  t.vals.resize(A.vals.size());
  detail::check_csr(impm_csr_transposed(A.n, A.row_ptr.data(), A.cols.data(), A.vals.data(), t.row_ptr.data(),
                                        t.cols.data(), t.vals.data(), device));
  return t;
}

}  // namespace impm_gpu
