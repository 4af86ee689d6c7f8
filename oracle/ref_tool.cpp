// ref_tool — driver linked against the UNMODIFIED reference core
// (/root/reference/proj/src/*.cpp + include/impm/*.hpp), built by
// oracle/Makefile into oracle/_ref/impm_ref.
//
// TEST INFRASTRUCTURE ONLY. It is the results oracle (golden fixtures under
// tests/golden/ are generated with it by tests/golden/make_golden.py) and the
// CPU baseline arm of bench.py ("kind": "reference"). Nothing in the product
// links or calls it.
//
//   impm_ref run   <cfg> [section.key=value ...]   run_scenario (tools/main.cpp:25-89)
//   impm_ref check <cfg> [section.key=value ...]   run_scenario with checks
//   impm_ref dump  <spec> <outdir>                 per-stage golden arrays (.npy)
//   impm_ref bench <spec> <seconds>                MpmSim::step timing (JSON line)
//
// <spec> is a tiny key=value file (see tests/golden/specs/*.spec) describing a
// seed_box problem (particle.hpp:33-69) on the survey's grid convention
// (origin -h, cells+3 nodes per axis, scenarios.cpp:96-98).
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "impm/config.hpp"
#include "impm/mpm_solver.hpp"
#include "impm/porous.hpp"
#include "impm/scenarios.hpp"

using namespace impm;
namespace fs = std::filesystem;

namespace {

// ---------------------------------------------------------------- npy out --
template <class T>
const char* npy_descr();
template <>
const char* npy_descr<double>() { return "<f8"; }
template <>
const char* npy_descr<std::int32_t>() { return "<i4"; }
template <>
const char* npy_descr<std::int64_t>() { return "<i8"; }
template <>
const char* npy_descr<std::uint8_t>() { return "|u1"; }

template <class T>
void write_npy(const std::string& path, const T* data, std::vector<std::size_t> shape) {
  std::string sh = "(";
  std::size_t count = 1;
  for (std::size_t i = 0; i < shape.size(); ++i) {
    sh += std::to_string(shape[i]);
    sh += (shape.size() == 1 || i + 1 < shape.size()) ? "," : "";
    if (i + 1 < shape.size()) sh += " ";
    count *= shape[i];
  }
  sh += ")";
  std::string header = std::string("{'descr': '") + npy_descr<T>() +
                       "', 'fortran_order': False, 'shape': " + sh + ", }";
  const std::size_t base = 10 + header.size() + 1;
  header.append((64 - base % 64) % 64, ' ');
  header += '\n';
  std::ofstream f(path, std::ios::binary);
  f.write("\x93NUMPY\x01\x00", 8);
  const std::uint16_t hl = static_cast<std::uint16_t>(header.size());
  f.write(reinterpret_cast<const char*>(&hl), 2);
  f.write(header.data(), header.size());
  f.write(reinterpret_cast<const char*>(data), count * sizeof(T));
}
template <class T>
void write_vec(const std::string& dir, const std::string& name, const std::vector<T>& v) {
  write_npy(dir + "/" + name + ".npy", v.data(), {v.size()});
}

// ------------------------------------------------------------------ spec --
struct Spec {
  std::map<std::string, std::string> kv;
  std::string get(const std::string& k, const std::string& d) const {
    auto it = kv.find(k);
    return it == kv.end() ? d : it->second;
  }
  double num(const std::string& k, double d) const {
    auto it = kv.find(k);
    return it == kv.end() ? d : std::stod(it->second);
  }
  std::vector<double> list(const std::string& k, std::vector<double> d) const {
    auto it = kv.find(k);
    if (it == kv.end()) return d;
    std::vector<double> out;
    std::stringstream ss(it->second);
    std::string item;
    while (std::getline(ss, item, ',')) out.push_back(std::stod(item));
    return out;
  }
};

Spec read_spec(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw std::runtime_error("cannot open spec " + path);
  Spec s;
  std::string line;
  while (std::getline(f, line)) {
    const auto hash = line.find('#');
    if (hash != std::string::npos) line = line.substr(0, hash);
    const auto eq = line.find('=');
    if (eq == std::string::npos) continue;
    auto trim = [](std::string x) {
      while (!x.empty() && std::isspace(static_cast<unsigned char>(x.back()))) x.pop_back();
      std::size_t a = 0;
      while (a < x.size() && std::isspace(static_cast<unsigned char>(x[a]))) ++a;
      return x.substr(a);
    };
    s.kv[trim(line.substr(0, eq))] = trim(line.substr(eq + 1));
  }
  return s;
}

MaterialKind kind_of(const std::string& m) {
  if (m == "hencky") return MaterialKind::hencky;
  if (m == "hencky_j2") return MaterialKind::hencky_j2;
  if (m == "neo_hookean") return MaterialKind::neo_hookean;
  throw ConfigError("unknown material " + m);
}

template <int D>
MpmSim<D> build(const Spec& s) {
  const auto cells = s.list("cells", {8, 8, 8});
  const double h = s.num("h", 1.0);
  const int ppc = static_cast<int>(s.num("ppc", 2));
  Grid<D> grid;
  grid.h = h;
  Vec<double, D> lo{}, hi{};
  for (int a = 0; a < D; ++a) {
    grid.origin[a] = -h;
    grid.nodes[a] = static_cast<int>(cells[a]) + 3;
    lo[a] = 0.0;
    hi[a] = cells[a] * h;
  }
  auto parts = seed_box<D>(grid, lo, hi, ppc, s.num("rho", 2000.0));
  // slope filter (cfg 2): keep y <= y0 + (x - x0) tan(beta) measured from the toe
  const double slope_deg = s.num("slope_deg", 0.0);
  if (slope_deg > 0.0 && D >= 2) {
    const double tb = std::tan(slope_deg * M_PI / 180.0);
    const double x0 = s.num("slope_x0", 0.0), y0 = s.num("slope_y0", 0.0);
    std::vector<Particle<D>> kept;
    for (const auto& p : parts)
      if (p.X[1] <= y0 + (p.X[0] - x0) * tb || p.X[1] <= y0) kept.push_back(p);
    parts.swap(kept);
  }
  const double jitter = s.num("jitter", 0.0);
  if (jitter > 0.0) {
    std::mt19937 rng(static_cast<unsigned>(s.num("seed", 2507)));
    std::uniform_real_distribution<double> U(-jitter, jitter);
    const double spacing = h / ppc;
    for (auto& p : parts)
      for (int a = 0; a < D; ++a) {
        p.X[a] += U(rng) * spacing;
        p.x[a] = p.X[a];
      }
  }
  MaterialSpec mat;
  mat.kind = kind_of(s.get("material", "neo_hookean"));
  mat.elastic = {s.num("E", 10e6), s.num("nu", 0.3)};
  mat.kappa = s.num("kappa", 0.0);
  SolverOptions opt;
  opt.tol = s.num("tol", 1e-10);
  opt.max_iterations = static_cast<int>(s.num("max_iterations", 20));
  opt.total_lagrangian = s.num("total_lagrangian", 0) != 0;
  MpmSim<D> sim(grid, std::move(parts), mat, opt);
  const std::string bc = s.get("bc", "column");
  if (bc == "column") {
    // base fixed, lateral rollers (src/inverse.cpp:33-36 pattern)
    const int up = D - 1;
    sim.fix_nodes([up](const Vec<double, D>& x) { return x[up] <= 1e-12; });
    for (int a = 0; a < D - 1; ++a) {
      const double w = cells[a] * h;
      sim.fix_nodes([a, w](const Vec<double, D>& x) { return x[a] <= 1e-12 || x[a] >= w - 1e-12; }, a);
    }
  } else if (bc == "wall") {
    sim.fix_nodes([](const Vec<double, D>& x) { return x[0] <= 1e-12; });
  }
  const auto g = s.list("gravity", {});
  if (!g.empty()) {
    for (int a = 0; a < D; ++a) sim.gravity[a] = g[a];
  } else {
    sim.gravity[D - 1] = -9.81;
  }
  // strip traction on the top particle layer (footing, src/inverse.cpp:45-61 pattern)
  const double t_hat = s.num("t_hat", 0.0);
  if (t_hat != 0.0) {
    const double frac = s.num("strip_fraction", 0.25);
    // strip_axes = number of leading lateral axes the strip is narrow in
    // (default all D-1: a centred patch; 1: a strip along axis 0 only, the
    // cfg 4 footing of paper_2507_09435_b200/workloads.py:_strip_traction)
    const int narrow = static_cast<int>(s.num("strip_axes", D - 1));
    double top = -1e300;
    for (const auto& p : sim.particles) top = std::max(top, p.X[D - 1]);
    std::vector<std::size_t> strip;
    for (std::size_t pi = 0; pi < sim.particles.size(); ++pi) {
      const auto& p = sim.particles[pi];
      bool in = p.X[D - 1] >= top - 1e-9;
      for (int a = 0; a < narrow && in; ++a) {
        const double w = cells[a] * h;
        in = p.X[a] >= 0.5 * w * (1 - frac) && p.X[a] <= 0.5 * w * (1 + frac);
      }
      if (in) strip.push_back(pi);
    }
    double area = 1.0;
    for (int a = 0; a < D - 1; ++a) area *= cells[a] * h * (a < narrow ? frac : 1.0);
    for (std::size_t pi : strip)
      sim.particles[pi].traction_force[D - 1] = -t_hat * area / strip.size();
  }
  return sim;
}

template <int D>
std::vector<double> particle_blob(const std::vector<Particle<D>>& ps) {
  constexpr std::size_t nd = sizeof(Particle<D>) / sizeof(double);
  static_assert(sizeof(Particle<D>) % sizeof(double) == 0);
  std::vector<double> out(ps.size() * nd);
  std::memcpy(out.data(), ps.data(), ps.size() * sizeof(Particle<D>));
  return out;
}

template <int D>
void dump_case(const Spec& s, const std::string& dir) {
  fs::create_directories(dir);
  auto sim = build<D>(s);
  constexpr std::size_t nd = sizeof(Particle<D>) / sizeof(double);
  {
    // [origin x3, h, nodes x3], padded with (0, 1) beyond D
    std::vector<double> g{0.0, 0.0, 0.0, sim.grid.h, 1.0, 1.0, 1.0};
    for (int a = 0; a < D; ++a) {
      g[a] = sim.grid.origin[a];
      g[4 + a] = sim.grid.nodes[a];
    }
    write_vec(dir, "grid", g);
    std::vector<double> grav(sim.gravity.e.begin(), sim.gravity.e.end());
    write_vec(dir, "gravity", grav);
    write_vec(dir, "fixed", sim.fixed);
    const auto blob = particle_blob<D>(sim.particles);
    write_npy(dir + "/particles0.npy", blob.data(), {sim.particles.size(), nd});
    std::vector<double> mat{double(static_cast<int>(sim.material.kind)), sim.material.elastic.E,
                            sim.material.elastic.nu, sim.material.kappa, sim.options.tol,
                            double(sim.options.max_iterations), sim.options.total_lagrangian ? 1.0 : 0.0};
    write_vec(dir, "material", mat);
  }
  const double s0 = s.num("probe_scale", 0.5);
  sim.begin_step();
  write_vec(dir, "node_mass", sim.node_mass());
  write_vec(dir, "dof_of", sim.dofs().dof_of);
  write_vec(dir, "node_of", sim.dofs().node_of);
  write_vec(dir, "field_of", sim.dofs().field_of);
  const int n = sim.n_dofs();
  {
    const auto& pat = sim.assembler().pattern();
    std::vector<std::int64_t> rp(n + 1, 0);
    std::vector<std::int32_t> cols;
    for (int d = 0; d < n; ++d) {
      rp[d + 1] = rp[d] + static_cast<std::int64_t>(pat[d].size());
      cols.insert(cols.end(), pat[d].begin(), pat[d].end());
    }
    write_vec(dir, "row_ptr", rp);
    write_vec(dir, "cols", cols);
  }
  std::vector<double> u0(n, 0.0);
  write_vec(dir, "r0", sim.residual(u0, s0));
  // probe state: small smooth random displacement
  std::mt19937 rng(7);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  const double amp = s.num("probe_amp", 1e-3) * sim.grid.h;
  std::vector<double> u1(n);
  for (int d = 0; d < n; ++d) u1[d] = amp * U(rng);
  write_vec(dir, "u1", u1);
  write_vec(dir, "r1", sim.residual(u1, s0));
  {
    ad::Tape tape;
    sim.record_residual(u1, s0, tape);
    JacobianStats st;
    const CsrMatrix J = sim.assembler().sparse(tape, &st, InterferenceCheck::always);
    write_vec(dir, "J1_vals", J.vals);
    std::vector<std::int32_t> passes{st.total_passes, st.passes_per_field};
    write_vec(dir, "passes", passes);
    // colour groups (jacobian.hpp:101-110), observed through the reference's
    // own sparse(): on a probe tape r_i = w_i * sum_j u_j (generic weights
    // w_i), every entry of seeded row d equals the sum of w over d's group,
    // so two dofs share a group iff their rows hold the same value
    {
      ad::Tape probe_tape;
      std::vector<ad::Var> in;
      in.reserve(n);
      for (int d = 0; d < n; ++d) in.push_back(probe_tape.input(0.0));
      ad::Var sum = in.empty() ? ad::Var() : in[0];
      for (int d = 1; d < n; ++d) sum = sum + in[d];
      std::mt19937 wr(2507);
      std::uniform_real_distribution<double> W(1.0, 2.0);
      std::vector<ad::Var> outs;
      outs.reserve(n);
      for (int d = 0; d < n; ++d) outs.push_back(sum * W(wr));
      probe_tape.set_outputs(outs);
      JacobianStats pst;
      const CsrMatrix G = sim.assembler().sparse(probe_tape, &pst);
      std::vector<double> colour_probe(n);
      for (int d = 0; d < n; ++d) colour_probe[d] = G.vals[G.row_ptr[d]];
      write_vec(dir, "colour_probe", colour_probe);
      std::vector<std::int32_t> cpasses{pst.total_passes, pst.passes_per_field};
      write_vec(dir, "colour_passes", cpasses);
    }
    // the linear solve at the probe (the seam sparse_lu_solve replaces)
    std::vector<double> r1 = sim.residual(u1, s0), rhs(n);
    for (int i = 0; i < n; ++i) rhs[i] = -r1[i];
    write_vec(dir, "delta1", sparse_lu_solve(J, rhs));
  }
  // G2P at the probe state on a copy (commit_step, mpm_solver.hpp:359-400)
  {
    MpmSim<D> probe = sim;
    probe.set_nodal_solution(u1);
    probe.commit_step();
    const auto blob = particle_blob<D>(probe.particles);
    write_npy(dir + "/particles_commit1.npy", blob.data(), {probe.particles.size(), nd});
  }
  // Newton trace over the load schedule
  const int steps = static_cast<int>(s.num("steps", 2));
  std::vector<std::int32_t> iters;
  std::vector<double> rels, r0s;
  std::vector<std::int32_t> ndofs;
  std::vector<double> u_last;
  for (int k = 1; k <= steps; ++k) {
    const StepRecord rec = sim.step(static_cast<double>(k) / steps);
    iters.push_back(rec.iterations);
    ndofs.push_back(sim.n_dofs());
    r0s.push_back(rec.r0_norm);
    for (double r : rec.rel_residuals) rels.push_back(r);
    if (k == 1) {
      u_last = sim.nodal_solution();
      write_vec(dir, "u_step1", u_last);
      const auto blob = particle_blob<D>(sim.particles);
      write_npy(dir + "/particles_step1.npy", blob.data(), {sim.particles.size(), nd});
    }
  }
  write_vec(dir, "newton_iters", iters);
  write_vec(dir, "newton_rel", rels);
  write_vec(dir, "newton_r0", r0s);
  write_vec(dir, "step_ndofs", ndofs);
  const auto blob = particle_blob<D>(sim.particles);
  write_npy(dir + "/particles_final.npy", blob.data(), {sim.particles.size(), nd});
}

// coupled u-p column (scenarios.cpp:387-418 build_column), small
void dump_coupled(const Spec& s, const std::string& dir) {
  fs::create_directories(dir);
  const std::string cfg_text =
      "scenario = consolidation\n[geometry]\nheight = " + s.get("height", "10") +
      "\ncells = " + s.get("cells", "10") +
      "\nparticles_per_cell = 2\n[material]\nlambda = 600 kPa\nmu = 600 kPa\nk = 1e-12\nmu_f = 0.1\n"
      "[schedule]\nt_hat = 1 kPa\ndt0 = 100 s\nTv_checkpoints = 0.05\nTv_end = 0.05\n";
  (void)cfg_text;
  const double H = s.num("height", 10.0);
  const int cells = static_cast<int>(s.num("cells", 10));
  const double h = H / cells;
  Grid<2> grid;
  grid.h = h;
  grid.origin = Vec2d{{-h, -h}};
  grid.nodes = {static_cast<int>(s.num("width_cells", 1)) + 3, cells + 3};
  PoroParams pp{s.num("lambda", 600e3), s.num("mu", 600e3), s.num("k", 1e-12), s.num("mu_f", 0.1),
                s.num("rho_f", 1000.0)};
  const double W = s.num("width_cells", 1) * h;
  auto parts = seed_box<2>(grid, Vec2d{{0.0, 0.0}}, Vec2d{{W, H}}, 2, 2000.0);
  SolverOptions opt;
  opt.tol = s.num("tol", 1e-10);
  CoupledSim sim(grid, std::move(parts), pp, opt);
  sim.fix_displacement([](const Vec2d&) { return true; }, 0);
  sim.fix_displacement([](const Vec2d& x) { return x[1] <= 1e-12; });
  sim.fix_pressure([H](const Vec2d& x) { return x[1] >= H - 1e-9; });
  sim.gravity = Vec2d{{0.0, s.num("gy", 0.0)}};
  const double t_hat = s.num("t_hat", 1e3);
  double top_y = -1e300;
  for (const auto& p : sim.particles) top_y = std::max(top_y, p.X[1]);
  std::vector<std::size_t> top;
  for (std::size_t pi = 0; pi < sim.particles.size(); ++pi)
    if (sim.particles[pi].X[1] >= top_y - 1e-9) top.push_back(pi);
  for (std::size_t pi : top)
    sim.particles[pi].traction_force = Vec2d{{0.0, -t_hat * W / top.size()}};
  {
    std::vector<double> g{grid.origin[0], grid.origin[1], 0.0, grid.h, double(grid.nodes[0]),
                          double(grid.nodes[1]), 1.0};
    write_vec(dir, "grid", g);
    std::vector<double> grav(sim.gravity.e.begin(), sim.gravity.e.end());
    write_vec(dir, "gravity", grav);
    write_vec(dir, "fixed_u", sim.fixed_u);
    write_vec(dir, "fixed_p", sim.fixed_p);
    std::vector<double> poro{pp.lambda, pp.mu, pp.k, pp.mu_f, pp.rho_f, opt.tol};
    write_vec(dir, "poro", poro);
    const auto blob = particle_blob<2>(sim.particles);
    write_npy(dir + "/particles0.npy", blob.data(), {sim.particles.size(), sizeof(Particle<2>) / 8});
  }
  sim.initialize();
  const int n = sim.n_dofs();
  write_vec(dir, "dof_of", sim.dofs().dof_of);
  {
    const auto& pat = sim.assembler().pattern();
    std::vector<std::int64_t> rp(n + 1, 0);
    std::vector<std::int32_t> cols;
    for (int d = 0; d < n; ++d) {
      rp[d + 1] = rp[d] + static_cast<std::int64_t>(pat[d].size());
      cols.insert(cols.end(), pat[d].begin(), pat[d].end());
    }
    write_vec(dir, "row_ptr", rp);
    write_vec(dir, "cols", cols);
  }
  const double dt = s.num("dt", 100.0);
  std::mt19937 rng(11);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  std::vector<double> x1(n);
  for (int d = 0; d < n; ++d) x1[d] = (sim.dofs().field_of[d] == 2 ? 500.0 : 1e-4) * U(rng);
  write_vec(dir, "x1", x1);
  write_vec(dir, "r1", sim.residual(x1, dt));
  {
    ad::Tape tape;
    sim.record_residual(x1, dt, tape);
    JacobianStats st;
    const CsrMatrix J = sim.assembler().sparse(tape, &st, InterferenceCheck::always);
    write_vec(dir, "J1_vals", J.vals);
  }
  const int steps = static_cast<int>(s.num("steps", 5));
  std::vector<std::int32_t> iters;
  std::vector<double> rels, settle;
  for (int k = 1; k <= steps; ++k) {
    const StepRecord rec = sim.step(dt);
    iters.push_back(rec.iterations);
    for (double r : rec.rel_residuals) rels.push_back(r);
    settle.push_back(sim.top_settlement());
  }
  write_vec(dir, "newton_iters", iters);
  write_vec(dir, "newton_rel", rels);
  write_vec(dir, "settlement", settle);
  write_vec(dir, "p_nodes", sim.nodal_pressure());
  const auto blob = particle_blob<2>(sim.particles);
  write_npy(dir + "/particles_final.npy", blob.data(), {sim.particles.size(), sizeof(Particle<2>) / 8});
}

// Times MpmSim::step on the spec'd problem until `budget` seconds are spent;
// prints one JSON line with the reference's own StepRecord counters.
template <int D>
int bench_case(const Spec& s, double budget) {
  auto sim = build<D>(s);
  const int steps = static_cast<int>(s.num("steps", 10));
  long iters = 0;
  double secs = 0.0, diff = 0.0;
  int done = 0;
  std::int64_t nnz = 0;
  const auto t0 = std::chrono::steady_clock::now();
  for (int k = 1; k <= steps; ++k) {
    const auto ts = std::chrono::steady_clock::now();
    const StepRecord rec = sim.step(static_cast<double>(k) / steps);
    secs += std::chrono::duration<double>(std::chrono::steady_clock::now() - ts).count();
    iters += rec.iterations;
    diff += rec.diff_seconds;
    ++done;
    // nnz of the pattern used by this step (assembler is rebuilt at begin_step)
    std::int64_t z = 0;
    for (const auto& row : sim.assembler().pattern()) z += static_cast<std::int64_t>(row.size());
    nnz += z * rec.iterations;
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > budget) break;
  }
  std::printf(
      "{\"particles\": %zu, \"load_steps\": %d, \"newton_iterations\": %ld, \"step_seconds\": %.6f, "
      "\"diff_seconds\": %.6f, \"nnz_assembled\": %lld, \"newton_per_s\": %.6g, \"nnz_per_s\": %.6g}\n",
      sim.particles.size(), done, iters, secs, diff, static_cast<long long>(nnz),
      iters / secs, diff > 0 ? nnz / diff : 0.0);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 3) {
      std::fprintf(stderr, "usage: impm_ref run|check|dump|bench ...\n");
      return 2;
    }
    const std::string cmd = argv[1];
    if (cmd == "run" || cmd == "check") {
      Config cfg = Config::parse_file(argv[2]);
      for (int i = 3; i < argc; ++i) cfg.set_override(argv[i]);
      const RunReport rep = run_scenario(cfg, cmd == "check");
      for (const auto& c : rep.checks)
        std::printf("[%s] %s measured %.9g expected %.9g\n", c.pass ? "PASS" : "FAIL",
                    c.name.c_str(), c.measured, c.expected);
      std::printf("%s: %d steps in %.3f s\n", rep.scenario.c_str(), rep.steps, rep.wall_s);
      return rep.all_pass() ? 0 : 1;
    }
    const Spec s = read_spec(argv[2]);
    const int dim = static_cast<int>(s.num("dim", 2));
    if (cmd == "dump") {
      if (argc < 4) return 2;
      if (s.get("kind", "mpm") == "coupled") {
        dump_coupled(s, argv[3]);
      } else if (dim == 1) {
        dump_case<1>(s, argv[3]);
      } else if (dim == 2) {
        dump_case<2>(s, argv[3]);
      } else {
        dump_case<3>(s, argv[3]);
      }
      return 0;
    }
    if (cmd == "bench") {
      const double budget = argc > 3 ? std::stod(argv[3]) : 20.0;
      if (dim == 1) return bench_case<1>(s, budget);
      if (dim == 2) return bench_case<2>(s, budget);
      return bench_case<3>(s, budget);
    }
    std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
    return 2;
  } catch (const NonConvergenceError& e) {
    std::fprintf(stderr, "solver did not converge: %s\n", e.what());
    for (double r : e.residual_history) std::fprintf(stderr, "  rel %.3e\n", r);
    return 2;
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
}
