// The reference's bar scenario (src/scenarios.cpp:92-142: build_bar + the
// stepping loop of run_bar) with exactly one change: the simulation type is
// impm_gpu::MpmSim<1> (include/impm_gpu.hpp in IMPM_GPU_REFERENCE_TYPES mode)
// instead of impm::MpmSim<1>. Every other type is the reference's own
// (impm::Grid, impm::Vec, impm::seed_box, impm::MaterialSpec,
// impm::SolverOptions, impm::StepRecord). Compiled against
// /root/reference/proj/include by __graft_entry__.build(); run by
// tests/test_gpu_facade.py against the committed out/bar_elastic outputs.
//
//   bar_swap height cells ppc E nu rho0 steps gravity tol max_iterations
// prints "it <step> <iterations>" per load step, then one
// "p Y_ref y sigma_yy sigma_xx F_yy V" line per particle (particles.csv).
#define IMPM_GPU_REFERENCE_TYPES
#include "impm_gpu.hpp"

#include <cstdio>
#include <cstdlib>

namespace scenarios {
using namespace impm;
template <int D>
using MpmSim = impm_gpu::MpmSim<D>;  // <- the swap

struct BarCfg {
  double height, E, nu, rho0, gravity, tol;
  int cells, ppc, steps, max_iterations;
};

MpmSim<1> build_bar(const BarCfg& cfg, int cells) {  // scenarios.cpp:92-106
  const double l0 = cfg.height;
  const int ppc = cfg.ppc;
  Grid<1> grid;
  grid.h = l0 / cells;
  grid.origin = Vec<double, 1>{{-grid.h}};
  grid.nodes = {cells + 3};
  auto parts = seed_box<1>(grid, Vec<double, 1>{{0.0}}, Vec<double, 1>{{l0}}, ppc, cfg.rho0);
  MaterialSpec mat;  // bar_material (scenarios.cpp:78-90), model = hencky
  mat.kind = MaterialKind::hencky;
  mat.elastic = {cfg.E, cfg.nu};
  SolverOptions opt;  // solver_options (scenarios.cpp:66-72)
  opt.tol = cfg.tol;
  opt.max_iterations = cfg.max_iterations;
  opt.strategy = JacobianStrategy::sparse;
  MpmSim<1> sim(grid, std::move(parts), mat, opt);
  sim.fix_nodes([](const Vec<double, 1>& x) { return x[0] <= 1e-12; });
  sim.gravity = Vec<double, 1>{{-cfg.gravity}};
  return sim;
}

}  // namespace scenarios

int main(int argc, char** argv) {
  using namespace scenarios;
  if (argc < 11) {
    std::fprintf(stderr, "usage: bar_swap height cells ppc E nu rho0 steps gravity tol max_iterations\n");
    return 2;
  }
  BarCfg cfg{std::atof(argv[1]), std::atof(argv[4]), std::atof(argv[5]), std::atof(argv[6]),
             std::atof(argv[8]), std::atof(argv[9]), std::atoi(argv[2]), std::atoi(argv[3]),
             std::atoi(argv[7]), std::atoi(argv[10])};
  try {
    auto sim = build_bar(cfg, cfg.cells);  // run_bar (scenarios.cpp:119-142)
    for (int k = 1; k <= cfg.steps; ++k) {
      const StepRecord rec = sim.step(static_cast<double>(k) / cfg.steps);
      std::printf("it %d %d\n", rec.step, rec.iterations);
    }
    for (const auto& p : sim.particles)
      std::printf("p %.17g %.17g %.17g %.17g %.17g %.17g\n", p.X[0], p.x[0], p.sigma(0, 0), p.sigma(1, 1), p.F(0, 0),
                  p.V);
  } catch (const Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
