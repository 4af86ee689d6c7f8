// Drop-in check of include/impm_gpu.hpp: the smoke3d scenario
// (scenarios.cpp:690-716) written against the facade exactly as a caller of
// impm::MpmSim<3> would, stepped on the GPU. Prints "n_dof iterations".
#include <cstdio>

#include "impm_gpu.hpp"

int main() {
  using namespace impm_gpu;
  const double h = 0.25;
  Grid<3> grid;
  grid.h = h;
  grid.origin = {-h, -h, -h};
  grid.nodes = {7, 7, 7};
  std::vector<Particle<3>> parts;
  const double sp = h / 2, vol = sp * sp * sp;
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j)
      for (int k = 0; k < 8; ++k) {  // seed_box (particle.hpp:33-69), last axis fastest
        Particle<3> p;
        p.X = {(i + 0.5) * sp, (j + 0.5) * sp, (k + 0.5) * sp};
        p.x = p.X;
        p.lp0 = p.lp = {0.5 * sp, 0.5 * sp, 0.5 * sp};
        p.V0 = p.V = vol;
        p.m = 1500.0 * vol;
        parts.push_back(p);
      }
  MaterialSpec mat;
  mat.kind = MaterialKind::neo_hookean;
  mat.elastic = {1e6, 0.3};
  SolverOptions opt;
  opt.tol = 1e-9;
  MpmSim<3> sim(grid, parts, mat, opt);
  sim.fix_nodes([](const std::array<double, 3>& x) { return x[2] <= 1e-12; });
  sim.gravity = {0.0, 0.0, -9.81};
  try {
    const StepRecord rec = sim.step(1.0);
    // link-level seam: the 2x2 hand solve of test_linear_solver.cpp:60-65, and
    // the singular matrix of :92-97 -> LinearSolverError
    CsrMatrix A;
    A.n = 2;
    A.row_ptr = {0, 2, 4};
    A.cols = {0, 1, 0, 1};
    A.vals = {2.0, 1.0, 1.0, 2.0};
    const std::vector<double> b{3.0, 3.0};
    const std::vector<double> x = sparse_lu_solve(A, b);
    A.vals = {1.0, 2.0, 2.0, 4.0};
    bool threw = false;
    try {
      (void)sparse_lu_solve(A, std::vector<double>{1.0, 2.0});
    } catch (const LinearSolverError&) {
      threw = true;
    }
    std::printf("%d %d %.17g %.17g %d\n", sim.n_dofs(), rec.iterations, x[0], x[1], threw ? 1 : 0);
  } catch (const Error& e) {
    std::printf("error: %s\n", e.what());
    return 1;
  }
  return 0;
}
