// Substitute for the reference's Eigen-backed `impm::sparse_lu_solve`
// (/root/reference/proj/src/linear_solver.cpp:11-88). Eigen3 is not present
// in this image, so the reference core is linked against this file instead.
//
// TEST INFRASTRUCTURE ONLY: compiled into oracle/_ref (the reference build used
// as the results oracle and the CPU baseline); never linked into the product.
//
// Contract kept from linear_solver.cpp:
//   * row equilibration by max |a_ij| (linear_solver.cpp:16-23), empty row ->
//     LinearSolverError;
//   * pivoted LU of the scaled matrix (here: banded LU with partial pivoting,
//     LAPACK dgbtrf layout, instead of Eigen SparseLU's supernodal LU);
//   * normwise backward error |Ax-b| / (|A|_inf |x|_inf + |b|), up to two
//     refinement sweeps while it exceeds 1e-14, LinearSolverError above 1e-10
//     (linear_solver.cpp:55-85).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "impm/sparse.hpp"

namespace impm {

namespace {

struct BandLU {
  int n = 0, kl = 0, ku = 0, ldab = 0;
  std::vector<double> ab;  // column-major band storage, (2kl+ku+1) x n
  std::vector<int> piv;

  double& at(int i, int j) { return ab[static_cast<std::size_t>(j) * ldab + (kl + ku + i - j)]; }

  void factor() {
    const int kv = ku + kl;
    piv.assign(n, 0);
    for (int j = 0; j < n; ++j) {
      const int km = std::min(kl, n - 1 - j);
      // pivot search in column j, rows j..j+km
      int p = j;
      double best = std::abs(at(j, j));
      for (int i = j + 1; i <= j + km; ++i)
        if (std::abs(at(i, j)) > best) {
          best = std::abs(at(i, j));
          p = i;
        }
      piv[j] = p;
      if (best == 0.0) throw LinearSolverError("singular factorization: zero pivot in column " + std::to_string(j));
      const int jlast = std::min(n - 1, j + kv);
      if (p != j)
        for (int c = j; c <= jlast; ++c) std::swap(at(j, c), at(p, c));
      const double inv = 1.0 / at(j, j);
      for (int i = j + 1; i <= j + km; ++i) at(i, j) *= inv;
      for (int c = j + 1; c <= jlast; ++c) {
        const double ujc = at(j, c);
        if (ujc == 0.0) continue;
        for (int i = j + 1; i <= j + km; ++i) at(i, c) -= at(i, j) * ujc;
      }
    }
  }

  void solve(std::vector<double>& x) {
    const int kv = ku + kl;
    for (int j = 0; j < n; ++j) {
      const int p = piv[j];
      if (p != j) std::swap(x[j], x[p]);
      const int km = std::min(kl, n - 1 - j);
      for (int i = j + 1; i <= j + km; ++i) x[i] -= at(i, j) * x[j];
    }
    for (int j = n - 1; j >= 0; --j) {
      x[j] /= at(j, j);
      const int lo = std::max(0, j - kv);
      for (int i = lo; i < j; ++i) x[i] -= at(i, j) * x[j];
    }
  }
};

}  // namespace

std::vector<double> sparse_lu_solve(const CsrMatrix& A, std::span<const double> b) {
  if (A.n == 0) return {};
  if (static_cast<int>(b.size()) != A.n)
    throw LinearSolverError("right-hand side size does not match the matrix dimension");
  std::vector<double> row_scale(A.n, 0.0);
  int kl = 0, ku = 0;
  for (int i = 0; i < A.n; ++i) {
    for (std::int64_t k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k) {
      row_scale[i] = std::max(row_scale[i], std::abs(A.vals[k]));
      kl = std::max(kl, i - A.cols[k]);
      ku = std::max(ku, A.cols[k] - i);
    }
    if (row_scale[i] == 0.0) throw LinearSolverError("empty matrix row " + std::to_string(i));
  }
  BandLU lu;
  lu.n = A.n;
  lu.kl = kl;
  lu.ku = ku;
  lu.ldab = 2 * kl + ku + 1;
  lu.ab.assign(static_cast<std::size_t>(lu.ldab) * A.n, 0.0);
  for (int i = 0; i < A.n; ++i)
    for (std::int64_t k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k)
      lu.at(i, A.cols[k]) = A.vals[k] / row_scale[i];
  lu.factor();

  std::vector<double> x(b.begin(), b.end());
  for (int i = 0; i < A.n; ++i) x[i] /= row_scale[i];
  lu.solve(x);

  double rhs_norm = 0.0;
  for (double v : b) rhs_norm += v * v;
  rhs_norm = std::sqrt(rhs_norm);
  if (rhs_norm > 0.0) {
    double mat_norm = 0.0;
    for (int i = 0; i < A.n; ++i) {
      double row = 0.0;
      for (std::int64_t k = A.row_ptr[i]; k < A.row_ptr[i + 1]; ++k) row += std::abs(A.vals[k]);
      mat_norm = std::max(mat_norm, row);
    }
    auto residual = [&](const std::vector<double>& sol) {
      std::vector<double> r = A.multiply(sol);
      for (int i = 0; i < A.n; ++i) r[i] = b[i] - r[i];
      return r;
    };
    auto backward_error = [&](const std::vector<double>& sol) {
      const std::vector<double> r = residual(sol);
      double rn = 0.0, xinf = 0.0;
      for (double v : r) rn += v * v;
      for (double v : sol) xinf = std::max(xinf, std::abs(v));
      return std::sqrt(rn) / (mat_norm * xinf + rhs_norm);
    };
    double res = backward_error(x);
    for (int sweep = 0; sweep < 2 && res > 1e-14; ++sweep) {
      std::vector<double> rs = residual(x);
      for (int i = 0; i < A.n; ++i) rs[i] /= row_scale[i];
      lu.solve(rs);
      for (int i = 0; i < A.n; ++i) x[i] += rs[i];
      res = backward_error(x);
    }
    if (!(res <= 1e-10)) {
      char buf[32];
      std::snprintf(buf, sizeof buf, "%.3e", res);
      throw LinearSolverError("solution backward error " + std::string(buf) +
                              " exceeds 1e-10; matrix is ill-conditioned or singular");
    }
  }
  return x;
}

}  // namespace impm
