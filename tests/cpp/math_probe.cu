// Host-side probe of the device constitutive code (csrc/impm_math.cuh is
// __host__ __device__): compiled by nvcc for the HOST only and loaded by
// tests/test_math_cpu.py to check the 3x3 spectral log/exp and the Cam-Clay /
// Drucker-Prager / J2 return maps (values, dual-number tangents vs finite
// differences, admissibility, objectivity) without a GPU. Test harness only;
// the product runs these functions inside libimpm_gpu.so's kernels.
#include <cmath>
#include <cstring>

#include "../../paper_2507_09435_b200/csrc/impm_math.cuh"

using namespace impm_gpu;

extern "C" {

// out = f(B) (fn 0 = log, 1 = exp); dout[k*9..] = directional derivative along dB[k] (K = 3 directions)
void probe_sym_fun3(const double* B, const double* dB, int fn, double* out, double* dout) {
  Mat<Dual<3>, 3> b;
  for (int i = 0; i < 9; ++i) {
    b.e[i].v = B[i];
    for (int k = 0; k < 3; ++k) b.e[i].d[k] = dB[k * 9 + i];
  }
  const Mat<Dual<3>, 3> r = sym_fun3(b, fn);
  Mat<double, 3> bv;
  for (int i = 0; i < 9; ++i) bv.e[i] = B[i];
  const Mat<double, 3> rv = sym_fun3(bv, fn);
  for (int i = 0; i < 9; ++i) {
    out[i] = rv.e[i];
    for (int k = 0; k < 3; ++k) dout[k * 9 + i] = r.e[i].d[k];
  }
  // the value path of the dual overload must equal the double overload
  for (int i = 0; i < 9; ++i)
    if (r.e[i].v != rv.e[i]) out[i] = NAN;
}

void probe_eig3(const double* B, double* l, double* Q) { sym_eig3(B, l, Q); }

// kind: 0 hencky, 1 j2, 3 DP, 4 Cam-Clay, 2 neo-Hookean; 3D, total F = f_inc * F_n.
// params: lam, mu, kappa, dp_alpha, dp_ec, M, pc0, theta, pt
// Be_n[10] (alpha at [9]). Outputs sigma[9], J, Be_out[9], dg, and dsigma/dG[9][9] by duals (K = 9).
void probe_stress3(int kind, const double* f_inc, const double* F_n, const double* Be_n, const double* prm,
                   double* sigma, double* J, double* Be_out, double* dg, double* dsig) {
  const double lam = prm[0], mu = prm[1];
  auto eval = [&](auto tag, const double* seed_dirs, double* s_out, double* d_out, double* Jo, double* Bo,
                  double* dgo) {
    using T = decltype(tag);
    Mat<T, 3> f, Fn, Fnew;
    for (int i = 0; i < 9; ++i) {
      f.e[i] = T(f_inc[i]);
      Fn.e[i] = T(F_n[i]);
    }
    if constexpr (!std::is_same_v<T, double>) {
      for (int i = 0; i < 9; ++i)
        for (int k = 0; k < 9; ++k) f.e[i].d[k] = seed_dirs[k * 9 + i];
    }
    Fnew = matmul(f, Fn);
    StressOut<T> su;
    const T L = T(lam), Mu = T(mu);
    if (kind == 0) su = hencky_update<T, 3>(Fnew, L, Mu);
    else if (kind == 1) su = j2_update<T, 3>(f, Be_n, L, Mu, prm[2], Bo, dgo);
    else if (kind == 2) su = neo_hookean_update<T, 3>(Fnew, L, Mu);
    else if (kind == 3) su = dp_update<T, 3>(Fnew, f, Be_n, L, Mu, prm[3], prm[4], Bo, dgo);
    else su = mcc_update<T, 3>(Fnew, f, Be_n, lam + 2.0 * mu / 3.0, mu, prm[5], prm[6], prm[7], prm[8], Bo, dgo);
    for (int i = 0; i < 9; ++i) s_out[i] = value_of(su.sigma.e[i]);
    *Jo = value_of(su.J);
    if constexpr (!std::is_same_v<T, double>) {
      for (int i = 0; i < 9; ++i)
        for (int k = 0; k < 9; ++k) d_out[i * 9 + k] = su.sigma.e[i].d[k];
    }
  };
  double seeds[81] = {0};
  for (int k = 0; k < 9; ++k) seeds[k * 9 + k] = 1.0;  // d/d f_inc_k
  double s2[9], J2v, Bdummy[9], dgd = 0.0;
  eval(0.0, nullptr, sigma, nullptr, J, Be_out, dg);
  eval(Dual<9>(), seeds, s2, dsig, &J2v, Bdummy, &dgd);
}

// 2D (plane strain) closed-form path of the same kinds: f_inc, F_n 2x2 row-major
void probe_stress2(int kind, const double* f_inc, const double* F_n, const double* Be_n, const double* prm,
                   double* sigma, double* J, double* Be_out, double* dg) {
  Mat<double, 2> f, Fn;
  for (int i = 0; i < 4; ++i) {
    f.e[i] = f_inc[i];
    Fn.e[i] = F_n[i];
  }
  const Mat<double, 2> Fnew = matmul(f, Fn);
  StressOut<double> su;
  const double lam = prm[0], mu = prm[1];
  if (kind == 0) su = hencky_update<double, 2>(Fnew, lam, mu);
  else if (kind == 1) su = j2_update<double, 2>(f, Be_n, lam, mu, prm[2], Be_out, dg);
  else if (kind == 2) su = neo_hookean_update<double, 2>(Fnew, lam, mu);
  else if (kind == 3) su = dp_update<double, 2>(Fnew, f, Be_n, lam, mu, prm[3], prm[4], Be_out, dg);
  else su = mcc_update<double, 2>(Fnew, f, Be_n, lam + 2.0 * mu / 3.0, mu, prm[5], prm[6], prm[7], prm[8], Be_out, dg);
  for (int i = 0; i < 9; ++i) sigma[i] = su.sigma.e[i];
  *J = su.J;
}

}  // extern "C"
