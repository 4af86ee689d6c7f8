// Device math for the implicit MPM Newton step: forward-mode dual numbers,
// fixed-size matrices, the cpGIMP transfer and the constitutive updates.
//
// Every function here is written once over a scalar type T (double or
// Dual<K>) so the residual kernel (T = double) and the tangent kernel
// (T = Dual<K>, K seeded directions of the displacement gradient G) evaluate
// the SAME expression graph the reference records on its AD tape
// (/root/reference/proj/include/impm/tape.hpp:67-176). Branches are taken on
// values, exactly like the tape records the active branch
// (materials.hpp:160-164, small_math.hpp:193).
#pragma once

#include <cmath>
#include <cstdint>
#include <type_traits>

#ifndef IMPM_HD
#define IMPM_HD __host__ __device__ __forceinline__
#endif

namespace impm_gpu {

// ------------------------------------------------------------------ dual --
// value + K tangent components; the K directions are seeded entries of G.
template <int K>
struct Dual {
  double v;
  double d[K];
  IMPM_HD Dual() : v(0.0) {
#pragma unroll
    for (int i = 0; i < K; ++i) d[i] = 0.0;
  }
  IMPM_HD Dual(double x) : v(x) {  // NOLINT: constants mix freely, like ad::Var
#pragma unroll
    for (int i = 0; i < K; ++i) d[i] = 0.0;
  }
};

IMPM_HD double value_of(double x) { return x; }
template <int K>
IMPM_HD double value_of(const Dual<K>& x) { return x.v; }

template <int K>
IMPM_HD Dual<K> operator+(const Dual<K>& a, const Dual<K>& b) {
  Dual<K> r;
  r.v = a.v + b.v;
#pragma unroll
  for (int i = 0; i < K; ++i) r.d[i] = a.d[i] + b.d[i];
  return r;
}
template <int K>
IMPM_HD Dual<K> operator-(const Dual<K>& a, const Dual<K>& b) {
  Dual<K> r;
  r.v = a.v - b.v;
#pragma unroll
  for (int i = 0; i < K; ++i) r.d[i] = a.d[i] - b.d[i];
  return r;
}
template <int K>
IMPM_HD Dual<K> operator-(const Dual<K>& a) {
  Dual<K> r;
  r.v = -a.v;
#pragma unroll
  for (int i = 0; i < K; ++i) r.d[i] = -a.d[i];
  return r;
}
template <int K>
IMPM_HD Dual<K> operator*(const Dual<K>& a, const Dual<K>& b) {
  Dual<K> r;
  r.v = a.v * b.v;
#pragma unroll
  for (int i = 0; i < K; ++i) r.d[i] = a.d[i] * b.v + a.v * b.d[i];
  return r;
}
template <int K>
IMPM_HD Dual<K> operator/(const Dual<K>& a, const Dual<K>& b) {
  Dual<K> r;
  r.v = a.v / b.v;
  const double inv = 1.0 / b.v;
#pragma unroll
  for (int i = 0; i < K; ++i) r.d[i] = (a.d[i] - r.v * b.d[i]) * inv;
  return r;
}
// mixed forms (constant on one side): no tangent from the constant
template <int K>
IMPM_HD Dual<K> operator+(const Dual<K>& a, double c) {
  Dual<K> r = a;
  r.v = a.v + c;
  return r;
}
template <int K>
IMPM_HD Dual<K> operator+(double c, const Dual<K>& a) { return a + c; }
template <int K>
IMPM_HD Dual<K> operator-(const Dual<K>& a, double c) {
  Dual<K> r = a;
  r.v = a.v - c;
  return r;
}
template <int K>
IMPM_HD Dual<K> operator-(double c, const Dual<K>& a) {
  Dual<K> r;
  r.v = c - a.v;
#pragma unroll
  for (int i = 0; i < K; ++i) r.d[i] = -a.d[i];
  return r;
}
template <int K>
IMPM_HD Dual<K> operator*(const Dual<K>& a, double c) {
  Dual<K> r;
  r.v = a.v * c;
#pragma unroll
  for (int i = 0; i < K; ++i) r.d[i] = a.d[i] * c;
  return r;
}
template <int K>
IMPM_HD Dual<K> operator*(double c, const Dual<K>& a) {
  Dual<K> r;
  r.v = c * a.v;
#pragma unroll
  for (int i = 0; i < K; ++i) r.d[i] = c * a.d[i];
  return r;
}
template <int K>
IMPM_HD Dual<K> operator/(const Dual<K>& a, double c) {
  Dual<K> r;
  r.v = a.v / c;
#pragma unroll
  for (int i = 0; i < K; ++i) r.d[i] = a.d[i] / c;
  return r;
}
template <int K>
IMPM_HD Dual<K> operator/(double c, const Dual<K>& a) {
  Dual<K> r;
  r.v = c / a.v;
  const double s = -r.v / a.v;
#pragma unroll
  for (int i = 0; i < K; ++i) r.d[i] = s * a.d[i];
  return r;
}
template <int K>
IMPM_HD Dual<K>& operator+=(Dual<K>& a, const Dual<K>& b) { return a = a + b; }
template <int K>
IMPM_HD Dual<K>& operator-=(Dual<K>& a, const Dual<K>& b) { return a = a - b; }
template <int K>
IMPM_HD Dual<K>& operator+=(Dual<K>& a, double c) {
  a.v += c;
  return a;
}
template <int K>
IMPM_HD Dual<K>& operator-=(Dual<K>& a, double c) {
  a.v -= c;
  return a;
}

IMPM_HD double dlog(double x) { return log(x); }
IMPM_HD double dexp(double x) { return exp(x); }
IMPM_HD double dsqrt(double x) { return sqrt(x); }
template <int K>
IMPM_HD Dual<K> dlog(const Dual<K>& a) {
  Dual<K> r;
  r.v = log(a.v);
  const double s = 1.0 / a.v;
#pragma unroll
  for (int i = 0; i < K; ++i) r.d[i] = a.d[i] * s;
  return r;
}
template <int K>
IMPM_HD Dual<K> dexp(const Dual<K>& a) {
  Dual<K> r;
  r.v = exp(a.v);
#pragma unroll
  for (int i = 0; i < K; ++i) r.d[i] = a.d[i] * r.v;
  return r;
}
template <int K>
IMPM_HD Dual<K> dsqrt(const Dual<K>& a) {
  Dual<K> r;
  r.v = sqrt(a.v);
  const double s = 0.5 / r.v;
#pragma unroll
  for (int i = 0; i < K; ++i) r.d[i] = a.d[i] * s;
  return r;
}

// --------------------------------------------------------------- matrices --
template <class T, int R, int C = R>
struct Mat {
  T e[R * C];
  IMPM_HD T& operator()(int i, int j) { return e[i * C + j]; }
  IMPM_HD const T& operator()(int i, int j) const { return e[i * C + j]; }
  IMPM_HD static Mat identity() {
    Mat m;
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int j = 0; j < C; ++j) m(i, j) = T(i == j ? 1.0 : 0.0);
    return m;
  }
  IMPM_HD static Mat zero() {
    Mat m;
#pragma unroll
    for (int i = 0; i < R * C; ++i) m.e[i] = T(0.0);
    return m;
  }
};

// small_math.hpp:302-312 (same left-to-right accumulation)
template <class T, int R, int K, int C>
IMPM_HD Mat<T, R, C> matmul(const Mat<T, R, K>& a, const Mat<T, K, C>& b) {
  Mat<T, R, C> m;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < C; ++j) {
      T s = a(i, 0) * b(0, j);
#pragma unroll
      for (int k = 1; k < K; ++k) s += a(i, k) * b(k, j);
      m(i, j) = s;
    }
  return m;
}

template <class T, int N>
IMPM_HD Mat<T, N> transpose(const Mat<T, N>& a) {
  Mat<T, N> m;
#pragma unroll
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < N; ++j) m(i, j) = a(j, i);
  return m;
}

template <class T, int N>
IMPM_HD T trace(const Mat<T, N>& a) {
  T s = a(0, 0);
#pragma unroll
  for (int i = 1; i < N; ++i) s += a(i, i);
  return s;
}

// small_math.hpp:348-363
template <class T>
IMPM_HD T det(const Mat<T, 1>& a) { return a(0, 0); }
template <class T>
IMPM_HD T det(const Mat<T, 2>& a) { return a(0, 0) * a(1, 1) - a(0, 1) * a(1, 0); }
template <class T>
IMPM_HD T det(const Mat<T, 3>& a) {
  return a(0, 0) * (a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1)) -
         a(0, 1) * (a(1, 0) * a(2, 2) - a(1, 2) * a(2, 0)) +
         a(0, 2) * (a(1, 0) * a(2, 1) - a(1, 1) * a(2, 0));
}

// small_math.hpp:365-397
template <class T>
IMPM_HD Mat<T, 1> inverse(const Mat<T, 1>& a) {
  Mat<T, 1> m;
  m(0, 0) = 1.0 / a(0, 0);
  return m;
}
template <class T>
IMPM_HD Mat<T, 2> inverse(const Mat<T, 2>& a) {
  const T d = det(a);
  Mat<T, 2> m;
  m(0, 0) = a(1, 1) / d;
  m(0, 1) = (-1.0) * a(0, 1) / d;
  m(1, 0) = (-1.0) * a(1, 0) / d;
  m(1, 1) = a(0, 0) / d;
  return m;
}
template <class T>
IMPM_HD Mat<T, 3> inverse(const Mat<T, 3>& a) {
  const T d = det(a);
  Mat<T, 3> m;
  m(0, 0) = (a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1)) / d;
  m(0, 1) = (a(0, 2) * a(2, 1) - a(0, 1) * a(2, 2)) / d;
  m(0, 2) = (a(0, 1) * a(1, 2) - a(0, 2) * a(1, 1)) / d;
  m(1, 0) = (a(1, 2) * a(2, 0) - a(1, 0) * a(2, 2)) / d;
  m(1, 1) = (a(0, 0) * a(2, 2) - a(0, 2) * a(2, 0)) / d;
  m(1, 2) = (a(0, 2) * a(1, 0) - a(0, 0) * a(1, 2)) / d;
  m(2, 0) = (a(1, 0) * a(2, 1) - a(1, 1) * a(2, 0)) / d;
  m(2, 1) = (a(0, 1) * a(2, 0) - a(0, 0) * a(2, 1)) / d;
  m(2, 2) = (a(0, 0) * a(1, 1) - a(0, 1) * a(1, 0)) / d;
  return m;
}

// ------------------------------------------------------------------ GIMP --
struct WeightValue {
  double w, dw;
};

// cpGIMP 1D weight (src/gimp.cpp:27-44): hat function averaged over the
// particle domain [xi - lp, xi + lp]; half-open branches in |xi|.
IMPM_HD WeightValue gimp_weight_1d(double xi, double lp, double h) {
  const double ax = fabs(xi);
  const double sgn = xi >= 0.0 ? 1.0 : -1.0;
  if (ax < lp) return {1.0 - (xi * xi + lp * lp) / (2.0 * h * lp), -xi / (h * lp)};
  if (ax < h - lp) return {1.0 - ax / h, -sgn / h};
  if (ax < h + lp) {
    const double t = h + lp - ax;
    return {t * t / (4.0 * h * lp), -sgn * t / (2.0 * h * lp)};
  }
  return {0.0, 0.0};
}

// Quadratic B-spline (extension, parity unpinned: the reference registers the
// kind for block_size only, src/gimp.cpp:11). Same 3-node support.
IMPM_HD WeightValue bspline2_weight_1d(double xi, double h) {
  const double q = fabs(xi) / h;
  const double sgn = xi >= 0.0 ? 1.0 : -1.0;
  if (q < 0.5) return {0.75 - q * q, -2.0 * q * sgn / h};
  if (q < 1.5) {
    const double t = 1.5 - q;
    return {0.5 * t * t, -t * sgn / h};
  }
  return {0.0, 0.0};
}

// Integer support along one axis (src/gimp.cpp:46-53). Built from IEEE
// add/sub/div only (no multiply => no FMA contraction), so the floor/ceil
// decisions are bit-exact against the reference's double arithmetic.
__device__ __forceinline__ void gimp_support_1d(double x, double lp, double origin, double h, int& first, int& count) {
  const double lo = __dsub_rn(__dsub_rn(x, origin), __dadd_rn(h, lp));
  const double hi = __dadd_rn(__dsub_rn(x, origin), __dadd_rn(h, lp));
  const int f = static_cast<int>(floor(__ddiv_rn(lo, h))) + 1;
  const int l = static_cast<int>(ceil(__ddiv_rn(hi, h))) - 1;
  first = f;
  count = l - f + 1;
}

// ---------------------------------------------------------- constitutive --
enum MaterialKind : int { kHencky = 0, kHenckyJ2 = 1, kNeoHookean = 2, kDruckerPrager = 3, kCamClay = 4 };

template <class T>
struct StressOut {
  Mat<T, 3> sigma;  // embedded Cauchy stress
  T J;
};

// plane-strain / uniaxial embedding (materials.hpp:51-57)
template <class T, int D>
IMPM_HD Mat<T, 3> embed_F(const Mat<T, D>& F) {
  Mat<T, 3> out = Mat<T, 3>::identity();
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) out(i, j) = F(i, j);
  return out;
}

// closed-form SPD 2x2 log (small_math.hpp:185-210)
template <class T>
IMPM_HD Mat<T, 2> sym_log_2x2(const Mat<T, 2>& a) {
  const T m = 0.5 * (a(0, 0) + a(1, 1));
  const T h = 0.5 * (a(0, 0) - a(1, 1));
  const T r2 = h * h + a(0, 1) * a(1, 0);
  T p, q;
  if (value_of(r2) < 1e-8 * value_of(m) * value_of(m)) {
    const T s = r2 / (m * m);
    p = dlog(m) - 0.5 * s * (1.0 + 0.5 * s);
    q = (1.0 + s * (1.0 / 3.0 + s * (1.0 / 5.0))) / m;
  } else {
    const T r = dsqrt(r2);
    const T log_hi = dlog(m + r);
    const T log_lo = dlog(m - r);
    p = 0.5 * (log_hi + log_lo);
    q = (log_hi - log_lo) / (2.0 * r);
  }
  Mat<T, 2> out;
  out(0, 0) = p + q * h;
  out(1, 1) = p - q * h;
  out(0, 1) = q * a(0, 1);
  out(1, 0) = q * a(1, 0);
  return out;
}

// closed-form symmetric 2x2 exp (small_math.hpp:213-237)
template <class T>
IMPM_HD Mat<T, 2> sym_exp_2x2(const Mat<T, 2>& a) {
  const T m = 0.5 * (a(0, 0) + a(1, 1));
  const T h = 0.5 * (a(0, 0) - a(1, 1));
  const T r2 = h * h + a(0, 1) * a(1, 0);
  T p, q;
  if (value_of(r2) < 1e-8) {
    p = dexp(m) * (1.0 + 0.5 * r2 * (1.0 + r2 * (1.0 / 12.0)));
    q = dexp(m) * (1.0 + r2 * (1.0 / 6.0 + r2 * (1.0 / 120.0)));
  } else {
    const T r = dsqrt(r2);
    const T exp_hi = dexp(m + r);
    const T exp_lo = dexp(m - r);
    p = 0.5 * (exp_hi + exp_lo);
    q = (exp_hi - exp_lo) / (2.0 * r);
  }
  Mat<T, 2> out;
  out(0, 0) = p + q * h;
  out(1, 1) = p - q * h;
  out(0, 1) = q * a(0, 1);
  out(1, 0) = q * a(1, 0);
  return out;
}


// ------------------------------------------------- 3x3 spectral functions --
// Extension beyond the reference, whose embedded closed forms stop at D <= 2
// (materials.hpp:61-62 static_assert "use the 3x3 spectral path"): f(B) for a
// symmetric 3x3 B with f = log (Hencky strain) or exp (B_e from strain).
// Values: cyclic Jacobi eigen-decomposition B = Q diag(l) Q^T (orthogonal Q to
// roundoff, no branch on eigenvalue multiplicity), f(B) = Q diag(f(l)) Q^T.
// Tangents (T = Dual<K>): the Daleckii-Krein formula
//   df(B)[dB] = Q (F o (Q^T dB Q)) Q^T,  F_ij = f[l_i, l_j],
// with first divided differences in cancellation-free forms that tend to
// f'(l) as l_i -> l_j, so repeated eigenvalues (B = I at rest) are exact.
IMPM_HD void sym_eig3(const double Bin[9], double l[3], double Q[9]) {
  double a[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) a[i * 3 + j] = 0.5 * (Bin[i * 3 + j] + Bin[j * 3 + i]);
#pragma unroll
  for (int i = 0; i < 9; ++i) Q[i] = (i % 4 == 0) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 12; ++sweep) {
    const double off = a[1] * a[1] + a[2] * a[2] + a[5] * a[5];
    const double dia = a[0] * a[0] + a[4] * a[4] + a[8] * a[8];
    if (!(off > 1e-34 * dia)) break;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int p = r == 2 ? 1 : 0, q = r == 0 ? 1 : 2;
      const double apq = a[p * 3 + q];
      if (apq == 0.0) continue;
      const double theta = (a[q * 3 + q] - a[p * 3 + p]) / (2.0 * apq);
      const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
      const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
      // A <- J^T A J with J = rotation in the (p, q) plane
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double akp = a[k * 3 + p], akq = a[k * 3 + q];
        a[k * 3 + p] = c * akp - sn * akq;
        a[k * 3 + q] = sn * akp + c * akq;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double apk = a[p * 3 + k], aqk = a[q * 3 + k];
        a[p * 3 + k] = c * apk - sn * aqk;
        a[q * 3 + k] = sn * apk + c * aqk;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double qkp = Q[k * 3 + p], qkq = Q[k * 3 + q];
        Q[k * 3 + p] = c * qkp - sn * qkq;
        Q[k * 3 + q] = sn * qkp + c * qkq;
      }
    }
  }
  l[0] = a[0];
  l[1] = a[4];
  l[2] = a[8];
}

enum SymFn : int { kSymLog = 0, kSymExp = 1 };

IMPM_HD double sym_fn(int fn, double x) { return fn == kSymLog ? log(x) : exp(x); }

// first divided difference f[a, b] (f'(a) at a == b)
IMPM_HD double sym_fn_dd(int fn, double a, double b) {
  if (fn == kSymLog) {
    const double r = (a - b) / (a + b);  // log(a/b) = 2 atanh(r)
    if (fabs(r) < 1e-3) {
      const double r2 = r * r;
      return 2.0 / (a + b) * (1.0 + r2 * (1.0 / 3.0 + r2 * (1.0 / 5.0 + r2 * (1.0 / 7.0))));
    }
    return (log(a) - log(b)) / (a - b);
  }
  const double d = a - b;  // exp[a, b] = exp(b) expm1(d) / d
  if (fabs(d) < 1e-3) return exp(b) * (1.0 + d * (0.5 + d * (1.0 / 6.0 + d * (1.0 / 24.0 + d * (1.0 / 120.0)))));
  return exp(b) * expm1(d) / d;
}

IMPM_HD Mat<double, 3> sym_fun3(const Mat<double, 3>& B, int fn) {
  double l[3], Q[9];
  sym_eig3(B.e, l, Q);
  const double f[3] = {sym_fn(fn, l[0]), sym_fn(fn, l[1]), sym_fn(fn, l[2])};
  Mat<double, 3> out;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      out(i, j) = Q[i * 3 + 0] * f[0] * Q[j * 3 + 0] + Q[i * 3 + 1] * f[1] * Q[j * 3 + 1] +
                  Q[i * 3 + 2] * f[2] * Q[j * 3 + 2];
  return out;
}

template <int K>
IMPM_HD Mat<Dual<K>, 3> sym_fun3(const Mat<Dual<K>, 3>& B, int fn) {
  Mat<double, 3> Bv;
#pragma unroll
  for (int i = 0; i < 9; ++i) Bv.e[i] = B.e[i].v;
  double l[3], Q[9];
  sym_eig3(Bv.e, l, Q);
  double f[3], dd[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i) f[i] = sym_fn(fn, l[i]);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) dd[i][j] = j < i ? dd[j][i] : sym_fn_dd(fn, l[i], l[j]);
  Mat<Dual<K>, 3> out;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      out(i, j).v = Q[i * 3 + 0] * f[0] * Q[j * 3 + 0] + Q[i * 3 + 1] * f[1] * Q[j * 3 + 1] +
                    Q[i * 3 + 2] * f[2] * Q[j * 3 + 2];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double dB[9], M[9], T1[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) dB[i * 3 + j] = 0.5 * (B(i, j).d[k] + B(j, i).d[k]);
    // M = Q^T dB Q, scaled by the divided differences
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        T1[i * 3 + j] = dB[i * 3 + 0] * Q[0 * 3 + j] + dB[i * 3 + 1] * Q[1 * 3 + j] + dB[i * 3 + 2] * Q[2 * 3 + j];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        M[i * 3 + j] = dd[i][j] * (Q[0 * 3 + i] * T1[0 * 3 + j] + Q[1 * 3 + i] * T1[1 * 3 + j] +
                                   Q[2 * 3 + i] * T1[2 * 3 + j]);
    // out.d = Q M Q^T
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        T1[i * 3 + j] = Q[i * 3 + 0] * M[0 * 3 + j] + Q[i * 3 + 1] * M[1 * 3 + j] + Q[i * 3 + 2] * M[2 * 3 + j];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        out(i, j).d[k] = T1[i * 3 + 0] * Q[j * 3 + 0] + T1[i * 3 + 1] * Q[j * 3 + 1] + T1[i * 3 + 2] * Q[j * 3 + 2];
  }
  return out;
}

// embedded_sym_log / embedded_sym_exp (materials.hpp:61-105); D = 3 takes the
// spectral path above (extension, parity unpinned)
template <class T, int D>
IMPM_HD Mat<T, 3> embedded_sym_log(const Mat<T, 3>& b) {
  if constexpr (D == 3) {
    return sym_fun3(b, kSymLog);
  } else {
  Mat<T, 3> out = Mat<T, 3>::zero();
  if constexpr (D == 1) {
    out(0, 0) = dlog(b(0, 0));
  } else {
    Mat<T, 2> blk;
    blk(0, 0) = b(0, 0);
    blk(0, 1) = b(0, 1);
    blk(1, 0) = b(1, 0);
    blk(1, 1) = b(1, 1);
    const Mat<T, 2> l = sym_log_2x2(blk);
    out(0, 0) = l(0, 0);
    out(0, 1) = l(0, 1);
    out(1, 0) = l(1, 0);
    out(1, 1) = l(1, 1);
  }
#pragma unroll
  for (int i = D; i < 3; ++i) out(i, i) = dlog(b(i, i));
  return out;
  }
}

template <class T, int D>
IMPM_HD Mat<T, 3> embedded_sym_exp(const Mat<T, 3>& eps) {
  if constexpr (D == 3) {
    return sym_fun3(eps, kSymExp);
  } else {
  Mat<T, 3> out = Mat<T, 3>::zero();
  if constexpr (D == 1) {
    out(0, 0) = dexp(eps(0, 0));
  } else {
    Mat<T, 2> blk;
    blk(0, 0) = eps(0, 0);
    blk(0, 1) = eps(0, 1);
    blk(1, 0) = eps(1, 0);
    blk(1, 1) = eps(1, 1);
    const Mat<T, 2> e = sym_exp_2x2(blk);
    out(0, 0) = e(0, 0);
    out(0, 1) = e(0, 1);
    out(1, 0) = e(1, 0);
    out(1, 1) = e(1, 1);
  }
#pragma unroll
  for (int i = D; i < 3; ++i) out(i, i) = dexp(eps(i, i));
  return out;
  }
}

template <class T>
IMPM_HD Mat<T, 3> scale3(double s, const Mat<T, 3>& a) {
  Mat<T, 3> m;
#pragma unroll
  for (int i = 0; i < 9; ++i) m.e[i] = s * a.e[i];
  return m;
}

// Hencky (materials.hpp:117-136)
template <class T, int D>
IMPM_HD StressOut<T> hencky_update(const Mat<T, D>& F, const T& lam, const T& mu) {
  const Mat<T, 3> F3 = embed_F<T, D>(F);
  const Mat<T, 3> b = matmul(F3, transpose(F3));
  const Mat<T, 3> eps = scale3(0.5, embedded_sym_log<T, D>(b));
  const T tr = trace(eps);
  const T J = dexp(tr);
  StressOut<T> out;
  out.J = J;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      T tau = 2.0 * mu * eps(i, j);
      if (i == j) tau += lam * tr;
      out.sigma(i, j) = tau / J;
    }
  return out;
}

// neo-Hookean (materials.hpp:139-158)
template <class T, int D>
IMPM_HD StressOut<T> neo_hookean_update(const Mat<T, D>& F, const T& lam, const T& mu) {
  const T J = det(F);
  const Mat<T, 3> F3 = embed_F<T, D>(F);
  const Mat<T, 3> b = matmul(F3, transpose(F3));
  const T lnJ = dlog(J);
  StressOut<T> out;
  out.J = J;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      T tau = mu * (b(i, j) - (i == j ? T(1.0) : T(0.0)));
      if (i == j) tau += lam * lnJ;
      out.sigma(i, j) = tau / J;
    }
  return out;
}

// J2 radial return on Hencky strain (materials.hpp:165-219). Returns sigma,
// J; optionally the updated B_e and dgamma (commit only, plain doubles).
template <class T, int D>
IMPM_HD StressOut<T> j2_update(const Mat<T, D>& f_incr, const double* Be_n /*3x3*/, const T& lam,
                               const T& mu, double kappa, double* Be_out = nullptr,
                               double* dgamma_out = nullptr) {
  const Mat<T, 3> f3 = embed_F<T, D>(f_incr);
  Mat<T, 3> Ben;
#pragma unroll
  for (int i = 0; i < 9; ++i) Ben.e[i] = T(Be_n[i]);
  const Mat<T, 3> b_tr = matmul(matmul(f3, Ben), transpose(f3));
  const Mat<T, 3> eps_tr = scale3(0.5, embedded_sym_log<T, D>(b_tr));
  const T tr_eps = trace(eps_tr);
  const T J = dexp(tr_eps);
  Mat<T, 3> dev_eps = eps_tr;
#pragma unroll
  for (int i = 0; i < 3; ++i) dev_eps(i, i) -= tr_eps * (1.0 / 3.0);
  T s2 = T(0.0);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) s2 += dev_eps(i, j) * dev_eps(i, j);
  const T two_mu = 2.0 * mu;
  const T s_norm = two_mu * dsqrt(s2 + 1e-300);
  const T p_tau = lam * tr_eps + two_mu * tr_eps * (1.0 / 3.0);
  StressOut<T> out;
  out.J = J;
  if (value_of(s_norm) <= kappa) {
    if (Be_out) {
#pragma unroll
      for (int i = 0; i < 9; ++i) Be_out[i] = value_of(b_tr.e[i]);
      *dgamma_out = 0.0;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        T tau = two_mu * dev_eps(i, j);
        if (i == j) tau += p_tau;
        out.sigma(i, j) = tau / J;
      }
    return out;
  }
  const T scale = T(kappa) / s_norm;
  if (Be_out) {
    *dgamma_out = value_of((s_norm - kappa) / two_mu);
    Mat<double, 3> eps_e;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        eps_e(i, j) = value_of(scale * dev_eps(i, j));
        if (i == j) eps_e(i, j) += value_of(tr_eps * (1.0 / 3.0));
      }
    const Mat<double, 3> Be = embedded_sym_exp<double, D>(scale3(2.0, eps_e));
#pragma unroll
    for (int i = 0; i < 9; ++i) Be_out[i] = Be.e[i];
  }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      T tau = two_mu * scale * dev_eps(i, j);
      if (i == j) tau += p_tau;
      out.sigma(i, j) = tau / J;
    }
  return out;
}

// Drucker-Prager on Hencky strain, plane strain / uniaxial (D <= 2), with a
// non-associative return (Klar et al. 2016): extension -> tip projection
// (eps = 0); otherwise dgamma = |dev eps| + (3 lam + 2 mu)/(2 mu) tr(eps)
// alpha, radial return of the deviator when dgamma > 0. Extension beyond the
// reference (parity unpinned): no DP in /root/reference.
// J = det(F_new) (plastic flow is not isochoric here). B_e = exp(2 eps_e).
template <class T, int D>
IMPM_HD StressOut<T> dp_update(const Mat<T, D>& F_new, const Mat<T, D>& f_incr, const double* Be_n, const T& lam,
                               const T& mu, double alpha, double e_c, double* Be_out = nullptr,
                               double* dgamma_out = nullptr) {
  const Mat<T, 3> f3 = embed_F<T, D>(f_incr);
  Mat<T, 3> Ben;
#pragma unroll
  for (int i = 0; i < 9; ++i) Ben.e[i] = T(Be_n[i]);
  const Mat<T, 3> b_tr = matmul(matmul(f3, Ben), transpose(f3));
  const Mat<T, 3> eps_tr = scale3(0.5, embedded_sym_log<T, D>(b_tr));
  const T tr = trace(eps_tr);
  Mat<T, 3> dev = eps_tr;
#pragma unroll
  for (int i = 0; i < 3; ++i) dev(i, i) -= tr * (1.0 / 3.0);
  T s2 = T(0.0);
#pragma unroll
  for (int i = 0; i < 9; ++i) s2 += dev.e[i] * dev.e[i];
  const T dnorm = dsqrt(s2 + 1e-300);
  Mat<T, 3> eps = eps_tr;
  double dg = 0.0;
  // the stress-free apex (eps = 0 exactly) stays elastic so the initial
  // tangent is the elastic one; strict thresholds in strain units
  // cohesion shifts the apex to tr = e_c (mean Kirchhoff stress = cohesion)
  if (value_of(tr) > e_c + 1e-14) {  // extension: project to the cone tip
    eps = Mat<T, 3>::zero();
#pragma unroll
    for (int i = 0; i < 3; ++i) eps(i, i) = T(e_c / 3.0);
    // the tip carries no stiffness: a node whose particles all sit there makes
    // J singular. The TANGENT (dual parts only; the residual value is the exact
    // projection) keeps 1e-6 of the elastic response, a modified-Newton
    // regularisation that leaves converged states unchanged.
    if constexpr (!std::is_same<T, double>::value) {
#pragma unroll
      for (int i = 0; i < 9; ++i)
#pragma unroll
        for (int k = 0; k < (int)(sizeof(eps.e[i].d) / sizeof(double)); ++k) eps.e[i].d[k] = 1e-6 * eps_tr.e[i].d[k];
    }
    T e2 = T(0.0);
#pragma unroll
    for (int i = 0; i < 9; ++i) e2 += (eps_tr.e[i] - eps.e[i]) * (eps_tr.e[i] - eps.e[i]);
    dg = value_of(dsqrt(e2 + 1e-300));
  } else {
    const T gam = dnorm + (3.0 * lam + 2.0 * mu) / (2.0 * mu) * (tr - e_c) * alpha;
    if (value_of(gam) > 1e-14) {
      const T sc = gam / dnorm;
#pragma unroll
      for (int i = 0; i < 9; ++i) eps.e[i] = eps_tr.e[i] - sc * dev.e[i];
      dg = value_of(gam);
    }
  }
  const T tre = trace(eps);
  const T J = det(F_new);
  StressOut<T> out;
  out.J = J;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      T tau = 2.0 * mu * eps(i, j);
      if (i == j) tau += lam * tre;
      out.sigma(i, j) = tau / J;
    }
  if (Be_out) {
    Mat<double, 3> e2;
#pragma unroll
    for (int i = 0; i < 9; ++i) e2.e[i] = 2.0 * value_of(eps.e[i]);
    const Mat<double, 3> Be = embedded_sym_exp<double, D>(e2);
#pragma unroll
    for (int i = 0; i < 9; ++i) Be_out[i] = Be.e[i];
    *dgamma_out = dg;
  }
  return out;
}

// Modified Cam-Clay on Hencky strain (extension, parity unpinned: no
// critical-state model in /root/reference). Linear isotropic elasticity in
// Hencky strain (K, G), compression-positive invariants
//   P = -K tr(eps_e),  q = sqrt(3/2) |2 G dev(eps_e)|,
// yield f = q^2/M^2 + (P + p_t)(P - p_c) (ellipse from -p_t to p_c; p_t > 0
// keeps the stress-free state strictly elastic), associative flow, and
// exponential hardening p_c = p_c0 exp(theta a), a = accumulated plastic
// compaction (the particle's alpha). Return map: radial in the deviatoric
// plane (coaxial with the trial strain), Newton on (x = plastic compaction
// increment, g = plastic multiplier):
//   r1 = x - g (2P + p_t - p_c) = 0,   r2 = (q^2/M^2 + (P + p_t)(P - p_c)) / p_c,n^2 = 0,
//   P = P_tr - K x,  p_c = p_c,n exp(theta x),  q = q_tr / (1 + 6 G g / M^2).
// Run in T = Dual<K>, one extra Newton step after the values converge makes
// the dual parts the exact implicit derivative (the consistent tangent).
// Be_n[9] carries alpha_n. Outputs B_e = exp(2 eps_e) and x (added to alpha).
template <class T, int D>
IMPM_HD StressOut<T> mcc_update(const Mat<T, D>& F_new, const Mat<T, D>& f_incr, const double* Be_n, double K,
                                double G, double M, double pc0, double theta, double pt, double* Be_out = nullptr,
                                double* dgamma_out = nullptr) {
  const Mat<T, 3> f3 = embed_F<T, D>(f_incr);
  Mat<T, 3> Ben;
#pragma unroll
  for (int i = 0; i < 9; ++i) Ben.e[i] = T(Be_n[i]);
  const Mat<T, 3> b_tr = matmul(matmul(f3, Ben), transpose(f3));
  const Mat<T, 3> eps_tr = scale3(0.5, embedded_sym_log<T, D>(b_tr));
  const T tr = trace(eps_tr);
  Mat<T, 3> dev = eps_tr;
#pragma unroll
  for (int i = 0; i < 3; ++i) dev(i, i) -= tr * (1.0 / 3.0);
  T s2 = T(0.0);
#pragma unroll
  for (int i = 0; i < 9; ++i) s2 += dev.e[i] * dev.e[i];
  const T dn = dsqrt(s2 + 1e-300);
  const T P_tr = (-K) * tr;
  const T q_tr = (2.449489742783178 * G) * dn;  // sqrt(6) G |dev|
  const double pcn = pc0 * exp(theta * Be_n[9]);
  const double M2 = M * M;
  const T f_tr = q_tr * q_tr / M2 + (P_tr + pt) * (P_tr - pcn);
  T P = P_tr, scale_q = T(1.0);
  double xv = 0.0;
  if (value_of(f_tr) > 1e-12 * pcn * pcn) {
    T x = T(0.0), g = T(0.0);
    const double inv_pc2 = 1.0 / (pcn * pcn);
    int extra = -1;
    for (int it = 0; it < 60; ++it) {
      const T pc = pcn * dexp(theta * x);
      const T Pk = P_tr - K * x;
      const T den = 1.0 + (6.0 * G / M2) * g;
      const T q = q_tr / den;
      const T r1 = x - g * (2.0 * Pk + pt - pc);
      const T r2 = (q * q / M2 + (Pk + pt) * (Pk - pc)) * inv_pc2;
      const double rn = fabs(value_of(r1)) + fabs(value_of(r2));
      if (extra < 0 && rn <= 1e-14) extra = 0;
      if (extra >= 0 && extra++ >= 2) break;
      const T a11 = 1.0 + g * (2.0 * K + theta * pc);
      const T a12 = -(2.0 * Pk + pt - pc);
      const T a21 = ((-K) * (Pk - pc) + (Pk + pt) * ((-K) - theta * pc)) * inv_pc2;
      const T a22 = (2.0 * q / M2) * ((-6.0 * G / M2) * q / den) * inv_pc2;
      const T dt = a11 * a22 - a12 * a21;
      T dx = (a22 * r1 - a12 * r2) / dt;
      T dg = (a11 * r2 - a21 * r1) / dt;
      // keep the multiplier non-negative (den > 0) with a damped step
      double lam_s = 1.0;
      while (value_of(g) - lam_s * value_of(dg) < 0.0 && lam_s > 1e-6) lam_s *= 0.5;
      x = x - lam_s * dx;
      g = g - lam_s * dg;
    }
    P = P_tr - K * x;
    scale_q = 1.0 / (1.0 + (6.0 * G / M2) * g);
    xv = value_of(x);
  }
  const T J = det(F_new);
  StressOut<T> out;
  out.J = J;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      T tau = (2.0 * G) * scale_q * dev(i, j);
      if (i == j) tau -= P;
      out.sigma(i, j) = tau / J;
    }
  if (Be_out) {
    Mat<double, 3> e2;
    const double ev = -value_of(P) / K;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) e2(i, j) = 2.0 * (value_of(scale_q) * value_of(dev(i, j)) + (i == j ? ev / 3.0 : 0.0));
    const Mat<double, 3> Be = embedded_sym_exp<double, D>(e2);
#pragma unroll
    for (int i = 0; i < 9; ++i) Be_out[i] = Be.e[i];
    *dgamma_out = xv;
  }
  return out;
}

}  // namespace impm_gpu
