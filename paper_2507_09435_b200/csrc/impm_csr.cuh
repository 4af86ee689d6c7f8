// impm_csr.cuh — general CSR linear algebra on the device, behind the
// reference's only link-level hot-path seam:
//   impm::sparse_lu_solve   include/impm/sparse.hpp:43, src/linear_solver.cpp:11-88
//   CsrMatrix::multiply     src/sparse.cpp:44-53
//   CsrMatrix::transposed   src/sparse.cpp:55-70
// Included once into impm_sim.cu (shares SimError / DBuf / CK / g_launches).
//
// sparse_lu_solve keeps the reference contract statement by statement: row
// equilibration by max|a_ij| ("empty matrix row i" on a zero row), a solve of
// the scaled system, up to two refinement sweeps while the normwise backward
// error |Ax-b|_2 / (|A|_inf |x|_inf + |b|_2) exceeds 1e-14, and
// LinearSolverError when it ends above 1e-10. The factorisation is chosen by
// size:
//  * n <= kDenseMax: dense LU with partial pivoting in HBM (row-major, one
//    pivot kernel + one rank-1 trailing update per column). An exactly zero
//    pivot column is "singular factorization", the condition under which
//    Eigen's SparseLU::factorize fails.
//  * larger n: restarted GMRES(m) on the equilibrated system, right-
//    preconditioned by its diagonal, classical Gram-Schmidt twice with
//    batched fixed-order dot partials, iterated to the same 1e-14 backward
//    error. A singular system is reported through the backward-error check.
#pragma once

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

namespace csr {

constexpr int kDenseMax = 2048;
constexpr int kGmresM = 60;
constexpr int kGmresMaxRestarts = 400;
constexpr int kRedBlk = 148 * 2;  // fixed partial count: deterministic dots

// ----------------------------------------------------------- kernels ----

// y = A x, each row summed in column order with unfused multiply and add:
// bitwise the value CsrMatrix::multiply (src/sparse.cpp:44-53) produces on
// x86-64 (SSE2, no contraction). A warp owns 32 consecutive rows; lanes form
// the products of a 256-entry chunk in parallel (coalesced value / column
// loads) into shared memory, then each lane adds its own row's run in order.
// MODE 0: y = A x. MODE 1: y = (b - A x) / scale (scaled refinement residual).
// MODE 2: y = b - A x.
template <int MODE>
__global__ void __launch_bounds__(128) k_csr_spmv(int n, const int64_t* __restrict__ rp,
                                                  const int32_t* __restrict__ ci, const double* __restrict__ v,
                                                  const double* __restrict__ x, double* __restrict__ y,
                                                  const double* __restrict__ b, const double* __restrict__ scale) {
  constexpr int kChunk = 256;
  __shared__ double prod[4][kChunk];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = ((int64_t)blockIdx.x * 4 + w) * 32;
  if (r0 >= n) return;
  const int rows = (int)(n - r0 < 32 ? n - r0 : 32);
  const int64_t e0 = rp[r0], e1 = rp[r0 + rows];
  const int64_t my_b = lane < rows ? rp[r0 + lane] : e1;
  const int64_t my_e = lane < rows ? rp[r0 + lane + 1] : e1;
  double s = 0.0;
  for (int64_t c0 = e0; c0 < e1; c0 += kChunk) {
    const int cn = (int)(e1 - c0 < kChunk ? e1 - c0 : kChunk);
    for (int k = lane; k < cn; k += 32) prod[w][k] = __dmul_rn(__ldg(v + c0 + k), __ldg(x + __ldg(ci + c0 + k)));
    __syncwarp();
    const int64_t lo = max(my_b, c0), hi = min(my_e, c0 + cn);
    for (int64_t k = lo; k < hi; ++k) s = __dadd_rn(s, prod[w][k - c0]);
    __syncwarp();
  }
  if (lane < rows) {
    if constexpr (MODE == 0) y[r0 + lane] = s;
    else if constexpr (MODE == 1) y[r0 + lane] = (b[r0 + lane] - s) / scale[r0 + lane];
    else y[r0 + lane] = b[r0 + lane] - s;
  }
}

// row_scale[i] = max_k |a_ik| and row_abs[i] = sum_k |a_ik| (linear_solver.cpp:18-22,
// :57-62); empty row -> atomicMin of its index (the reference throws on the first).
__global__ void k_csr_row_stats(int n, const int64_t* __restrict__ rp, const double* __restrict__ v,
                                double* __restrict__ row_scale, double* __restrict__ row_abs, int* __restrict__ empty_row,
                                double* __restrict__ diag_out, const int32_t* __restrict__ ci) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = t >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double mx = 0.0, sm = 0.0, dg = 0.0;
  for (int64_t k = rp[row] + lane; k < rp[row + 1]; k += 32) {
    const double a = fabs(v[k]);
    mx = fmax(mx, a);
    sm += a;
    if (ci[k] == row) dg = v[k];
  }
  for (int o = 16; o; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
    dg += __shfl_xor_sync(0xffffffffu, dg, o);
  }
  if (lane == 0) {
    row_scale[row] = mx;
    row_abs[row] = sm;
    diag_out[row] = mx > 0.0 ? dg / mx : 0.0;
    if (mx == 0.0) atomicMin(empty_row, (int)row);
  }
}

// fixed-order partials over kRedBlk blocks: out[j*kRedBlk + blk]
// MODE 0: sum a_j . b  (nv vectors a_j = A + j*lda)   MODE 1: sum b^2 (nv=1)   MODE 2: max |b|
template <int MODE>
__global__ void __launch_bounds__(256) k_multi_reduce(int64_t n, const double* __restrict__ A, int64_t lda, int nv,
                                                      const double* __restrict__ b, double* __restrict__ out) {
  __shared__ double red[8];
  for (int j = 0; j < nv; ++j) {
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      if constexpr (MODE == 0) s += A[j * lda + i] * b[i];
      else if constexpr (MODE == 1) s += b[i] * b[i];
      else s = fmax(s, fabs(b[i]));
    }
    for (int o = 16; o; o >>= 1) {
      const double u = __shfl_xor_sync(0xffffffffu, s, o);
      s = MODE == 2 ? fmax(s, u) : s + u;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = red[0];
      for (int w = 1; w < 8; ++w) t = MODE == 2 ? fmax(t, red[w]) : t + red[w];
      out[(int64_t)j * gridDim.x + blockIdx.x] = t;
    }
    __syncthreads();
  }
}

// w -= sum_j h_j V_j   (classical Gram-Schmidt projection, h on the device)
__global__ void k_gs_sub(int64_t n, const double* __restrict__ V, int64_t ldv, int nv, const double* __restrict__ h,
                         double* __restrict__ w) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = w[i];
    for (int j = 0; j < nv; ++j) s -= h[j] * V[j * ldv + i];
    w[i] = s;
  }
}

// y = a*x (+ y if ACC)
template <bool ACC>
__global__ void k_axpy(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = ACC ? y[i] + a * x[i] : a * x[i];
}

// z = x / d (Jacobi of the equilibrated system; zero diagonal -> identity)
__global__ void k_jacobi(int64_t n, const double* __restrict__ d, const double* __restrict__ x, double* __restrict__ z) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z[i] = d[i] != 0.0 ? x[i] / d[i] : x[i];
}

// x += sum_j y_j Z_j  (GMRES update with the preconditioned basis, y on the device)
__global__ void k_gmres_update(int64_t n, const double* __restrict__ V, int64_t ldv, int k, const double* __restrict__ y,
                               const double* __restrict__ d, double* __restrict__ x) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < k; ++j) s += y[j] * V[j * ldv + i];
    x[i] += d[i] != 0.0 ? s / d[i] : s;
  }
}

// dense row-major M = A / row_scale (zero-filled beforehand)
__global__ void k_dense_scatter(int n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                const double* __restrict__ v, const double* __restrict__ scale, double* __restrict__ M) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = t >> 5;
  if (row >= n) return;
  const double s = scale[row];
  for (int64_t k = rp[row] + (threadIdx.x & 31); k < rp[row + 1]; k += 32) M[row * n + ci[k]] = v[k] / s;
}

// column k of the LU: partial pivot (first row of maximal |m_ik|, i >= k),
// full-row swap, multipliers l_ik = m_ik / m_kk. Zero pivot -> singular flag.
__global__ void __launch_bounds__(1024) k_lu_pivot(int n, int k, double* __restrict__ M, int* __restrict__ perm,
                                                   int* __restrict__ singular) {
  __shared__ double bv[32];
  __shared__ int bi[32];
  __shared__ int piv;
  if (*singular >= 0) return;
  double best = -1.0;
  int bidx = n;
  for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
    const double a = fabs(M[(int64_t)i * n + k]);
    if (a > best) { best = a; bidx = i; }
  }
  for (int o = 16; o; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; }
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { bv[w] = best; bi[w] = bidx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b0 = bv[0];
    int i0 = bi[0];
    for (int j = 1; j < (int)(blockDim.x >> 5); ++j)
      if (bv[j] > b0 || (bv[j] == b0 && bi[j] < i0)) { b0 = bv[j]; i0 = bi[j]; }
    if (!(b0 > 0.0)) { *singular = k; i0 = -1; }
    piv = i0;
    if (i0 >= 0 && i0 != k) { const int t = perm[k]; perm[k] = perm[i0]; perm[i0] = t; }
  }
  __syncthreads();
  const int p = piv;
  if (p < 0) return;
  if (p != k)
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const double t = M[(int64_t)k * n + j];
      M[(int64_t)k * n + j] = M[(int64_t)p * n + j];
      M[(int64_t)p * n + j] = t;
    }
  __syncthreads();
  const double inv = 1.0 / M[(int64_t)k * n + k];
  for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) M[(int64_t)i * n + k] *= inv;
}

// trailing update m_ij -= l_ik u_kj, i, j > k (32x32 tiles, j fastest: coalesced rows)
__global__ void __launch_bounds__(256) k_lu_update(int n, int k, double* __restrict__ M, const int* __restrict__ singular) {
  if (*singular >= 0) return;
  __shared__ double u[32], l[32];
  const int j0 = k + 1 + blockIdx.x * 32, i0 = k + 1 + blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  if (threadIdx.x < 32) u[tx] = j0 + tx < n ? M[(int64_t)k * n + j0 + tx] : 0.0;
  else if (threadIdx.x < 64) l[tx] = i0 + tx < n ? M[(int64_t)(i0 + tx) * n + k] : 0.0;
  __syncthreads();
  const int j = j0 + tx;
  if (j >= n) return;
  for (int r = ty; r < 32; r += 8) {
    const int i = i0 + r;
    if (i < n) M[(int64_t)i * n + j] -= l[r] * u[tx];
  }
}

// x = U^-1 L^-1 P rhs in one CTA (n <= kDenseMax; column-oriented sweeps)
__global__ void __launch_bounds__(1024) k_lu_solve(int n, const double* __restrict__ M, const int* __restrict__ perm,
                                                   const double* __restrict__ rhs, double* __restrict__ x) {
  extern __shared__ double y[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = rhs[perm[i]];
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const double yk = y[k];
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) y[i] -= M[(int64_t)i * n + k] * yk;
    __syncthreads();
  }
  for (int k = n - 1; k >= 0; --k) {
    if (threadIdx.x == 0) y[k] /= M[(int64_t)k * n + k];
    __syncthreads();
    const double yk = y[k];
    for (int i = threadIdx.x; i < k; i += blockDim.x) y[i] -= M[(int64_t)i * n + k] * yk;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = y[i];
}

// transposed(): entry keys (col, row) for a stable two-key radix sort, and the column histogram
__global__ void k_csr_keys(int n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           uint64_t* __restrict__ keys, int64_t* __restrict__ idx, int64_t* __restrict__ count) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = t >> 5;
  if (row >= n) return;
  for (int64_t k = rp[row] + (threadIdx.x & 31); k < rp[row + 1]; k += 32) {
    keys[k] = ((uint64_t)(uint32_t)ci[k] << 32) | (uint32_t)row;
    idx[k] = k;
    atomicAdd(reinterpret_cast<unsigned long long*>(count + ci[k]), 1ull);
  }
}

__global__ void k_csr_t_fill(int64_t nnz, const uint64_t* __restrict__ keys, const int64_t* __restrict__ idx,
                             const double* __restrict__ v, int32_t* __restrict__ tc, double* __restrict__ tv) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    tc[k] = (int32_t)(keys[k] & 0xffffffffu);
    tv[k] = v[idx[k]];
  }
}

// ------------------------------------------------------------- host -----

inline unsigned grid_rows_warp(int64_t n, int threads = 256) {
  return (unsigned)std::max<int64_t>(1, (n * 32 + threads - 1) / threads);
}
inline unsigned grid_stride(int64_t n) { return (unsigned)std::min<int64_t>(std::max<int64_t>(1, (n + 255) / 256), 148 * 8); }

#define CSR_LAUNCH(...)  \
  do {                   \
    __VA_ARGS__;         \
    ++g_launches;        \
    CKL();               \
  } while (0)

// A CSR matrix resident on one device (uploaded from host arrays).
struct DevCsr {
  int n = 0;
  int64_t nnz = 0;
  DBuf<int64_t> rp;
  DBuf<int32_t> ci;
  DBuf<double> v;
  cudaStream_t s = nullptr;

  void upload(int n_, const int64_t* row_ptr, const int32_t* cols, const double* vals, cudaStream_t st) {
    n = n_;
    s = st;
    if (n < 0) throw SimError(IMPM_ERR_CONFIG, "negative matrix dimension");
    if (row_ptr[0] != 0) throw SimError(IMPM_ERR_CONFIG, "CSR row_ptr[0] must be 0");
    nnz = row_ptr[n];
    for (int i = 0; i < n; ++i)
      if (row_ptr[i + 1] < row_ptr[i]) throw SimError(IMPM_ERR_CONFIG, "CSR row_ptr is not monotone");
    for (int64_t k = 0; k < nnz; ++k)
      if (cols[k] < 0 || cols[k] >= n)
        throw SimError(IMPM_ERR_CONFIG, "CSR column index " + std::to_string(cols[k]) + " out of range");
    rp.ensure(n + 1);
    ci.ensure(nnz);
    v.ensure(nnz);
    CK(cudaMemcpyAsync(rp.get(), row_ptr, (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    if (nnz) {
      CK(cudaMemcpyAsync(ci.get(), cols, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(v.get(), vals, nnz * sizeof(double), cudaMemcpyHostToDevice, s));
    }
  }

  // device-resident CSR (already validated by construction): device-to-device copies
  void upload_device(int n_, const int64_t* row_ptr, const int32_t* cols, const double* vals, int64_t nnz_,
                     cudaStream_t st) {
    n = n_;
    s = st;
    nnz = nnz_;
    rp.ensure(n + 1);
    ci.ensure(std::max<int64_t>(nnz, 1));
    v.ensure(std::max<int64_t>(nnz, 1));
    CK(cudaMemcpyAsync(rp.get(), row_ptr, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    if (nnz) {
      CK(cudaMemcpyAsync(ci.get(), cols, nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(v.get(), vals, nnz * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
  }

  template <int MODE>
  void spmv(const double* x, double* y, const double* b = nullptr, const double* scale = nullptr) const {
    if (n == 0) return;
    const unsigned g = (unsigned)((n + 127) / 128);
    CSR_LAUNCH((k_csr_spmv<MODE><<<g, 128, 0, s>>>(n, rp.get(), ci.get(), v.get(), x, y, b, scale)));
  }
};

struct Reducer {
  DBuf<double> part;
  std::vector<double> host;
  cudaStream_t s = nullptr;
  // returns nv values (fixed-order host finalize of the kRedBlk partials)
  template <int MODE>
  const std::vector<double>& run(int64_t n, const double* A, int64_t lda, int nv, const double* b) {
    part.ensure((size_t)kRedBlk * std::max(nv, 1));
    host.assign((size_t)kRedBlk * nv, 0.0);
    CSR_LAUNCH((k_multi_reduce<MODE><<<kRedBlk, 256, 0, s>>>(n, A, lda, nv, b, part.get())));
    CK(cudaMemcpyAsync(host.data(), part.get(), host.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    for (int j = 0; j < nv; ++j) {
      double t = MODE == 2 ? 0.0 : 0.0;
      for (int blk = 0; blk < kRedBlk; ++blk) {
        const double u = host[(size_t)j * kRedBlk + blk];
        t = MODE == 2 ? std::max(t, u) : t + u;
      }
      host[j] = t;
    }
    host.resize(nv);
    return host;
  }
};

struct LuSolver {
  DevCsr A;
  Reducer red;
  DBuf<double> b, x, r, corr, scale, rabs, diag, M, V, hdev, z, zero;
  DBuf<int> perm, flags;  // flags[0] = empty row (INT_MAX none), flags[1] = singular column (-1 none)
  double mat_norm = 0.0, rhs_norm = 0.0;
  int krylov_iterations = 0;

  double backward_error() {  // |Ax-b|_2 / (|A|_inf |x|_inf + |b|_2)   (linear_solver.cpp:63-66)
    const int n = A.n;
    A.spmv<0>(x.get(), r.get());
    CSR_LAUNCH((k_axpy<true><<<grid_stride(n), 256, 0, A.s>>>(n, -1.0, b.get(), r.get())));
    const double rn = std::sqrt(red.run<1>(n, nullptr, 0, 1, r.get())[0]);
    const double xinf = red.run<2>(n, nullptr, 0, 1, x.get())[0];
    return rn / (mat_norm * xinf + rhs_norm);
  }

  // dense: M = P^-1 L U of the equilibrated matrix
  void dense_factor() {
    const int n = A.n;
    M.ensure((size_t)n * n);
    CK(cudaMemsetAsync(M.get(), 0, (size_t)n * n * sizeof(double), A.s));
    CSR_LAUNCH((k_dense_scatter<<<grid_rows_warp(n), 256, 0, A.s>>>(n, A.rp.get(), A.ci.get(), A.v.get(), scale.get(),
                                                                     M.get())));
    perm.ensure(n);
    std::vector<int> id(n);
    for (int i = 0; i < n; ++i) id[i] = i;
    CK(cudaMemcpyAsync(perm.get(), id.data(), n * sizeof(int), cudaMemcpyHostToDevice, A.s));
    for (int k = 0; k < n; ++k) {
      CSR_LAUNCH((k_lu_pivot<<<1, 1024, 0, A.s>>>(n, k, M.get(), perm.get(), flags.get() + 1)));
      const int m = n - k - 1;
      if (m > 0) {
        const dim3 g((m + 31) / 32, (m + 31) / 32);
        CSR_LAUNCH((k_lu_update<<<g, 256, 0, A.s>>>(n, k, M.get(), flags.get() + 1)));
      }
    }
    int sing = -1;
    CK(cudaMemcpyAsync(&sing, flags.get() + 1, sizeof(int), cudaMemcpyDeviceToHost, A.s));
    CK(cudaStreamSynchronize(A.s));
    if (sing >= 0)
      throw SimError(IMPM_ERR_LINEAR_SOLVER, "singular factorization: structurally or numerically zero pivot in column " +
                                                 std::to_string(sing));
  }

  void dense_solve(const double* rhs, double* out) {
    const int n = A.n;
    CSR_LAUNCH((k_lu_solve<<<1, 1024, n * sizeof(double), A.s>>>(n, M.get(), perm.get(), rhs, out)));
  }

  // GMRES(m) on the equilibrated system A_s = S^-1 A (S = row_scale), right-
  // preconditioned by diag(A_s): sol ~= A^-1 bu for the UNSCALED right-hand
  // side bu (the scaled one is formed inside the residual SpMV). Stops at a
  // relative scaled residual `target` or when a restart gains < 1%.
  void gmres(const double* bu, double* sol, double target) {
    const int n = A.n;
    const int m = kGmresM;
    V.ensure((size_t)(m + 1) * n);
    z.ensure(n);
    hdev.ensure(m + 1);
    std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), g(m + 1), yv(m);
    CK(cudaMemsetAsync(sol, 0, n * sizeof(double), A.s));
    double bn = -1.0, prev = INFINITY;
    for (int restart = 0; restart < kGmresMaxRestarts; ++restart) {
      A.spmv<1>(sol, V.get(), bu, scale.get());  // v0 = S^-1 (bu - A sol)
      const double beta = std::sqrt(red.run<1>(n, nullptr, 0, 1, V.get())[0]);
      if (!(beta == beta)) throw SimError(IMPM_ERR_LINEAR_SOLVER, "GMRES breakdown: NaN residual");
      if (bn < 0.0) bn = beta;
      if (beta == 0.0 || beta <= target * bn || beta > 0.99 * prev) return;
      prev = beta;
      CSR_LAUNCH((k_axpy<false><<<grid_stride(n), 256, 0, A.s>>>(n, 1.0 / beta, V.get(), V.get())));
      std::fill(g.begin(), g.end(), 0.0);
      g[0] = beta;
      int k = 0;
      bool done = false;
      for (; k < m && !done; ++k) {
        double* vk = V.get() + (size_t)k * n;
        double* w = V.get() + (size_t)(k + 1) * n;
        CSR_LAUNCH((k_jacobi<<<grid_stride(n), 256, 0, A.s>>>(n, diag.get(), vk, z.get())));
        A.spmv<1>(z.get(), w, zero.get(), scale.get());  // w = -A_s z
        CSR_LAUNCH((k_axpy<false><<<grid_stride(n), 256, 0, A.s>>>(n, -1.0, w, w)));
        std::vector<double> h(k + 1, 0.0);
        for (int pass = 0; pass < 2; ++pass) {  // classical Gram-Schmidt, twice
          const std::vector<double>& d = red.run<0>(n, V.get(), n, k + 1, w);
          CK(cudaMemcpyAsync(hdev.get(), d.data(), (k + 1) * sizeof(double), cudaMemcpyHostToDevice, A.s));
          for (int j = 0; j <= k; ++j) h[j] += d[j];
          CSR_LAUNCH((k_gs_sub<<<grid_stride(n), 256, 0, A.s>>>(n, V.get(), n, k + 1, hdev.get(), w)));
        }
        const double hn = std::sqrt(red.run<1>(n, nullptr, 0, 1, w)[0]);
        for (int j = 0; j <= k; ++j) H[(size_t)j * m + k] = h[j];
        H[(size_t)(k + 1) * m + k] = hn;
        if (hn > 0.0) CSR_LAUNCH((k_axpy<false><<<grid_stride(n), 256, 0, A.s>>>(n, 1.0 / hn, w, w)));
        for (int j = 0; j < k; ++j) {  // previous Givens rotations
          const double a = H[(size_t)j * m + k], c = H[(size_t)(j + 1) * m + k];
          H[(size_t)j * m + k] = cs[j] * a + sn[j] * c;
          H[(size_t)(j + 1) * m + k] = -sn[j] * a + cs[j] * c;
        }
        const double a = H[(size_t)k * m + k], c = H[(size_t)(k + 1) * m + k];
        const double rr = std::hypot(a, c);
        cs[k] = rr > 0.0 ? a / rr : 1.0;
        sn[k] = rr > 0.0 ? c / rr : 0.0;
        H[(size_t)k * m + k] = rr;
        H[(size_t)(k + 1) * m + k] = 0.0;
        g[k + 1] = -sn[k] * g[k];
        g[k] = cs[k] * g[k];
        ++krylov_iterations;
        if (std::fabs(g[k + 1]) <= 0.5 * target * bn || hn == 0.0) done = true;
      }
      for (int i = k - 1; i >= 0; --i) {  // H y = g
        double t = g[i];
        for (int j = i + 1; j < k; ++j) t -= H[(size_t)i * m + j] * yv[j];
        yv[i] = H[(size_t)i * m + i] != 0.0 ? t / H[(size_t)i * m + i] : 0.0;
      }
      CK(cudaMemcpyAsync(hdev.get(), yv.data(), k * sizeof(double), cudaMemcpyHostToDevice, A.s));
      CSR_LAUNCH((k_gmres_update<<<grid_stride(n), 256, 0, A.s>>>(n, V.get(), n, k, hdev.get(), diag.get(), sol)));
      CK(cudaStreamSynchronize(A.s));
    }
  }

  // sparse_lu_solve (src/linear_solver.cpp:11-88); host right-hand side and solution
  void solve(const double* bh, double* xh) { solve_io(bh, cudaMemcpyHostToDevice, xh, cudaMemcpyDeviceToHost); }
  // the same on device vectors (the direct path of the GPU Newton solve)
  void solve_device(const double* bd, double* xd) {
    solve_io(bd, cudaMemcpyDeviceToDevice, xd, cudaMemcpyDeviceToDevice);
  }

  void solve_io(const double* bh, cudaMemcpyKind kin, double* xh, cudaMemcpyKind kout) {
    const int n = A.n;
    const cudaStream_t s = A.s;
    red.s = s;
    if (n == 0) return;
    b.ensure(n); x.ensure(n); r.ensure(n); corr.ensure(n); scale.ensure(n); rabs.ensure(n); diag.ensure(n);
    zero.ensure(n);
    CK(cudaMemsetAsync(zero.get(), 0, n * sizeof(double), s));
    flags.ensure(2);
    const int init[2] = {INT_MAX, -1};
    CK(cudaMemcpyAsync(flags.get(), init, sizeof(init), cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(b.get(), bh, n * sizeof(double), kin, s));
    CSR_LAUNCH((k_csr_row_stats<<<grid_rows_warp(n), 256, 0, s>>>(n, A.rp.get(), A.v.get(), scale.get(), rabs.get(),
                                                                   flags.get(), diag.get(), A.ci.get())));
    int empty = INT_MAX;
    CK(cudaMemcpyAsync(&empty, flags.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (empty != INT_MAX) throw SimError(IMPM_ERR_LINEAR_SOLVER, "empty matrix row " + std::to_string(empty));
    mat_norm = red.run<2>(n, nullptr, 0, 1, rabs.get())[0];
    rhs_norm = std::sqrt(red.run<1>(n, nullptr, 0, 1, b.get())[0]);
    const bool dense = n <= kDenseMax;
    if (dense) {
      A.spmv<1>(zero.get(), corr.get(), b.get(), scale.get());  // b / s
      dense_factor();
      dense_solve(corr.get(), x.get());
    } else {
      gmres(b.get(), x.get(), 1e-14);
    }
    if (rhs_norm > 0.0) {
      double res = backward_error();
      for (int sweep = 0; sweep < 2 && res > 1e-14; ++sweep) {
        if (dense) {
          A.spmv<1>(x.get(), r.get(), b.get(), scale.get());  // (b - A x) / s
          dense_solve(r.get(), corr.get());
        } else {
          A.spmv<2>(x.get(), r.get(), b.get());  // b - A x (gmres equilibrates)
          gmres(r.get(), corr.get(), 1e-14);
        }
        CSR_LAUNCH((k_axpy<true><<<grid_stride(n), 256, 0, s>>>(n, 1.0, corr.get(), x.get())));
        res = backward_error();
      }
      if (!(res <= 1e-10)) {
        char buf[32];
        std::snprintf(buf, sizeof buf, "%.3e", res);
        throw SimError(IMPM_ERR_LINEAR_SOLVER, "solution backward error " + std::string(buf) +
                                                   " exceeds 1e-10; matrix is ill-conditioned or singular");
      }
    }
    CK(cudaMemcpyAsync(xh, x.get(), n * sizeof(double), kout, s));
    CK(cudaStreamSynchronize(s));
  }
};

// CsrMatrix::transposed (src/sparse.cpp:55-70): stable order (column, then row)
inline void transposed(const DevCsr& A, int64_t* t_rp, int32_t* t_ci, double* t_v) {
  const int n = A.n;
  const int64_t nnz = A.nnz;
  const cudaStream_t s = A.s;
  DBuf<uint64_t> keys, keys2;
  DBuf<int64_t> idx, idx2, count, rowp;
  DBuf<int32_t> tc;
  DBuf<double> tv;
  DBuf<unsigned char> tmp;
  keys.ensure(nnz); keys2.ensure(nnz); idx.ensure(nnz); idx2.ensure(nnz); count.ensure(n + 1); rowp.ensure(n + 1);
  tc.ensure(nnz); tv.ensure(nnz);
  CK(cudaMemsetAsync(count.get(), 0, (n + 1) * sizeof(int64_t), s));
  if (n > 0)
    CSR_LAUNCH((k_csr_keys<<<grid_rows_warp(n), 256, 0, s>>>(n, A.rp.get(), A.ci.get(), keys.get(), idx.get(),
                                                              count.get())));
  int bits = 1;
  while ((1ll << bits) < std::max(n, 2)) ++bits;
  size_t tb = 0, tb2 = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.get(), keys2.get(), idx.get(), idx2.get(), (int64_t)nnz, 0, 32 + bits, s));
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb2, count.get(), rowp.get(), n + 1, s));
  tmp.ensure(std::max(tb, tb2));
  if (nnz > 0) {
    CK(cub::DeviceRadixSort::SortPairs(tmp.get(), tb, keys.get(), keys2.get(), idx.get(), idx2.get(), (int64_t)nnz, 0,
                                       32 + bits, s));
    ++g_launches;
    CSR_LAUNCH((k_csr_t_fill<<<grid_stride(nnz), 256, 0, s>>>(nnz, keys2.get(), idx2.get(), A.v.get(), tc.get(), tv.get())));
  }
  CK(cub::DeviceScan::ExclusiveSum(tmp.get(), tb2, count.get(), rowp.get(), n + 1, s));
  ++g_launches;
  CK(cudaMemcpyAsync(t_rp, rowp.get(), (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  if (nnz > 0) {
    CK(cudaMemcpyAsync(t_ci, tc.get(), nnz * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(t_v, tv.get(), nnz * sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
}

}  // namespace csr
