// sm_100a kernels of the implicit MPM Newton step (fp64, HBM-bound).
//
// Data layout in HBM:
//   particles   SoA pd[field * cap + i], fields in impm::Particle<D> order,
//               kept cell-sorted (counting sort on the first support node);
//   grid vectors [node][field] over ALL grid nodes, zero at non-free DOFs, so
//               a node's D components are one 8*D-byte record;
//   Jacobian    "box BSR": one row per active node, 5^D implicit block
//               columns (the reference pattern, jacobian.hpp:36-65), F x F
//               blocks, row length padded to a multiple of 4 doubles;
//   tangent     per-particle dP/dG, AoS [P][D^4] (read by 3^D rows).
//
// Reductions are deterministic: per-block partials in fixed order + one
// finalize block. No global float atomics anywhere on the path.
#pragma once
#include <cuda_fp16.h>

#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <type_traits>

#include "impm_math.cuh"

namespace impm_gpu {

// Checked build (-DIMPM_CHECKED, scripts/checked_cases.sh): the index math of
// the scattered accesses (assembly block updates, transpose pass, SpMV gathers,
// residual node updates) is range-checked on the device and violations are
// counted (impm_debug_oob_count). compute-sanitizer is closed on this pool.
#ifdef IMPM_CHECKED
__device__ unsigned long long g_oob_count = 0;
#define IMPM_CHECK_IDX(i, n)                                                              \
  do {                                                                                    \
    if (static_cast<unsigned long long>(i) >= static_cast<unsigned long long>(n))         \
      atomicAdd(&g_oob_count, 1ull);                                                      \
  } while (0)
#else
#define IMPM_CHECK_IDX(i, n) ((void)0)
#endif

__host__ __device__ constexpr int ipow_c(int b, int e) { return e == 0 ? 1 : b * ipow_c(b, e - 1); }
__host__ __device__ constexpr int pad4(int x) { return (x + 3) / 4 * 4; }
// Compacted rows are stored component-major: [c][block pos][d], each
// component chunk padded to an even length (16-byte aligned double2 loads).
__host__ __device__ constexpr int cpad(int nzb, int F) { return (nzb * F + 1) & ~1; }
__host__ __device__ constexpr int row_len_for(int S, int F) { return pad4(F * cpad(S, F)); }
// per-component chunk length of a compacted row: fp64 rows pad to 2 values
// (double2 loads), fp32 rows to 4 (float4 loads); both 16-byte aligned
template <class VT>
__host__ __device__ constexpr int chunk_len(int nzb, int F) {
  return sizeof(VT) == 8 ? cpad(nzb, F) : (sizeof(VT) == 4 ? ((nzb * F + 3) & ~3) : ((nzb * F + 7) & ~7));
}
template <class VT>
__host__ __device__ constexpr int64_t row_len_of(int S, int F) {
  return sizeof(VT) == 8 ? row_len_for(S, F) : static_cast<int64_t>(F) * chunk_len<VT>(S, F);
}

// Particle<D> field offsets (particle.hpp:10-29)
template <int D>
struct PF {
  static constexpr int X = 0, x = D, m = 2 * D, V0 = 2 * D + 1, V = 2 * D + 2, F = 2 * D + 3,
                       sigma = 2 * D + 3 + D * D, lp0 = 2 * D + 12 + D * D, lp = 3 * D + 12 + D * D,
                       Be = 4 * D + 12 + D * D, alpha = 4 * D + 21 + D * D,
                       trac = 4 * D + 22 + D * D, pload = 5 * D + 22 + D * D,
                       N = 6 * D + 22 + D * D;
};

struct GridC {
  int nodes[3];
  int stride[3];
  double origin[3];
  double h;
  int N;
  // global axis-0 index of local node 0 (slab decomposition): node positions
  // and supports stay relative to the GLOBAL origin, so a slab computes the
  // same fp64 weights, bit for bit, as the single-GPU grid
  int base0;
};

template <int D>
__device__ __forceinline__ void unflat(const GridC& g, int n, int* idx) {
#pragma unroll
  for (int a = 0; a < D; ++a) idx[a] = (n / g.stride[a]) % g.nodes[a];
}

__device__ __forceinline__ double node_coord(const GridC& g, int a, int i) {
  const int gi = a == 0 ? i + g.base0 : i;
  return __dadd_rn(g.origin[a], __dmul_rn(static_cast<double>(gi), g.h));  // grid.hpp:180-185
}

// packed support counts: 2 bits per axis
__device__ __forceinline__ int sup_cnt(int s, int a) { return (s >> (2 * a)) & 3; }

// weights of one axis for a particle at its support nodes [first, first+cnt)
struct AxisW {
  double w[3], dw[3];
};

template <int SHAPE>
__device__ __forceinline__ WeightValue weight_1d(double xi, double lp, double h) {
  if constexpr (SHAPE == 2) return bspline2_weight_1d(xi, h);
  return gimp_weight_1d(xi, lp, h);
}

// gimp_weight<D> (gimp.hpp:37-52): w = prod w_a, grad_a = dw_a prod_{b!=a} w_b
template <int D>
__device__ __forceinline__ void tensor_weight(const double* w, const double* dw, double& W, double* grad) {
  W = 1.0;
#pragma unroll
  for (int a = 0; a < D; ++a) W *= w[a];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double gg = dw[a];
#pragma unroll
    for (int b = 0; b < D; ++b)
      if (b != a) gg *= w[b];
    grad[a] = gg;
  }
}

// ------------------------------------------------------------ layout io --
__global__ void k_aos_to_soa(const double* __restrict__ aos, int64_t stride_dbl, int n, int nd,
                             double* __restrict__ soa, int64_t cap, int* __restrict__ orig) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int f = 0; f < nd; ++f) soa[f * cap + i] = aos[i * stride_dbl + f];
  orig[i] = i;
}

__global__ void k_soa_to_aos(const double* __restrict__ soa, int64_t cap, int n, int nd,
                             const int* __restrict__ orig, double* __restrict__ aos, int64_t stride_dbl) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t o = orig[i];
  for (int f = 0; f < nd; ++f) aos[o * stride_dbl + f] = soa[f * cap + i];
}

// chunked particle I/O (the copies of one chunk overlap the layout kernel of
// the next): inverse of the sorted -> original permutation, and AoS rows
// [o0, o1) in original order gathered from the sorted SoA
__global__ void k_invert_perm(const int* __restrict__ orig, int n, int* __restrict__ inv) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) inv[orig[i]] = i;
}
__global__ void k_rows_to_aos(const double* __restrict__ soa, int64_t cap, const int* __restrict__ inv, int o0,
                              int o1, int nd, double* __restrict__ aos) {
  const int64_t e0 = static_cast<int64_t>(o0) * nd, e1 = static_cast<int64_t>(o1) * nd;
  for (int64_t e = e0 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < e1;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = e / nd;
    const int f = static_cast<int>(e - row * nd);
    aos[e] = soa[f * cap + inv[row]];
  }
}
__global__ void k_aos_rows_to_soa(const double* __restrict__ aos, int r0, int r1, int nd, double* __restrict__ soa,
                                  int64_t cap, int* __restrict__ orig) {
  const int i = r0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r1) return;
  for (int f = 0; f < nd; ++f) soa[f * cap + i] = aos[static_cast<int64_t>(i) * nd + f];
  orig[i] = i;
}

// per-particle field in ORIGINAL order -> sorted slot
__global__ void k_set_field(double* __restrict__ col, const double* __restrict__ vals,
                            const int* __restrict__ orig, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) col[i] = vals[orig[i]];
}

// ------------------------------------------------------------ K1 binning --
// Device status words (one small struct read back per host decision).
struct DevStatus {
  double norm2;       // last reduction
  double max_mass;    // max particle mass (as ordered bits)
  int err_domain;     // min original particle id with det <= 0 (INT_MAX none)
  int err_ood;        // min (orig*4 + axis) with support outside the grid
  int err_cfg;        // min original id with lp outside (0, h/2)
  int perm_moved;     // counting sort moved at least one particle
  int err_lp;         // commit: min original id with lp >= h/2 or <= 0
  int err_migrate;    // slab migration: min original id that left the neighbour slabs
  int err_seed;       // min (orig*4 + axis) whose support exceeds the 3-node stencil (seeding hazard)
};

template <int D, int SHAPE>
__global__ void k_support(const double* __restrict__ pd, int64_t cap, int P, GridC g,
                          const int* __restrict__ orig, int* __restrict__ key, int* __restrict__ sup,
                          double* __restrict__ xs, DevStatus* st, int use_X = 0) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  int k = 0, packed = 0;
  bool ok = true;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const double x = pd[((use_X ? PF<D>::X : PF<D>::x) + a) * cap + i];
    const double lp = pd[(PF<D>::lp + a) * cap + i];
    xs[a * cap + i] = x;
    int first, count;
    if constexpr (SHAPE == 2) {
      // quadratic B-spline: nodes with |x - x_i| < 1.5 h
      const double lo = __dsub_rn(__dsub_rn(x, g.origin[a]), 1.5 * g.h);
      const double hi = __dadd_rn(__dsub_rn(x, g.origin[a]), 1.5 * g.h);
      first = static_cast<int>(floor(__ddiv_rn(lo, g.h))) + 1;
      count = static_cast<int>(ceil(__ddiv_rn(hi, g.h))) - 1 - first + 1;
    } else {
      gimp_support_1d(x, lp, g.origin[a], g.h, first, count);
    }
    if (a == 0) first -= g.base0;
    if (ok && (first < 0 || first + count > g.nodes[a])) {
      atomicMin(&st->err_ood, orig[i] * 4 + a);  // mpm_solver.hpp:105-110
      ok = false;
    }
    if (SHAPE != 2 && (!(lp > 0.0) || lp >= 0.5 * g.h)) atomicMin(&st->err_cfg, orig[i]);  // gimp.cpp:28-30
    if (count < 1) count = 1;
    // a support wider than 3 nodes would couple nodes beyond the +-2 pattern
    // (b = 5, gimp.cpp:7-15) and break the colour/owner separation of the
    // assembly: the GPU form of the reference's seeding hazard
    // (jacobian.hpp:167-182), reported as SeedingFault when checked
    if (count > 3) {
      atomicMin(&st->err_seed, orig[i] * 4 + a);
      count = 3;
    }
    if (first < 0) first = 0;
    if (first + count > g.nodes[a]) first = g.nodes[a] - count;
    k += first * g.stride[a];
    packed |= count << (2 * a);
  }
  key[i] = k;
  sup[i] = packed;
}

__global__ void k_bin_count(const int* __restrict__ key, int P, int* __restrict__ count, int* __restrict__ rank) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < P) rank[i] = atomicAdd(&count[key[i]], 1);
}

__global__ void k_bin_scatter(const int* __restrict__ key, const int* __restrict__ rank,
                              const int* __restrict__ start, int P, int* __restrict__ perm) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < P) perm[start[key[i]] + rank[i]] = i;
}

// stable order inside each bin (by previous slot) => deterministic sort
__global__ void k_bin_sort(const int* __restrict__ start, int N, int* __restrict__ perm) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= N) return;
  const int s = start[b], e = start[b + 1];
  for (int i = s + 1; i < e; ++i) {
    const int v = perm[i];
    int j = i - 1;
    while (j >= s && perm[j] > v) {
      perm[j + 1] = perm[j];
      --j;
    }
    perm[j + 1] = v;
  }
}

__global__ void k_perm_check(const int* __restrict__ perm, int P, DevStatus* st) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < P && perm[i] != i) st->perm_moved = 1;
}

// dst[f][i] = src[f][perm[i]] for all fields (blockIdx.y = field)
// blockIdx.y takes fields [fpb y, fpb y + fpb) of nf: one perm load per particle
// serves fpb fields, whose loads are in flight together
__global__ void k_gather_fields(const double* __restrict__ src, double* __restrict__ dst, int64_t cap,
                                const int* __restrict__ perm, int P, int nf = 1, int fpb = 1) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const int64_t j = perm[i];
  const int f0 = blockIdx.y * fpb, f1 = min(nf, f0 + fpb);
  constexpr int U = 8;
  for (int fb = f0; fb < f1; fb += U) {
    double v[U];
#pragma unroll
    for (int q = 0; q < U; ++q) v[q] = fb + q < f1 ? src[(fb + q) * cap + j] : 0.0;
#pragma unroll
    for (int q = 0; q < U; ++q)
      if (fb + q < f1) dst[(fb + q) * cap + i] = v[q];
  }
}
__global__ void k_gather_int(const int* __restrict__ src, int* __restrict__ dst, const int* __restrict__ perm, int P) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < P) dst[i] = src[perm[i]];
}

// external load per particle at unit schedule (mpm_solver.hpp:205-206) and max mass
template <int D>
__global__ void k_bext(const double* __restrict__ pd, int64_t cap, int P, double gx, double gy, double gz,
                       double* __restrict__ bext, DevStatus* st) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double m = 0.0;
  if (i < P) {
    m = pd[PF<D>::m * cap + i];
    const double g[3] = {gx, gy, gz};
#pragma unroll
    for (int c = 0; c < D; ++c)
      bext[c * cap + i] = m * g[c] + pd[(PF<D>::trac + c) * cap + i] + pd[(PF<D>::pload + c) * cap + i];
  }
  // block max, then one atomicMax on the (positive) double's bit pattern
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0 && m > 0.0)
      atomicMax(reinterpret_cast<unsigned long long*>(&st->max_mass), __double_as_longlong(m));
  }
}

// Visits the particles whose support contains node `idx`, in fixed order
// (3^D candidate bins lexicographic, then sorted slot order): fn(p, off[]).
template <int D, class Fn>
__device__ __forceinline__ void for_each_particle_of_node(const GridC& g, const int* idx,
                                                          const int* __restrict__ bin_start,
                                                          const int* __restrict__ sup, Fn&& fn) {
  constexpr int NB = ipow_c(3, D);
  for (int ob = 0; ob < NB; ++ob) {
    int off[3] = {0, 0, 0};
    int r = ob, b = 0;
    bool ok = true;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      off[a] = r % 3;
      r /= 3;
      const int bi = idx[a] - off[a];
      ok = ok && bi >= 0;
      b += bi * g.stride[a];
    }
    if (!ok) continue;
    const int s = bin_start[b], e = bin_start[b + 1];
    for (int p = s; p < e; ++p) {
      const int sp = sup[p];
      bool in = true;
#pragma unroll
      for (int a = 0; a < D; ++a) in = in && off[a] < sup_cnt(sp, a);
      if (in) fn(p, off);
    }
  }
}

// K2: node mass (pull, deterministic) + active flag + free flags
template <int D, int F, int SHAPE>
__global__ void k_node_mass(GridC g, const double* __restrict__ pd, int64_t cap, const double* __restrict__ xs,
                            const int* __restrict__ bin_start, const int* __restrict__ sup,
                            const uint8_t* __restrict__ fixed, const DevStatus* st, double* __restrict__ mass,
                            int* __restrict__ act_flag, int* __restrict__ free_flag) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.N) return;
  int idx[3];
  unflat<D>(g, n, idx);
  double M = 0.0;
  for_each_particle_of_node<D>(g, idx, bin_start, sup, [&](int p, const int*) {
    double w[3], dw[3];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const WeightValue wv = weight_1d<SHAPE>(xs[a * cap + p] - node_coord(g, a, idx[a]),
                                              pd[(PF<D>::lp + a) * cap + p], g.h);
      w[a] = wv.w;
      dw[a] = wv.dw;
    }
    double W, grad[3];
    tensor_weight<D>(w, dw, W, grad);
    M += W * pd[PF<D>::m * cap + p];
  });
  mass[n] = M;
  const int active = M > 1e-12 * st->max_mass ? 1 : 0;  // mpm_solver.hpp:131-133
  act_flag[n] = active;
#pragma unroll
  for (int c = 0; c < F; ++c) free_flag[n * F + c] = active && !fixed[n * F + c];
}

// K3: DofMap::build (grid.hpp:69-86) from exclusive scans
__global__ void k_dof_finalize(int NF, int F, const int* __restrict__ free_flag, const int* __restrict__ free_scan,
                               int* __restrict__ dof_of, int* __restrict__ node_of, int* __restrict__ field_of,
                               uint8_t* __restrict__ freem) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= NF) return;
  const int f = free_flag[j];
  freem[j] = static_cast<uint8_t>(f);
  if (f) {
    const int d = free_scan[j];
    dof_of[j] = d;
    node_of[d] = j / F;
    field_of[d] = j % F;
  } else {
    dof_of[j] = -1;
  }
}

__global__ void k_act_finalize(int N, const int* __restrict__ act_flag, const int* __restrict__ act_scan,
                               int* __restrict__ act_idx, int* __restrict__ act_list) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  if (act_flag[n]) {
    const int r = act_scan[n];
    act_idx[n] = r;
    act_list[r] = n;
  } else {
    act_idx[n] = -1;
  }
}

// Row order of the box-BSR: brick-major (4^D node bricks, flat order of bricks
// and of nodes inside a brick). A CTA's chunk of 64 rows is then one 4x4x4
// brick whose SpMV x-neighbourhood (8^3 nodes, 12 KB) stays in L1. Row order
// is internal: DOF numbering, grid vectors and exports are node-indexed.
template <int D>
__device__ __forceinline__ int brick_pos(const GridC& g, const int* idx) {
  int p = 0, l = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const int nb = (g.nodes[a] + 3) >> 2;
    p = p * nb + (idx[a] >> 2);
    l = l * 4 + (idx[a] & 3);
  }
  return (p << (2 * D)) | l;
}

template <int D>
__global__ void k_brick_flags(GridC g, const int* __restrict__ act_flag, int* __restrict__ bflags) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.N) return;
  int idx[3];
  unflat<D>(g, n, idx);
  bflags[brick_pos<D>(g, idx)] = act_flag[n];
}

template <int D>
__global__ void k_act_finalize_brick(GridC g, const int* __restrict__ act_flag, const int* __restrict__ bscan,
                                     int* __restrict__ act_idx, int* __restrict__ act_list) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.N) return;
  if (act_flag[n]) {
    int idx[3];
    unflat<D>(g, n, idx);
    const int r = bscan[brick_pos<D>(g, idx)];
    act_idx[n] = r;
    act_list[r] = n;
  } else {
    act_idx[n] = -1;
  }
}

// ------------------------------------------------------ block reductions --
template <int NV>
__device__ __forceinline__ void block_sum_store(double (&v)[NV], double* __restrict__ partials) {
  __shared__ double red[NV][32];
#pragma unroll
  for (int k = 0; k < NV; ++k)
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) red[k][w] = v[k];
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = l < nw ? red[k][l] : 0.0;
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (l == 0) partials[k * gridDim.x + blockIdx.x] = s;
    }
  }
}

// block partials of an int64 array (exact in fp64 while every partial < 2^53)
__global__ void k_sum_i64(int64_t n, const int64_t* __restrict__ v, double* __restrict__ partials) {
  double s[1] = {0.0};
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    s[0] += static_cast<double>(v[i]);
  block_sum_store<1>(s, partials);
}

// sums NV rows of `nb` partials in fixed order into out[0..NV)
template <int NV>
__global__ void k_finalize_sum(const double* __restrict__ partials, int nb, double* __restrict__ out) {
  double v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) s += partials[k * nb + i];
    v[k] = s;
  }
  __shared__ double red[NV][32];
#pragma unroll
  for (int k = 0; k < NV; ++k)
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k) red[k][w] = v[k];
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = l < nw ? red[k][l] : 0.0;
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (l == 0) out[k] = s;
    }
  }
}

// ---------------------------------------------------------- K5 residual --
// Displacement gradient at a particle from its support (mpm_solver.hpp:164-171),
// lexicographic support order, last axis fastest.
template <int D, int SHAPE>
__device__ __forceinline__ void particle_weights(const GridC& g, const double* __restrict__ pd, int64_t cap,
                                                 const double* __restrict__ xs, int p, int key, int sp,
                                                 int* first, int* cnt, AxisW* aw) {
  int rem = key;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    first[a] = rem / g.stride[a];
    rem -= first[a] * g.stride[a];
    cnt[a] = sup_cnt(sp, a);
    const double x = xs[a * cap + p];
    const double lp = pd[(PF<D>::lp + a) * cap + p];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (i < cnt[a]) {
        const WeightValue wv = weight_1d<SHAPE>(x - node_coord(g, a, first[a] + i), lp, g.h);
        aw[a].w[i] = wv.w;
        aw[a].dw[i] = wv.dw;
      } else {
        aw[a].w[i] = 0.0;
        aw[a].dw[i] = 0.0;
      }
    }
  }
}

// iterate the support of a particle: fn(node, W, grad)
template <int D, class Fn>
__device__ __forceinline__ void for_each_support(const GridC& g, const int* first, const int* cnt, const AxisW* aw,
                                                 Fn&& fn) {
  const int c0 = cnt[0], c1 = D > 1 ? cnt[1] : 1, c2 = D > 2 ? cnt[2] : 1;
  for (int i = 0; i < c0; ++i)
    for (int j = 0; j < c1; ++j)
      for (int k = 0; k < c2; ++k) {
        const int li[3] = {i, j, k};
        double w[3], dw[3];
        int node = 0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          w[a] = aw[a].w[li[a]];
          dw[a] = aw[a].dw[li[a]];
          node += (first[a] + li[a]) * g.stride[a];
        }
        double W, grad[3];
        tensor_weight<D>(w, dw, W, grad);
        fn(node, W, grad);
      }
}

struct MatParams {
  int kind;
  double lam, mu, kappa;
  double dp_alpha;  // Drucker-Prager sqrt(2/3) 2 sin(phi) / (3 - sin(phi))
  double dp_ec;     // apex strain shift 3 c / (3 lam + 2 mu)
  double mcc_M;     // Cam-Clay critical-state slope 6 sin(phi) / (3 - sin(phi))
  double mcc_pc0;   // initial preconsolidation pressure
  double mcc_theta; // hardening exponent (1 + e0) / (lambda - kappa)
  double mcc_pt;    // tensile intercept
};

__host__ __device__ __forceinline__ bool has_history(int kind) {
  return kind == kHenckyJ2 || kind == kDruckerPrager || kind == kCamClay;
}

// update_stress (mpm_solver.hpp:445-454) over scalar T. NHO: the kind is
// known to be neo-Hookean at compile time (keeps the 3D tangent lean).
template <class T, int D, bool NHO = false>
__device__ __forceinline__ StressOut<T> update_stress(const MatParams& mp, const Mat<T, D>& F_new,
                                                      const Mat<T, D>& f_inc, const double* Be_n,
                                                      double* Be_out = nullptr, double* dg_out = nullptr) {
  const T lam = T(mp.lam), mu = T(mp.mu);
  if constexpr (NHO) return neo_hookean_update<T, D>(F_new, lam, mu);
  if (mp.kind == kNeoHookean) return neo_hookean_update<T, D>(F_new, lam, mu);
  // D = 3 Hencky / J2 / Drucker-Prager / Cam-Clay take the 3x3 spectral
  // log/exp (extensions; the reference stops at D <= 2, mpm_solver.hpp:448-453)
  if (mp.kind == kHencky) return hencky_update<T, D>(F_new, lam, mu);
  if (mp.kind == kDruckerPrager) return dp_update<T, D>(F_new, f_inc, Be_n, lam, mu, mp.dp_alpha, mp.dp_ec, Be_out, dg_out);
  if (mp.kind == kCamClay)
    return mcc_update<T, D>(F_new, f_inc, Be_n, mp.lam + 2.0 * mp.mu / 3.0, mp.mu, mp.mcc_M, mp.mcc_pc0, mp.mcc_theta,
                            mp.mcc_pt, Be_out, dg_out);
  return j2_update<T, D>(f_inc, Be_n, lam, mu, mp.kappa, Be_out, dg_out);
}

// Residual phase A (particles): G, f_inc, F_new, det check, sigma, V and the
// nominal stress P = V sigma f_inc^{-T} so that the node-side gather is
// r_{k,c} = sum_b grad_{k,b} P_{cb} - w_k b_c s  (mpm_solver.hpp:164-208).
template <int D, int SHAPE, bool NHO>
#ifndef IMPM_RESP_MINB
#define IMPM_RESP_MINB 4  // resident 256-thread CTAs per SM (64 registers): 0.94 vs 1.06 ms per cfg 4 residual at 1 (80 registers); 5: 1.15
#endif
__global__ void __launch_bounds__(256, IMPM_RESP_MINB) k_residual_particles(GridC g, const double* __restrict__ pd, int64_t cap, int P,
                                     const double* __restrict__ xs, const int* __restrict__ key,
                                     const int* __restrict__ sup, const int* __restrict__ orig,
                                     const double* __restrict__ u, MatParams mp, int tl,
                                     double* __restrict__ Pst, DevStatus* st) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int first[3], cnt[3];
  AxisW aw[3];
  particle_weights<D, SHAPE>(g, pd, cap, xs, p, key[p], sup[p], first, cnt, aw);
  Mat<double, D> G = Mat<double, D>::zero();
  for_each_support<D>(g, first, cnt, aw, [&](int node, double, const double* grad) {
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double uc = u[node * D + c];
#pragma unroll
      for (int a = 0; a < D; ++a) G(c, a) += uc * grad[a];
    }
  });
  Mat<double, D> f_inc = G;
#pragma unroll
  for (int a = 0; a < D; ++a) f_inc(a, a) += 1.0;
  Mat<double, D> F_new;
  if (tl) {
    F_new = f_inc;
  } else {
    Mat<double, D> Fn;
#pragma unroll
    for (int i = 0; i < D * D; ++i) Fn.e[i] = pd[(PF<D>::F + i) * cap + p];
    F_new = matmul(f_inc, Fn);
  }
  double* out = Pst + static_cast<int64_t>(p) * D * D;
  if (!(det(F_new) > 0.0)) {  // mpm_solver.hpp:183-184
    atomicMin(&st->err_domain, orig[p]);
#pragma unroll
    for (int i = 0; i < D * D; ++i) out[i] = 0.0;
    return;
  }
  double Be_n[10];
  if (has_history(mp.kind))
#pragma unroll
    for (int i = 0; i < 9; ++i) Be_n[i] = pd[(PF<D>::Be + i) * cap + p];
  if (mp.kind == kCamClay) Be_n[9] = pd[PF<D>::alpha * cap + p];
  const StressOut<double> su = update_stress<double, D, NHO>(mp, F_new, f_inc, Be_n);
  const double V = su.J * pd[PF<D>::V0 * cap + p];
  const Mat<double, D> fi = inverse(f_inc);
#pragma unroll
  for (int c = 0; c < D; ++c)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double s = su.sigma(c, 0) * fi(b, 0);
#pragma unroll
      for (int a = 1; a < D; ++a) s += su.sigma(c, a) * fi(b, a);
      out[c * D + b] = V * s;
    }
}

// Residual phase B, bin-centric push in 3^D colour batches (bins of one
// colour have disjoint supports): a warp owns a bin, lane k < nk owns box
// node k and sums the bin's particle contributions
// sum_b grad_{k,b} P_cb - w_k b_c s in fixed order, then adds them to r[k]
// (exclusive within the colour; r zeroed first). Masking and r.r follow in
// k_mask_norm.
template <int D, int SHAPE, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_residual_bins(
    GridC g, const double* __restrict__ pd, int64_t cap, const double* __restrict__ xs,
    const int* __restrict__ bin_start, const uint8_t* __restrict__ bflag, const double* __restrict__ Pst,
    const double* __restrict__ bext, double load_scale, double* __restrict__ r, int c0, int c1, int c2, int nb0,
    int nb1, int nb2) {
  __shared__ double W1[WARPS][D][3][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbins = nb0 * nb1 * nb2;
  const int col[3] = {c0, c1, c2};
  const int nbv[3] = {nb0, nb1, nb2};
  for (int bi = blockIdx.x * WARPS + warp; bi < nbins; bi += gridDim.x * WARPS) {
    int bidx[3] = {0, 0, 0}, rr = bi, b = 0;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      bidx[a] = 3 * (rr % nbv[a]) + col[a];
      rr /= nbv[a];
      b += bidx[a] * g.stride[a];
    }
    const int fl = bflag[b];
    if (!(fl & 0x80)) continue;
    int cn[3] = {1, 1, 1};
#pragma unroll
    for (int a = 0; a < D; ++a) cn[a] = 2 + ((fl >> a) & 1);
    const int nk = cn[0] * cn[1] * cn[2];
    int li[3] = {0, 0, 0};
    {
      int rk = lane;
#pragma unroll
      for (int a = D - 1; a >= 0; --a) {
        li[a] = rk % cn[a];
        rk /= cn[a];
      }
    }
    double acc[3] = {0.0, 0.0, 0.0};
    const int p0 = bin_start[b], p1 = bin_start[b + 1];
    for (int p = p0; p < p1; ++p) {
      __syncwarp();
      if (lane < 3 * D) {
        const int a = lane / 3, i = lane % 3;
        double w = 0.0, dw = 0.0;
        if (i < cn[a]) {
          const WeightValue wv = weight_1d<SHAPE>(xs[a * cap + p] - node_coord(g, a, bidx[a] + i),
                                                  pd[(PF<D>::lp + a) * cap + p], g.h);
          w = wv.w;
          dw = wv.dw;
        }
        W1[warp][a][i][0] = w;
        W1[warp][a][i][1] = dw;
      }
      __syncwarp();
      if (lane < nk) {
        double w[3], dw[3], W, gr[3];
#pragma unroll
        for (int a = 0; a < D; ++a) {
          w[a] = W1[warp][a][li[a]][0];
          dw[a] = W1[warp][a][li[a]][1];
        }
        tensor_weight<D>(w, dw, W, gr);
        const double* Pp = Pst + static_cast<int64_t>(p) * D * D;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          double fint = gr[0] * __ldg(Pp + c * D);
#pragma unroll
          for (int bb = 1; bb < D; ++bb) fint += gr[bb] * __ldg(Pp + c * D + bb);
          const double fext = W * __ldg(bext + c * cap + p) * load_scale;
          acc[c] += fint - fext;
        }
      }
    }
    if (lane < nk) {
      int node = 0;
#pragma unroll
      for (int a = 0; a < D; ++a) node += (bidx[a] + li[a]) * g.stride[a];
#pragma unroll
      for (int c = 0; c < D; ++c) r[static_cast<int64_t>(node) * D + c] += acc[c];
    }
  }
}

// Staged variant of k_residual_bins: the bin's particles are processed in
// chunks of PCH with every global load of the chunk in flight at once
// (positions, lp, nominal stress P, external-force density) into shared
// memory, the 1D weights of all chunk particles computed in parallel, then the
// node lanes sum from shared memory in the same fixed particle order (bitwise
// the values of k_residual_bins). Removes the per-particle load->sync->FMA
// latency chain of the unstaged loop.
#ifndef IMPM_RESB_MINB
#define IMPM_RESB_MINB 0  // 0: the compiler's register choice
#endif
#if IMPM_RESB_MINB > 0
#define IMPM_RESB_LB(T) __launch_bounds__(T, IMPM_RESB_MINB)
#else
#define IMPM_RESB_LB(T) __launch_bounds__(T)
#endif
template <int D, int SHAPE, int WARPS, int PCH>
__global__ void IMPM_RESB_LB(WARPS * 32) k_residual_bins_staged(
    GridC g, const double* __restrict__ pd, int64_t cap, const double* __restrict__ xs,
    const int* __restrict__ bin_start, const uint8_t* __restrict__ bflag, const double* __restrict__ Pst,
    const double* __restrict__ bext, double load_scale, double* __restrict__ r, int c0, int c1, int c2, int nb0,
    int nb1, int nb2) {
  constexpr int DD = D * D;
  __shared__ double Ps[WARPS][PCH * DD];
  __shared__ double Bs[WARPS][PCH][D];
  __shared__ double W1[WARPS][PCH][D][3][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbins = nb0 * nb1 * nb2;
  const int col[3] = {c0, c1, c2};
  const int nbv[3] = {nb0, nb1, nb2};
  for (int bi = blockIdx.x * WARPS + warp; bi < nbins; bi += gridDim.x * WARPS) {
    int bidx[3] = {0, 0, 0}, rr = bi, b = 0;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      bidx[a] = 3 * (rr % nbv[a]) + col[a];
      rr /= nbv[a];
      b += bidx[a] * g.stride[a];
    }
    const int fl = bflag[b];
    if (!(fl & 0x80)) continue;
    int cn[3] = {1, 1, 1};
#pragma unroll
    for (int a = 0; a < D; ++a) cn[a] = 2 + ((fl >> a) & 1);
    const int nk = cn[0] * cn[1] * cn[2];
    int li[3] = {0, 0, 0};
    {
      int rk = lane;
#pragma unroll
      for (int a = D - 1; a >= 0; --a) {
        li[a] = rk % cn[a];
        rk /= cn[a];
      }
    }
    double acc[3] = {0.0, 0.0, 0.0};
    const int p0 = bin_start[b], p1 = bin_start[b + 1];
    for (int pc = p0; pc < p1; pc += PCH) {
      const int np = min(PCH, p1 - pc);
      __syncwarp();
      // P of the chunk is contiguous (particle-major, D*D per particle)
      const double* Pb = Pst + static_cast<int64_t>(pc) * DD;
      for (int e = lane; e < np * DD; e += 32) Ps[warp][e] = __ldg(Pb + e);
      for (int e = lane; e < np * D; e += 32) {
        const int pl = e / D, c = e - pl * D;
        Bs[warp][pl][c] = __ldg(bext + c * cap + pc + pl);
      }
      for (int e = lane; e < np * D * 3; e += 32) {
        const int pl = e / (D * 3), rem = e - pl * D * 3, a = rem / 3, i = rem - a * 3;
        double w = 0.0, dw = 0.0;
        if (i < cn[a]) {
          const int p = pc + pl;
          const WeightValue wv = weight_1d<SHAPE>(__ldg(xs + a * cap + p) - node_coord(g, a, bidx[a] + i),
                                                  __ldg(pd + (PF<D>::lp + a) * cap + p), g.h);
          w = wv.w;
          dw = wv.dw;
        }
        W1[warp][pl][a][i][0] = w;
        W1[warp][pl][a][i][1] = dw;
      }
      __syncwarp();
      if (lane < nk) {
        for (int pl = 0; pl < np; ++pl) {
          double w[3], dw[3], W, gr[3];
#pragma unroll
          for (int a = 0; a < D; ++a) {
            w[a] = W1[warp][pl][a][li[a]][0];
            dw[a] = W1[warp][pl][a][li[a]][1];
          }
          tensor_weight<D>(w, dw, W, gr);
          const double* Pp = &Ps[warp][pl * DD];
#pragma unroll
          for (int c = 0; c < D; ++c) {
            double fint = gr[0] * Pp[c * D];
#pragma unroll
            for (int bb = 1; bb < D; ++bb) fint += gr[bb] * Pp[c * D + bb];
            const double fext = W * Bs[warp][pl][c] * load_scale;  // same association as k_residual_bins
            acc[c] += fint - fext;
          }
        }
      }
    }
    if (lane < nk) {
      int node = 0;
#pragma unroll
      for (int a = 0; a < D; ++a) node += (bidx[a] + li[a]) * g.stride[a];
      IMPM_CHECK_IDX(node, g.N);
#pragma unroll
      for (int c = 0; c < D; ++c) atomicAdd(r + static_cast<int64_t>(node) * D + c, acc[c]);  // RED, one writer per colour
    }
  }
}

// r <- r at free DOFs, 0 elsewhere; partial sums of r.r
__global__ void k_mask_norm(int64_t n, const uint8_t* __restrict__ freem, double* __restrict__ r,
                            double* __restrict__ partials) {
  double v[1] = {0.0};
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double x = freem[i] ? r[i] : 0.0;
    r[i] = x;
    v[0] += x * x;
  }
  block_sum_store<1>(v, partials);
}

// ------------------------------------------------------- K6 tangent (AD) --
// dP/dG per particle by forward-mode duals over the same expression graph as
// the residual (hand-written AD replacing the tape, tape.hpp:107-122):
// A[p][(d*D+f)*D*D + (c*D+b)] = dP_cb / dG_df (direction-major: a pass writes
// whole contiguous runs, so the multi-pass 3D kernel writes full sectors).
template <int D, int SHAPE, int K, bool NHO>
__global__ void k_tangent(GridC g, const double* __restrict__ pd, int64_t cap, int P,
                          const double* __restrict__ xs, const int* __restrict__ key,
                          const int* __restrict__ sup, const double* __restrict__ u, MatParams mp, int tl,
                          double* __restrict__ A) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  using T = Dual<K>;
  constexpr int DD = D * D;
  int first[3], cnt[3];
  AxisW aw[3];
  particle_weights<D, SHAPE>(g, pd, cap, xs, p, key[p], sup[p], first, cnt, aw);
  Mat<double, D> G = Mat<double, D>::zero();
  for_each_support<D>(g, first, cnt, aw, [&](int node, double, const double* grad) {
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double uc = u[node * D + c];
#pragma unroll
      for (int a = 0; a < D; ++a) G(c, a) += uc * grad[a];
    }
  });
  double Fn[DD];
#pragma unroll
  for (int i = 0; i < DD; ++i) Fn[i] = pd[(PF<D>::F + i) * cap + p];
  double Be_n[10];
  if (has_history(mp.kind))
#pragma unroll
    for (int i = 0; i < 9; ++i) Be_n[i] = pd[(PF<D>::Be + i) * cap + p];
  if (mp.kind == kCamClay) Be_n[9] = pd[PF<D>::alpha * cap + p];
  const double V0 = pd[PF<D>::V0 * cap + p];
  double* out = A + static_cast<int64_t>(p) * DD * DD;
#pragma unroll 1
  for (int pass = 0; pass < DD / K; ++pass) {
    Mat<T, D> f_inc;
#pragma unroll
    for (int i = 0; i < DD; ++i) {
      f_inc.e[i] = T(G.e[i]);
      const int j = i - pass * K;
      if (j >= 0 && j < K) f_inc.e[i].d[j] = 1.0;
    }
#pragma unroll
    for (int a = 0; a < D; ++a) f_inc(a, a) += 1.0;
    Mat<T, D> F_new;
    if (tl) {
      F_new = f_inc;
    } else {
      Mat<T, D> FnT;
#pragma unroll
      for (int i = 0; i < DD; ++i) FnT.e[i] = T(Fn[i]);
      F_new = matmul(f_inc, FnT);
    }
    if (!(value_of(det(F_new)) > 0.0)) {
#pragma unroll
      for (int i = 0; i < DD * DD; ++i) out[i] = 0.0;
      return;
    }
    const StressOut<T> su = update_stress<T, D, NHO>(mp, F_new, f_inc, Be_n);
    const T V = su.J * V0;
    const Mat<T, D> fi = inverse(f_inc);
#pragma unroll
    for (int c = 0; c < D; ++c)
#pragma unroll
      for (int b = 0; b < D; ++b) {
        T s = su.sigma(c, 0) * fi(b, 0);
#pragma unroll
        for (int a = 1; a < D; ++a) s += su.sigma(c, a) * fi(b, a);
        const T Pcb = V * s;
#pragma unroll
        for (int j = 0; j < K; ++j) out[(pass * K + j) * DD + c * D + b] = Pcb.d[j];
      }
  }
}

// Analytic neo-Hookean tangent (3D), the closed form of what k_tangent's
// dual numbers compute on the same expression graph: with f = I + G,
// F = f F_n (updated Lagrangian; F = f total Lagrangian), b = F F^T,
// tau = mu (b - I) + lam ln J I (neo_hookean_update, materials.hpp:139-158)
// and P = V sigma f^-T = V0 tau f^-T (mpm_solver.hpp:187-198),
//   dP_cb/dG_df = V0 [ mu d_cd (Fi b Fi^T)_fb + mu (Fi b)_fc Fi_bd
//                      + lam Fi_fd Fi_bc - Fi_bd (tau Fi^T)_cf ],  Fi = f^-1.
// ~900 flops per particle instead of nine dual-number passes of the stress
// update; A is written through a per-warp transpose in contiguous 216-byte
// runs (one output direction d at a time), same layout as k_tangent.
// The neo-Hookean factors of one particle at displacement u: Fi = f^-1,
// X = Fi b, Y = Fi b Fi^T, Z = tau Fi^T (false when det F <= 0).
template <int SHAPE>
__device__ __forceinline__ bool nh3_factors(const GridC& g, const double* __restrict__ pd, int64_t cap,
                                            const double* __restrict__ xs, int p, int key, int sup,
                                            const double* __restrict__ u, double lam, double mu, int tl, double* Fi,
                                            double* X, double* Y, double* Z, double& V0) {
  constexpr int D = 3;
  int first[3], cnt[3];
  AxisW aw[3];
  particle_weights<D, SHAPE>(g, pd, cap, xs, p, key, sup, first, cnt, aw);
  Mat<double, D> G = Mat<double, D>::zero();
  for_each_support<D>(g, first, cnt, aw, [&](int node, double, const double* grad) {
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double uc = u[node * D + c];
#pragma unroll
      for (int a = 0; a < D; ++a) G(c, a) += uc * grad[a];
    }
  });
  Mat<double, D> f = G;
#pragma unroll
  for (int a = 0; a < D; ++a) f(a, a) += 1.0;
  Mat<double, D> F = f;
  if (!tl) {
    Mat<double, D> Fn;
#pragma unroll
    for (int i = 0; i < 9; ++i) Fn.e[i] = pd[(PF<D>::F + i) * cap + p];
    F = matmul(f, Fn);
  }
  const double J = det(F);
  V0 = pd[PF<D>::V0 * cap + p];
  if (!(J > 0.0)) return false;
  const Mat<double, D> fi = inverse(f);
  const Mat<double, D> b = matmul(F, transpose(F));
  const double lnJ = log(J);
#pragma unroll
  for (int i = 0; i < 9; ++i) Fi[i] = fi.e[i];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double x = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) x += fi(i, a) * b(a, j);
      X[i * 3 + j] = x;  // (Fi b)_ij
    }
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      double y = 0.0, z = 0.0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        y += X[i * 3 + a] * fi(j, a);  // (Fi b Fi^T)_ij
        const double tau = mu * (b(i, a) - (i == a ? 1.0 : 0.0)) + (i == a ? lam * lnJ : 0.0);
        z += tau * fi(j, a);  // (tau Fi^T)_ij
      }
      Y[i * 3 + j] = y;
      Z[i * 3 + j] = z;
    }
  return true;
}

template <int SHAPE>
__global__ void __launch_bounds__(128) k_tangent_nh3(GridC g, const double* __restrict__ pd, int64_t cap, int P,
                                                     const double* __restrict__ xs, const int* __restrict__ key,
                                                     const int* __restrict__ sup, const double* __restrict__ u,
                                                     MatParams mp, int tl, double* __restrict__ A) {
  __shared__ double tb[4][32][28];  // [warp][particle][27 values of one direction d] (+1 pad)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p0 = (blockIdx.x * 4 + warp) * 32;
  const int p = p0 + lane;
  double Fi[9] = {}, Y[9] = {}, X[9] = {}, Z[9] = {}, V0 = 0.0;
  const double lam = mp.lam, mu = mp.mu;
  const bool ok = p < P && nh3_factors<SHAPE>(g, pd, cap, xs, p, key[p], sup[p], u, lam, mu, tl, Fi, X, Y, Z, V0);
  double* tw = &tb[warp][0][0];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    // this lane's particle: the 27 values of direction d, index (f, c, b)
#pragma unroll
    for (int f = 0; f < 3; ++f)
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int bb = 0; bb < 3; ++bb) {
          double v = 0.0;
          if (ok)
            v = V0 * ((c == d ? mu * Y[f * 3 + bb] : 0.0) + mu * X[f * 3 + c] * Fi[bb * 3 + d] +
                      lam * Fi[f * 3 + d] * Fi[bb * 3 + c] - Fi[bb * 3 + d] * Z[c * 3 + f]);
          tw[lane * 28 + f * 9 + c * 3 + bb] = v;
        }
    __syncwarp();
    // write the warp's 32 particles, 27 contiguous doubles each (df = d*3 + f)
    for (int q = 0; q < 32 && p0 + q < P; ++q)
      if (lane < 27) A[static_cast<int64_t>(p0 + q) * 81 + d * 27 + lane] = tw[q * 28 + lane];
    __syncwarp();
  }
}

// Factored form of the same tangent for the 3D neo-Hookean assembly
// (k_assemble_nh3f). With v = Fi^T g and Fi b Fi^T = (Fi F)(Fi F)^T = Fn Fn^T
// (Fn = I total Lagrangian), the four terms of dP/dG above contract with the
// node gradients g^k (index b) and g^l (index f) to
//   J_kl = sum_p [ (e_k . e_l) I + w_l v_k^T + V0 lam v_k v_l^T ],
//   e = sqrt(V0 mu) Fn^T g,  w = V0 (mu X^T - Z) g,
// so per particle the assembly needs Q = {Fi, sqrt(V0 mu) Fn^T, V0 (mu X^T - Z),
// V0 lam} (28 doubles) instead of the 81 entries of dP/dG. Same values as
// sum_bf g^k_b A[cb][df] g^l_f up to rounding. (Carrying the particle's 1D
// weights in Q as well, 46 doubles, measured slower: 19.8 vs 19.4 ms per cfg 4
// tangent + assembly, and 20.0 with Q component-major.)
constexpr int kNhQ = 28;
template <int SHAPE>
// (min-blocks hints measured: none 1.27 ms per cfg 4 tangent, 1: 1.50, 8: 1.31)
__global__ void __launch_bounds__(128) k_tangent_nh3q(GridC g, const double* __restrict__ pd, int64_t cap, int P,
                                                      const double* __restrict__ xs, const int* __restrict__ key,
                                                      const int* __restrict__ sup, const double* __restrict__ u,
                                                      MatParams mp, int tl, double* __restrict__ Q) {
  __shared__ double tb[4][32 * kNhQ];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p0 = (blockIdx.x * 4 + warp) * 32;
  const int p = p0 + lane;
  double Fi[9] = {}, Y[9] = {}, X[9] = {}, Z[9] = {}, V0 = 0.0;
  const double lam = mp.lam, mu = mp.mu;
  const bool ok = p < P && nh3_factors<SHAPE>(g, pd, cap, xs, p, key[p], sup[p], u, lam, mu, tl, Fi, X, Y, Z, V0);
  const double sq = ok ? sqrt(V0 * mu) : 0.0;
  double* q = &tb[warp][lane * kNhQ];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const double fn = tl ? (i == j ? 1.0 : 0.0) : (ok ? pd[(PF<3>::F + j * 3 + i) * cap + p] : 0.0);
      q[i * 3 + j] = ok ? Fi[i * 3 + j] : 0.0;
      q[9 + i * 3 + j] = sq * fn;                                                 // E[i][j] = sqrt(V0 mu) Fn_ji
      q[18 + i * 3 + j] = ok ? V0 * (mu * X[j * 3 + i] - Z[i * 3 + j]) : 0.0;  // [c][f]
    }
  q[27] = ok ? V0 * lam : 0.0;
  __syncwarp();
  // the warp's 32 records are one contiguous run
  const int nq = min(32, P - p0) * kNhQ;
  for (int e = lane; e < nq; e += 32) Q[static_cast<int64_t>(p0) * kNhQ + e] = tb[warp][e];
}

// ------------------------------------------- K6 Jacobian: structure ------
// Per bin (= first support node): bit a set when some particle of the bin
// has a 3-node support on axis a; bit 7 = bin non-empty.
__global__ void k_bin_flags(int N, int D, const int* __restrict__ bin_start, const int* __restrict__ sup,
                            uint8_t* __restrict__ bflag) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= N) return;
  const int s0 = bin_start[b], e0 = bin_start[b + 1];
  int f = 0;
  for (int p = s0; p < e0; ++p)
    for (int a = 0; a < D; ++a)
      if (sup_cnt(sup[p], a) == 3) f |= 1 << a;
  bflag[b] = static_cast<uint8_t>(e0 > s0 ? (0x80 | f) : 0);
}

// Row structure (once per load step: it does not depend on u): the stored
// block columns of row k are the box offsets l - k of every bin support box
// containing k (a superset of the particle-pair couplings; the reference
// pattern, jacobian.hpp:36-65, is the full +-2 box). Ascending slot list,
// count and a 128-bit slot mask (position = popcount below the slot).
template <int D>
__global__ void k_row_structure(GridC g, const int* __restrict__ act_list, int n_act,
                                const uint8_t* __restrict__ bflag, uint8_t* __restrict__ row_slots,
                                int* __restrict__ row_nzb, unsigned* __restrict__ row_mask,
                                unsigned long long* __restrict__ nzb_total) {
  constexpr int S = ipow_c(5, D);
  constexpr int NB = ipow_c(3, D);
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long cnt = 0;
  if (row < n_act) {
    const int k = act_list[row];
    int kidx[3];
    unflat<D>(g, k, kidx);
    unsigned m[4] = {0u, 0u, 0u, 0u};
    for (int ob = 0; ob < NB; ++ob) {
      int off[3] = {0, 0, 0}, r = ob, b = 0;
      bool ok = true;
#pragma unroll
      for (int a = D - 1; a >= 0; --a) {
        off[a] = r % 3;
        r /= 3;
        ok = ok && kidx[a] - off[a] >= 0;
        b += (kidx[a] - off[a]) * g.stride[a];
      }
      if (!ok) continue;
      const int fl = bflag[b];
      if (!(fl & 0x80)) continue;
      int cn[3] = {1, 1, 1};
#pragma unroll
      for (int a = 0; a < D; ++a) {
        cn[a] = 2 + ((fl >> a) & 1);
        ok = ok && off[a] < cn[a];
      }
      if (!ok) continue;
      for (int i0 = 0; i0 < cn[0]; ++i0)
        for (int i1 = 0; i1 < (D > 1 ? cn[1] : 1); ++i1)
          for (int i2 = 0; i2 < (D > 2 ? cn[2] : 1); ++i2) {
            const int li[3] = {i0, i1, i2};
            int sl = 0;
#pragma unroll
            for (int a = 0; a < D; ++a) sl = sl * 5 + (li[a] - off[a] + 2);
            m[sl >> 5] |= 1u << (sl & 31);
          }
    }
    int pos = 0;
    uint8_t* out = row_slots + static_cast<int64_t>(row) * S;
    for (int w = 0; w < 4; ++w) {
      unsigned bits = m[w];
      row_mask[static_cast<int64_t>(row) * 4 + w] = bits;
      while (bits) {
        const int bt = __ffs(bits) - 1;
        bits &= bits - 1;
        out[pos++] = static_cast<uint8_t>(w * 32 + bt);
      }
    }
    row_nzb[row] = pos;
    cnt = pos;
  }
  // one atomic per warp (integer: order-independent)
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(nzb_total, cnt);
}

__device__ __forceinline__ int mask_pos(const unsigned* m, int sl) {
  int pos = 0;
  const int w = sl >> 5;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (i < w) pos += __popc(m[i]);
  return pos + __popc(m[w] & ((1u << (sl & 31)) - 1u));
}

// 8-byte asynchronous global -> shared copy (LDGSTS): no register staging,
// so the copies of a whole bin are in flight while the warp does other work
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// mask_pos over a register copy of the row's 128-bit slot mask (no dynamic
// indexing, so the words stay in registers)
__device__ __forceinline__ int mask_pos_r(const unsigned (&m)[4], int sl) {
  const int w = sl >> 5;
  int pos = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
    if (i < w) pos += __popc(m[i]);
  const unsigned mw = w == 0 ? m[0] : (w == 1 ? m[1] : (w == 2 ? m[2] : m[3]));
  return pos + __popc(mw & ((1u << (sl & 31)) - 1u));
}

// zero the stored part of every row (component chunks incl. padding)
// row_mask != nullptr: zero only the upper blocks (slot >= the centre slot
// S/2; the assembly then forms only those and k_mirror_lower writes the rest)
__global__ void k_zero_rows(int n_act, int F, const int* __restrict__ row_nzb, double* __restrict__ vals,
                            int64_t row_len, const unsigned* __restrict__ row_mask = nullptr, int center = 0) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= n_act) return;
  const int nzb = row_nzb[warp], cp = cpad(nzb, F);
  int lo = 0;  // first stored position at or above the centre slot
  if (row_mask) {
    const unsigned* m = row_mask + static_cast<int64_t>(warp) * 4;
    for (int w = 0; w < 4; ++w) {
      const int b0 = w * 32;
      unsigned bits = m[w];
      if (b0 + 32 <= center) {
        lo += __popc(bits);
      } else if (b0 < center) {
        lo += __popc(bits & ((1u << (center - b0)) - 1u));
      }
    }
  }
  double* r = vals + static_cast<int64_t>(warp) * row_len;
  const int len = cp - lo * F;
  for (int c = 0; c < F; ++c)
    for (int j = lane; j < len; j += 32) r[c * cp + lo * F + j] = 0.0;
}

// ------------------------------------------- K6 Jacobian: numeric ---------
// Colour-batched, bin-centric assembly. Bins of colour (c_a = idx_a mod 3)
// are >= 3 nodes apart per axis, so their support boxes (<= 3 nodes/axis)
// and hence their (k, l) blocks are disjoint: one warp owns a bin and adds
// its element blocks straight into the BSR rows, no atomics, fixed order.
// Per particle: 1D weights (lanes < 3D), node gradients g^k (lane per box
// node), H_k[c][d][f] = sum_b g^k_b A_p[cb][df] (lanes over (k, cdf)); then
// every lane accumulates its PPL block pairs (k, l) += H_k . g^l over the
// bin's particles in registers before one read-modify-write.
template <int D, int SHAPE, int PPL, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_assemble_bins(
    GridC g, const double* __restrict__ pd, int64_t cap, const double* __restrict__ xs,
    const int* __restrict__ bin_start, const uint8_t* __restrict__ bflag, const double* __restrict__ A,
    const int* __restrict__ act_idx, const unsigned* __restrict__ row_mask, const int* __restrict__ row_nzb,
    double* __restrict__ vals, int64_t row_len, int c0, int c1, int c2, int nb0, int nb1, int nb2) {
  constexpr int DD = D * D;
  constexpr int D3 = D * D * D;
  constexpr int NK = ipow_c(3, D);
  __shared__ double W1s[WARPS][3][3], DW1s[WARPS][3][3];
  __shared__ double Gs[WARPS][NK][3];
  __shared__ double Hs[WARPS][NK * D3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbins = nb0 * nb1 * nb2;
  const int col[3] = {c0, c1, c2};
  const int nbv[3] = {nb0, nb1, nb2};
  for (int bi = blockIdx.x * WARPS + warp; bi < nbins; bi += gridDim.x * WARPS) {
    int bidx[3] = {0, 0, 0}, r = bi, b = 0;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      bidx[a] = 3 * (r % nbv[a]) + col[a];
      r /= nbv[a];
      b += bidx[a] * g.stride[a];
    }
    const int fl = bflag[b];
    if (!(fl & 0x80)) continue;
    int cn[3] = {1, 1, 1};
#pragma unroll
    for (int a = 0; a < D; ++a) cn[a] = 2 + ((fl >> a) & 1);
    const int nk = cn[0] * cn[1] * cn[2];
    const int npairs = nk * nk;
    const int p0 = bin_start[b], p1 = bin_start[b + 1];
    for (int q0 = 0; q0 < npairs; q0 += 32 * PPL) {
      double acc[PPL][DD];
#pragma unroll
      for (int t = 0; t < PPL; ++t)
#pragma unroll
        for (int e = 0; e < DD; ++e) acc[t][e] = 0.0;
      for (int p = p0; p < p1; ++p) {
        if (lane < 3 * D) {
          const int a = lane / 3, i = lane % 3;
          double w = 0.0, dw = 0.0;
          if (i < cn[a]) {
            const WeightValue wv = weight_1d<SHAPE>(xs[a * cap + p] - node_coord(g, a, bidx[a] + i),
                                                    pd[(PF<D>::lp + a) * cap + p], g.h);
            w = wv.w;
            dw = wv.dw;
          }
          W1s[warp][a][i] = w;
          DW1s[warp][a][i] = dw;
        }
        __syncwarp();
        for (int k = lane; k < nk; k += 32) {
          int li[3] = {0, 0, 0}, rr = k;
#pragma unroll
          for (int a = D - 1; a >= 0; --a) {
            li[a] = rr % cn[a];
            rr /= cn[a];
          }
          double w[3], dw[3], W, gk[3];
#pragma unroll
          for (int a = 0; a < D; ++a) {
            w[a] = W1s[warp][a][li[a]];
            dw[a] = DW1s[warp][a][li[a]];
          }
          tensor_weight<D>(w, dw, W, gk);
#pragma unroll
          for (int a = 0; a < D; ++a) Gs[warp][k][a] = gk[a];
        }
        __syncwarp();
        const double* Ap = A + static_cast<int64_t>(p) * DD * DD;
        for (int e = lane; e < nk * D3; e += 32) {
          const int k = e / D3, cdf = e - k * D3, c = cdf / DD, df = cdf - c * DD;
          double sacc = 0.0;
#pragma unroll
          for (int bb = 0; bb < D; ++bb) sacc += Gs[warp][k][bb] * __ldg(Ap + (c * D + bb) * DD + df);
          Hs[warp][e] = sacc;
        }
        __syncwarp();
#pragma unroll
        for (int t = 0; t < PPL; ++t) {
          const int q = q0 + lane + 32 * t;
          if (q < npairs) {
            const int k = q / nk, l = q - k * nk;
            const double* Hk = &Hs[warp][k * D3];
            double gl[3];
#pragma unroll
            for (int f = 0; f < D; ++f) gl[f] = Gs[warp][l][f];
#pragma unroll
            for (int cd = 0; cd < DD; ++cd) {
              double sacc = 0.0;
#pragma unroll
              for (int f = 0; f < D; ++f) sacc += Hk[cd * D + f] * gl[f];
              acc[t][cd] += sacc;
            }
          }
        }
        __syncwarp();
      }
      // read-modify-write of the owned blocks (exclusive within this colour)
#pragma unroll
      for (int t = 0; t < PPL; ++t) {
        const int q = q0 + lane + 32 * t;
        if (q >= npairs) continue;
        const int k = q / nk, l = q - k * nk;
        int lk[3] = {0, 0, 0}, ll[3] = {0, 0, 0}, rk = k, rl = l, node = 0, sl = 0;
#pragma unroll
        for (int a = D - 1; a >= 0; --a) {
          lk[a] = rk % cn[a];
          rk /= cn[a];
          ll[a] = rl % cn[a];
          rl /= cn[a];
        }
#pragma unroll
        for (int a = 0; a < D; ++a) {
          node += (bidx[a] + lk[a]) * g.stride[a];
          sl = sl * 5 + (ll[a] - lk[a] + 2);
        }
        const int row = act_idx[node];
        if (row < 0) continue;
        const unsigned* m = row_mask + static_cast<int64_t>(row) * 4;
        const int pos = mask_pos(m, sl);
        const int cp = cpad(row_nzb[row], D);
        double* rv = vals + static_cast<int64_t>(row) * row_len + pos * D;
#pragma unroll
        for (int c = 0; c < D; ++c)
#pragma unroll
          for (int d = 0; d < D; ++d) rv[c * cp + d] += acc[t][c * D + d];
      }
    }
  }
}

// Staged variant of k_assemble_bins: the bin's particles are processed in
// chunks of PCH; per chunk the tangent blocks A_p (contiguous for a bin's
// sorted particles) and the 1D weights / node gradients of every particle
// are staged in shared memory with all loads in flight at once, so the
// per-particle loop (H_k = g^k . A_p, then the lane-owned block pairs) runs
// from shared memory only.
//
// SYM: the single-field J is symmetric (hyperelastic / associative J2: the
// per-particle tangent has major symmetry), so only blocks with l >= k are
// computed and the transpose is mirrored into row l: ~45% fewer task rounds.
//
// A bin with at most PCH particles (the common case: PCH = 8 = ppc^3 in 3D) is
// staged once and stays resident across all of its task rounds; larger bins
// restage per round and chunk.
// RMW: flush through a per-warp shared-memory transpose and plain coalesced
// read-modify-writes instead of per-lane RED.ADD.F64 (exclusive per colour, so
// no atomics are needed; same one add per block per colour, bitwise the same
// sums). A RED costs ~1.3 LSU cycles per lane; a transposed RMW moves the
// 27 values of one task with one load and one store instruction.
template <int PPL, int DD>
struct AsmFlush {
  static constexpr int NV = PPL * DD;
  double F[32][NV];
  long long DB[32][PPL], MB[32][PPL];
  int DCP[32], MCP[32][PPL];
};

// MIRROR (SYM only): add K_kl^T into row l inside the kernel (RED); false:
// only the upper blocks (flat(l) >= flat(k)) are formed and k_mirror_lower
// copies the transposes once after the last colour (half the reductions)
template <int D, int SHAPE, int PPL, int WARPS, int PCH, bool SYM = false, bool RMW = false, bool MIRROR = true>
#ifndef IMPM_ASM_MINB
#define IMPM_ASM_MINB 4  // resident CTAs per SM the 3D assembly is compiled for
#endif
__global__ void __launch_bounds__(WARPS * 32, D == 3 ? (RMW ? 2 : IMPM_ASM_MINB) : 1) k_assemble_bins_staged(
    GridC g, const double* __restrict__ pd, int64_t cap, const double* __restrict__ xs,
    const int* __restrict__ bin_start, const uint8_t* __restrict__ bflag, const double* __restrict__ A,
    const int* __restrict__ act_idx, const unsigned* __restrict__ row_mask, const int* __restrict__ row_nzb,
    double* __restrict__ vals, int64_t row_len, int c0, int c1, int c2, int nb0, int nb1, int nb2) {
  constexpr int DD = D * D;
  constexpr int D3 = D * D * D;
  constexpr int NA = DD * DD;
  constexpr int NK = ipow_c(3, D);
  constexpr int NW1 = PCH * D * 6;  // 1D weights [pl][a][i][w|dw]
  __shared__ double As[WARPS][PCH * NA];
  __shared__ double Gs[WARPS][PCH][NK][D];
  __shared__ double HWs[WARPS][NW1];  // 1D weights of the staged chunk
  // row metadata of the bin's box nodes: row index, slot mask, component pitch
  __shared__ int Rrow[WARPS][NK];
  __shared__ int Rcp[WARPS][NK];
  __shared__ uint4 Rmask[WARPS][NK];
  static_assert(sizeof(As) + sizeof(Gs) + sizeof(HWs) + sizeof(Rrow) + sizeof(Rcp) + sizeof(Rmask) <= 48 * 1024,
                "k_assemble_bins_staged: static shared memory above the 48 KB launch limit");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  extern __shared__ __align__(16) unsigned char asm_dyn[];
  using FL = AsmFlush<PPL, DD>;
  FL& fls = reinterpret_cast<FL*>(asm_dyn)[RMW ? warp : 0];
  const int nbins = nb0 * nb1 * nb2;
  const int col[3] = {c0, c1, c2};
  const int nbv[3] = {nb0, nb1, nb2};
  for (int bi = blockIdx.x * WARPS + warp; bi < nbins; bi += gridDim.x * WARPS) {
    int bidx[3] = {0, 0, 0}, r = bi, b = 0;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      bidx[a] = 3 * (r % nbv[a]) + col[a];
      r /= nbv[a];
      b += bidx[a] * g.stride[a];
    }
    const int fl = bflag[b];
    if (!(fl & 0x80)) continue;
    int cn[3] = {1, 1, 1};
#pragma unroll
    for (int a = 0; a < D; ++a) cn[a] = 2 + ((fl >> a) & 1);
    const int nk = cn[0] * cn[1] * cn[2];
    // lane task = (row node k, run of PPL column nodes l0..l0+PPL-1); SYM:
    // runs start at l = k (row k has ceil((nk - k) / PPL) runs)
    const int nchunk = (nk + PPL - 1) / PPL;
    int ntasks = nk * nchunk;
    if constexpr (SYM) {
      ntasks = 0;
      for (int k = 0; k < nk; ++k) ntasks += (nk - k + PPL - 1) / PPL;
    }
    // (row, first column) of task t
    auto task_of = [&](int t, int& k_out, int& l_out) {
      if constexpr (SYM) {
        int k = 0, n = (nk + PPL - 1) / PPL;
        while (t >= n) {
          t -= n;
          ++k;
          n = (nk - k + PPL - 1) / PPL;
        }
        k_out = k;
        l_out = k + t * PPL;
      } else {
        k_out = t / nchunk;
        l_out = (t - k_out * nchunk) * PPL;
      }
    };
    // resident bin (<= PCH particles): its tangent blocks go to shared memory
    // by asynchronous copies now, so that they are in flight during the row
    // metadata and 1D-weight staging below (global A is direction-major
    // [df][cb]; As keeps [cb][df] for the H loop)
    const int p0 = bin_start[b], p1 = bin_start[b + 1];
    const bool resident = p1 - p0 <= PCH;
    __syncwarp();
    if (resident) {
      const int np0 = p1 - p0;
      const double* Ab = A + static_cast<int64_t>(p0) * NA;
      for (int e = lane; e < np0 * NA; e += 32) {
        const int pl = e / NA, r = e - pl * NA, df = r / DD, cb = r - df * DD;
        cp_async8(&As[warp][pl * NA + cb * DD + df], Ab + e);
      }
    }
    // stage the box nodes' row metadata once per bin (all lanes in parallel)
    // so that the per-task block lookups read shared memory only
    if (lane < nk) {
      int rk = lane, node = 0;
      int li[3] = {0, 0, 0};
#pragma unroll
      for (int a = D - 1; a >= 0; --a) {
        li[a] = rk % cn[a];
        rk /= cn[a];
      }
#pragma unroll
      for (int a = 0; a < D; ++a) node += (bidx[a] + li[a]) * g.stride[a];
      const int rw = act_idx[node];
      Rrow[warp][lane] = rw;
      if (rw >= 0) {
        Rmask[warp][lane] = *reinterpret_cast<const uint4*>(row_mask + static_cast<int64_t>(rw) * 4);
        Rcp[warp][lane] = cpad(row_nzb[rw], D);
      }
    }
    __syncwarp();
    for (int r0 = 0; r0 < ntasks; r0 += 32) {
      const int task = r0 + lane;
      const bool has_task = task < ntasks;
      int tk = 0, tl0 = nk;
      if (has_task) task_of(task, tk, tl0);
      double acc[PPL][DD];
#pragma unroll
      for (int t = 0; t < PPL; ++t)
#pragma unroll
        for (int e = 0; e < DD; ++e) acc[t][e] = 0.0;
      // the task's row metadata (staged per bin in shared memory)
      int lk[3] = {0, 0, 0}, row = -1, cp = 0;
      unsigned rm[4] = {0u, 0u, 0u, 0u};
      if (has_task) {
        int rk = tk;
#pragma unroll
        for (int a = D - 1; a >= 0; --a) {
          lk[a] = rk % cn[a];
          rk /= cn[a];
        }
        row = Rrow[warp][tk];
        if (row >= 0) {
          const uint4 m4 = Rmask[warp][tk];
          rm[0] = m4.x;
          rm[1] = m4.y;
          rm[2] = m4.z;
          rm[3] = m4.w;
          cp = Rcp[warp][tk];
        }
      }
      for (int pc = p0; pc < p1; pc += PCH) {
        const int np = min(PCH, p1 - pc);
        if (!resident || r0 == 0) {
        __syncwarp();
        // stage A_p (contiguous) and the 1D weights of the chunk; the A loads
        // go to registers first (4 particles at a time) so that they are in
        // flight together (resident bins: already copied asynchronously)
        const double* Ab = A + static_cast<int64_t>(pc) * NA;
#pragma unroll 1
        for (int q0 = 0; q0 < (resident ? 0 : PCH); q0 += 4) {
          constexpr int NL = (4 * NA + 31) / 32;
          double ta[NL];
#pragma unroll
          for (int i = 0; i < NL; ++i) {
            const int e = q0 * NA + lane + 32 * i;
            ta[i] = (e < np * NA && e < (q0 + 4) * NA) ? __ldg(Ab + e) : 0.0;
          }
          // global A is direction-major [df][cb]; As keeps [cb][df] for the H loop
#pragma unroll
          for (int i = 0; i < NL; ++i) {
            const int e = q0 * NA + lane + 32 * i;
            if (e < np * NA && e < (q0 + 4) * NA) {
              const int pl = e / NA, r = e - pl * NA, df = r / DD, cb = r - df * DD;
              As[warp][pl * NA + cb * DD + df] = ta[i];
            }
          }
        }
        double* W1 = HWs[warp];
        for (int e = lane; e < np * D * 3; e += 32) {
          const int pl = e / (D * 3), rem = e - pl * D * 3, a = rem / 3, i = rem - a * 3;
          double w = 0.0, dw = 0.0;
          if (i < cn[a]) {
            const int p = pc + pl;
            const WeightValue wv = weight_1d<SHAPE>(xs[a * cap + p] - node_coord(g, a, bidx[a] + i),
                                                    pd[(PF<D>::lp + a) * cap + p], g.h);
            w = wv.w;
            dw = wv.dw;
          }
          W1[((pl * D + a) * 3 + i) * 2] = w;
          W1[((pl * D + a) * 3 + i) * 2 + 1] = dw;
        }
        if (resident) cp_async_wait_all();  // this lane's tangent copies have landed
        __syncwarp();
        for (int e = lane; e < np * nk; e += 32) {
          const int pl = e / nk, k = e - pl * nk;
          int li[3] = {0, 0, 0}, rr = k;
#pragma unroll
          for (int a = D - 1; a >= 0; --a) {
            li[a] = rr % cn[a];
            rr /= cn[a];
          }
          double w[3], dw[3], W, gk[3];
#pragma unroll
          for (int a = 0; a < D; ++a) {
            w[a] = W1[((pl * D + a) * 3 + li[a]) * 2];
            dw[a] = W1[((pl * D + a) * 3 + li[a]) * 2 + 1];
          }
          tensor_weight<D>(w, dw, W, gk);
#pragma unroll
          for (int a = 0; a < D; ++a) Gs[warp][pl][k][a] = gk[a];
        }
        }
        __syncwarp();
        // each lane forms its own row's H_k = g^k . A_p one component row c at
        // a time (A_p and g^k are warp-uniform shared-memory broadcasts), so the
        // particle loop needs no warp barrier
        if (has_task) {
          for (int pl = 0; pl < np; ++pl) {
            const double* Ap = &As[warp][pl * NA];
            double gk[3], gl[PPL][3];
#pragma unroll
            for (int bb = 0; bb < D; ++bb) gk[bb] = Gs[warp][pl][tk][bb];
#pragma unroll
            for (int t = 0; t < PPL; ++t)
#pragma unroll
              for (int f = 0; f < D; ++f) gl[t][f] = (tl0 + t < nk) ? Gs[warp][pl][tl0 + t][f] : 0.0;
#pragma unroll
            for (int cd = 0; cd < DD; ++cd) {
              const int c = cd / D, d = cd - c * D;
              double h[3];  // H_k[c][d * D + f]
#pragma unroll
              for (int f = 0; f < D; ++f) {
                double sacc = 0.0;
#pragma unroll
                for (int bb = 0; bb < D; ++bb) sacc = fma(gk[bb], Ap[(c * D + bb) * DD + d * D + f], sacc);
                h[f] = sacc;
              }
#pragma unroll
              for (int t = 0; t < PPL; ++t)
#pragma unroll
                for (int f = 0; f < D; ++f) acc[t][cd] = fma(h[f], gl[t][f], acc[t][cd]);
            }
          }
        }
      }
      if constexpr (RMW) {
        // publish the task's blocks (values + element offsets) to the warp's
        // transpose buffer, then move them with coalesced RMWs
#pragma unroll
        for (int t = 0; t < PPL; ++t) {
          long long db = -1, mb = -1;
          int mcp = 0;
          const int l = tl0 + t;
          if (has_task && l < nk) {
            int ll[3] = {0, 0, 0}, rl = l, sl = 0, slm = 0;
#pragma unroll
            for (int a = D - 1; a >= 0; --a) {
              ll[a] = rl % cn[a];
              rl /= cn[a];
            }
#pragma unroll
            for (int a = 0; a < D; ++a) {
              sl = sl * 5 + (ll[a] - lk[a] + 2);
              slm = slm * 5 + (lk[a] - ll[a] + 2);
            }
            if (row >= 0) db = static_cast<long long>(row) * row_len + mask_pos_r(rm, sl) * D;
            if constexpr (SYM) {
              const int rowl = Rrow[warp][l];
              if (l != tk && rowl >= 0) {
                const uint4 m4 = Rmask[warp][l];
                const unsigned ml[4] = {m4.x, m4.y, m4.z, m4.w};
                mb = static_cast<long long>(rowl) * row_len + mask_pos_r(ml, slm) * D;
                mcp = Rcp[warp][l];
              }
            }
          }
          fls.DB[lane][t] = db;
          fls.MB[lane][t] = mb;
          fls.MCP[lane][t] = mcp;
#pragma unroll
          for (int e = 0; e < DD; ++e) fls.F[lane][t * DD + e] = acc[t][e];
        }
        fls.DCP[lane] = cp;
        __syncwarp();
        const int tq = lane / DD, cq = (lane % DD) / D, dq = lane % D;
        const bool vl = lane < FL::NV;
        const int ntr = min(32, ntasks - r0);
        for (int i0 = 0; i0 < ntr; i0 += 4) {
          long long oa[4], ma[4];
          double ov[4], mv[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int i = i0 + q;
            oa[q] = -1;
            ma[q] = -1;
            if (vl && i < ntr) {
              const long long db = fls.DB[i][tq];
              if (db >= 0) oa[q] = db + static_cast<long long>(cq) * fls.DCP[i] + dq;
              if constexpr (SYM) {
                const long long mb = fls.MB[i][tq];
                if (mb >= 0) ma[q] = mb + static_cast<long long>(cq) * fls.MCP[i][tq] + dq;
              }
            }
            ov[q] = oa[q] >= 0 ? __ldcg(vals + oa[q]) : 0.0;
            mv[q] = ma[q] >= 0 ? __ldcg(vals + ma[q]) : 0.0;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int i = i0 + q;
            if (oa[q] >= 0) __stcg(vals + oa[q], ov[q] + fls.F[i][tq * DD + cq * D + dq]);
            if (ma[q] >= 0) __stcg(vals + ma[q], mv[q] + fls.F[i][tq * DD + dq * D + cq]);
          }
        }
        __syncwarp();
        continue;
      }
      if (has_task) {
        if (row >= 0) {
          double* rbase = vals + static_cast<int64_t>(row) * row_len;
#pragma unroll
          for (int t = 0; t < PPL; ++t) {
            const int l = tl0 + t;
            if (l >= nk) continue;
            int ll[3] = {0, 0, 0}, rl = l, sl = 0;
#pragma unroll
            for (int a = D - 1; a >= 0; --a) {
              ll[a] = rl % cn[a];
              rl /= cn[a];
            }
#pragma unroll
            for (int a = 0; a < D; ++a) sl = sl * 5 + (ll[a] - lk[a] + 2);
            IMPM_CHECK_IDX((D - 1) * cp + mask_pos_r(rm, sl) * D + D - 1, row_len);
            double* rv = rbase + mask_pos_r(rm, sl) * D;
            // fire-and-forget L2 reductions (RED.ADD.F64, result unused): one
            // writer per address per colour launch and launches in stream
            // order, so the sum is the same deterministic RMW without the
            // warp waiting on the DRAM read
#pragma unroll
            for (int c = 0; c < D; ++c)
#pragma unroll
              for (int d = 0; d < D; ++d) atomicAdd(rv + c * cp + d, acc[t][c * D + d]);
          }
        }
        if constexpr (SYM && MIRROR) {
          // mirrored blocks: row l, column k, K_lk = K_kl^T
#pragma unroll
          for (int t = 0; t < PPL; ++t) {
            const int l = tl0 + t;
            if (l >= nk || l == tk) continue;
            int ll[3] = {0, 0, 0}, rl = l, nodel = 0, sl = 0;
#pragma unroll
            for (int a = D - 1; a >= 0; --a) {
              ll[a] = rl % cn[a];
              rl /= cn[a];
            }
#pragma unroll
            for (int a = 0; a < D; ++a) {
              nodel += (bidx[a] + ll[a]) * g.stride[a];
              sl = sl * 5 + (lk[a] - ll[a] + 2);
            }
            (void)nodel;
            const int rowl = Rrow[warp][l];
            if (rowl < 0) continue;
            const uint4 m4 = Rmask[warp][l];
            const unsigned ml[4] = {m4.x, m4.y, m4.z, m4.w};
            const int cpl = Rcp[warp][l];
            IMPM_CHECK_IDX((D - 1) * cpl + mask_pos_r(ml, sl) * D + D - 1, row_len);
            double* rv = vals + static_cast<int64_t>(rowl) * row_len + mask_pos_r(ml, sl) * D;
#pragma unroll
            for (int c = 0; c < D; ++c)
#pragma unroll
              for (int d = 0; d < D; ++d) atomicAdd(rv + c * cpl + d, acc[t][d * D + c]);
          }
        }
      }
    }
  }
}

// 3D neo-Hookean assembly on the factored tangent (k_tangent_nh3q): same
// colour batches, bins and block addressing as k_assemble_bins_staged (upper
// blocks, SYM), but one CTA per bin and one block pair (k, l >= k) per thread.
// For the bin's particles the CTA builds, per (particle, box node), e, v and
// w (k_tangent_nh3q) in shared memory, component-major with the node index
// fastest (the pair loop's loads are conflict-free); a pair then costs 24 FMA
// per particle instead of the g^k A g^l contraction over 81 tangent entries.
// The bins of a CTA are software-pipelined: while bin j is assembled, the
// row indices of bin j+2 and the row masks, factors Q, positions and sizes of
// bin j+1 are in flight as asynchronous copies (LDGSTS), so a bin's chain of
// dependent loads (bin -> rows -> masks, bin -> particles) is off the
// critical path. Bins with more than PCH particles stage chunk by chunk.
// MIRROR: also add K_kl^T into row l (slabs); false: k_mirror_lower fills the
// lower blocks.
#ifndef IMPM_ASMF_WARPS
#define IMPM_ASMF_WARPS 6  // 192 threads: the 171 pairs of an 18-node box in one round (ms per cfg 4 Jacobian, assembly + transpose: 3 warps 19.25, 6 warps 18.92, 8 warps 19.43; 4 warps 0.3 below 3)
#endif
#ifndef IMPM_ASMF_MINB
#define IMPM_ASMF_MINB 4  // 80 registers, 4 x 25 KB shared per SM
#endif
struct BinHdr {
  int fl, p0, p1;
};
template <int SHAPE, int WARPS, int PCH, bool MIRROR>
__global__ void __launch_bounds__(WARPS * 32, IMPM_ASMF_MINB) k_assemble_nh3f(
    GridC g, const double* __restrict__ pd, int64_t cap, const double* __restrict__ xs,
    const int* __restrict__ bin_start, const uint8_t* __restrict__ bflag, const double* __restrict__ Q,
    const int* __restrict__ act_idx, const unsigned* __restrict__ row_mask, const int* __restrict__ row_nzb,
    double* __restrict__ vals, int64_t row_len, int c0, int c1, int c2, int nb0, int nb1, int nb2) {
  constexpr int D = 3, NK = 27, NT = WARPS * 32;
  __shared__ double T[PCH][9][NK];     // [particle][e0..2 v0..2 w0..2][box node]
  __shared__ double Qs[2][PCH][kNhQ];  // factors of the bin's particles (double-buffered)
  __shared__ double XL[2][PCH][6];     // positions and half sizes (double-buffered)
  __shared__ double W1[PCH][D][3][2];  // 1D weights [particle][axis][node][w|dw]
  __shared__ int Hs[3][4];             // bin header: bflag word, first particle, end
  __shared__ int Ridx[3][NK];          // row of each node of the 3x3x3 superset box (-1: none)
  __shared__ uint4 Rmask[2][NK];
  __shared__ int Rnzb[2][NK];
  // index tables (no runtime integer division in the per-bin code): box
  // shape code cc = 4 (cn0 - 2) + 2 (cn1 - 2) + (cn2 - 2); local node -> its
  // superset index; superset index -> packed axis offsets and its 5^3 slot base
  __shared__ uint8_t s_sup[8][NK];
  __shared__ uint8_t s_lpk[NK];
  __shared__ uint8_t s_b25[NK];
  const int tid = threadIdx.x;
  for (int e = tid; e < 8 * NK; e += NT) {
    const int cc = e / NK, kk = e - cc * NK;
    const int n0 = 2 + (cc >> 2), n1 = 2 + ((cc >> 1) & 1), n2 = 2 + (cc & 1);
    const int l2 = kk % n2, l1 = (kk / n2) % n1, l0 = kk / (n2 * n1);
    s_sup[cc][kk] = static_cast<uint8_t>(kk < n0 * n1 * n2 ? l0 * 9 + l1 * 3 + l2 : 0);
  }
  for (int e = tid; e < NK; e += NT) {
    const int l0 = e / 9, l1 = (e / 3) % 3, l2 = e % 3;
    s_lpk[e] = static_cast<uint8_t>(l0 | (l1 << 2) | (l2 << 4));
    s_b25[e] = static_cast<uint8_t>(l0 * 25 + l1 * 5 + l2);
  }
  // (visible after the first __syncthreads below)
  const int nbins = nb0 * nb1 * nb2;
  const int G = gridDim.x;
  auto bin_node = [&](int bi, int* bidx) {
    int r = bi;
    bidx[2] = 3 * (r % nb2) + c2;
    r /= nb2;
    bidx[1] = 3 * (r % nb1) + c1;
    bidx[0] = 3 * (r / nb1) + c0;
    return bidx[0] * g.stride[0] + bidx[1] * g.stride[1] + bidx[2] * g.stride[2];
  };
  auto read_hdr = [&](int bi, int buf) {
    BinHdr h{0, 0, 0};
    if (bi < nbins) {
      int bidx[3];
      const int b = bin_node(bi, bidx);
      h.fl = (Hs[buf][0] >> (8 * (b & 3))) & 0xff;
      h.p0 = Hs[buf][1];
      h.p1 = Hs[buf][2];
    }
    return h;
  };
  // stage A (depends on the bin index only): the bin's header and the rows of
  // the superset box nodes
  auto issue_rows = [&](int bi, int buf) {
    if (bi < nbins && tid < NK) {
      int bidx[3];
      const int b = bin_node(bi, bidx);
      if (tid == 0) cp_async4(&Hs[buf][0], bflag + (b & ~3));  // the aligned word holding the flag byte
      if (tid == 1) cp_async4(&Hs[buf][1], bin_start + b);
      if (tid == 2) cp_async4(&Hs[buf][2], bin_start + b + 1);
      const int i0 = tid / 9, i1 = (tid / 3) % 3, i2 = tid % 3;
      if (bidx[0] + i0 < g.nodes[0] && bidx[1] + i1 < g.nodes[1] && bidx[2] + i2 < g.nodes[2])
        cp_async4(&Ridx[buf][tid],
                  act_idx + (bidx[0] + i0) * g.stride[0] + (bidx[1] + i1) * g.stride[1] + bidx[2] + i2);
      else
        Ridx[buf][tid] = -1;
    }
  };
  // stage B: masks of those rows + the particles of a resident bin (needs stage A and the header)
  auto issue_data = [&](const BinHdr& h, int abuf, int buf) {
    if (!(h.fl & 0x80)) return;
    if (tid < NK) {
      const int rw = Ridx[abuf][tid];
      if (rw >= 0) {
        cp_async16(&Rmask[buf][tid], row_mask + static_cast<int64_t>(rw) * 4);
        cp_async4(&Rnzb[buf][tid], row_nzb + rw);
      }
    }
    const int np = h.p1 - h.p0;
    if (np <= PCH) {
      for (int e = tid; e < np * kNhQ; e += NT)
        cp_async8(&Qs[buf][0][0] + e, Q + static_cast<int64_t>(h.p0) * kNhQ + e);
      for (int e = tid; e < np * 6; e += NT) {
        const int pl = e / 6, jj = e - pl * 6;
        const int p = h.p0 + pl;
        cp_async8(&XL[buf][pl][jj], jj < 3 ? xs + jj * cap + p : pd + (PF<D>::lp + jj - 3) * cap + p);
      }
    }
  };
  // the staged particles (Qs/XL[buf], np of them) -> 1D weights -> T
  auto build_table = [&](int np, int buf, const int* bidx, const int* cn, int nk, int cc) {
    for (int e = tid; e < np * D * 3; e += NT) {
      const int pl = e / (D * 3), rem = e - pl * D * 3, a = rem / 3, i = rem - a * 3;
      // (selects instead of runtime-indexed grid arrays: no stack frame)
      const int cna = a == 0 ? cn[0] : (a == 1 ? cn[1] : cn[2]);
      const int ba = a == 0 ? bidx[0] + g.base0 : (a == 1 ? bidx[1] : bidx[2]);
      const double oa = a == 0 ? g.origin[0] : (a == 1 ? g.origin[1] : g.origin[2]);
      double w = 0.0, dw = 0.0;
      if (i < cna) {
        // node_coord (grid.hpp:180-185) with the selected axis
        const double xn = __dadd_rn(oa, __dmul_rn(static_cast<double>(ba + i), g.h));
        const WeightValue wv = weight_1d<SHAPE>(XL[buf][pl][a] - xn, XL[buf][pl][3 + a], g.h);
        w = wv.w;
        dw = wv.dw;
      }
      W1[pl][a][i][0] = w;
      W1[pl][a][i][1] = dw;
    }
    __syncthreads();
    // e / nk = umulhi(e, mg) for e < 2^16, mg = 2^32 / nk rounded up (nk is 8, 12, 18 or 27)
    const unsigned mg = nk == 8 ? 0x20000000u : (nk == 12 ? 0x15555556u : (nk == 18 ? 0x0E38E38Fu : 0x097B425Fu));
    for (int e = tid; e < np * nk; e += NT) {
      const int pl = static_cast<int>(__umulhi(static_cast<unsigned>(e), mg)), k = e - pl * nk;
      const int pk = s_lpk[s_sup[cc][k]];
      const int l0 = pk & 3, l1 = (pk >> 2) & 3, l2 = pk >> 4;
      const double w[3] = {W1[pl][0][l0][0], W1[pl][1][l1][0], W1[pl][2][l2][0]};
      const double dw[3] = {W1[pl][0][l0][1], W1[pl][1][l1][1], W1[pl][2][l2][1]};
      double W, gk[3];
      tensor_weight<D>(w, dw, W, gk);
      const double* q = Qs[buf][pl];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        double v = 0.0, ee = 0.0, ww = 0.0;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          v = fma(q[a * 3 + i], gk[a], v);         // (Fi^T g)_i
          ee = fma(q[9 + i * 3 + a], gk[a], ee);   // (sqrt(V0 mu) Fn^T g)_i
          ww = fma(q[18 + i * 3 + a], gk[a], ww);  // (V0 (mu X^T - Z) g)_i
        }
        T[pl][i][k] = ee;
        T[pl][3 + i][k] = v;
        T[pl][6 + i][k] = ww;
      }
    }
    __syncthreads();
  };

  int bi = blockIdx.x;
  issue_rows(bi, 0);
  issue_rows(bi + G, 1);
  cp_async_wait_all();
  __syncthreads();
  issue_data(read_hdr(bi, 0), 0, 0);
  for (int j = 0; bi < nbins; ++j, bi += G) {
    const int ab = j % 3, db = j & 1;
    cp_async_wait_all();
    __syncthreads();  // this bin's stage B and the next bin's stage A have landed; bin j-1 is done
    const BinHdr hc = read_hdr(bi, ab);
    issue_data(read_hdr(bi + G, (j + 1) % 3), (j + 1) % 3, db ^ 1);
    issue_rows(bi + 2 * G, (j + 2) % 3);
    if (hc.fl & 0x80) {
      int bidx[3], cn[3];
      bin_node(bi, bidx);
#pragma unroll
      for (int a = 0; a < D; ++a) cn[a] = 2 + ((hc.fl >> a) & 1);
      const int nk = cn[0] * cn[1] * cn[2];
      const int cc = ((hc.fl & 1) << 2) | (hc.fl & 2) | ((hc.fl >> 2) & 1);
      const int ntasks = nk * (nk + 1) / 2;
      const bool resident = hc.p1 - hc.p0 <= PCH;
      if (resident) build_table(hc.p1 - hc.p0, db, bidx, cn, nk, cc);
      for (int r0 = 0; r0 < ntasks; r0 += NT) {
        // this thread's pair: row-major over k, l = k .. nk-1
        const int task = r0 + tid;
        const bool has = task < ntasks;
        int tk = 0, tl = 0;
        if (has) {
          // row k of the upper triangle starts at off(k) = k nk - k (k - 1) / 2:
          // the root of off(k) = task, then an exact integer correction
          const float b2 = static_cast<float>(2 * nk + 1);
          tk = static_cast<int>(0.5f * (b2 - sqrtf(b2 * b2 - 8.0f * static_cast<float>(task))));
          tk = max(0, min(nk - 1, tk));
          if (tk * nk - tk * (tk - 1) / 2 > task) --tk;
          if ((tk + 1) * nk - (tk + 1) * tk / 2 <= task) ++tk;
          tl = tk + task - (tk * nk - tk * (tk - 1) / 2);
        }
        double acc[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) acc[e] = 0.0;
        for (int pc = hc.p0; pc < hc.p1; pc += PCH) {
          const int np = min(PCH, hc.p1 - pc);
          if (!resident) {
            // chunk by chunk, synchronously, in this bin's half of the double
            // buffers (the other half holds the next bin's copies)
            __syncthreads();
            for (int e = tid; e < np * kNhQ; e += NT)
              (&Qs[db][0][0])[e] = __ldg(Q + static_cast<int64_t>(pc) * kNhQ + e);
            for (int e = tid; e < np * 6; e += NT) {
              const int pl = e / 6, jj = e - pl * 6;
              XL[db][pl][jj] = jj < 3 ? xs[jj * cap + pc + pl] : pd[(PF<D>::lp + jj - 3) * cap + pc + pl];
            }
            __syncthreads();
            build_table(np, db, bidx, cn, nk, cc);
          }
          if (has) {
            for (int pl = 0; pl < np; ++pl) {
              const double lv = Qs[db][pl][27];
              double ek[3], vk[3], el[3], vl[3], wl[3];
#pragma unroll
              for (int i = 0; i < 3; ++i) {
                ek[i] = T[pl][i][tk];
                vk[i] = T[pl][3 + i][tk];
                el[i] = T[pl][i][tl];
                vl[i] = T[pl][3 + i][tl];
                wl[i] = T[pl][6 + i][tl];
              }
              const double sk = fma(ek[0], el[0], fma(ek[1], el[1], ek[2] * el[2]));
#pragma unroll
              for (int c = 0; c < 3; ++c) {
                const double Lc = lv * vk[c];
#pragma unroll
                for (int d = 0; d < 3; ++d) acc[c * 3 + d] = fma(wl[c], vk[d], fma(Lc, vl[d], acc[c * 3 + d]));
                acc[c * 3 + c] += sk;
              }
            }
          }
        }
        if (has) {
          const int sk9 = s_sup[cc][tk], sl9 = s_sup[cc][tl];
          const int sl = 62 + s_b25[sl9] - s_b25[sk9];  // slot of the offset l - k in the 5^3 box
          const int row = Ridx[ab][sk9];
          if (row >= 0) {
            const uint4 m4 = Rmask[db][sk9];
            const unsigned rm[4] = {m4.x, m4.y, m4.z, m4.w};
            const int cp = cpad(Rnzb[db][sk9], D);
            IMPM_CHECK_IDX((D - 1) * cp + mask_pos_r(rm, sl) * D + D - 1, row_len);
            double* rv = vals + static_cast<int64_t>(row) * row_len + mask_pos_r(rm, sl) * D;
#pragma unroll
            for (int c = 0; c < D; ++c)
#pragma unroll
              for (int d = 0; d < D; ++d) atomicAdd(rv + c * cp + d, acc[c * D + d]);
          }
          if constexpr (MIRROR) {
            const int rowl = Ridx[ab][sl9];
            if (tl != tk && rowl >= 0) {
              const int slm = 124 - sl;  // the mirrored offset k - l
              const uint4 m4 = Rmask[db][sl9];
              const unsigned ml[4] = {m4.x, m4.y, m4.z, m4.w};
              const int cpl = cpad(Rnzb[db][sl9], D);
              IMPM_CHECK_IDX((D - 1) * cpl + mask_pos_r(ml, slm) * D + D - 1, row_len);
              double* rv = vals + static_cast<int64_t>(rowl) * row_len + mask_pos_r(ml, slm) * D;
#pragma unroll
              for (int c = 0; c < D; ++c)
#pragma unroll
                for (int d = 0; d < D; ++d) atomicAdd(rv + c * cpl + d, acc[d * D + c]);
            }
          }
        }
      }
    }
  }
  cp_async_wait_all();  // no copy outlives the CTA
}

// Lower blocks of a symmetric J from the upper ones (the assembly ran with
// MIRROR = false): K_ab = K_ba^T for flat(b) < flat(a). One warp per row.
// First each lane resolves one lower block's source (row b, position of
// -delta in row b, its component pitch) into shared memory, so the per-value
// loop is one load and one coalesced store. A column node that is not a row
// (no DOF) gets a zero block.
// F16: the warp then also writes its row's fp16 smoother copy (k_vals_to_f16's
// row scale and rounding): the row is in L2 from the mirror, so the copy
// costs no second pass over the fp64 matrix.
template <int D, bool F16 = false>
__global__ void __launch_bounds__(256) k_mirror_lower(GridC g, int n_act, const int* __restrict__ act_list,
                                                      const int* __restrict__ act_idx, const int* __restrict__ row_nzb,
                                                      const uint8_t* __restrict__ row_slots,
                                                      const unsigned* __restrict__ row_mask,
                                                      double* __restrict__ vals, int64_t row_len,
                                                      __half* __restrict__ v16 = nullptr, int64_t row_len16 = 0,
                                                      float* __restrict__ rscale = nullptr) {
  constexpr int S = ipow_c(5, D);
  constexpr int center = (S - 1) / 2;  // slot of delta = 0
  __shared__ long long src_s[8][center];
  __shared__ int cpb_s[8][center];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  if (row >= n_act) return;
  const int node = act_list[row];
  const int nzb = row_nzb[row], cp = cpad(nzb, D);
  const uint8_t* sl = row_slots + static_cast<int64_t>(row) * S;
  // stored slots ascend, so the lower blocks are the first nl positions
  int nl = 0;
  {
    const unsigned* m = row_mask + static_cast<int64_t>(row) * 4;
    for (int w = 0; w < 4; ++w) {
      const int b0 = w * 32;
      if (b0 + 32 <= center)
        nl += __popc(m[w]);
      else if (b0 < center)
        nl += __popc(m[w] & ((1u << (center - b0)) - 1u));
    }
  }
  for (int j = lane; j < nl; j += 32) {
    int r = sl[j], off = 0;
    const int slot = r;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      off += (r % 5 - 2) * g.stride[a];
      r /= 5;
    }
    const int rb = act_idx[node + off];
    long long src = -1;
    int cpb = 0;
    if (rb >= 0) {
      const int ms = S - 1 - slot;  // the slot of -delta in row b
      const uint4 m4 = *reinterpret_cast<const uint4*>(row_mask + static_cast<int64_t>(rb) * 4);
      const unsigned mw[4] = {m4.x, m4.y, m4.z, m4.w};
      const int w = ms >> 5;
      int pb = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (k < w) pb += __popc(mw[k]);
        if (k == w) pb += __popc(mw[k] & ((1u << (ms & 31)) - 1u));
      }
      cpb = cpad(row_nzb[rb], D);
      IMPM_CHECK_IDX(pb, row_nzb[rb]);
      IMPM_CHECK_IDX(rb, n_act);
      src = static_cast<long long>(rb) * row_len + pb * D;
    }
    src_s[warp][j] = src;
    cpb_s[warp][j] = cpb;
  }
  __syncwarp();
  double* out = vals + static_cast<int64_t>(row) * row_len;
  // value (c, j, d) of the lower part: component chunk c is contiguous
  for (int c = 0; c < D; ++c)
    for (int e = lane; e < nl * D; e += 32) {
      const int j = e / D, d = e - j * D;
      const long long src = src_s[warp][j];
      out[c * cp + e] = src >= 0 ? vals[src + d * cpb_s[warp][j] + c] : 0.0;
    }
  if constexpr (F16) {
    __syncwarp();  // the lower blocks this warp stored (read back through L2: __ldcg)
    const int cq = chunk_len<__half>(nzb, D);
    __half* dst = v16 + static_cast<int64_t>(row) * row_len16;
    double mx = 0.0;
    for (int c = 0; c < D; ++c)
      for (int e = lane; e < nzb * D; e += 32) mx = fmax(mx, fabs(__ldcg(out + c * cp + e)));
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float sc = mx > 0.0 ? static_cast<float>(mx / 1024.0) : 1.0f;
    const float inv = 1.0f / sc;
    if (lane == 0) rscale[row] = sc;
    const int h2 = cq >> 1;  // __half2 per chunk
    for (int e = lane; e < D * h2; e += 32) {
      const int c = e / h2, j2 = e - c * h2;
      float2 o = make_float2(0.0f, 0.0f);
      if (2 * j2 < nzb * D) {
        const double2 v = __ldcg(reinterpret_cast<const double2*>(out + c * cp) + j2);
        o = make_float2(static_cast<float>(v.x) * inv, 2 * j2 + 1 < nzb * D ? static_cast<float>(v.y) * inv : 0.0f);
      }
      reinterpret_cast<__half2*>(dst + c * cq)[j2] = __float22half2_rn(o);
    }
  }
}

// Block inverse for the smoother / block-Jacobi preconditioner, safeguarded:
// a free component can carry an exactly zero diagonal (a lone particle with
// dw = 0 at that node), making the block singular; then fall back to the
// inverse of the positive diagonal entries (0 for a zero diagonal).
// 4x4 (3D u-p node blocks): Gauss-Jordan with partial pivoting; the
// determinant is the signed product of the pivots
__device__ __forceinline__ double det(const Mat<double, 4>& a) {
  double m[4][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) m[i / 4][i % 4] = a.e[i];
  double d = 1.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    int piv = k;
#pragma unroll
    for (int i = k + 1; i < 4; ++i)
      if (fabs(m[i][k]) > fabs(m[piv][k])) piv = i;
    if (m[piv][k] == 0.0) return 0.0;
    if (piv != k) {
      d = -d;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double t = m[k][j];
        m[k][j] = m[piv][j];
        m[piv][j] = t;
      }
    }
    d *= m[k][k];
#pragma unroll
    for (int i = k + 1; i < 4; ++i) {
      const double f = m[i][k] / m[k][k];
#pragma unroll
      for (int j = k; j < 4; ++j) m[i][j] -= f * m[k][j];
    }
  }
  return d;
}
__device__ __forceinline__ Mat<double, 4> inverse(const Mat<double, 4>& a) {
  double m[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      m[i][j] = a.e[i * 4 + j];
      m[i][4 + j] = i == j ? 1.0 : 0.0;
    }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    int piv = k;
#pragma unroll
    for (int i = k + 1; i < 4; ++i)
      if (fabs(m[i][k]) > fabs(m[piv][k])) piv = i;
    if (piv != k)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double t = m[k][j];
        m[k][j] = m[piv][j];
        m[piv][j] = t;
      }
    const double inv = 1.0 / m[k][k];
#pragma unroll
    for (int j = 0; j < 8; ++j) m[k][j] *= inv;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (i != k) {
        const double f = m[i][k];
#pragma unroll
        for (int j = 0; j < 8; ++j) m[i][j] -= f * m[k][j];
      }
  }
  Mat<double, 4> out;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) out.e[i * 4 + j] = m[i][4 + j];
  return out;
}

template <int F>
__device__ __forceinline__ Mat<double, F> safe_block_inverse(const Mat<double, F>& Mb) {
  double mx = 0.0;
#pragma unroll
  for (int i = 0; i < F * F; ++i) mx = fmax(mx, fabs(Mb.e[i]));
  const double d = det(Mb);
  double tol = 1e-13;
#pragma unroll
  for (int i = 0; i < F; ++i) tol *= mx;
  if (fabs(d) > tol && isfinite(d)) {
    const Mat<double, F> Mi = inverse(Mb);
    bool ok = true;
#pragma unroll
    for (int i = 0; i < F * F; ++i) ok = ok && isfinite(Mi.e[i]);
    if (ok) return Mi;
  }
  Mat<double, F> Mi = Mat<double, F>::zero();
#pragma unroll
  for (int c = 0; c < F; ++c) Mi(c, c) = Mb(c, c) > 0.0 ? 1.0 / Mb(c, c) : 0.0;
  return Mi;
}

// masked diagonal block inverse per row (block-Jacobi / MG smoother)
template <int D, int F = D>
__global__ void k_diag_inverse(int n_act, const int* __restrict__ act_list, const uint8_t* __restrict__ freem,
                               const unsigned* __restrict__ row_mask, const int* __restrict__ row_nzb,
                               const double* __restrict__ vals, int64_t row_len, double* __restrict__ dinv) {
  constexpr int S = ipow_c(5, D);
  constexpr int DD = F * F;
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n_act) return;
  const int k = act_list[row];
  const unsigned* m = row_mask + static_cast<int64_t>(row) * 4;
  const int sc = (S - 1) / 2;
  const bool has = (m[sc >> 5] >> (sc & 31)) & 1u;
  const int pos = mask_pos(m, sc);
  const int cp = cpad(row_nzb[row], F);
  const double* rv = vals + static_cast<int64_t>(row) * row_len + pos * F;
  Mat<double, F> Mb;
#pragma unroll
  for (int c = 0; c < F; ++c)
#pragma unroll
    for (int d = 0; d < F; ++d) {
      const bool fr = freem[static_cast<int64_t>(k) * F + c] && freem[static_cast<int64_t>(k) * F + d];
      Mb(c, d) = (has && fr) ? rv[c * cp + d] : (c == d ? 1.0 : 0.0);
    }
  const Mat<double, F> Mi = safe_block_inverse<F>(Mb);
#pragma unroll
  for (int i = 0; i < DD; ++i) dinv[static_cast<int64_t>(row) * DD + i] = Mi.e[i];
}

// -------------------------------------------------------------- K7 SpMV --
// y = J x on the box BSR: one warp per active row. The row's 5^D neighbour
// x-records are staged once in shared memory, then the row (S*F*F fp64,
// 16-byte aligned) is streamed with coalesced 16-byte loads; a per-block
// table maps value j -> (x slot, output component). Masked to free DOFs;
// fused partial of dotv . y for the CG step.
template <int D, int F>
struct SpmvTab {
  static constexpr int S = ipow_c(5, D);
  static constexpr int NV = S * F * F;
};

// MODE 0: y = A x (+ partial dotv.y); MODE 1: damped block-Jacobi sweep
// y = x + omega Dinv (b - A x); MODE 2: residual y = b - A x.
enum SpmvMode { kSpmvY = 0, kSpmvJacobi = 1, kSpmvResid = 2 };


// VT = double: the Jacobian itself; VT = float: the preconditioner's copy of
// a level matrix (values rounded once, vectors and sums stay fp64); VT =
// __half: the fine level's smoother copy, each row stored as fp16(a / s_row)
// with an fp32 row scale s_row = max|a| / 1024 (rscale), products in fp32
// against the fp32-staged x, row sums rescaled once
// RPW: rows per warp and chunk (0: the runtime rows_per_warp argument)
#ifndef IMPM_HW16
#define IMPM_HW16 16  // 8 measured slower (level 0: 49 vs 41 ms per load step)
#endif
constexpr int HW16 = IMPM_HW16;  // lanes per fp16 row on the big levels
#ifndef IMPM_SPMV_AHEAD
#define IMPM_SPMV_AHEAD 1  // load each row's head one row ahead
#endif
#ifndef IMPM_SPMV_HALF_MINB
#define IMPM_SPMV_HALF_MINB 8  // resident 4-warp CTAs per SM the half-warp (level) variants are compiled for
#endif
template <int D, int F, int WARPS, int MODE = kSpmvY, class VT = double, int RPW = 16, bool HALF = false>
__global__ void __launch_bounds__(WARPS * 32, HALF ? IMPM_SPMV_HALF_MINB : 1024 / (WARPS * 32)) k_spmv(GridC g, const int* __restrict__ act_list, int n_act,
                                                     const VT* __restrict__ vals, int64_t row_len,
                                                     const uint8_t* __restrict__ row_slots,
                                                     const int* __restrict__ row_nzb,
                                                     const double* __restrict__ x, const uint8_t* __restrict__ freem,
                                                     double* __restrict__ y, const double* __restrict__ dotv,
                                                     double* __restrict__ partials, const int* __restrict__ done,
                                                     const double* __restrict__ b = nullptr,
                                                     const double* __restrict__ dinv = nullptr, double omega = 0.0,
                                                     int rows_per_warp = 16,
                                                     const float* __restrict__ x4 = nullptr,
                                                     float* __restrict__ y4 = nullptr,
                                                     const float* __restrict__ rscale = nullptr) {
  constexpr int S = ipow_c(5, D);
  constexpr int FF = F * F;
  constexpr int XS = chunk_len<VT>(S, F);
  constexpr int VW = 16 / sizeof(VT);  // values per 16-byte load
  constexpr int TAIL_UNROLL = sizeof(VT) == 8 ? 4 : 2;
  using V16 = typename std::conditional<sizeof(VT) == 8, double2,
                                        typename std::conditional<sizeof(VT) == 4, float4, uint4>::type>::type;
  using XT = typename std::conditional<sizeof(VT) == 8, double, float>::type;  // staged x
  // double2 per lane buffered ahead of the x gathers (the Jacobi sweep keeps
  // its Dinv row and rhs in registers too: smaller head under the 64-reg cap)
  // fp32 rows carry half the bytes (~5 float4 per lane at 73 blocks/row)
#ifndef IMPM_SPMV16_NB
#define IMPM_SPMV16_NB 0  // 0: as fp32/fp64; > 0: buffered 16-byte loads per lane of the fp16 sweeps
#endif
  constexpr int NB = (sizeof(VT) == 2 && IMPM_SPMV16_NB > 0) ? IMPM_SPMV16_NB
                     : sizeof(VT) == 8                     ? (MODE == kSpmvJacobi ? 4 : 6)
                                                           : (MODE == kSpmvJacobi ? 4 : 6);
  // lanes per row: fp32 rows carry half the bytes, so on big levels (HALF) a
  // half-warp streams one row and each warp keeps two rows (two latency
  // chains) in flight
  constexpr int HW = (sizeof(VT) == 2 && HALF) ? HW16 : ((sizeof(VT) == 4 && HALF) ? 16 : 32);
  constexpr int RW = 32 / HW;  // rows per warp in flight
  __shared__ int offt[S];
  // x neighbourhood staged in the matrix precision (fp32 copies: products in
  // fp32, each 4-term partial added to the fp64 row sum)
  __shared__ __align__(16) XT xs_all[WARPS * RW][XS];
  for (int sl = threadIdx.x; sl < S; sl += blockDim.x) {
    int rs = sl, off = 0;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      off += (rs % 5 - 2) * g.stride[a];
      rs /= 5;
    }
    offt[sl] = off;  // stored blocks always couple in-grid nodes
  }
  __syncthreads();
  double part[1] = {0.0};
  if (done == nullptr || *done == 0) {
    const int warp = threadIdx.x >> 5, wl = threadIdx.x & 31;
    const int lane = wl % HW, sub = wl / HW;  // lane within the row group, row slot in the warp
    XT* xs = xs_all[warp * RW + sub];
    // contiguous row chunks per CTA: consecutive rows share 4/5 of their x
    // neighbourhood, so the x gathers of a chunk hit in this SM's L1 (small
    // coarse levels use short chunks so that every warp gets a row)
    const int CH = (RPW > 0 ? RPW : rows_per_warp) * WARPS;
    const int nchunks = (n_act + CH - 1) / CH;
    for (int ci = blockIdx.x; ci < nchunks; ci += gridDim.x) {
    const int rend = min(n_act, (ci + 1) * CH);
    // the head of a row (node, block count, row scale, the lane's first slot)
    // is loaded one row ahead, so it is in flight while the previous row runs
    int kq = 0, nzq = 0, slq = 0;
    float rsq = 1.0f;
    auto head = [&](int r) {
      kq = 0;
      nzq = 0;
      slq = 0;
      rsq = 1.0f;
      if (r < rend) {
        kq = act_list[r];
        nzq = row_nzb[r];
        slq = lane < S ? row_slots[static_cast<int64_t>(r) * S + lane] : 0;
        if constexpr (sizeof(VT) == 2) rsq = __ldg(rscale + r);
      }
    };
    // (the level sweeps: 0.518 vs 0.535 ms per level-0 scope; the fp64 CG
    // SpMV is HBM-bound and loses 1.5% with it)
    constexpr bool AHEAD = IMPM_SPMV_AHEAD && HALF;
    if (AHEAD) head(ci * CH + warp * RW + sub);
    for (int row0 = ci * CH + warp * RW; row0 < rend; row0 += WARPS * RW) {
      const int row = row0 + sub;
      const bool live = row < rend;  // the last pair may be half empty
      int k, nzb, sl0;
      float rsc;
      if (AHEAD) {
        k = kq;
        nzb = nzq;
        sl0 = slq;
        rsc = rsq;
        head(row + WARPS * RW);
      } else {
        k = live ? act_list[row] : 0;
        nzb = live ? row_nzb[row] : 0;
        sl0 = 0;
        rsc = (sizeof(VT) == 2 && live) ? __ldg(rscale + row) : 1.0f;
      }
      const int cp = chunk_len<VT>(nzb, F);
      const int h = cp / VW, tot2 = F * h;
      const int64_t base = static_cast<int64_t>(k) * F;
      // 0. epilogue operands go in flight first: lane c < F holds component
      //    c's free mask, its dot / rhs operand, its own x and row c of Dinv
      bool fm = false;
      double e0 = 0.0, e1 = 0.0;
      double di[F];
#pragma unroll
      for (int d = 0; d < F; ++d) di[d] = 0.0;
      if (live && lane < F) {
        fm = freem[base + lane] != 0;
        if constexpr (MODE == kSpmvY) {
          if (dotv) e0 = dotv[base + lane];
        } else {
          e0 = b[base + lane];
          if constexpr (MODE == kSpmvJacobi) {
            e1 = x[base + lane];
#pragma unroll
            for (int d = 0; d < F; ++d) di[d] = dinv[static_cast<int64_t>(row) * FF + lane * F + d];
          }
        }
      }
      // 1. the first NB double2 per lane of the row (independent of x) go in
      //    flight before the x gathers
      const V16* rv = reinterpret_cast<const V16*>(vals + static_cast<int64_t>(row) * row_len);
      V16 buf[NB];
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        const int j2 = lane + HW * t;
        buf[t] = j2 < tot2 ? __ldcs(rv + j2) : V16{};  // streamed once: evict-first
      }
      // 2. stage the x records of the stored neighbours
      const uint8_t* rsl = row_slots + static_cast<int64_t>(row) * S;
      if constexpr (sizeof(VT) <= 4 && F <= 4) {
        if (x4 != nullptr) {
          // fp32 twin of x, one 16-byte record per node: one load per neighbour
          for (int pos = lane; pos < nzb; pos += HW) {
            const int sl = AHEAD && pos == lane ? sl0 : rsl[pos];
            IMPM_CHECK_IDX(k + offt[sl], g.N);
            const float4 v = __ldg(reinterpret_cast<const float4*>(x4) + (k + offt[sl]));
            xs[pos * F + 0] = v.x;
            if (F > 1) xs[pos * F + 1] = v.y;
            if (F > 2) xs[pos * F + 2] = v.z;
            if (F > 3) xs[pos * F + 3] = v.w;
          }
        } else {
          for (int pos = lane; pos < nzb; pos += HW) {
            const int sl = AHEAD && pos == lane ? sl0 : rsl[pos];
            IMPM_CHECK_IDX(k + offt[sl], g.N);
            const int64_t nb = static_cast<int64_t>(k + offt[sl]) * F;
#pragma unroll
            for (int d = 0; d < F; ++d) xs[pos * F + d] = static_cast<XT>(__ldg(x + nb + d));
          }
        }
      } else {
        for (int pos = lane; pos < nzb; pos += HW) {
          const int sl = AHEAD && pos == lane ? sl0 : rsl[pos];
          IMPM_CHECK_IDX(k + offt[sl], g.N);
          const int64_t nb = static_cast<int64_t>(k + offt[sl]) * F;
#pragma unroll
          for (int d = 0; d < F; ++d) xs[pos * F + d] = static_cast<XT>(__ldg(x + nb + d));
        }
      }
      for (int e = lane; e < cp - nzb * F; e += HW) xs[nzb * F + e] = XT(0);
      __syncwarp();
      // 3. component-major dot products (buffered head, streamed tail)
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      using XV = typename std::conditional<sizeof(VT) == 8, double2, float4>::type;
      constexpr int XSTEP = sizeof(VT) == 2 ? 2 : 1;  // x vectors per value vector
      const XV* xv = reinterpret_cast<const XV*>(xs);
      auto consume = [&](int j2, const V16 v) {
        const int c = F == 1   ? 0
                      : F == 2 ? (j2 >= h)
                      : F == 3 ? (j2 >= h) + (j2 >= 2 * h)
                               : (j2 >= h) + (j2 >= 2 * h) + (j2 >= 3 * h);
        double p;
        const XV xx = xv[XSTEP * (j2 - c * h)];
        if constexpr (sizeof(VT) == 8) {
          p = fma(v.x, xx.x, v.y * xx.y);
        } else if constexpr (sizeof(VT) == 4) {
          p = static_cast<double>(fmaf(v.x, xx.x, fmaf(v.y, xx.y, fmaf(v.z, xx.z, v.w * xx.w))));
        } else {
          const __half2* hv = reinterpret_cast<const __half2*>(&v);
          const float2 a0 = __half22float2(hv[0]), a1 = __half22float2(hv[1]);
          const float2 a2 = __half22float2(hv[2]), a3 = __half22float2(hv[3]);
          const float4 xb = xv[XSTEP * (j2 - c * h) + 1];
          p = static_cast<double>(fmaf(a0.x, xx.x, fmaf(a0.y, xx.y, fmaf(a1.x, xx.z, a1.y * xx.w)))) +
              static_cast<double>(fmaf(a2.x, xb.x, fmaf(a2.y, xb.y, fmaf(a3.x, xb.z, a3.y * xb.w))));
        }
        acc[0] += c == 0 ? p : 0.0;
        if (F > 1) acc[1] += c == 1 ? p : 0.0;
        if (F > 2) acc[2] += c == 2 ? p : 0.0;
        if (F > 3) acc[3] += c == 3 ? p : 0.0;
      };
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        const int j2 = lane + HW * t;
        if (j2 < tot2) consume(j2, buf[t]);
      }
#pragma unroll TAIL_UNROLL
      for (int j2 = lane + HW * NB; j2 < tot2; j2 += HW) consume(j2, __ldcs(rv + j2));
      // butterfly within the row group: every lane holds the row sums; lane
      // c < F finishes component c
#pragma unroll
      for (int c = 0; c < F; ++c)
        for (int o = HW / 2; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
      double mine = acc[0];
      if (F > 1 && lane == 1) mine = acc[1];
      if (F > 2 && lane == 2) mine = acc[2];
      if (F > 3 && lane == 3) mine = acc[3];
      if constexpr (sizeof(VT) == 2) mine *= static_cast<double>(rsc);
      if constexpr (MODE == kSpmvY) {
        if (live && lane < F) {
          const double v = fm ? mine : 0.0;
          y[base + lane] = v;
          if (dotv) part[0] += v * e0;
        }
      } else if constexpr (MODE == kSpmvResid) {
        if (live && lane < F) y[base + lane] = fm ? e0 - mine : 0.0;
      } else {
        const double rown = (lane < F && fm) ? e0 - mine : 0.0;
        double rr[F];
#pragma unroll
        for (int d = 0; d < F; ++d) rr[d] = __shfl_sync(0xffffffffu, rown, sub * HW + d);
        if (live && lane < F) {
          double sacc = 0.0;
#pragma unroll
          for (int d = 0; d < F; ++d) sacc += di[d] * rr[d];
          const double yv = fm ? e1 + omega * sacc : 0.0;
          y[base + lane] = yv;
          if (y4) y4[static_cast<int64_t>(k) * 4 + lane] = static_cast<float>(yv);
        }
      }
      __syncwarp();
    }
    }
  }
  if (partials) block_sum_store<1>(part, partials);
}

// fp32 copy of a compacted level matrix for the preconditioner (one pass per
// assembly / Galerkin product: read 8 B + write 4 B per stored value)
template <int F>
__global__ void k_vals_to_f32(int n_act, const int* __restrict__ row_nzb, const double* __restrict__ vals,
                              int64_t row_len, float* __restrict__ v32, int64_t row_len32, int f16sim = 0) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int row = warp; row < n_act; row += nw) {
    const int nzb = row_nzb[row];
    const int cp = chunk_len<double>(nzb, F), cq = chunk_len<float>(nzb, F);
    const double* src = vals + static_cast<int64_t>(row) * row_len;
    float* dst = v32 + static_cast<int64_t>(row) * row_len32;
    if (f16sim) {  // A/B experiment: values rounded to fp16 with a per-row scale
      double mx = 0.0;
      for (int e = lane; e < F * cp; e += 32) mx = fmax(mx, fabs(src[e]));
      for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float sc = mx > 0.0 ? static_cast<float>(mx / 1024.0) : 1.0f;
      const int h2 = cq >> 1;
      for (int e = lane; e < F * h2; e += 32) {
        const int c = e / h2, j2 = e - c * h2;
        float2 o = make_float2(0.0f, 0.0f);
        if (2 * j2 < nzb * F) {
          const double2 v = reinterpret_cast<const double2*>(src + c * cp)[j2];
          o.x = __half2float(__float2half_rn(static_cast<float>(v.x) / sc)) * sc;
          o.y = 2 * j2 + 1 < nzb * F ? __half2float(__float2half_rn(static_cast<float>(v.y) / sc)) * sc : 0.0f;
        }
        reinterpret_cast<float2*>(dst + c * cq)[j2] = o;
      }
      continue;
    }
    // pairs: both chunk starts are 16-byte aligned (cp even, cq % 4 == 0)
    const int h2 = cq >> 1;  // float2 per fp32 chunk
    for (int e = lane; e < F * h2; e += 32) {
      const int c = e / h2, j2 = e - c * h2;
      float2 o = make_float2(0.0f, 0.0f);
      if (2 * j2 < nzb * F) {  // pads (fp64 or fp32) become exact zeros
        const double2 v = __ldcs(reinterpret_cast<const double2*>(src + c * cp) + j2);
        o = make_float2(static_cast<float>(v.x), 2 * j2 + 1 < nzb * F ? static_cast<float>(v.y) : 0.0f);
      }
      reinterpret_cast<float2*>(dst + c * cq)[j2] = o;
    }
  }
}

// fp16 copy of the fine level matrix for the smoother: per row s = max|a| /
// 1024 (fp32), values fp16(a / s) -- the MG V-cycle is a preconditioner,
// CG's own SpMV stays fp64 (tests: Krylov and Newton counts unchanged)
template <int F>
__global__ void k_vals_to_f16(int n_act, const int* __restrict__ row_nzb, const double* __restrict__ vals,
                              int64_t row_len, __half* __restrict__ v16, int64_t row_len16,
                              float* __restrict__ rscale) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int row = warp; row < n_act; row += nw) {
    const int nzb = row_nzb[row];
    const int cp = chunk_len<double>(nzb, F), cq = chunk_len<__half>(nzb, F);
    const double* src = vals + static_cast<int64_t>(row) * row_len;
    __half* dst = v16 + static_cast<int64_t>(row) * row_len16;
    double mx = 0.0;
    for (int c = 0; c < F; ++c)
      for (int e = lane; e < nzb * F; e += 32) mx = fmax(mx, fabs(__ldg(src + c * cp + e)));  // kept in L1 for the 2nd pass
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float sc = mx > 0.0 ? static_cast<float>(mx / 1024.0) : 1.0f;
    const float inv = 1.0f / sc;
    if (lane == 0) rscale[row] = sc;
    const int h2 = cq >> 1;  // __half2 per chunk
    for (int e = lane; e < F * h2; e += 32) {
      const int c = e / h2, j2 = e - c * h2;
      float2 o = make_float2(0.0f, 0.0f);
      if (2 * j2 < nzb * F) {
        const double2 v = __ldcs(reinterpret_cast<const double2*>(src + c * cp) + j2);
        o = make_float2(static_cast<float>(v.x) * inv, 2 * j2 + 1 < nzb * F ? static_cast<float>(v.y) * inv : 0.0f);
      }
      reinterpret_cast<__half2*>(dst + c * cq)[j2] = __float22half2_rn(o);
    }
  }
}

// ------------------------------------------------------- K7 PCG vectors --
// scalar slots of the device-resident CG state
enum CgSlot { kRz = 0, kPq, kRzNew, kRr, kBb, kAlpha, kBeta, kIters, kDone, kNSlots };

// r = b, x = 0, z = Minv r, p = z; partials of r.z and b.b
template <int F>
__global__ void k_cg_init(int N, const int* __restrict__ act_idx, const double* __restrict__ dinv,
                          const double* __restrict__ b, double* __restrict__ x, double* __restrict__ r,
                          double* __restrict__ z, double* __restrict__ p, double* __restrict__ partials) {
  double v[2] = {0.0, 0.0};
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    const int row = act_idx[n];
    double rl[F], zl[F];
#pragma unroll
    for (int c = 0; c < F; ++c) rl[c] = row >= 0 ? b[n * F + c] : 0.0;
#pragma unroll
    for (int c = 0; c < F; ++c) {
      double s = 0.0;
      if (row >= 0)
#pragma unroll
        for (int d = 0; d < F; ++d) s += dinv[static_cast<int64_t>(row) * F * F + c * F + d] * rl[d];
      zl[c] = s;
    }
#pragma unroll
    for (int c = 0; c < F; ++c) {
      x[n * F + c] = 0.0;
      r[n * F + c] = rl[c];
      z[n * F + c] = zl[c];
      p[n * F + c] = zl[c];
      v[0] += rl[c] * zl[c];
      v[1] += rl[c] * rl[c];
    }
  }
  block_sum_store<2>(v, partials);
}

__global__ void k_cg_start(const double* __restrict__ sums, double* __restrict__ sc, double rtol) {
  // sums = {r.z, b.b}
  sc[kRz] = sums[0];
  sc[kBb] = sums[1];
  sc[kRr] = sums[1];
  sc[kIters] = 0.0;
  sc[kDone] = (sums[1] == 0.0) ? 1.0 : 0.0;
  (void)rtol;
}

// alpha = rz / (p.q); breakdown (p.q <= 0) -> done = 2
__global__ void k_cg_alpha(const double* __restrict__ sums, double* __restrict__ sc, int* __restrict__ done) {
  if (*done) return;
  const double pq = sums[0];
  sc[kPq] = pq;
  if (!(pq > 0.0)) {
    sc[kDone] = 2.0;
    *done = 2;
    return;
  }
  sc[kAlpha] = sc[kRz] / pq;
}

// x += a p; r -= a q; z = Minv r; partials of r.z and r.r
template <int F>
__global__ void k_cg_update(int N, const int* __restrict__ act_idx, const double* __restrict__ dinv,
                            const double* __restrict__ sc, const int* __restrict__ done, double* __restrict__ x,
                            double* __restrict__ r, double* __restrict__ z, const double* __restrict__ p,
                            const double* __restrict__ q, double* __restrict__ partials) {
  double v[2] = {0.0, 0.0};
  if (*done == 0) {
    const double alpha = sc[kAlpha];
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
      const int row = act_idx[n];
      if (row >= 0) {
        double rl[F];
#pragma unroll
        for (int c = 0; c < F; ++c) {
          x[n * F + c] += alpha * p[n * F + c];
          rl[c] = r[n * F + c] - alpha * q[n * F + c];
          r[n * F + c] = rl[c];
        }
#pragma unroll
        for (int c = 0; c < F; ++c) {
          double s = 0.0;
#pragma unroll
          for (int d = 0; d < F; ++d) s += dinv[static_cast<int64_t>(row) * F * F + c * F + d] * rl[d];
          z[n * F + c] = s;
          v[0] += rl[c] * s;
          v[1] += rl[c] * rl[c];
        }
      }
    }
  }
  block_sum_store<2>(v, partials);
}

__global__ void k_cg_beta(const double* __restrict__ sums, double* __restrict__ sc, int* __restrict__ done,
                          double rtol2, int max_iter) {
  if (*done) return;
  const double rz_new = sums[0], rr = sums[1];
  sc[kIters] += 1.0;
  sc[kRr] = rr;
  if (!(rr == rr)) {  // NaN
    sc[kDone] = 3.0;
    *done = 3;
    return;
  }
  if (rr <= rtol2 * sc[kBb]) {
    sc[kDone] = 1.0;
    *done = 1;
    return;
  }
  if (sc[kIters] >= max_iter) {
    sc[kDone] = 4.0;
    *done = 4;
    return;
  }
  sc[kBeta] = rz_new / sc[kRz];
  sc[kRz] = rz_new;
}

template <int F>
__global__ void k_cg_p(int N, const int* __restrict__ act_idx, const double* __restrict__ sc,
                       const int* __restrict__ done, const double* __restrict__ z, double* __restrict__ p) {
  if (*done) return;
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N || act_idx[n] < 0) return;
  const double beta = sc[kBeta];
#pragma unroll
  for (int c = 0; c < F; ++c) p[n * F + c] = z[n * F + c] + beta * p[n * F + c];
}

// Sum of `nb` partials (row k of NV rows) by one block, fixed order: every
// block of the consumer kernel computes the same value (deterministic, no
// separate finalize launch).
template <int NV>
__device__ __forceinline__ void block_reduce_partials(const double* __restrict__ partials, int nb, double (&out)[NV]) {
  __shared__ double red[NV][32];
  __shared__ double res[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) s += partials[k * nb + i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[k][threadIdx.x >> 5] = s;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = threadIdx.x < nw ? red[k][threadIdx.x] : 0.0;
      for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
      if (threadIdx.x == 0) res[k] = s;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < NV; ++k) out[k] = res[k];
}

// CG step part 1: alpha = rz / p.q (from the SpMV partials); x += a p;
// r -= a q; z = Minv r; partials of r.z and r.r.  rz lives in sc[kRz + par].
template <int F>
__global__ void k_cg_update2(int N, const int* __restrict__ act_idx, const double* __restrict__ dinv,
                             double* __restrict__ sc, int* __restrict__ done, int par, const double* __restrict__ pq_part,
                             int nb, double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
                             const double* __restrict__ p, const double* __restrict__ q,
                             double* __restrict__ partials) {
  double v[2] = {0.0, 0.0};
  const int was_done = *done;
  double pq[1];
  block_reduce_partials<1>(pq_part, nb, pq);
  if (!was_done) {
    const double rz = sc[par ? kBeta : kRz];  // ping-pong slot holding the current r.z
    if (!(pq[0] > 0.0)) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        sc[kDone] = 2.0;
        *done = 2;
      }
    } else {
      const double alpha = rz / pq[0];
      for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
        const int row = act_idx[n];
        if (row < 0) continue;
        double rl[F];
#pragma unroll
        for (int c = 0; c < F; ++c) {
          x[n * F + c] += alpha * p[n * F + c];
          rl[c] = r[n * F + c] - alpha * q[n * F + c];
          r[n * F + c] = rl[c];
        }
#pragma unroll
        for (int c = 0; c < F; ++c) {
          double s = 0.0;
#pragma unroll
          for (int d = 0; d < F; ++d) s += dinv[static_cast<int64_t>(row) * F * F + c * F + d] * rl[d];
          z[n * F + c] = s;
          v[0] += rl[c] * s;
          v[1] += rl[c] * rl[c];
        }
      }
    }
  }
  block_sum_store<2>(v, partials);
}

// CG step part 2: convergence test on r.r, beta = rz_new / rz, p = z + beta p.
// Block 0 records rz_new in the other ping-pong slot and the iteration count.
template <int F>
__global__ void k_cg_p2(int N, const int* __restrict__ act_idx, double* __restrict__ sc, int* __restrict__ done,
                        int par, int it, const double* __restrict__ part, int nb, double rtol2, int max_iter,
                        const double* __restrict__ z, double* __restrict__ p) {
  if (*done) return;
  double v[2];
  block_reduce_partials<2>(part, nb, v);
  const double rz_new = v[0], rr = v[1];
  const double rz = sc[par ? kBeta : kRz];
  const double iters = it + 1.0;
  int stop = 0;
  if (!(rr == rr)) stop = 3;
  else if (rr <= rtol2 * sc[kBb]) stop = 1;
  else if (iters >= max_iter) stop = 4;
  // every block takes the same decision from the same sums
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc[kIters] = iters;
    sc[kRr] = rr;
    sc[par ? kRz : kBeta] = rz_new;
    if (stop) {
      sc[kDone] = stop;
      *done = stop;
    }
  }
  if (stop) return;
  const double beta = rz_new / rz;
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    if (act_idx[n] < 0) continue;
#pragma unroll
    for (int c = 0; c < F; ++c) p[n * F + c] = z[n * F + c] + beta * p[n * F + c];
  }
}

// generic BLAS-1 on grid vectors (nonsymmetric Krylov path)
__global__ void k_dot2(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                       const double* __restrict__ c, const double* __restrict__ d, double* __restrict__ partials) {
  double v[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    v[0] += a[i] * b[i];
    if (c) v[1] += c[i] * d[i];
  }
  block_sum_store<2>(v, partials);
}

// h_i = V_i . w for i < nv (blockIdx.y = i), per-block partials [i][block]
__global__ void k_vdot(int64_t n, const double* __restrict__ V, int64_t ldv, const double* __restrict__ w,
                       double* __restrict__ partials) {
  const double* Vi = V + static_cast<int64_t>(blockIdx.y) * ldv;
  double v[1] = {0.0};
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    v[0] += Vi[i] * w[i];
  block_sum_store<1>(v, partials + static_cast<int64_t>(blockIdx.y) * gridDim.x);
}
// out[row] = sum of partials row (one block per row, fixed order)
__global__ void k_finalize_rows(const double* __restrict__ partials, int nb, double* __restrict__ out) {
  const double* p = partials + static_cast<int64_t>(blockIdx.x) * nb;
  double v = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) v += p[i];
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) out[blockIdx.x] = v;
  }
}
// w -= sum_i h_i V_i  (h on the device)
__global__ void k_vsub(int64_t n, const double* __restrict__ V, int64_t ldv, int nv, const double* __restrict__ h,
                       double* __restrict__ w) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double acc = w[i];
    for (int j = 0; j < nv; ++j) acc -= h[j] * V[static_cast<int64_t>(j) * ldv + i];
    w[i] = acc;
  }
}

// y = a*x + b*y + c*z  (z optional)
__global__ void k_axpbypcz(int64_t n, double a, const double* __restrict__ x, double b, double* __restrict__ y,
                           double c, const double* __restrict__ z) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = a * x[i] + b * y[i] + (z ? c * z[i] : 0.0);
}

// z = Minv r (block Jacobi on active rows)
template <int F>
__global__ void k_precond(int N, const int* __restrict__ act_idx, const double* __restrict__ dinv,
                          const double* __restrict__ r, double* __restrict__ z) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const int row = act_idx[n];
#pragma unroll
  for (int c = 0; c < F; ++c) {
    double s = 0.0;
    if (row >= 0)
#pragma unroll
      for (int d = 0; d < F; ++d) s += dinv[static_cast<int64_t>(row) * F * F + c * F + d] * r[n * F + d];
    z[n * F + c] = s;
  }
}

// ------------------------------------------------- K7 multigrid (Galerkin) --
// Vertex-centred factor-2 coarsening of the structured grid: coarse node I
// sits on fine node 2I; trilinear prolongation P (weights 1 / 0.5 per axis).
// The coarse operator A_c = P^T M A M P (M = free-DOF mask) is again a 5^D
// box-BSR (|2I-2J| <= 1+2+1), stored compacted like the fine Jacobian, so the
// same SpMV / smoother kernel serves every level.
__device__ __forceinline__ double p1w(int e) { return e == 0 ? 1.0 : 0.5; }

// coarse node active iff an active fine row lies in supp(P_I)
template <int D>
__global__ void k_coarse_active(GridC gf, GridC gc, const int* __restrict__ fine_act_idx, int* __restrict__ cflag) {
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= gc.N) return;
  int ci[3];
  unflat<D>(gc, I, ci);
  int act = 0;
  constexpr int NE = ipow_c(3, D);
  for (int e = 0; e < NE && !act; ++e) {
    int r = e, fi = 0;
    bool ok = true;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      const int ia = 2 * ci[a] + (r % 3) - 1;
      r /= 3;
      ok = ok && ia >= 0 && ia < gf.nodes[a];
      fi += ia * gf.stride[a];
    }
    if (ok && fine_act_idx[fi] >= 0) act = 1;
  }
  cflag[I] = act;
}

// Galerkin step 1 (one warp per fine row i): T[i][J] = sum_j A_ij M_j P_jJ
// for the <= 4^D coarse nodes J whose support meets the +-2 box of i
// (J_a in [(i_a-2)>>1, +4)); lanes own the coarse slots (deterministic).
template <int D, int F, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_galerkin_ap(GridC gf, GridC gc, int f_n_act,
                                                            const int* __restrict__ f_act_list,
                                                            const double* __restrict__ fvals, int64_t f_row_len,
                                                            const uint8_t* __restrict__ f_slots,
                                                            const int* __restrict__ f_nzb,
                                                            const uint8_t* __restrict__ f_freem,
                                                            double* __restrict__ T) {
  constexpr int S = ipow_c(5, D);
  constexpr int FF = F * F;
  constexpr int NT = ipow_c(4, D);
  constexpr int NTL = (NT + 31) / 32;
  __shared__ short inv_all[WARPS][S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  short* inv = inv_all[warp];
  for (int row = blockIdx.x * WARPS + warp; row < f_n_act; row += gridDim.x * WARPS) {
    const int i = f_act_list[row];
    int fi[3];
    unflat<D>(gf, i, fi);
    const int nzb = f_nzb[row];
    const uint8_t* fs = f_slots + static_cast<int64_t>(row) * S;
    for (int sl = lane; sl < S; sl += 32) inv[sl] = -1;
    __syncwarp();
    for (int pos = lane; pos < nzb; pos += 32) inv[fs[pos]] = static_cast<short>(pos);
    __syncwarp();
    const double* fv = fvals + static_cast<int64_t>(row) * f_row_len;
    const int cpf = cpad(nzb, F);
    double* Ti = T + static_cast<int64_t>(row) * NT * FF;
#pragma unroll
    for (int u = 0; u < NTL; ++u) {
      const int tl = lane + 32 * u;
      if (tl >= NT) continue;
      double acc[FF];
#pragma unroll
      for (int e = 0; e < FF; ++e) acc[e] = 0.0;
      // per axis: coarse J_a = ((fi_a - 2) >> 1) + t_a; fine j_a = 2 J_a + f, |j_a - fi_a| <= 2
      int Ja[3], lo[3], hi[3];
      bool ok = true;
      int r = tl;
#pragma unroll
      for (int a = D - 1; a >= 0; --a) {
        const int t = r % 4;
        r /= 4;
        Ja[a] = ((fi[a] - 2) >> 1) + t;
        ok = ok && Ja[a] >= 0 && Ja[a] < gc.nodes[a];
        lo[a] = max(-1, fi[a] - 2 - 2 * Ja[a]);
        hi[a] = min(1, fi[a] + 2 - 2 * Ja[a]);
        ok = ok && lo[a] <= hi[a];
      }
      if (ok) {
        const int f1lo = D > 1 ? lo[1] : 0, f1hi = D > 1 ? hi[1] : 0;
        const int f2lo = D > 2 ? lo[2] : 0, f2hi = D > 2 ? hi[2] : 0;
        for (int f0 = lo[0]; f0 <= hi[0]; ++f0)
          for (int f1 = f1lo; f1 <= f1hi; ++f1)
            for (int f2 = f2lo; f2 <= f2hi; ++f2) {
              const int fo[3] = {f0, f1, f2};
              int sl = 0, j = 0;
              double w = 1.0;
              bool in = true;
#pragma unroll
              for (int a = 0; a < D; ++a) {
                const int ja = 2 * Ja[a] + fo[a];
                in = in && ja >= 0 && ja < gf.nodes[a];
                sl = sl * 5 + (ja - fi[a] + 2);
                j += ja * gf.stride[a];
                w *= p1w(fo[a]);
              }
              if (!in) continue;
              const int pos = inv[sl];
              if (pos < 0) continue;
              const double* blk = fv + pos * F;
#pragma unroll
              for (int d = 0; d < F; ++d) {
                if (!f_freem[static_cast<int64_t>(j) * F + d]) continue;
#pragma unroll
                for (int c = 0; c < F; ++c) acc[c * F + d] += w * blk[c * cpf + d];
              }
            }
      }
#pragma unroll
      for (int e = 0; e < FF; ++e) Ti[tl * FF + e] = acc[e];
    }
    __syncwarp();
  }
}

// Galerkin step 2 (one warp per coarse row I): A_c[I][J] = sum_i w_i M_i T[i][J]
// over the 3^D fine rows i in supp(P_I); lanes own coarse box slots J.
// Compacts nonzero blocks, sets the coarse free mask from the diagonal and
// the masked block inverse.
#ifndef IMPM_PTAP_MINB
#define IMPM_PTAP_MINB 0  // 0: the compiler's register choice
#endif
#if IMPM_PTAP_MINB > 0
#define IMPM_PTAP_LB(T) __launch_bounds__(T, IMPM_PTAP_MINB)
#else
#define IMPM_PTAP_LB(T) __launch_bounds__(T)
#endif
template <int D, int F, int WARPS>
__global__ void IMPM_PTAP_LB(WARPS * 32) k_galerkin_ptap(GridC gf, GridC gc, const int* __restrict__ f_act_idx,
                                                              const uint8_t* __restrict__ f_freem,
                                                              const double* __restrict__ T,
                                                              const int* __restrict__ c_act_list, int c_n_act,
                                                              double* __restrict__ cvals, int64_t c_row_len,
                                                              uint8_t* __restrict__ c_slots, int* __restrict__ c_nzb,
                                                              uint8_t* __restrict__ c_freem, double* __restrict__ c_dinv,
                                                              unsigned long long* __restrict__ nzb_total) {
  constexpr int S = ipow_c(5, D);
  constexpr int FF = F * F;
  constexpr int NE = ipow_c(3, D);
  constexpr int NT = ipow_c(4, D);
  constexpr int NJ = (S + 31) / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int row = blockIdx.x * WARPS + warp; row < c_n_act; row += gridDim.x * WARPS) {
    const int I = c_act_list[row];
    int ci[3];
    unflat<D>(gc, I, ci);
    double acc[NJ][FF];
#pragma unroll
    for (int t = 0; t < NJ; ++t)
#pragma unroll
      for (int e = 0; e < FF; ++e) acc[t][e] = 0.0;
    for (int e = 0; e < NE; ++e) {
      int r = e, fi[3], eo[3], i = 0;
      bool ok = true;
      double wi = 1.0;
#pragma unroll
      for (int a = D - 1; a >= 0; --a) {
        eo[a] = (r % 3) - 1;
        r /= 3;
        fi[a] = 2 * ci[a] + eo[a];
        ok = ok && fi[a] >= 0 && fi[a] < gf.nodes[a];
        i += fi[a] * gf.stride[a];
      }
      if (!ok) continue;
      const int frow = f_act_idx[i];
      if (frow < 0) continue;
#pragma unroll
      for (int a = 0; a < D; ++a) wi *= p1w(eo[a]);
      bool mi[F];
#pragma unroll
      for (int c = 0; c < F; ++c) mi[c] = f_freem[static_cast<int64_t>(i) * F + c] != 0;
      const double* Ti = T + static_cast<int64_t>(frow) * NT * FF;
#pragma unroll
      for (int t = 0; t < NJ; ++t) {
        const int js = lane + 32 * t;
        if (js >= S) continue;
        int rs = js, tl = 0;
        bool in = true;
#pragma unroll
        for (int a = D - 1; a >= 0; --a) {
          const int Ja = ci[a] + rs % 5 - 2;
          rs /= 5;
          const int ta = Ja - ((fi[a] - 2) >> 1);
          in = in && ta >= 0 && ta < 4;
          tl += ta * (a == D - 1 ? 1 : (a == D - 2 ? 4 : 16));
        }
        if (!in) continue;
        const double* tb = Ti + tl * FF;
#pragma unroll
        for (int c = 0; c < F; ++c) {
          if (!mi[c]) continue;
#pragma unroll
          for (int d = 0; d < F; ++d) acc[t][c * F + d] += wi * tb[c * F + d];
        }
      }
    }
    int base = 0;
    int posv[NJ];
    bool flag[NJ];
#pragma unroll
    for (int t = 0; t < NJ; ++t) {
      const int js = lane + 32 * t;
      bool f = false;
      if (js < S)
#pragma unroll
        for (int e = 0; e < FF; ++e) f = f || acc[t][e] != 0.0;
      const unsigned m = __ballot_sync(0xffffffffu, f);
      posv[t] = base + __popc(m & ((1u << lane) - 1u));
      flag[t] = f;
      base += __popc(m);
    }
    const int cpc = cpad(base, F);
    double* rowv = cvals + static_cast<int64_t>(row) * c_row_len;
    if (lane < F && (base * F) % 2) rowv[lane * cpc + base * F] = 0.0;  // chunk pad
#pragma unroll
    for (int t = 0; t < NJ; ++t) {
      const int js = lane + 32 * t;
      if (flag[t]) {
        const int pos = posv[t];
        c_slots[static_cast<int64_t>(row) * S + pos] = static_cast<uint8_t>(js);
#pragma unroll
        for (int c = 0; c < F; ++c)
#pragma unroll
          for (int d = 0; d < F; ++d) rowv[c * cpc + pos * F + d] = acc[t][c * F + d];
      }
      if (js == (S - 1) / 2) {
        bool fr[F];
#pragma unroll
        for (int c = 0; c < F; ++c) {
          fr[c] = acc[t][c * F + c] > 0.0;
          c_freem[static_cast<int64_t>(I) * F + c] = fr[c] ? 1 : 0;
        }
        Mat<double, F> Mb;
#pragma unroll
        for (int c = 0; c < F; ++c)
#pragma unroll
          for (int d = 0; d < F; ++d) Mb(c, d) = (fr[c] && fr[d]) ? acc[t][c * F + d] : (c == d ? 1.0 : 0.0);
        const Mat<double, F> Mi = safe_block_inverse<F>(Mb);
#pragma unroll
        for (int e2 = 0; e2 < FF; ++e2) c_dinv[static_cast<int64_t>(row) * FF + e2] = Mi.e[e2];
      }
    }
    if (lane == 0) {
      c_nzb[row] = base;
      atomicAdd(nzb_total, static_cast<unsigned long long>(base));
    }
  }
}

// b_c = P^T r (masked to coarse free components)
template <int D, int F>
__global__ void k_restrict(GridC gf, GridC gc, const int* __restrict__ done, const double* __restrict__ rf,
                           const uint8_t* __restrict__ c_freem, double* __restrict__ bc) {
  if (done && *done) return;
  const int I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I >= gc.N) return;
  int ci[3];
  unflat<D>(gc, I, ci);
  double acc[F];
#pragma unroll
  for (int c = 0; c < F; ++c) acc[c] = 0.0;
  constexpr int NE = ipow_c(3, D);
  for (int e = 0; e < NE; ++e) {
    int r = e, fi = 0;
    bool ok = true;
    double w = 1.0;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      const int eo = (r % 3) - 1;
      r /= 3;
      const int ia = 2 * ci[a] + eo;
      ok = ok && ia >= 0 && ia < gf.nodes[a];
      fi += ia * gf.stride[a];
      w *= p1w(eo);
    }
    if (!ok) continue;
#pragma unroll
    for (int c = 0; c < F; ++c) acc[c] += w * rf[static_cast<int64_t>(fi) * F + c];
  }
#pragma unroll
  for (int c = 0; c < F; ++c) bc[static_cast<int64_t>(I) * F + c] = c_freem[static_cast<int64_t>(I) * F + c] ? acc[c] : 0.0;
}

// x_f += P x_c (masked to fine free components)
template <int D, int F>
__global__ void k_prolong_add(GridC gf, GridC gc, const int* __restrict__ done, const double* __restrict__ xc,
                              const uint8_t* __restrict__ f_freem, double* __restrict__ xf,
                              float* __restrict__ xf4 = nullptr) {
  if (done && *done) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= gf.N) return;
  int fi[3];
  unflat<D>(gf, i, fi);
  double acc[F];
#pragma unroll
  for (int c = 0; c < F; ++c) acc[c] = 0.0;
  constexpr int NC = ipow_c(2, D);
  for (int e = 0; e < NC; ++e) {
    int I = 0;
    double w = 1.0;
    bool ok = true;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const int bit = (e >> a) & 1;
      int Ia;
      if (fi[a] % 2 == 0) {
        if (bit) { ok = false; Ia = 0; } else { Ia = fi[a] / 2; }
      } else {
        Ia = (fi[a] - 1) / 2 + bit;
        w *= 0.5;
      }
      ok = ok && Ia >= 0 && Ia < gc.nodes[a];
      I += Ia * gc.stride[a];
    }
    if (!ok) continue;
#pragma unroll
    for (int c = 0; c < F; ++c) acc[c] += w * xc[static_cast<int64_t>(I) * F + c];
  }
#pragma unroll
  for (int c = 0; c < F; ++c)
    if (f_freem[static_cast<int64_t>(i) * F + c]) {
      const double v = xf[static_cast<int64_t>(i) * F + c] + acc[c];
      xf[static_cast<int64_t>(i) * F + c] = v;
      if (F <= 4 && xf4) xf4[static_cast<int64_t>(i) * 4 + c] = static_cast<float>(v);
    }
}

__global__ void k_fill_free(int64_t n, const uint8_t* __restrict__ freem, double* __restrict__ v) {
  const int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i < n) v[i] = freem[i] ? 1.0 : 0.0;
}

// power-iteration step: lam = |t| / |v|, v = t / |t|  (sums = {t.t, v.v})
__global__ void k_power_step(int64_t n, const double* __restrict__ sums, const double* __restrict__ t,
                             double* __restrict__ v, double* __restrict__ lam) {
  const double tt = sums[0], vv = sums[1];
  const double inv = tt > 0.0 ? rsqrt(tt) : 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    v[i] = t[i] * inv;
  if (blockIdx.x == 0 && threadIdx.x == 0) *lam = vv > 0.0 ? sqrt(tt / vv) : 1.0;
}

// first smoothing sweep from x = 0: x = omega Dinv b (masked)
template <int F>
__global__ void k_jacobi0(int n_act, const int* __restrict__ done, const int* __restrict__ act_list,
                          const double* __restrict__ dinv, const uint8_t* __restrict__ freem, double omega,
                          const double* __restrict__ b, double* __restrict__ x, float* __restrict__ x4 = nullptr) {
  if (done && *done) return;
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < n_act; row += gridDim.x * blockDim.x) {
    const int64_t node = act_list[row];
    const int64_t base = node * F;
#pragma unroll
    for (int c = 0; c < F; ++c) {
      double s = 0.0;
#pragma unroll
      for (int d = 0; d < F; ++d) s += dinv[static_cast<int64_t>(row) * F * F + c * F + d] * b[base + d];
      const double v = freem[base + c] ? omega * s : 0.0;
      x[base + c] = v;
      if (F <= 4 && x4) x4[node * 4 + c] = static_cast<float>(v);
    }
  }
}

// coarsest level: x = Ainv b with a dense inverse over (active row, component)
__global__ void k_dense_apply(int n, int F, const int* __restrict__ done, const int* __restrict__ act_list,
                              const double* __restrict__ Ainv, const double* __restrict__ b, double* __restrict__ x) {
  if (done && *done) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) s += Ainv[static_cast<int64_t>(i) * n + j] * b[static_cast<int64_t>(act_list[j / F]) * F + j % F];
    x[static_cast<int64_t>(act_list[i / F]) * F + i % F] = s;
  }
}

// CG (MG-preconditioned) step part 1: alpha from p.q; x += a p; r -= a q;
// partial r.r into row 1 of `partials`.
template <int F>
__global__ void k_cg_update_mg(int N, const int* __restrict__ act_idx, double* __restrict__ sc, int* __restrict__ done,
                               int par, const double* __restrict__ pq_part, int nb, double* __restrict__ x,
                               double* __restrict__ r, const double* __restrict__ p, const double* __restrict__ q,
                               double* __restrict__ partials_rr) {
  double v[1] = {0.0};
  const int was_done = *done;
  double pq[1];
  block_reduce_partials<1>(pq_part, nb, pq);
  if (!was_done) {
    const double rz = sc[par ? kBeta : kRz];
    if (!(pq[0] > 0.0)) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        sc[kDone] = 2.0;
        *done = 2;
      }
    } else {
      const double alpha = rz / pq[0];
      for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
        if (act_idx[n] < 0) continue;
#pragma unroll
        for (int c = 0; c < F; ++c) {
          x[n * F + c] += alpha * p[n * F + c];
          const double rl = r[n * F + c] - alpha * q[n * F + c];
          r[n * F + c] = rl;
          v[0] += rl * rl;
        }
      }
    }
  }
  block_sum_store<1>(v, partials_rr);
}

// partial a.b over grid vectors (row 0 of `partials`)
__global__ void k_dot1(int64_t n, const int* __restrict__ done, const double* __restrict__ a,
                       const double* __restrict__ b, double* __restrict__ partials) {
  double v[1] = {0.0};
  if (!(done && *done))
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
      v[0] += a[i] * b[i];
  block_sum_store<1>(v, partials);
}

// --------------------------------------------------------------- K9 G2P --
template <int D, int SHAPE, bool NHO>
#ifndef IMPM_COMMIT_MINB
#define IMPM_COMMIT_MINB 4  // resident 256-thread CTAs per SM (64 registers): 1.16 vs 1.26 ms per cfg 4 commit
#endif
__global__ void __launch_bounds__(256, IMPM_COMMIT_MINB) k_commit(GridC g, double* __restrict__ pd, int64_t cap, int P, const double* __restrict__ xs,
                         const int* __restrict__ key, const int* __restrict__ sup, const int* __restrict__ orig,
                         const double* __restrict__ u, MatParams mp, int tl, DevStatus* st) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int first[3], cnt[3];
  AxisW aw[3];
  particle_weights<D, SHAPE>(g, pd, cap, xs, p, key[p], sup[p], first, cnt, aw);
  double du[3] = {0.0, 0.0, 0.0};
  Mat<double, D> G = Mat<double, D>::zero();
  for_each_support<D>(g, first, cnt, aw, [&](int node, double W, const double* grad) {
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double uv = u[node * D + c];
      du[c] += W * uv;
#pragma unroll
      for (int a = 0; a < D; ++a) G(c, a) += uv * grad[a];
    }
  });
  Mat<double, D> f_inc = G;
#pragma unroll
  for (int a = 0; a < D; ++a) f_inc(a, a) += 1.0;
  if (!(det(f_inc) > 0.0)) {  // mpm_solver.hpp:377-379
    atomicMin(&st->err_domain, orig[p]);
    return;
  }
  Mat<double, D> F_new;
  if (tl) {
    F_new = f_inc;
  } else {
    Mat<double, D> Fn;
#pragma unroll
    for (int i = 0; i < D * D; ++i) Fn.e[i] = pd[(PF<D>::F + i) * cap + p];
    F_new = matmul(f_inc, Fn);
  }
  double Be_n[10], Be_new[9], dg = 0.0;
  if (has_history(mp.kind))
#pragma unroll
    for (int i = 0; i < 9; ++i) Be_n[i] = pd[(PF<D>::Be + i) * cap + p];
  if (mp.kind == kCamClay) Be_n[9] = pd[PF<D>::alpha * cap + p];
  const StressOut<double> su = update_stress<double, D, NHO>(mp, F_new, f_inc, Be_n, Be_new, &dg);
#pragma unroll
  for (int a = 0; a < D; ++a) {
    if (tl)
      pd[(PF<D>::x + a) * cap + p] = pd[(PF<D>::X + a) * cap + p] + du[a];
    else
      pd[(PF<D>::x + a) * cap + p] += du[a];
  }
#pragma unroll
  for (int i = 0; i < D * D; ++i) pd[(PF<D>::F + i) * cap + p] = F_new.e[i];
  pd[PF<D>::V * cap + p] = su.J * pd[PF<D>::V0 * cap + p];
#pragma unroll
  for (int i = 0; i < 9; ++i) pd[(PF<D>::sigma + i) * cap + p] = su.sigma.e[i];
  if (has_history(mp.kind)) {
#pragma unroll
    for (int i = 0; i < 9; ++i) pd[(PF<D>::Be + i) * cap + p] = Be_new[i];
    pd[PF<D>::alpha * cap + p] += dg;
  }
  if (!tl) {  // update_particle_domain (gimp.hpp:65-77)
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double lp = pd[(PF<D>::lp0 + a) * cap + p] * F_new(a, a);
      if (!(lp > 0.0) || lp >= 0.5 * g.h) atomicMin(&st->err_lp, orig[p]);
      pd[(PF<D>::lp + a) * cap + p] = lp;
    }
  }
}


// ================================================= coupled u-p (2D / 3D) ==
// CoupledSim (porous.hpp:48-186, src/porous.cpp:25-168): small-strain u-p on
// weights frozen at the reference configuration, 3 fields per node (ux, uy,
// p), F = 3 blocks. Grid vectors are [node][3].
struct PoroC {
  double lam, mu, mob, rho_f, g0, g1, g2;
};

// coupled u-p (porous.hpp:127-186) for D = 2 (the reference) and D = 3
// (extension, parity unpinned): fields (u_0 .. u_{D-1}, p) per node, F = D + 1.
// Particle record of phase A: Q = {V0 sigma'(c,b) (D*D), V0 p_w, V0 tr G, V0 mob grad p (D)}
template <int D>
struct UpQ {
  static constexpr int F = D + 1, DD = D * D, N = DD + 2 + D;
};

__host__ __device__ __forceinline__ double poro_g(const PoroC& pc, int a) { return a == 0 ? pc.g0 : (a == 1 ? pc.g1 : pc.g2); }

// residual phase A (per particle)
template <int D, int SHAPE>
__global__ void k_up_particles(GridC g, const double* __restrict__ pd, int64_t cap, int P,
                               const double* __restrict__ xs, const int* __restrict__ key,
                               const int* __restrict__ sup, const int* __restrict__ orig,
                               const double* __restrict__ x, PoroC pc, double* __restrict__ Q,
                               DevStatus* st) {
  constexpr int F = UpQ<D>::F, DD = UpQ<D>::DD, QN = UpQ<D>::N;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int first[3], cnt[3];
  AxisW aw[3];
  particle_weights<D, SHAPE>(g, pd, cap, xs, p, key[p], sup[p], first, cnt, aw);
  Mat<double, D> G = Mat<double, D>::zero();
  double pw = 0.0, gp[3] = {0.0, 0.0, 0.0};
  for_each_support<D>(g, first, cnt, aw, [&](int node, double W, const double* grad) {
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double uc = x[node * F + c];
#pragma unroll
      for (int a = 0; a < D; ++a) G(c, a) += uc * grad[a];
    }
    const double pv = x[node * F + D];
    pw += W * pv;
#pragma unroll
    for (int a = 0; a < D; ++a) gp[a] += pv * grad[a];
  });
  Mat<double, D> f_inc = G;
#pragma unroll
  for (int a = 0; a < D; ++a) f_inc(a, a) += 1.0;
  Mat<double, D> Fn;
#pragma unroll
  for (int i = 0; i < DD; ++i) Fn.e[i] = pd[(PF<D>::F + i) * cap + p];
  const Mat<double, D> F_new = matmul(f_inc, Fn);
  double* q = Q + static_cast<int64_t>(p) * QN;
  if (!(det(F_new) > 0.0)) {  // porous.hpp:159-160
    atomicMin(&st->err_domain, orig[p]);
#pragma unroll
    for (int i = 0; i < QN; ++i) q[i] = 0.0;
    return;
  }
  const StressOut<double> su = neo_hookean_update<double, D>(F_new, pc.lam, pc.mu);
  const double V0 = pd[PF<D>::V0 * cap + p];
#pragma unroll
  for (int c = 0; c < D; ++c)
#pragma unroll
    for (int b = 0; b < D; ++b) q[c * D + b] = V0 * su.sigma(c, b);
  q[DD] = V0 * pw;
  double trg = G(0, 0);
#pragma unroll
  for (int a = 1; a < D; ++a) trg += G(a, a);
  q[DD + 1] = V0 * trg;
#pragma unroll
  for (int a = 0; a < D; ++a) q[DD + 2 + a] = V0 * (pc.mob * gp[a]);
}

// residual phase B (nodes), porous.hpp:165-184 (masked, + partial r.r)
template <int D, int SHAPE>
__global__ void k_up_nodes(GridC g, const double* __restrict__ pd, int64_t cap, const double* __restrict__ xs,
                           const int* __restrict__ bin_start, const int* __restrict__ sup,
                           const double* __restrict__ Q, const double* __restrict__ bext,
                           const int* __restrict__ act_flag, const uint8_t* __restrict__ freem, PoroC pc, double dt,
                           double* __restrict__ r, double* __restrict__ partials) {
  constexpr int F = UpQ<D>::F, DD = UpQ<D>::DD, QN = UpQ<D>::N;
  double rr[1] = {0.0};
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < g.N; n += gridDim.x * blockDim.x) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (act_flag[n]) {
      int idx[3];
      unflat<D>(g, n, idx);
      for_each_particle_of_node<D>(g, idx, bin_start, sup, [&](int p, const int*) {
        double w[3], dw[3];
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const WeightValue wv = weight_1d<SHAPE>(xs[a * cap + p] - node_coord(g, a, idx[a]),
                                                  pd[(PF<D>::lp + a) * cap + p], g.h);
          w[a] = wv.w;
          dw[a] = wv.dw;
        }
        double W, gr[3];
        tensor_weight<D>(w, dw, W, gr);
        const double* q = Q + static_cast<int64_t>(p) * QN;
#pragma unroll
        for (int c = 0; c < D; ++c) {
          double fint = gr[0] * q[c * D];
#pragma unroll
          for (int b = 1; b < D; ++b) fint += gr[b] * q[c * D + b];
          fint -= gr[c] * q[DD];
          acc[c] += fint - W * bext[c * cap + p];
        }
        const double V0 = pd[PF<D>::V0 * cap + p];
        double fl = gr[0] * q[DD + 2], gg = gr[0] * pc.g0;
#pragma unroll
        for (int a = 1; a < D; ++a) {
          fl += gr[a] * q[DD + 2 + a];
          gg += gr[a] * poro_g(pc, a);
        }
        const double flux = fl - V0 * pc.mob * pc.rho_f * gg;
        acc[D] += W * q[DD + 1] + dt * flux;
      });
    }
#pragma unroll
    for (int c = 0; c < F; ++c) {
      const double v = freem[static_cast<int64_t>(n) * F + c] ? acc[c] : 0.0;
      r[static_cast<int64_t>(n) * F + c] = v;
      rr[0] += v * v;
    }
  }
  block_sum_store<1>(rr, partials);
}

// dP/dG with P = V0 sigma'(f_inc F_n) (the u-p internal force uses reference
// gradients and V0, porous.hpp:171-173); duals over the D*D entries of G.
template <int D, int SHAPE>
__global__ void k_up_tangent(GridC g, const double* __restrict__ pd, int64_t cap, int P,
                             const double* __restrict__ xs, const int* __restrict__ key,
                             const int* __restrict__ sup, const double* __restrict__ x, PoroC pc,
                             double* __restrict__ A) {
  constexpr int F = UpQ<D>::F, DD = UpQ<D>::DD;
  using T = Dual<DD>;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int first[3], cnt[3];
  AxisW aw[3];
  particle_weights<D, SHAPE>(g, pd, cap, xs, p, key[p], sup[p], first, cnt, aw);
  Mat<double, D> G = Mat<double, D>::zero();
  for_each_support<D>(g, first, cnt, aw, [&](int node, double, const double* grad) {
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double uc = x[node * F + c];
#pragma unroll
      for (int a = 0; a < D; ++a) G(c, a) += uc * grad[a];
    }
  });
  Mat<T, D> f_inc;
#pragma unroll
  for (int i = 0; i < DD; ++i) {
    f_inc.e[i] = T(G.e[i]);
    f_inc.e[i].d[i] = 1.0;
  }
#pragma unroll
  for (int a = 0; a < D; ++a) f_inc(a, a) += 1.0;
  Mat<T, D> FnT;
#pragma unroll
  for (int i = 0; i < DD; ++i) FnT.e[i] = T(pd[(PF<D>::F + i) * cap + p]);
  const Mat<T, D> F_new = matmul(f_inc, FnT);
  double* out = A + static_cast<int64_t>(p) * DD * DD;
  if (!(value_of(det(F_new)) > 0.0)) {
#pragma unroll
    for (int i = 0; i < DD * DD; ++i) out[i] = 0.0;
    return;
  }
  const StressOut<T> su = neo_hookean_update<T, D>(F_new, T(pc.lam), T(pc.mu));
  const double V0 = pd[PF<D>::V0 * cap + p];
#pragma unroll
  for (int c = 0; c < D; ++c)
#pragma unroll
    for (int b = 0; b < D; ++b)
#pragma unroll
      for (int j = 0; j < DD; ++j) out[(c * D + b) * DD + j] = V0 * su.sigma(c, b).d[j];
}

// colour-batched bin-centric assembly of the F x F u-p blocks:
//   uu(c,d) = sum_f H_k[c][d][f] g^l_f,   up(c) = -V0 g^k_c w^l,
//   pu(d)   = V0 w^k g^l_d,               pp    = V0 dt mob g^k . g^l
// one writer per block per colour launch: fire-and-forget RED adds
template <int D, int SHAPE, int PPL, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) k_up_assemble_bins(
    GridC g, const double* __restrict__ pd, int64_t cap, const double* __restrict__ xs,
    const int* __restrict__ bin_start, const uint8_t* __restrict__ bflag, const double* __restrict__ A,
    const int* __restrict__ act_idx, const unsigned* __restrict__ row_mask, const int* __restrict__ row_nzb,
    double* __restrict__ vals, int64_t row_len, double dtmob, int c0, int c1, int c2, int nb0, int nb1, int nb2) {
  constexpr int F = UpQ<D>::F, DD = UpQ<D>::DD, D3 = DD * D, NK = ipow_c(3, D), FF = F * F;
  __shared__ double W1s[WARPS][3][3], DW1s[WARPS][3][3];
  __shared__ double Gs[WARPS][NK][4];
  __shared__ double Hs[WARPS][NK * D3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbins = nb0 * nb1 * nb2;
  const int col[3] = {c0, c1, c2};
  const int nbv[3] = {nb0, nb1, nb2};
  for (int bi = blockIdx.x * WARPS + warp; bi < nbins; bi += gridDim.x * WARPS) {
    int bidx[3] = {0, 0, 0}, rr = bi, b = 0;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      bidx[a] = 3 * (rr % nbv[a]) + col[a];
      rr /= nbv[a];
      b += bidx[a] * g.stride[a];
    }
    const int fl = bflag[b];
    if (!(fl & 0x80)) continue;
    int cn[3] = {1, 1, 1};
#pragma unroll
    for (int a = 0; a < D; ++a) cn[a] = 2 + ((fl >> a) & 1);
    const int nk = cn[0] * cn[1] * cn[2];
    const int npairs = nk * nk;
    const int p0 = bin_start[b], p1 = bin_start[b + 1];
    for (int q0 = 0; q0 < npairs; q0 += 32 * PPL) {
      double acc[PPL][FF];
#pragma unroll
      for (int t = 0; t < PPL; ++t)
#pragma unroll
        for (int e = 0; e < FF; ++e) acc[t][e] = 0.0;
      for (int p = p0; p < p1; ++p) {
        if (lane < 3 * D) {
          const int a = lane / 3, i = lane % 3;
          double w = 0.0, dw = 0.0;
          if (i < cn[a]) {
            const WeightValue wv = weight_1d<SHAPE>(xs[a * cap + p] - node_coord(g, a, bidx[a] + i),
                                                    pd[(PF<D>::lp + a) * cap + p], g.h);
            w = wv.w;
            dw = wv.dw;
          }
          W1s[warp][a][i] = w;
          DW1s[warp][a][i] = dw;
        }
        __syncwarp();
        if (lane < nk) {
          int li[3] = {0, 0, 0}, rk = lane;
#pragma unroll
          for (int a = D - 1; a >= 0; --a) {
            li[a] = rk % cn[a];
            rk /= cn[a];
          }
          double w[3], dw[3];
#pragma unroll
          for (int a = 0; a < D; ++a) {
            w[a] = W1s[warp][a][li[a]];
            dw[a] = DW1s[warp][a][li[a]];
          }
          double W, gk[3];
          tensor_weight<D>(w, dw, W, gk);
#pragma unroll
          for (int a = 0; a < D; ++a) Gs[warp][lane][a] = gk[a];
          Gs[warp][lane][3] = W;
        }
        __syncwarp();
        const double* Ap = A + static_cast<int64_t>(p) * DD * DD;
        for (int e = lane; e < nk * D3; e += 32) {
          const int k = e / D3, cdf = e - k * D3, c = cdf / DD, df = cdf - c * DD;
          double h = Gs[warp][k][0] * __ldg(Ap + (c * D + 0) * DD + df);
#pragma unroll
          for (int bb = 1; bb < D; ++bb) h += Gs[warp][k][bb] * __ldg(Ap + (c * D + bb) * DD + df);
          Hs[warp][e] = h;
        }
        __syncwarp();
        const double V0 = pd[PF<D>::V0 * cap + p];
#pragma unroll
        for (int t = 0; t < PPL; ++t) {
          const int q = q0 + lane + 32 * t;
          if (q < npairs) {
            const int k = q / nk, l = q - k * nk;
            const double* Hk = &Hs[warp][k * D3];
            double gl[3], gk[3];
#pragma unroll
            for (int a = 0; a < D; ++a) {
              gl[a] = Gs[warp][l][a];
              gk[a] = Gs[warp][k][a];
            }
            const double wl = Gs[warp][l][3], wk = Gs[warp][k][3];
#pragma unroll
            for (int c = 0; c < D; ++c)
#pragma unroll
              for (int d = 0; d < D; ++d) {
                double sacc = Hk[(c * D + d) * D] * gl[0];
#pragma unroll
                for (int f = 1; f < D; ++f) sacc += Hk[(c * D + d) * D + f] * gl[f];
                acc[t][c * F + d] += sacc;
              }
#pragma unroll
            for (int c = 0; c < D; ++c) acc[t][c * F + D] += -V0 * gk[c] * wl;
#pragma unroll
            for (int d = 0; d < D; ++d) acc[t][D * F + d] += V0 * wk * gl[d];
            double gg = gk[0] * gl[0];
#pragma unroll
            for (int a = 1; a < D; ++a) gg += gk[a] * gl[a];
            acc[t][D * F + D] += V0 * dtmob * gg;
          }
        }
        __syncwarp();
      }
#pragma unroll
      for (int t = 0; t < PPL; ++t) {
        const int q = q0 + lane + 32 * t;
        if (q >= npairs) continue;
        const int k = q / nk, l = q - k * nk;
        int lk[3] = {0, 0, 0}, ll[3] = {0, 0, 0}, rk = k, rl = l, node = 0, sl = 0;
#pragma unroll
        for (int a = D - 1; a >= 0; --a) {
          lk[a] = rk % cn[a];
          rk /= cn[a];
          ll[a] = rl % cn[a];
          rl /= cn[a];
        }
#pragma unroll
        for (int a = 0; a < D; ++a) {
          node += (bidx[a] + lk[a]) * g.stride[a];
          sl = sl * 5 + (ll[a] - lk[a] + 2);
        }
        const int row = act_idx[node];
        if (row < 0) continue;
        const unsigned* m = row_mask + static_cast<int64_t>(row) * 4;
        const int pos = mask_pos(m, sl);
        const int cp = cpad(row_nzb[row], F);
        double* rv = vals + static_cast<int64_t>(row) * row_len + pos * F;
#pragma unroll
        for (int c = 0; c < F; ++c)
#pragma unroll
          for (int d = 0; d < F; ++d) atomicAdd(rv + c * cp + d, acc[t][c * F + d]);
      }
    }
  }
}

// commit (src/porous.cpp:139-151): F, V, sigma, accumulated vertical
// (last-axis) displacement
template <int D, int SHAPE>
__global__ void k_up_commit(GridC g, double* __restrict__ pd, int64_t cap, int P, const double* __restrict__ xs,
                            const int* __restrict__ key, const int* __restrict__ sup, const double* __restrict__ x,
                            PoroC pc, double* __restrict__ uty) {
  constexpr int F = UpQ<D>::F, DD = UpQ<D>::DD;
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  int first[3], cnt[3];
  AxisW aw[3];
  particle_weights<D, SHAPE>(g, pd, cap, xs, p, key[p], sup[p], first, cnt, aw);
  Mat<double, D> G = Mat<double, D>::zero();
  double duy = 0.0;
  for_each_support<D>(g, first, cnt, aw, [&](int node, double W, const double* grad) {
#pragma unroll
    for (int c = 0; c < D; ++c) {
      const double uv = x[node * F + c];
      if (c == D - 1) duy += W * uv;
#pragma unroll
      for (int a = 0; a < D; ++a) G(c, a) += uv * grad[a];
    }
  });
  Mat<double, D> f_inc = G;
#pragma unroll
  for (int a = 0; a < D; ++a) f_inc(a, a) += 1.0;
  Mat<double, D> Fn;
#pragma unroll
  for (int i = 0; i < DD; ++i) Fn.e[i] = pd[(PF<D>::F + i) * cap + p];
  const Mat<double, D> Fm = matmul(f_inc, Fn);
#pragma unroll
  for (int i = 0; i < DD; ++i) pd[(PF<D>::F + i) * cap + p] = Fm.e[i];
  pd[PF<D>::V * cap + p] = det(Fm) * pd[PF<D>::V0 * cap + p];
  const StressOut<double> su = neo_hookean_update<double, D>(Fm, pc.lam, pc.mu);
#pragma unroll
  for (int i = 0; i < 9; ++i) pd[(PF<D>::sigma + i) * cap + p] = su.sigma.e[i];
  uty[p] += duy;
}

// dst[n] field f of a grid vector (only where free), other entries untouched
__global__ void k_copy_field(int N, int F, int f, const uint8_t* __restrict__ freem, const double* __restrict__ src,
                             double* __restrict__ dst) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n < N && freem[static_cast<int64_t>(n) * F + f]) dst[static_cast<int64_t>(n) * F + f] = src[static_cast<int64_t>(n) * F + f];
}

// per-particle accumulator in ORIGINAL order
__global__ void k_gather_orig(const double* __restrict__ v, const int* __restrict__ orig, int n, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[orig[i]] = v[i];
}

// -------------------------------------------------- parity taps / export --
// dof vector <-> grid vector
__global__ void k_dof_to_grid(int n, const double* __restrict__ v, const int* __restrict__ node_of,
                              const int* __restrict__ field_of, int F, double* __restrict__ gvec) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d < n) gvec[static_cast<int64_t>(node_of[d]) * F + field_of[d]] = v[d];
}
__global__ void k_grid_to_dof(int n, const double* __restrict__ gvec, const int* __restrict__ node_of,
                              const int* __restrict__ field_of, int F, double* __restrict__ v) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d < n) v[d] = gvec[static_cast<int64_t>(node_of[d]) * F + field_of[d]];
}

// reference CSR pattern row lengths: free DOFs in the +-2 node box (jacobian.hpp:38-63)
template <int D>
__device__ __forceinline__ int box_slot_node(const GridC& g, const int* kidx, int s, int& nb) {
  int rs = s;
  nb = 0;
  bool ok = true;
  int rel[3];
#pragma unroll
  for (int a = D - 1; a >= 0; --a) {
    rel[a] = rs % 5 - 2;
    rs /= 5;
  }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const int ia = kidx[a] + rel[a];
    ok = ok && ia >= 0 && ia < g.nodes[a];
    nb += ia * g.stride[a];
  }
  return ok;
}

template <int D, int F>
__global__ void k_csr_count(GridC g, int n, const int* __restrict__ node_of, const int* __restrict__ dof_of,
                            int64_t* __restrict__ rowlen) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  constexpr int S = ipow_c(5, D);
  int kidx[3];
  unflat<D>(g, node_of[d], kidx);
  int64_t c = 0;
  for (int s = 0; s < S; ++s) {
    int nb;
    if (!box_slot_node<D>(g, kidx, s, nb)) continue;
    for (int f = 0; f < F; ++f) c += dof_of[nb * F + f] >= 0;
  }
  rowlen[d] = c;
}

template <int D, int F>
__global__ void k_csr_fill(GridC g, int n, const int* __restrict__ node_of, const int* __restrict__ field_of,
                           const int* __restrict__ dof_of, const int* __restrict__ act_idx,
                           const double* __restrict__ vals, int64_t row_len, const uint8_t* __restrict__ row_slots,
                           const int* __restrict__ row_nzb, const int64_t* __restrict__ row_ptr,
                           int* __restrict__ cols, double* __restrict__ out) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  constexpr int S = ipow_c(5, D);
  const int k = node_of[d], c = field_of[d];
  int kidx[3];
  unflat<D>(g, k, kidx);
  const int64_t row = act_idx[k];
  int64_t o = row_ptr[d];
  const int nzb = row_nzb[row];
  int pos = 0;
  for (int s = 0; s < S; ++s) {
    int nb;
    while (pos < nzb && row_slots[row * S + pos] < s) ++pos;
    const bool stored = pos < nzb && row_slots[row * S + pos] == s;
    if (!box_slot_node<D>(g, kidx, s, nb)) continue;
    for (int f = 0; f < F; ++f) {
      const int col = dof_of[nb * F + f];
      if (col < 0) continue;
      cols[o] = col;
      if (out) out[o] = stored ? vals[row * row_len + c * cpad(nzb, F) + pos * F + f] : 0.0;
      ++o;
    }
  }
}

// p2g_map (mpm_solver.hpp:142-152), pull form
template <int D, int SHAPE>
__global__ void k_p2g_map(GridC g, const double* __restrict__ pd, int64_t cap, const double* __restrict__ xs,
                          const int* __restrict__ bin_start, const int* __restrict__ sup,
                          const double* __restrict__ mass, const double* __restrict__ f, double* __restrict__ out) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= g.N) return;
  int idx[3];
  unflat<D>(g, n, idx);
  double acc = 0.0;
  for_each_particle_of_node<D>(g, idx, bin_start, sup, [&](int p, const int*) {
    double w[3], dw[3];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const WeightValue wv = weight_1d<SHAPE>(xs[a * cap + p] - node_coord(g, a, idx[a]),
                                              pd[(PF<D>::lp + a) * cap + p], g.h);
      w[a] = wv.w;
      dw[a] = wv.dw;
    }
    double W, grad[3];
    tensor_weight<D>(w, dw, W, grad);
    acc += W * pd[PF<D>::m * cap + p] * f[p];
  });
  out[n] = mass[n] > 0.0 ? acc / mass[n] : acc;
}

// ------------------------------------------------------------ scans (int) --
// exclusive scan, 1024 threads x 4 items per block, then block sums
template <class T>
__global__ void k_scan_block(const int* __restrict__ in, int64_t n, T* __restrict__ out, T* __restrict__ block_sums) {
  __shared__ T s[1024];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * 4096 + threadIdx.x * 4;
  T v[4];
  T t = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[i] = base + i < n ? static_cast<T>(in[base + i]) : 0;
    t += v[i];
  }
  s[threadIdx.x] = t;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    T add = threadIdx.x >= off ? s[threadIdx.x - off] : 0;
    __syncthreads();
    s[threadIdx.x] += add;
    __syncthreads();
  }
  T run = s[threadIdx.x] - t;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (threadIdx.x == 1023) block_sums[blockIdx.x] = s[1023];
}

template <class T>
__global__ void k_scan_sums(T* __restrict__ sums, int nb, T* __restrict__ total) {
  // single block, sequential per thread chunk (nb is small: n / 4096)
  __shared__ T s[1024];
  const int per = (nb + 1023) / 1024;
  const int lo = threadIdx.x * per, hi = min(nb, lo + per);
  T t = 0;
  for (int i = lo; i < hi; ++i) t += sums[i];
  s[threadIdx.x] = t;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    T add = threadIdx.x >= off ? s[threadIdx.x - off] : 0;
    __syncthreads();
    s[threadIdx.x] += add;
    __syncthreads();
  }
  T run = s[threadIdx.x] - t;
  for (int i = lo; i < hi; ++i) {
    const T v = sums[i];
    sums[i] = run;
    run += v;
  }
  if (threadIdx.x == 1023) *total = s[1023];
}

template <class T>
__global__ void k_scan_add(T* __restrict__ out, int64_t n, const T* __restrict__ sums, const T* __restrict__ total,
                           T* __restrict__ out_total_slot) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] += sums[i / 4096];
  if (i == 0 && out_total_slot) *out_total_slot = *total;
}

// ------------------------------------------------- slab decomposition (§8e) --
// Nodes outside the owned axis-0 range [own_lo, own_hi) are neither rows nor
// DOFs of this rank: their activity and freedom belong to the owner.
__global__ void k_mask_owned(int N, int F, int stride0, int own_lo, int own_hi, int* __restrict__ act_flag,
                             int* __restrict__ free_flag) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  const int i0 = n / stride0;
  if (i0 >= own_lo && i0 < own_hi) return;
  act_flag[n] = 0;
  for (int c = 0; c < F; ++c) free_flag[n * F + c] = 0;
}

// Destinations of every particle this rank OWNED during the step (first
// support node along axis 0 in [own_lo, own_hi) at begin_step) from its
// committed position: rank r keeps f in [A-2, B); r-1 needs f < A; r+1 needs
// f >= B-2 (f = new global first support node). Ghost copies are dropped.
template <int D, int SHAPE>
__global__ void k_migrate_flags(const double* __restrict__ pd, int64_t cap, int P, GridC g,
                                const int* __restrict__ key, int use_X, int own_lo, int own_hi, int A, int B,
                                int has_left, int has_right, int lo_ok, int hi_ok, const int* __restrict__ orig,
                                int* __restrict__ fk, int* __restrict__ fl, int* __restrict__ fr, DevStatus* st) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  const int f0 = key[i] / g.stride[0];
  int k = 0, l = 0, r = 0;
  if (f0 >= own_lo && f0 < own_hi) {
    const double x = pd[((use_X ? PF<D>::X : PF<D>::x) + 0) * cap + i];
    const double lp = pd[(PF<D>::lp + 0) * cap + i];
    int first, count;
    if constexpr (SHAPE == 2) {
      const double lo = __dsub_rn(__dsub_rn(x, g.origin[0]), 1.5 * g.h);
      first = static_cast<int>(floor(__ddiv_rn(lo, g.h))) + 1;
    } else {
      gimp_support_1d(x, lp, g.origin[0], g.h, first, count);
    }
    k = (!has_left || first >= A - 2) && (!has_right || first < B);
    l = has_left && first < A;
    r = has_right && first >= B - 2;
    if (first < lo_ok || first >= hi_ok) atomicMin(&st->err_migrate, orig[i]);
  }
  fk[i] = k;
  fl[i] = l;
  fr[i] = r;
}

// record = nd particle doubles + the global id (exact in fp64)
__global__ void k_pack_records(const double* __restrict__ pd, int64_t cap, int P, int nd,
                               const int* __restrict__ orig, const int* __restrict__ flag,
                               const int* __restrict__ pos, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P || !flag[i]) return;
  const int64_t o = static_cast<int64_t>(pos[i]) * (nd + 1);
  for (int f = 0; f < nd; ++f) out[o + f] = pd[f * cap + i];
  out[o + nd] = static_cast<double>(orig[i]);
}

__global__ void k_unpack_records(const double* __restrict__ in, int n, int nd, double* __restrict__ pd,
                                 int64_t cap, int off, int* __restrict__ orig) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t o = static_cast<int64_t>(j) * (nd + 1);
  for (int f = 0; f < nd; ++f) pd[f * cap + off + j] = in[o + f];
  orig[off + j] = static_cast<int>(in[o + nd]);
}

// stable compaction of the kept particles into the new SoA block at `off`
__global__ void k_keep_gather(const double* __restrict__ pd, int64_t cap, int P, int nd,
                              const int* __restrict__ orig, const int* __restrict__ flag,
                              const int* __restrict__ pos, double* __restrict__ pd_new, int64_t cap_new, int off,
                              int* __restrict__ orig_new) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P || !flag[i]) return;
  const int j = off + pos[i];
  for (int f = 0; f < nd; ++f) pd_new[f * cap_new + j] = pd[f * cap + i];
  orig_new[j] = orig[i];
}

// local particles -> AoS in local (sorted) order + their global ids
__global__ void k_soa_to_aos_ids(const double* __restrict__ soa, int64_t cap, int n, int nd,
                                 const int* __restrict__ orig, double* __restrict__ aos, int64_t stride_dbl,
                                 long long* __restrict__ ids) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int f = 0; f < nd; ++f) aos[static_cast<int64_t>(i) * stride_dbl + f] = soa[f * cap + i];
  ids[i] = orig[i];
}

}  // namespace impm_gpu
