// K6 Jacobian assembly, owner-computes z-sweep (3D, single field).
//
// Replaces the colour-batched bin kernel (k_assemble_bins_staged), whose 27
// colour launches read-modify-wrote every stored block up to 27 times through
// L2 reductions (RED.F64 issue-bound, ~8x the algorithmic DRAM traffic).
// Same result as JacobianAssembler::sparse (jacobian.hpp:95-137) on the
// reference pattern; the element stiffness of particle p is
//   K_ab += sum_f H_a^p[c][d][f] g_b^p[f],  H_a^p[c][d][f] = sum_e g_a^p[e] A_p[(c,e),(d,f)],
// A_p = dP_ce/dG_df from k_tangent (dual numbers over the residual's graph).
//
// Decomposition. A CTA owns a 2x2 tile of grid-node COLUMNS (x, y) and sweeps
// z upward. Bins are keyed by the first support node (k_support), so the
// particles of layer kz touch rows at levels kz .. kz+2 only; the CTA keeps
// those three row levels of its four columns as dense fp64 accumulators in
// shared memory (a ring of 3 levels x 125 slots x 9 values per column). After
// layer kz every row at level kz is complete and is written to the BSR exactly
// once (stored slots only, coalesced), then its ring level is reused for
// kz+3. No atomics, no colour launches, no zero pass.
//
// Work. Inside a bin particles are sorted by support signature (k_bin_sort),
// so each run of equal (bin, signature) -- a "group", <= kGMax particles -- has
// one exact support box: per particle the work is s_p^2 block products (not
// the bin box^2; on cfg 4 that halves it). The layer's particles (the 16 bins
// that reach the tile) are staged in chunks of kChunk: A_p and the 1D weights.
// Warp w owns column w of the tile. Its units are (group, row level) pairs
// whose box holds the column; a unit has one task per (x, y) node column of
// the group box, and a task accumulates the z-run of <= 3 blocks in registers
// over the group's particles. H_a^p is formed once per (unit, particle) in a
// per-warp scratch and broadcast to the unit's tasks. Rows are flushed into
// the ring unit by unit (tasks of one unit own disjoint blocks): every value is
// summed in a fixed order, so the result is deterministic.
//
// SYM (hyperelastic / associative J2: dP/dG has major symmetry, J = J^T):
// only blocks with flat(b) >= flat(a) are formed; k_mirror_lower copies
// K_ba^T into the rest.
#pragma once

#include "impm_kernels.cuh"

namespace impm_gpu {

namespace sweep {
constexpr int kWarps = 4;       // one warp per tile column (2 x 2 tile)
constexpr int kBins = 16;       // bins of one layer that reach the tile (4 x 4)
constexpr int kChunk = 64;      // staged particles per chunk
constexpr int kGMax = 16;       // particles per group (longer runs are split)
constexpr int kHMax = 48;       // (unit, particle) H vectors per task round
constexpr int kMaxUnits = 3 * kChunk;
constexpr int kNA = 81;
constexpr int kAccRow = 125 * 9;  // dense accumulator of one row: [slot][c*3+d]

struct Smem {
  double acc[kWarps][3][kAccRow];   // 108000 B
  double A[kChunk][kNA];            //  41472 B
  double W[kChunk][3][3][2];        //   9216 B: [slot][axis][node][w|dw]
  double H[kWarps][kHMax][27];      //  41472 B
  int bstart[kBins], bnp[kBins], lpre[kBins + 1];
  unsigned char sbin[kChunk], ssig[kChunk];
  unsigned char gstart[kChunk + 1];
  int ngroups;
  // per warp unit list of the chunk: group, ox, oy, oz; first task; H offset in round
  unsigned char ugrp[kWarps][kMaxUnits], uox[kWarps][kMaxUnits], uoy[kWarps][kMaxUnits], uoz[kWarps][kMaxUnits];
  short utask0[kWarps][kMaxUnits + 1];
  unsigned char uh[kWarps][kMaxUnits + 1];
  int nunits[kWarps];
  int rowact[kWarps][3];  // act_idx of the column's rows at levels kz .. kz+2
};
}  // namespace sweep

constexpr size_t sweep_smem_bytes() { return sizeof(sweep::Smem); }

template <int SHAPE, bool SYM>
__global__ void __launch_bounds__(sweep::kWarps * 32, 1)
    k_assemble_sweep(GridC g, const double* __restrict__ pd, int64_t cap, const double* __restrict__ xs,
                     const int* __restrict__ bin_start, const int* __restrict__ sup,
                     const double* __restrict__ A, const int* __restrict__ act_idx,
                     const int* __restrict__ row_nzb, const uint8_t* __restrict__ row_slots,
                     double* __restrict__ vals, int64_t row_len) {
  using namespace sweep;
  constexpr int D = 3;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = g.nodes[0], n1 = g.nodes[1], n2 = g.nodes[2];
  const int nt0 = (n0 + 1) / 2, nt1 = (n1 + 1) / 2;
  const int ntiles = nt0 * nt1;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int X0 = 2 * (tile / nt1), Y0 = 2 * (tile % nt1);
    const int cx = X0 + (warp >> 1), cy = Y0 + (warp & 1);
    const bool col_in = cx < n0 && cy < n1;
    const int col_node = cx * g.stride[0] + cy * g.stride[1];
    for (int e = lane; e < 3 * kAccRow; e += 32) (&S.acc[warp][0][0])[e] = 0.0;
    for (int kz = 0; kz < n2; ++kz) {
      __syncthreads();  // the previous layer's staging is free
      if (tid < kBins) {
        const int bx = X0 - 2 + (tid >> 2), by = Y0 - 2 + (tid & 3);
        int np = 0, st = 0;
        if (bx >= 0 && by >= 0 && bx < n0 && by < n1) {
          const int b = bx * g.stride[0] + by * g.stride[1] + kz;
          st = bin_start[b];
          np = bin_start[b + 1] - st;
        }
        S.bstart[tid] = st;
        S.bnp[tid] = np;
      }
      if (lane < 3) S.rowact[warp][lane] = col_in && kz + lane < n2 ? act_idx[col_node + kz + lane] : -1;
      __syncthreads();
      if (tid == 0) {
        int t = 0;
        for (int i = 0; i < kBins; ++i) {
          S.lpre[i] = t;
          t += S.bnp[i];
        }
        S.lpre[kBins] = t;
      }
      __syncthreads();
      const int nlayer = S.lpre[kBins];
      for (int c0 = 0; c0 < nlayer; c0 += kChunk) {
        if (c0 > 0) __syncthreads();  // all warps are done with the previous chunk
        const int nc = min(kChunk, nlayer - c0);
        // ---- stage: slot -> (bin, particle), A_p, 1D weights of the box nodes
        if (tid < kChunk) {
          int i = 0, sig = 0;
          if (tid < nc) {
            const int L = c0 + tid;
            while (S.lpre[i + 1] <= L) ++i;
            sig = sup[S.bstart[i] + L - S.lpre[i]] & 63;
          }
          S.sbin[tid] = static_cast<unsigned char>(i);
          S.ssig[tid] = static_cast<unsigned char>(sig);
        }
        __syncthreads();
        for (int e = tid; e < nc * kNA; e += kWarps * 32) {
          const int s = e / kNA, r = e - s * kNA, i = S.sbin[s];
          const int p = S.bstart[i] + c0 + s - S.lpre[i];
          S.A[s][r] = __ldg(A + static_cast<int64_t>(p) * kNA + r);
        }
        for (int e = tid; e < nc * 9; e += kWarps * 32) {
          const int s = e / 9, r = e - s * 9, a = r / 3, k = r - a * 3, i = S.sbin[s];
          double w = 0.0, dw = 0.0;
          if (k < sup_cnt(S.ssig[s], a)) {
            const int p = S.bstart[i] + c0 + s - S.lpre[i];
            const int base = a == 0 ? X0 - 2 + (i >> 2) : (a == 1 ? Y0 - 2 + (i & 3) : kz);
            const WeightValue wv =
                weight_1d<SHAPE>(xs[a * cap + p] - node_coord(g, a, base + k), pd[(PF<D>::lp + a) * cap + p], g.h);
            w = wv.w;
            dw = wv.dw;
          }
          S.W[s][a][k][0] = w;
          S.W[s][a][k][1] = dw;
        }
        if (tid == 0) {  // groups: runs of equal (bin, signature), <= kGMax long
          int ng = 0;
          for (int s = 0; s < nc; ++s)
            if (s == 0 || S.sbin[s] != S.sbin[s - 1] || S.ssig[s] != S.ssig[s - 1] ||
                s - S.gstart[ng - 1] >= kGMax)
              S.gstart[ng++] = static_cast<unsigned char>(s);
          S.gstart[ng] = static_cast<unsigned char>(nc);
          S.ngroups = ng;
        }
        __syncthreads();
        // ---- this warp's units: (group, row level) pairs whose box holds the column
        if (lane == 0) {
          int nu = 0, nt = 0;
          if (col_in) {
            for (int gi = 0; gi < S.ngroups; ++gi) {
              const int s0 = S.gstart[gi], i = S.sbin[s0], sg = S.ssig[s0];
              const int cnx = sup_cnt(sg, 0), cny = sup_cnt(sg, 1), cnz = sup_cnt(sg, 2);
              const int ox = cx - (X0 - 2 + (i >> 2)), oy = cy - (Y0 - 2 + (i & 3));
              if (ox < 0 || oy < 0 || ox >= cnx || oy >= cny) continue;
              for (int oz = 0; oz < cnz; ++oz) {
                if (S.rowact[warp][oz] < 0) continue;
                // SYM: (ibx, iby) with (ibx - ox, iby - oy) >= (0, 0) lexicographically
                const int ntk = SYM ? (cnx - ox - 1) * cny + (cny - oy) : cnx * cny;
                S.ugrp[warp][nu] = static_cast<unsigned char>(gi);
                S.uox[warp][nu] = static_cast<unsigned char>(ox);
                S.uoy[warp][nu] = static_cast<unsigned char>(oy);
                S.uoz[warp][nu] = static_cast<unsigned char>(oz);
                S.utask0[warp][nu] = static_cast<short>(nt);
                nt += ntk;
                ++nu;
              }
            }
          }
          S.utask0[warp][nu] = static_cast<short>(nt);
          S.nunits[warp] = nu;
        }
        __syncwarp();
        const int nu = S.nunits[warp];
        // ---- rounds: whole units, <= 32 tasks and <= kHMax H vectors
        int u0 = 0;
        while (u0 < nu) {
          int u1 = u0, nh = 0;
          while (u1 < nu) {
            const int gi = S.ugrp[warp][u1];
            const int gn = S.gstart[gi + 1] - S.gstart[gi];
            if (S.utask0[warp][u1 + 1] - S.utask0[warp][u0] > 32 || nh + gn > kHMax) break;
            if (lane == 0) S.uh[warp][u1] = static_cast<unsigned char>(nh);
            nh += gn;
            ++u1;
          }
          __syncwarp();
          const int t0 = S.utask0[warp][u0], ntask = S.utask0[warp][u1] - t0;
          // H_a^p for every (unit, particle) of the round
          for (int e = lane; e < nh * 27; e += 32) {
            const int hv = e / 27, cdf = e - hv * 27;
            int u = u0;
            while (u + 1 < u1 && S.uh[warp][u + 1] <= hv) ++u;
            const int gi = S.ugrp[warp][u];
            const int s = S.gstart[gi] + hv - S.uh[warp][u];
            const int ox = S.uox[warp][u], oy = S.uoy[warp][u], oz = S.uoz[warp][u];
            const double wx = S.W[s][0][ox][0], dwx = S.W[s][0][ox][1];
            const double wy = S.W[s][1][oy][0], dwy = S.W[s][1][oy][1];
            const double wz = S.W[s][2][oz][0], dwz = S.W[s][2][oz][1];
            const int c = cdf / 9, df = cdf - c * 9;  // H[c][d][f], df = d*3+f
            const double* Ap = &S.A[s][df * 9 + c * 3];
            double h = (dwx * wy * wz) * Ap[0];
            h = fma(wx * dwy * wz, Ap[1], h);
            h = fma(wx * wy * dwz, Ap[2], h);
            S.H[warp][hv][cdf] = h;
          }
          __syncwarp();
          // this lane's task: (unit, ibx, iby), a z-run of the group box
          const bool has = lane < ntask;
          int u = u0, ibx = 0, iby = 0;
          if (has) {
            const int t = t0 + lane;
            while (S.utask0[warp][u + 1] <= t) ++u;
            int k = t - S.utask0[warp][u];
            const int sg = S.ssig[S.gstart[S.ugrp[warp][u]]];
            const int cny = sup_cnt(sg, 1);
            if constexpr (SYM) {
              const int ox = S.uox[warp][u], oy = S.uoy[warp][u];
              if (k < cny - oy) {  // the delta_x = 0 column row: iby >= oy
                ibx = ox;
                iby = oy + k;
              } else {
                k -= cny - oy;
                ibx = ox + 1 + k / cny;
                iby = k - (k / cny) * cny;
              }
            } else {
              ibx = k / cny;
              iby = k - ibx * cny;
            }
          }
          double acc[3][9];
#pragma unroll
          for (int z = 0; z < 3; ++z)
#pragma unroll
            for (int e = 0; e < 9; ++e) acc[z][e] = 0.0;
          if (has) {
            const int gi = S.ugrp[warp][u];
            const int s0 = S.gstart[gi], gn = S.gstart[gi + 1] - s0;
            const double* Hu = S.H[warp][S.uh[warp][u]];
            for (int j = 0; j < gn; ++j) {
              const int s = s0 + j;
              const double wx = S.W[s][0][ibx][0], dwx = S.W[s][0][ibx][1];
              const double wy = S.W[s][1][iby][0], dwy = S.W[s][1][iby][1];
              const double gxy0 = dwx * wy, gxy1 = wx * dwy, gxy2 = wx * wy;
              double gb[3][3];
#pragma unroll
              for (int z = 0; z < 3; ++z) {
                const double wz = S.W[s][2][z][0], dwz = S.W[s][2][z][1];
                gb[z][0] = gxy0 * wz;
                gb[z][1] = gxy1 * wz;
                gb[z][2] = gxy2 * dwz;
              }
              const double* Hp = Hu + j * 27;
#pragma unroll
              for (int cd = 0; cd < 9; ++cd) {
                const double h0 = Hp[cd * 3], h1 = Hp[cd * 3 + 1], h2 = Hp[cd * 3 + 2];
#pragma unroll
                for (int z = 0; z < 3; ++z)
                  acc[z][cd] = fma(h2, gb[z][2], fma(h1, gb[z][1], fma(h0, gb[z][0], acc[z][cd])));
              }
            }
          }
          // flush unit by unit (tasks of one unit own disjoint blocks)
          for (int uf = u0; uf < u1; ++uf) {
            if (has && u == uf) {
              const int sg = S.ssig[S.gstart[S.ugrp[warp][u]]];
              const int cnz = sup_cnt(sg, 2);
              const int ox = S.uox[warp][u], oy = S.uoy[warp][u], oz = S.uoz[warp][u];
              const int sxy = (ibx - ox + 2) * 25 + (iby - oy + 2) * 5;
              const bool diag_col = SYM && ibx == ox && iby == oy;
              double* row = S.acc[warp][(kz + oz) % 3];
#pragma unroll
              for (int z = 0; z < 3; ++z) {
                if (z >= cnz || (diag_col && z < oz)) continue;
                double* blk = row + (sxy + z - oz + 2) * 9;
#pragma unroll
                for (int e = 0; e < 9; ++e) blk[e] += acc[z][e];
              }
            }
            __syncwarp();
          }
          u0 = u1;
        }
      }
      // ---- rows at level kz are complete: write their stored slots once, reset
      if (col_in) {
        const int row = S.rowact[warp][0];
        double* racc = S.acc[warp][kz % 3];
        if (row >= 0) {
          const int nzb = row_nzb[row];
          const int cp = cpad(nzb, D);
          const uint8_t* sl = row_slots + static_cast<int64_t>(row) * 125;
          double* out = vals + static_cast<int64_t>(row) * row_len;
          for (int c = 0; c < D; ++c)
            for (int e = lane; e < nzb * D; e += 32) {
              const int pos = e / D, d = e - pos * D;
              out[c * cp + e] = racc[sl[pos] * 9 + c * D + d];
            }
        }
        for (int e = lane; e < kAccRow; e += 32) racc[e] = 0.0;
      }
      __syncwarp();
    }
  }
}

// Lower blocks of a symmetric J from the upper ones written by the SYM sweep:
// K_ab = K_ba^T for flat(b) < flat(a). One warp per row, a lane per value.
template <int D>
__global__ void k_mirror_lower(GridC g, int n_act, const int* __restrict__ act_list, const int* __restrict__ act_idx,
                               const int* __restrict__ row_nzb, const uint8_t* __restrict__ row_slots,
                               const unsigned* __restrict__ row_mask, double* __restrict__ vals, int64_t row_len) {
  constexpr int S = ipow_c(5, D);
  constexpr int DD = D * D;
  constexpr int center = (S - 1) / 2;  // slot of delta = 0
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= n_act) return;
  const int node = act_list[row];
  const int nzb = row_nzb[row], cp = cpad(nzb, D);
  const uint8_t* sl = row_slots + static_cast<int64_t>(row) * S;
  double* out = vals + static_cast<int64_t>(row) * row_len;
  // stored slots are ascending, so the lower ones (slot < center) come first
  for (int e = lane; e < nzb * DD; e += 32) {
    const int pos = e / DD, cd = e - pos * DD, c = cd / D, d = cd - c * D;
    const int slot = sl[pos];
    if (slot >= center) break;
    int r = slot, off = 0;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      off += (r % 5 - 2) * g.stride[a];
      r /= 5;
    }
    const int rb = act_idx[node + off];
    if (rb < 0) {  // an inactive column node (box corner no particle reaches): not a DOF
      out[c * cp + pos * D + d] = 0.0;
      continue;
    }
    const int ms = S - 1 - slot;  // the slot of -delta in row b
    const unsigned* m = row_mask + static_cast<int64_t>(rb) * 4;
    const int w = ms >> 5;
    int pb = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (k < w) pb += __popc(m[k]);
    pb += __popc(m[w] & ((1u << (ms & 31)) - 1u));
    const int cpb = cpad(row_nzb[rb], D);
    out[c * cp + pos * D + d] = vals[static_cast<int64_t>(rb) * row_len + d * cpb + pb * D + c];
  }
}

}  // namespace impm_gpu
