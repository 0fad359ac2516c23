// K6 prolongation and K7 restriction kernels (non-nested transfer).
//
// Records are grouped by owning coarse cell (CSR cell_start / pt_dof / xhat),
// one warp per coarse cell.  See DESIGN.md "Transfers".
#pragma once

#include "nnmg_kernels.cuh"

namespace nnmg {

static constexpr int kTransferWarps = 4;  // coarse cells (one per warp) per thread block

// ---------------------------------------------------------------------------
// K6: u_f[pt] (+)= sum_l u_c[gather[pt,l]] prod_j phi_{l_j}(xhat_j)
// (transfer.py:31-44, 87-102).  The cell's coarse values are staged once in
// shared memory and broadcast; each lane evaluates two points per round so two
// independent load/store chains are in flight.  Contraction order x, y, z as
// transfer.py:93-95.
// ---------------------------------------------------------------------------
template <int DIM, int N1>
__device__ __forceinline__ double contract(const double* __restrict__ U, const double (&X)[DIM][N1]) {
  if constexpr (DIM == 2) {
    double val = 0.0;
#pragma unroll
    for (int i1 = 0; i1 < N1; ++i1) {
      double s = 0.0;
#pragma unroll
      for (int i0 = 0; i0 < N1; ++i0) s = fma(U[i0 + N1 * i1], X[0][i0], s);
      val = fma(s, X[1][i1], val);
    }
    return val;
  } else {
    double val = 0.0;
#pragma unroll
    for (int i2 = 0; i2 < N1; ++i2) {
      double s2 = 0.0;
#pragma unroll
      for (int i1 = 0; i1 < N1; ++i1) {
        double s = 0.0;
#pragma unroll
        for (int i0 = 0; i0 < N1; ++i0) s = fma(U[i0 + N1 * i1 + N1 * N1 * i2], X[0][i0], s);
        s2 = fma(s, X[1][i1], s2);
      }
      val = fma(s2, X[2][i2], val);
    }
    return val;
  }
}

template <int DIM, int PC, int NCOMP, int CBC>
__global__ void __launch_bounds__(kTransferWarps * 32, 6)
    k_prolongate(Tables tab, const double* __restrict__ uc, double* __restrict__ uf, int accumulate,
                 const int* __restrict__ cidx, const int* __restrict__ cell_start, const int* __restrict__ pt_dof,
                 const double* __restrict__ xhat, int64_t ncc) {
  constexpr int N1 = PC + 1;
  constexpr int NLOC = ipow(N1, DIM);
  __shared__ double su[kTransferWarps][NCOMP * NLOC];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t cell = blockIdx.x * (int64_t)kTransferWarps + warp;
  if (cell >= ncc) return;
  const int64_t blk = cell / CBC, cl = cell % CBC;
  for (int l = lane; l < NLOC; l += 32) {
    const int g = cidx[(blk * NLOC + l) * CBC + cl];
#pragma unroll
    for (int c = 0; c < NCOMP; ++c) su[warp][c * NLOC + l] = g >= 0 ? uc[(int64_t)g * NCOMP + c] : 0.0;
  }
  __syncwarp();
  constexpr int PPL = ((DIM == 2 || N1 <= 2) && NCOMP == 1) ? 2 : 1;  // points per lane per round
  const int p0 = cell_start[cell], p1 = cell_start[cell + 1];
  for (int base = p0; base < p1; base += 32 * PPL) {
    int pp[PPL], dd[PPL];
    bool vv[PPL];
    double X[PPL][DIM][N1];
#pragma unroll
    for (int k = 0; k < PPL; ++k) {
      pp[k] = base + 32 * k + lane;
      vv[k] = pp[k] < p1;
      dd[k] = vv[k] ? __ldcs(pt_dof + pp[k]) : 0;
#pragma unroll
      for (int j = 0; j < DIM; ++j)
        lagrange_values<N1>(tab, vv[k] ? __ldcs(xhat + (int64_t)pp[k] * DIM + j) : 0.5, X[k][j]);
    }
#pragma unroll
    for (int c = 0; c < NCOMP; ++c) {
      const double* U = su[warp] + c * NLOC;
#pragma unroll
      for (int k = 0; k < PPL; ++k) {
        const double a = contract<DIM, N1>(U, X[k]);
        if (vv[k]) {
          double* o = uf + (int64_t)dd[k] * NCOMP + c;
          *o = accumulate ? *o + a : a;
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K7 phase 1: per owning coarse cell the local vector
//   R_l = sum_pt r_f[pt] W_l(pt),  W = phi_{l2}(z) (phi_{l1}(y) phi_{l0}(x))
// (transfer.py:104-109, 115).  Deterministic, no atomics:
//  * NLOC <= 32: every lane accumulates the full local vector over a fixed
//    subset of the cell's points in registers, then a butterfly reduction
//    (fixed order) sums the lanes; one pass per component;
//  * larger NLOC: lanes own local outputs and sweep the cell's points staged
//    in shared memory.
// ---------------------------------------------------------------------------
template <int DIM, int PC, int NCOMP>
__global__ void __launch_bounds__(kTransferWarps * 32)
    k_restrict_cells(Tables tab, const double* __restrict__ rf, const int* __restrict__ cell_start,
                     const int* __restrict__ pt_dof, const double* __restrict__ xhat, int64_t ncc,
                     double* __restrict__ cellbuf) {
  constexpr int N1 = PC + 1;
  constexpr int NLOC = ipow(N1, DIM);
  constexpr int NOUT = NLOC * NCOMP;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t cell = blockIdx.x * (int64_t)kTransferWarps + warp;
  if (cell >= ncc) return;
  const int p0 = cell_start[cell], p1 = cell_start[cell + 1];
  if constexpr (NLOC <= 32) {
#pragma unroll 1
    for (int c = 0; c < NCOMP; ++c) {
      double acc[NLOC];
#pragma unroll
      for (int l = 0; l < NLOC; ++l) acc[l] = 0.0;
      for (int p = p0 + lane; p < p1; p += 32) {
        const int64_t dof = __ldcs(pt_dof + p);
        const double v = rf[dof * NCOMP + c];
        double X[DIM][N1];
#pragma unroll
        for (int j = 0; j < DIM; ++j) lagrange_values<N1>(tab, __ldcs(xhat + (int64_t)p * DIM + j), X[j]);
#pragma unroll
        for (int l = 0; l < NLOC; ++l) {
          const int i0 = l % N1, i1 = (l / N1) % N1, i2 = l / (N1 * N1);
          double w = X[1][i1] * X[0][i0];
          if constexpr (DIM == 3) w = X[2][i2] * w;
          acc[l] = fma(v, w, acc[l]);
        }
      }
#pragma unroll
      for (int l = 0; l < NLOC; ++l) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[l] += __shfl_xor_sync(0xffffffffu, acc[l], o);
      }
      double mine = 0.0;
#pragma unroll
      for (int l = 0; l < NLOC; ++l)
        if (lane == l) mine = acc[l];
      if (lane < NLOC) cellbuf[cell * NOUT + lane * NCOMP + c] = mine;
    }
  } else {
    constexpr int NPL = (NOUT + 31) / 32;
    __shared__ double sv[kTransferWarps][32][NCOMP];
    __shared__ double sx[kTransferWarps][32][DIM][N1];
    double acc[NPL];
#pragma unroll
    for (int k = 0; k < NPL; ++k) acc[k] = 0.0;
    for (int start = p0; start < p1; start += 32) {
      const int p = start + lane;
      if (p < p1) {
        const int64_t dof = __ldcs(pt_dof + p);
#pragma unroll
        for (int c = 0; c < NCOMP; ++c) sv[warp][lane][c] = rf[dof * NCOMP + c];
#pragma unroll
        for (int j = 0; j < DIM; ++j) lagrange_values<N1>(tab, __ldcs(xhat + (int64_t)p * DIM + j), sx[warp][lane][j]);
      }
      __syncwarp();
      const int cnt = min(32, p1 - start);
#pragma unroll
      for (int k = 0; k < NPL; ++k) {
        const int o = lane + 32 * k;
        if (o < NOUT) {
          const int l = o / NCOMP, c = o % NCOMP;
          const int i0 = l % N1, i1 = (l / N1) % N1, i2 = l / (N1 * N1);
          double a = acc[k];
          for (int j = 0; j < cnt; ++j) {
            double w = sx[warp][j][1][i1] * sx[warp][j][0][i0];
            if constexpr (DIM == 3) w = sx[warp][j][2][i2] * w;
            a = fma(sv[warp][j][c], w, a);
          }
          acc[k] = a;
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int k = 0; k < NPL; ++k) {
      const int o = lane + 32 * k;
      if (o < NOUT) cellbuf[cell * NOUT + o] = acc[k];
    }
  }
}

// K7 phase 2: r_c[g] = sum over the (cell, l) slots holding g, fixed order
__global__ void k_restrict_gather(const int* __restrict__ t_off, const int* __restrict__ t_ent,
                                  const double* __restrict__ cellbuf, int64_t nsc, int ncomp, double* __restrict__ rc) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= nsc) return;
  const int e0 = t_off[g], e1 = t_off[g + 1];
  for (int c = 0; c < ncomp; ++c) {
    double s = 0.0;
    for (int e = e0; e < e1; ++e) s += cellbuf[(int64_t)t_ent[e] * ncomp + c];
    rc[g * ncomp + c] = s;
  }
}

}  // namespace nnmg
