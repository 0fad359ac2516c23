// K6 prolongation and K7 restriction kernels (non-nested transfer).
//
// Records are grouped by owning coarse cell (CSR cell_start / pt_dof / xhat),
// one warp per coarse cell.  See DESIGN.md "Transfers".
#pragma once

#include "nnmg_kernels.cuh"

namespace nnmg {

static constexpr int kTransferWarps = 4;  // coarse cells (one per warp) per thread block

// Software-pipelined stream over a lane's points p = first, first+stride, ...
// (< end): point indices and coordinates are loaded two points ahead and the
// gathered fine value one point ahead, so the dependent pt_dof -> r_f[dof]
// chain overlaps the arithmetic of the current point.
template <int DIM, int NCOMP, int VSTRIDE = NCOMP>
struct PointStream {
  const int* __restrict__ pt_dof;
  const double* __restrict__ xhat;
  const double* __restrict__ rf;
  int end, stride;
  int p0, p1, p2;
  int64_t d0, d1, d2;
  double x0[DIM], x1[DIM], x2[DIM];
  double v0[NCOMP], v1[NCOMP];

  __device__ __forceinline__ void load_idx(int p, int64_t& d, double (&x)[DIM]) {
    const bool ok = p < end;
    d = ok ? __ldcs(pt_dof + p) : 0;
#pragma unroll
    for (int j = 0; j < DIM; ++j) x[j] = ok ? __ldcs(xhat + (int64_t)p * DIM + j) : 0.5;
  }
  __device__ __forceinline__ void load_val(int p, int64_t d, double (&v)[NCOMP]) {
#pragma unroll
    for (int c = 0; c < NCOMP; ++c) v[c] = p < end ? rf[d * VSTRIDE + c] : 0.0;
  }
  __device__ __forceinline__ void start(int first) {
    p0 = first;
    p1 = first + stride;
    p2 = first + 2 * stride;
    load_idx(p0, d0, x0);
    load_idx(p1, d1, x1);
    load_val(p0, d0, v0);
  }
  __device__ __forceinline__ bool valid() const { return p0 < end; }
  // issue the next loads; call before computing on (x0, v0)
  __device__ __forceinline__ void prefetch() {
    load_val(p1, d1, v1);
    load_idx(p2, d2, x2);
  }
  __device__ __forceinline__ void advance() {
    p0 = p1;
    p1 = p2;
    p2 += stride;
    d0 = d1;
    d1 = d2;
#pragma unroll
    for (int j = 0; j < DIM; ++j) {
      x0[j] = x1[j];
      x1[j] = x2[j];
    }
#pragma unroll
    for (int c = 0; c < NCOMP; ++c) v0[c] = v1[c];
  }
};

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
  // measured: two independent points per lane per round beat a pipelined
  // single-point stream here (C3: 0.195 vs 0.251 ms)
  constexpr int PPL = ((DIM == 2 || N1 <= 2) && NCOMP == 1) ? 2 : 1;
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
      // component c of the interleaved vector: values rf[dof*NCOMP + c]
      PointStream<DIM, 1, NCOMP> ps{pt_dof, xhat, rf + c, p1, 32};
      for (ps.start(p0 + lane); ps.valid(); ps.advance()) {
        ps.prefetch();
        const double v = ps.v0[0];
        double X[DIM][N1];
#pragma unroll
        for (int j = 0; j < DIM; ++j) lagrange_values<N1>(tab, ps.x0[j], X[j]);
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
    // G lanes share a point; lane slice g owns the outermost-axis planes
    // [g*PPG, (g+1)*PPG) of the local vector, all components, in registers.
    // Every register index is compile-time: the per-point inner-plane table
    // IN[i] (x, or x*y in 3D) is static, only the plane's 1D value is
    // evaluated at a runtime node index.  32/G points per round; fixed-order
    // butterfly over the point slots at the end.
    constexpr int INNER = DIM == 3 ? N1 * N1 : N1;  // points per plane
    // power of two so the xor butterfly keeps each slice's lanes together
    constexpr int G = (N1 * INNER * NCOMP <= 64) ? 1
                      : ((N1 + 1) / 2 * INNER * NCOMP <= 80 ? 2 : (N1 <= 4 ? 4 : 8));
    constexpr int PPG = (N1 + G - 1) / G;             // planes per lane
    constexpr int SLOTS = 32 / G;
    const int slice = lane % G, slot = lane / G;
    double acc[PPG][INNER][NCOMP];
#pragma unroll
    for (int a = 0; a < PPG; ++a)
#pragma unroll
      for (int i = 0; i < INNER; ++i)
#pragma unroll
        for (int c = 0; c < NCOMP; ++c) acc[a][i][c] = 0.0;
    PointStream<DIM, NCOMP> ps{pt_dof, xhat, rf, p1, SLOTS};
    for (ps.start(slot < SLOTS ? p0 + slot : p1); ps.valid(); ps.advance()) {
      ps.prefetch();
      {
        const double* v = ps.v0;
        double X[DIM - 1][N1];
#pragma unroll
        for (int j = 0; j < DIM - 1; ++j) lagrange_values<N1>(tab, ps.x0[j], X[j]);
        // inner table, reference product order X1[i1] * X0[i0] (transfer.py:104-109)
        double IN[INNER];
#pragma unroll
        for (int i = 0; i < INNER; ++i) IN[i] = DIM == 3 ? X[1][i / N1] * X[0][i % N1] : X[0][i];
        const double tz = ps.x0[DIM - 1];
#pragma unroll
        for (int a = 0; a < PPG; ++a) {
          const int plane = slice * PPG + a;
          if (plane < N1) {
            // phi_plane(tz) with a runtime node index (no register-array indexing)
            double z = 1.0;
#pragma unroll
            for (int j = 0; j < N1; ++j) z *= (j == plane) ? tab.rdenom[plane < N1 ? plane : 0] : (tz - tab.nodes[j]);
            double vz[NCOMP];
#pragma unroll
            for (int c = 0; c < NCOMP; ++c) vz[c] = v[c] * z;
#pragma unroll
            for (int i = 0; i < INNER; ++i)
#pragma unroll
              for (int c = 0; c < NCOMP; ++c) acc[a][i][c] = fma(vz[c], IN[i], acc[a][i][c]);
          }
        }
      }
    }
#pragma unroll
    for (int a = 0; a < PPG; ++a)
#pragma unroll
      for (int i = 0; i < INNER; ++i)
#pragma unroll
        for (int c = 0; c < NCOMP; ++c) {
          double s = acc[a][i][c];
#pragma unroll
          for (int off = G; off < 32; off <<= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
          acc[a][i][c] = s;
        }
    if (slot == 0) {
#pragma unroll
      for (int a = 0; a < PPG; ++a) {
        const int plane = slice * PPG + a;
        if (plane < N1) {
#pragma unroll
          for (int i = 0; i < INNER; ++i)
#pragma unroll
            for (int c = 0; c < NCOMP; ++c) cellbuf[cell * NOUT + (plane * INNER + i) * NCOMP + c] = acc[a][i][c];
        }
      }
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
