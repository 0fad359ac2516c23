// Register-resident cell kernel (one thread per cell) for low orders.
//
// The pencil kernel (nnmg_cellkernel.cuh) exchanges every intermediate through
// shared memory; ncu shows it L1/shared-pipe bound on 3D Q2 (l1tex 96% busy,
// DRAM 70%).  For NLOC <= 27 a whole cell fits in registers: the thread
// gathers its cell, runs all sum-factorisation sweeps in registers, visits the
// quadrature points slice by slice (gradients by collocation, flux, and the
// transposed derivative sweeps accumulated immediately), and scatters.  No
// shared memory, no block barriers; loads of the index table and geometry are
// coalesced across the warp (32 consecutive cells = one cell block of the
// blocked layout).
#pragma once

#include "nnmg_kernels.cuh"

namespace nnmg {

template <int DIM, int P>
struct CellReg {
  static constexpr int N1 = P + 1;
  static constexpr int NLOC = ipow(N1, DIM);
  static constexpr int CB = 32;
  static constexpr int NG = DIM * (DIM + 1) / 2;
  static constexpr bool kSupported = NLOC <= 27;
  // fp32 stored geometry in (k, k+1) pairs (level_enable_f32): even NG only (3D)
  template <class TG>
  static constexpr bool kPairedGeo = sizeof(TG) == sizeof(float) && NG % 2 == 0;

  __host__ __device__ static constexpr int at(int i0, int i1, int i2) { return i0 + N1 * (i1 + N1 * i2); }

  // in-register sweep along axis K with matrix M (trans: M^T)
  template <int K, bool TRANS, class TA = double>
  __device__ __forceinline__ static void sweep_axis(const TA (&M)[kMaxN1][kMaxN1], TA (&v)[NLOC]) {
    constexpr int S0 = K == 0 ? 1 : (K == 1 ? N1 : N1 * N1);
    constexpr int NL = NLOC / N1;  // lines along axis K
#pragma unroll
    for (int line = 0; line < NL; ++line) {
      // base position of the line: enumerate the other axes
      int base;
      if constexpr (K == 0)
        base = line * N1;
      else if constexpr (K == 1)
        base = (line % N1) + (line / N1) * N1 * N1;
      else
        base = line;
      TA in[N1], out[N1];
#pragma unroll
      for (int i = 0; i < N1; ++i) in[i] = v[base + i * S0];
#pragma unroll
      for (int q = 0; q < N1; ++q) {
        TA s = 0;
#pragma unroll
        for (int i = 0; i < N1; ++i) s = fma(TRANS ? M[i][q] : M[q][i], in[i], s);
        out[q] = s;
      }
#pragma unroll
      for (int i = 0; i < N1; ++i) v[base + i * S0] = out[i];
    }
  }

  // number of cell edge-vector components: 2^(d-1) edges per direction
  static constexpr int NE = DIM * (1 << (DIM - 1)) * DIM;

  // G = J^-1 J^-T |det J| w at a quadrature point, recomputed from the cell's
  // edge vectors E[b][k][a] (edge k along reference direction b):
  // J[a][b] = sum_k w_bk(xi) E[b][k][a] (the multilinear map, mesh.py:138-143),
  // C = cofactors of J, G = C^T C * w / det.
  __device__ __forceinline__ static void recompute_g(const Tables& tab, const double (&E)[NE], int qx, int qy, int qz,
                                                     double (&g)[NG]) {
    const double xi[3] = {tab.xq[qx], tab.xq[qy], DIM == 3 ? tab.xq[qz] : 0.0};
    const double wq = tab.w[qx] * tab.w[qy] * (DIM == 3 ? tab.w[qz] : 1.0);
    double J[DIM][DIM];
#pragma unroll
    for (int b = 0; b < DIM; ++b) {
      // the other axes in increasing order
      const int o0 = b == 0 ? 1 : 0;
      const int o1 = b == 2 ? 1 : 2;
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < (1 << (DIM - 1)); ++k) {
          double wk = (k & 1) ? xi[o0] : 1.0 - xi[o0];
          if constexpr (DIM == 3) wk *= (k & 2) ? xi[o1] : 1.0 - xi[o1];
          s = fma(wk, E[(b * (1 << (DIM - 1)) + k) * DIM + a], s);
        }
        J[a][b] = s;
      }
    }
    if constexpr (DIM == 3) {
      double C[3][3];
      C[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
      C[0][1] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
      C[0][2] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
      C[1][0] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
      C[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
      C[1][2] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
      C[2][0] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
      C[2][1] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
      C[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      const double det = J[0][0] * C[0][0] + J[0][1] * C[0][1] + J[0][2] * C[0][2];
      const double s = wq * __drcp_rn(det);
      int k = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = a; b < 3; ++b) g[k++] = s * (C[0][a] * C[0][b] + C[1][a] * C[1][b] + C[2][a] * C[2][b]);
    } else {
      const double det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      const double s = wq * __drcp_rn(det);
      // cofactors: C00 = J11, C01 = -J10, C10 = -J01, C11 = J00
      g[0] = s * (J[1][1] * J[1][1] + J[0][1] * J[0][1]);
      g[1] = -s * (J[1][1] * J[1][0] + J[0][1] * J[0][0]);
      g[2] = s * (J[1][0] * J[1][0] + J[0][0] * J[0][0]);
    }
  }

  // Laplace only.  Returns the thread's cell energy sum_l u_l (A_K u)_l.
  // GEO 0: stored G;  GEO 1: G recomputed from the cell's edge vectors held in
  // registers (naive per point);  GEO 2: recomputed, sum-factorised (3D)
  // GEO 3 (3D): stored G streamed through shared memory by TMA bulk copies,
  // one z-slice (N1^2 points x NG x CB doubles) per copy, two slots per warp
  // with an mbarrier each: the G loads of the point loop become shared-memory
  // reads whose data were in flight since the gather.  `wsm` = this warp's
  // WARP_SMEM bytes.
  static constexpr int SLICE_Q = DIM == 3 ? N1 * N1 : NLOC;
  static constexpr unsigned SLICE_BYTES = unsigned(SLICE_Q) * NG * CB * sizeof(double);
  static constexpr size_t WARP_SMEM = 2 * size_t(SLICE_BYTES) + 16;
  // GEO 4: the whole fp32 chunk of a warp's 32 cells plus its mbarrier
  static constexpr unsigned CHUNK32_BYTES = unsigned(NLOC) * NG * CB * sizeof(float);
  static constexpr size_t WARP_SMEM32 = size_t(CHUNK32_BYTES) + 16;

  // TD / TG: storage types of dst and of the stored geometry (double, or
  // float in the mixed-precision V-cycle); TA: the arithmetic type (double;
  // float = the paper's single-precision V-cycle: with fp64
  // arithmetic on fp32 storage the kernel is bound by its DFMAs and its
  // 248 registers, 543 us against 597 us for fp64 storage on C3)
  // XNB (warp-neighbour faces): lane c and lane c + 1 hold x-adjacent cells on
  // structured rows, so the last x-node of every line of cell c IS the first
  // x-node of cell c + 1.  Checked per line and lane pair at run time (index
  // comparison through one shuffle, no setup tables, any mesh): where it
  // holds the first node's value comes from the left neighbour's register
  // (no gather) and the last node's contribution is handed to the right
  // neighbour's first node before the scatter (no atomic): N1^(d-1) of the
  // N1^d gathers and atomics of a cell disappear (9 of 27 for 3D Q2).  The
  // L2 atomic units see 57M fp32 REDs per C3 apply otherwise.
  template <bool kStream, bool kEnergy, bool kNeg = false, int GEO = 0, class TA = double, int XNB = 0,
            class Src, class TD, class TG>
  __device__ __forceinline__ static double run(const Tables& tab, const Src& src, TD* __restrict__ dst,
                                               const int* __restrict__ idx, const TG* __restrict__ geo,
                                               int64_t blk, int lane, const double* __restrict__ edges = nullptr,
                                               double* wsm = nullptr, double* __restrict__ cellout = nullptr) {
    static_assert(GEO != 3 || sizeof(TG) == sizeof(double), "TMA slice staging is fp64");
    static_assert(GEO != 4 || (kPairedGeo<TG> && DIM == 3), "whole-chunk staging: paired fp32 geometry");
    static_assert(GEO == 0 || GEO == 4 || sizeof(TA) == sizeof(double),
                  "recomputed / slice-staged geometry is fp64 arithmetic");
    static_assert(!kEnergy || sizeof(TA) == sizeof(double), "cell energies are fp64");
    double* gbuf = wsm;
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(wsm + 2 * SLICE_Q * NG * CB);
    unsigned long long* mbar4 =
        reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(wsm) + CHUNK32_BYTES);  // GEO 4
    const TG* gchunk = geo + blk * (int64_t)NLOC * NG * CB;
    if constexpr (GEO == 3) {
      static_assert(DIM == 3, "slice staging is 3D");
      if (lane == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        fence_proxy_async();
#pragma unroll
        for (int s = 0; s < 2 && s < N1; ++s) {
          mbar_expect_tx(&mbar[s], SLICE_BYTES);
          tma_load_1d(gbuf + s * SLICE_Q * NG * CB, gchunk + s * SLICE_Q * NG * CB, SLICE_BYTES, &mbar[s]);
        }
      }
      __syncwarp();
    }
    if constexpr (GEO == 4) {
      // GEO 4 (fp32 geometry, 3D): the warp's whole chunk (NLOC x NG x CB
      // floats, 20.7 KB for Q2) by ONE TMA bulk copy issued before the gather:
      // every geometry byte is in flight while the gathers and the sweeps
      // run, and the point loop reads shared memory
      if (lane == 0) {
        mbar_init(mbar4, 1);
        fence_proxy_async();
        mbar_expect_tx(mbar4, CHUNK32_BYTES);
        tma_load_1d(wsm, gchunk, CHUNK32_BYTES, mbar4);
      }
      __syncwarp();
    }
    double E[GEO == 1 ? NE : 1];
    if constexpr (GEO == 1) {
      const double* eb = edges + blk * (int64_t)NE * CB + lane;
#pragma unroll
      for (int e = 0; e < NE; ++e) E[e] = ld_geo<kStream>(eb + e * CB);
    } else if constexpr (kStream && GEO == 0) {
      // the warp's geometry chunk (32 cells, 85% of the bytes) streams into L2
      // while the gathers and interpolation sweeps run
      constexpr unsigned kGeoBytes = unsigned(NLOC) * NG * CB * sizeof(TG);
      if (lane == 0) prefetch_l2_bulk(geo + blk * (int64_t)NLOC * NG * CB, kGeoBytes);
    }
    TA v[NLOC];
    const int* ib = idx + blk * NLOC * CB + lane;
    constexpr int NLINE = NLOC / N1;
    unsigned share_r = 0;  // XNB bit per line: my last x-node is the right neighbour's first
    if constexpr (XNB == 1) {
      constexpr unsigned kFull = 0xffffffffu;
      // phases, so that every load of a phase is in flight together: all
      // indices, the match bits (shuffles of indices), all values, then the
      // shuffles of the shared values
      int gi[NLOC];
#pragma unroll
      for (int l = 0; l < NLOC; ++l) gi[l] = ld_geo<kStream>(ib + l * CB);
      unsigned share_l = 0;
#pragma unroll
      for (int line = 0; line < NLINE; ++line) {
        const int gf = gi[line * N1], gl = gi[line * N1 + N1 - 1];
        const int nbf = __shfl_down_sync(kFull, gf, 1);
        share_r |= ((lane < 31 && gl >= 0 && nbf == gl) ? 1u : 0u) << line;
      }
      share_l = __shfl_up_sync(kFull, share_r, 1);  // every lane takes part in the shuffle
      if (lane == 0) share_l = 0u;
#pragma unroll
      for (int l = 0; l < NLOC; ++l) {
        const bool from_left = l % N1 == 0 && ((share_l >> (l / N1)) & 1u);
        v[l] = (gi[l] >= 0 && !from_left) ? TA(src((int64_t)gi[l])) : TA(0);
      }
#pragma unroll
      for (int line = 0; line < NLINE; ++line) {
        const TA recv = __shfl_up_sync(kFull, v[line * N1 + N1 - 1], 1);
        if ((share_l >> line) & 1u) v[line * N1] = recv;
      }
    } else {
#pragma unroll
      for (int l = 0; l < NLOC; ++l) {
        const int g = ld_geo<kStream>(ib + l * CB);
        v[l] = g >= 0 ? TA(src((int64_t)g)) : TA(0);
      }
    }
    TA u0[kEnergy ? NLOC : 1];
    if constexpr (kEnergy) {
#pragma unroll
      for (int l = 0; l < NLOC; ++l) u0[l] = v[l];
    }
    // values at the Gauss points
    const auto& tS = TabSel<TA>::S(tab);
    const auto& tDc = TabSel<TA>::Dc(tab);
    sweep_axis<0, false, TA>(tS, v);
    sweep_axis<1, false, TA>(tS, v);
    if constexpr (DIM == 3) sweep_axis<2, false, TA>(tS, v);
    TA w[NLOC];
#pragma unroll
    for (int l = 0; l < NLOC; ++l) w[l] = 0;
    // one quadrature point: collocation gradient, flux (G g), transposed
    // collocation derivatives accumulated at once
    auto point = [&](int qx, int qy, int qz, auto&& flux) {
      TA gx = 0, gy = 0, gz = 0;
#pragma unroll
      for (int r = 0; r < N1; ++r) {
        gx = fma(tDc[qx][r], v[at(r, qy, qz)], gx);
        gy = fma(tDc[qy][r], v[at(qx, r, qz)], gy);
        if constexpr (DIM == 3) gz = fma(tDc[qz][r], v[at(qx, qy, r)], gz);
      }
      TA fx, fy, fz = 0;
      flux(gx, gy, gz, fx, fy, fz);
#pragma unroll
      for (int r = 0; r < N1; ++r) {
        w[at(r, qy, qz)] = fma(tDc[qx][r], fx, w[at(r, qy, qz)]);
        w[at(qx, r, qz)] = fma(tDc[qy][r], fy, w[at(qx, r, qz)]);
        if constexpr (DIM == 3) w[at(qx, qy, r)] = fma(tDc[qz][r], fz, w[at(qx, qy, r)]);
      }
    };
    if constexpr (GEO == 2) {
      // 3D: G from the cell's edge vectors, sum-factorised along z-pencils of
      // the trilinear map (dx/dz constant along a pencil, dx/dx and dx/dy
      // affine in z); edges read through L1 (coalesced across the warp)
      static_assert(DIM == 3, "GEO 2 is 3D");
      const double* eb = edges + blk * (int64_t)NE * CB + lane;
      auto e = [&](int b, int k, int a) { return __ldg(eb + ((b * 4 + k) * 3 + a) * CB); };
#pragma unroll
      for (int qy = 0; qy < N1; ++qy) {
        const double y = tab.xq[qy];
        double A0[3], B0[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          A0[a] = fma(y, e(0, 1, a) - e(0, 0, a), e(0, 0, a));
          B0[a] = fma(y, e(0, 3, a) - e(0, 2, a), e(0, 2, a)) - A0[a];
        }
#pragma unroll
        for (int qx = 0; qx < N1; ++qx) {
          const double x = tab.xq[qx];
          const double wxy = tab.w[qx] * tab.w[qy];
          double A1[3], B1[3], J2[3];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            A1[a] = fma(x, e(1, 1, a) - e(1, 0, a), e(1, 0, a));
            B1[a] = fma(x, e(1, 3, a) - e(1, 2, a), e(1, 2, a)) - A1[a];
            J2[a] = (1.0 - y) * fma(x, e(2, 1, a) - e(2, 0, a), e(2, 0, a)) +
                    y * fma(x, e(2, 3, a) - e(2, 2, a), e(2, 2, a));
          }
#pragma unroll
          for (int qz = 0; qz < N1; ++qz) {
            point(qx, qy, qz, [&](double gx, double gy, double gz, double& fx, double& fy, double& fz) {
              const double z = tab.xq[qz];
              double J[3][3];
#pragma unroll
              for (int a = 0; a < 3; ++a) {
                J[a][0] = fma(z, B0[a], A0[a]);
                J[a][1] = fma(z, B1[a], A1[a]);
                J[a][2] = J2[a];
              }
              double C[3][3];
              C[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
              C[0][1] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
              C[0][2] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
              C[1][0] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
              C[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
              C[1][2] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
              C[2][0] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
              C[2][1] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
              C[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
              const double det = J[0][0] * C[0][0] + J[0][1] * C[0][1] + J[0][2] * C[0][2];
              const double sc = wxy * tab.w[qz] * __drcp_rn(det);
              const double h0 = sc * (C[0][0] * gx + C[0][1] * gy + C[0][2] * gz);
              const double h1 = sc * (C[1][0] * gx + C[1][1] * gy + C[1][2] * gz);
              const double h2 = sc * (C[2][0] * gx + C[2][1] * gy + C[2][2] * gz);
              fx = C[0][0] * h0 + C[1][0] * h1 + C[2][0] * h2;
              fy = C[0][1] * h0 + C[1][1] * h1 + C[2][1] * h2;
              fz = C[0][2] * h0 + C[1][2] * h1 + C[2][2] * h2;
            });
          }
        }
      }
    } else {
      const TG* g0 = geo + blk * (int64_t)NLOC * NG * CB + lane;
#pragma unroll
      for (int q = 0; q < NLOC; ++q) {
        const int qx = q % N1, qy = (q / N1) % N1, qz = DIM == 3 ? q / (N1 * N1) : 0;
        if constexpr (GEO == 3) {
          if (q % SLICE_Q == 0) {
            // slice qz lands in slot qz & 1, completion phase qz >> 1
            mbar_wait(&mbar[qz & 1], (qz >> 1) & 1);
          }
        }
        if constexpr (GEO == 4) {
          if (q == 0) mbar_wait(mbar4, 0);
        }
        point(qx, qy, qz, [&](TA gx, TA gy, TA gz, TA& fx, TA& fy, TA& fz) {
          TA gg[NG];
          if constexpr (GEO == 1) {
            recompute_g(tab, E, qx, qy, qz, gg);
          } else if constexpr (GEO == 3) {
            const double* G = gbuf + ((qz & 1) * SLICE_Q + q % SLICE_Q) * NG * CB + lane;
#pragma unroll
            for (int k = 0; k < NG; ++k) gg[k] = G[k * CB];
          } else if constexpr (GEO == 4) {
            const float2* G2 = reinterpret_cast<const float2*>(wsm) + q * (NG / 2) * CB + lane;
#pragma unroll
            for (int k = 0; k < NG / 2; ++k) {
              const float2 t = G2[k * CB];
              gg[2 * k] = TA(t.x);
              gg[2 * k + 1] = TA(t.y);
            }
          } else if constexpr (kPairedGeo<TG>) {
            // fp32 geometry of the 3D levels is stored in pairs [q][k/2][CB][2]:
            // 8-byte loads, 256 bytes per warp instruction like the fp64 stream
            const float2* G2 = reinterpret_cast<const float2*>(geo) + blk * (int64_t)NLOC * (NG / 2) * CB + lane +
                               q * (NG / 2) * CB;
#pragma unroll
            for (int k = 0; k < NG / 2; ++k) {
              const float2 t = ld_geo<kStream>(G2 + k * CB);
              gg[2 * k] = TA(t.x);
              gg[2 * k + 1] = TA(t.y);
            }
          } else {
            const TG* G = g0 + q * NG * CB;
#pragma unroll
            for (int k = 0; k < NG; ++k) gg[k] = TA(ld_geo<kStream>(G + k * CB));
          }
          if constexpr (DIM == 3) {
            fx = gg[0] * gx + gg[1] * gy + gg[2] * gz;
            fy = gg[1] * gx + gg[3] * gy + gg[4] * gz;
            fz = gg[2] * gx + gg[4] * gy + gg[5] * gz;
          } else {
            fx = gg[0] * gx + gg[1] * gy;
            fy = gg[1] * gx + gg[2] * gy;
          }
        });
        if constexpr (GEO == 3) {
          if (q % SLICE_Q == SLICE_Q - 1 && qz + 2 < N1) {
            // every lane has read slot qz & 1: refill it with slice qz + 2
            __syncwarp();
            if (lane == 0) {
              fence_proxy_async();
              mbar_expect_tx(&mbar[qz & 1], SLICE_BYTES);
              tma_load_1d(gbuf + (qz & 1) * SLICE_Q * NG * CB, gchunk + (qz + 2) * SLICE_Q * NG * CB, SLICE_BYTES,
                          &mbar[qz & 1]);
            }
          }
        }
      }
    }
    // back to the nodal basis: S^T sweeps
    if constexpr (DIM == 3) sweep_axis<2, true, TA>(tS, w);
    sweep_axis<1, true, TA>(tS, w);
    sweep_axis<0, true, TA>(tS, w);
    double energy = 0.0;
    if constexpr (XNB != 0) {
      static_assert(!kEnergy, "warp-neighbour sharing is for the plain apply");
      constexpr unsigned kFull = 0xffffffffu;
      if constexpr (XNB == 2) {
        // scatter-only sharing: the match bits from the first / last indices of every line
#pragma unroll
        for (int line = 0; line < NLINE; ++line) {
          const int gf = kStream ? __ldg(ib + (line * N1) * CB) : ib[(line * N1) * CB];
          const int gl = kStream ? __ldg(ib + (line * N1 + N1 - 1) * CB) : ib[(line * N1 + N1 - 1) * CB];
          const int nbf = __shfl_down_sync(kFull, gf, 1);
          share_r |= ((lane < 31 && gl >= 0 && nbf == gl) ? 1u : 0u) << line;
        }
      }
      // hand the last-node contributions of shared faces to the right neighbour
      if (cellout) share_r = 0;  // deterministic mode keeps every slot: no hand-over (warp-uniform)
      const unsigned share_l = __shfl_up_sync(kFull, share_r, 1);
#pragma unroll
      for (int line = 0; line < NLINE; ++line) {
        const int lf = line * N1, ll = line * N1 + N1 - 1;
        const bool mr = (share_r >> line) & 1u;
        const TA recv = __shfl_up_sync(kFull, mr ? w[ll] : TA(0), 1);
        if (lane > 0 && ((share_l >> line) & 1u)) w[lf] += recv;
      }
    }
    // the index table is re-read (L1/L2 hit) rather than kept live across the
    // sweeps; XNB reads it as one batch (its lane-dependent skips otherwise
    // serialise the reloads: 918 vs 625 us measured) and marks the shared
    // last nodes, which were handed over, as skipped
    int gs[XNB ? NLOC : 1];
    if constexpr (XNB != 0) {
#pragma unroll
      for (int l = 0; l < NLOC; ++l) gs[l] = kStream ? __ldg(ib + l * CB) : ib[l * CB];
#pragma unroll
      for (int line = 0; line < NLINE; ++line)
        if ((share_r >> line) & 1u) gs[line * N1 + N1 - 1] = -1;
    }
#pragma unroll
    for (int l = 0; l < NLOC; ++l) {
      int g;
      if constexpr (XNB != 0)
        g = gs[l];
      else
        g = kStream ? __ldg(ib + l * CB) : ib[l * CB];
      if (g >= 0) {
        // deterministic mode: the cell's result goes to the cell buffer in
        // the idx layout (coalesced), a fixed-order gather sums it later
        if (cellout)
          cellout[(blk * NLOC + l) * CB + lane] = w[l];
        else
          atomicAdd(dst + g, TD(kNeg ? -w[l] : w[l]));
        if constexpr (kEnergy) energy = fma(double(u0[l]), double(w[l]), energy);
      }
    }
    return energy;
  }
};

}  // namespace nnmg
