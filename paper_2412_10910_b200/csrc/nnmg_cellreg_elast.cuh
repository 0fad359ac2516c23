// Register-resident elasticity cell kernel (K2, 3D, NLOC <= 27): one thread
// per (cell, component).
//
// The pencil kernel (nnmg_cellkernel.cuh) keeps every sweep intermediate of
// the 3 x 27 cell values in shared memory; ncu shows it L1/shared-pipe bound
// on C5 (l1tex 92% busy, mio_throttle the top stall, DRAM 33%).  Here a CTA of
// 3 warps owns one block of 32 cells and warp w holds component w of them:
// gather, the three interpolation sweeps, the collocation gradient, the
// transposed sweeps and the scatter all run in registers exactly as the
// Laplace register kernel (nnmg_cellreg.cuh).  Only the quadrature-point
// physics couples the components (mfoperator.py:183-191); it runs per
// z-slice of 9 points with two shared-memory exchanges:
//   A  every thread writes d u_w / d xhat (3 values) at the 9 points;
//   B  thread w evaluates the full stress at points s = w, w+3, w+6 of the
//      slice (so each geometry entry J^-1, |det J| w_q is loaded exactly once)
//      and writes the reference flux of all 3 components;
//   C  every thread reads its component's flux and applies the transposed
//      collocation derivatives.
// Shared memory is [point][component][direction][cell] (cell fastest: no bank
// conflicts), 2 x 20.7 KB per CTA.
#pragma once

#include "nnmg_kernels.cuh"

namespace nnmg {

// block-local node tables (Level::bln_*), see the BLN variant below
struct BlnTables {
  const int* node = nullptr;
  const int* cnt = nullptr;
  const unsigned* slot = nullptr;  // [blk][(nloc+1)/2][cb]: staging positions of local points 2i (low half), 2i+1 (high)
  int kp = 0;
};

template <int P>
struct CellRegElast {
  static constexpr int DIM = 3;
  static constexpr int N1 = P + 1;
  static constexpr int NLOC = N1 * N1 * N1;
  static constexpr int CB = 32;
  static constexpr int NG = DIM * DIM + 1;  // J^-1 row-major, then |det J| w_q
  static constexpr int SLICE = N1 * N1;     // quadrature points per z-slice
  static constexpr int PER = (SLICE + 2) / 3;  // points per thread in phase B
  static constexpr bool kSupported = NLOC <= 27;
  // GSM variant (geometry slices staged by TMA): the flux overwrites the
  // gradients in place, so the second phase buffer holds the current
  // z-slice of J^-1 / dv instead: [exchange | geometry slice | mbarrier]
  static constexpr int KS_BLN = NLOC * CB + NLOC * CB / 8 + 1;  // block-local node staging row (see run)
  __host__ __device__ static constexpr int cmax(int a, int b) { return a > b ? a : b; }
  static constexpr int XB = (cmax(cmax(NLOC * 3 * (CB + 1), SLICE * 9 * CB), 3 * KS_BLN) + 15) / 16 * 16;
  static constexpr int GEO_DOUBLES = SLICE * NG * CB;
  static constexpr int SMEM_GSM = XB + GEO_DOUBLES + 2;
  static constexpr int SMEM_DOUBLES = 2 * SLICE * 9 * CB > SMEM_GSM ? 2 * SLICE * 9 * CB : SMEM_GSM;

  __host__ __device__ static constexpr int at(int i0, int i1, int i2) { return i0 + N1 * (i1 + N1 * i2); }
  __host__ __device__ __forceinline__ static unsigned bln_phys(unsigned k) { return k + (k >> 3); }

  template <int K, bool TRANS, class TA = double>
  __device__ __forceinline__ static void sweep_axis(const TA (&M)[kMaxN1][kMaxN1], TA (&v)[NLOC]) {
    constexpr int S0 = K == 0 ? 1 : (K == 1 ? N1 : N1 * N1);
    constexpr int NL = NLOC / N1;
#pragma unroll
    for (int line = 0; line < NL; ++line) {
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

  // one cell block; threads: w = threadIdx.x / 32 (component), lane = cell.
  // GEO 0: J^-1 and |det J| w streamed from HBM.  GEO 2 (Q2): J recomputed
  // from the cell's 12 edge vectors (`geo` is then the edge table
  // [blk][36][CB]): 288 B per cell instead of 2,160 B.  In phase B thread w
  // evaluates the points (qx, qy) = (w, k) of each z-slice, so on the
  // trilinear map dx/dz is affine in qy, dx/dy constant per slice and dx/dx
  // affine in qy per slice; with cofactors C: J^-1 = C^T / det,
  // pg = g C^T / det and flux = w_q sigma C.
  // TV / TG: storage types of the vectors and of the stored geometry (double,
  // or float in the mixed-precision V-cycle); the arithmetic is fp64
  // XCH (node-major exchange): the gather and the scatter go through shared
  // memory so that the 96 threads of the CTA access global memory as
  // (cell = t / 3, component = t % 3): the three components of a node are
  // adjacent in the interleaved vector, so a warp instruction touches ~16
  // sectors instead of 32 (the component-per-warp mapping), halving the L1
  // wavefronts of the two scattered phases (ncu r1: L1 80% busy).
  // padded row of the exchange buffer [l][comp][XS].  Node-major thread t
  // touches row t % 3, column t / 3: with 3 XS = 1 (mod 16) its 8-byte bank is
  // XS t (mod 16), a bijection over any 16 consecutive threads, so the
  // node-major side is conflict-free like the lane-contiguous side (XS = 33
  // measured 3.5k shared wavefronts per CTA against 2.6k of payload).  The
  // TMA-staged variant keeps 33: its exchange shares the 48 KB with a
  // geometry slice.
  template <bool GSM>
  __host__ __device__ static constexpr int xs() {
    return GSM ? CB + 1 : CB + 11;
  }
  static_assert(NLOC * 3 * (CB + 11) <= SMEM_DOUBLES && NLOC * 3 * (CB + 1) <= XB, "exchange buffer fits");

  // GSM (GEO 0): the block's stored geometry is streamed through shared
  // memory one z-slice at a time by TMA bulk copies (cp.async.bulk +
  // mbarrier): slice 0 is in flight during the gather and the interpolation
  // sweeps, slice qz+1 during phase C of slice qz and phase A of slice qz+1,
  // so phase B reads J^-1 / dv from shared memory instead of waiting on 30
  // global loads per thread (ncu r2: long scoreboard 3.6 warps per issue, the
  // phase-B DFMAs on top of the sampled stalls).
  // BLN (block-local nodes): the 32 cells of a block share most of their
  // nodes (585 distinct of 864 slots on a structured Q2 row), and consecutive
  // list entries are mostly consecutive in memory.  The CTA gathers the
  // block's distinct node values once into shared memory (thread i -> entry
  // i / 3, component i % 3: contiguous runs instead of 27 scattered warp
  // loads per thread), every thread picks its 27 values by list position, and
  // after the transposed sweeps thread i sums the slots of entry i / 3 in a
  // fixed order and issues ONE atomic per node component and block.
  // TA: the arithmetic type (double; float = single-precision arithmetic of
  // the mixed-precision V-cycle: registers, the exchange buffers and with
  // them the L1 wavefronts of the three phases halve)
  // XNB (with XCH): x-adjacent cells of the block share the last x-node of
  // every line with the next cell's first one where the index tables say so
  // (checked per line and cell pair, any mesh): the shared value is read from
  // the left neighbour's exchange slot instead of gathered, and the shared
  // contribution is added into the right neighbour's first node instead of
  // scattered: N1^2 of the N1^3 gathers and atomics per cell and component.
  template <bool kNeg, int GEO = 0, class TV, class TG, bool XCH = false, bool GSM = false, bool BLN = false,
            class TA = double, bool XNB = false>
  __device__ __forceinline__ static void run(const Tables& tab, const TV* __restrict__ src, TV* __restrict__ dst,
                                             const int* __restrict__ idx, const TG* __restrict__ geo, int64_t blk,
                                             double lam, double mu, double* sm, double* __restrict__ cellout = nullptr,
                                             const BlnTables bln = {}) {
    static_assert(GEO == 0 || sizeof(TG) == sizeof(double), "edge recompute reads fp64 edges");
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    static_assert(GEO == 0 || N1 == 3, "edge recompute relies on qx == component in phase B");
    constexpr int NE = 36;
    if (w == 0 && lane == 0) {
      if constexpr (GEO == 0) {
        constexpr unsigned kGeoBytes = unsigned(NLOC) * NG * CB * sizeof(TG);
        if constexpr (!GSM) prefetch_l2_bulk(geo + blk * (int64_t)NLOC * NG * CB, kGeoBytes);
      } else {
        prefetch_l2_bulk(geo + blk * (int64_t)NE * CB, unsigned(NE) * CB * sizeof(double));
      }
    }
    static_assert(!GSM || GEO == 0, "TMA staging streams the stored geometry");
    static_assert(sizeof(TA) == sizeof(double) || (GEO == 0 && !BLN && !GSM),
                  "single-precision arithmetic: stored geometry, node-major exchange (the buffers are sized in TA)");
    constexpr int XS = xs<GSM>();
    TA* gbuf = reinterpret_cast<TA*>(sm);  // [SLICE][3 comps][3 dirs][CB]
    TA* fbuf = GSM ? gbuf : gbuf + SLICE * 9 * CB;  // same layout, reference flux (GSM: in place)
    TA* smt = gbuf;                        // node-major exchange buffer [l][comp][XS]
    const auto& tS = TabSel<TA>::S(tab);
    const auto& tDc = TabSel<TA>::Dc(tab);
    const TA lamT = TA(lam), muT = TA(mu);
    const TG* gsm = reinterpret_cast<const TG*>(sm + XB);  // GSM: [SLICE][NG][CB] of the current slice
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + XB + GEO_DOUBLES);
    constexpr unsigned kSliceBytes = unsigned(SLICE) * NG * CB * sizeof(TG);
    const TG* gblock = geo + blk * (int64_t)NLOC * NG * CB;
    if constexpr (GSM) {
      if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_proxy_async();
        mbar_expect_tx(bar, kSliceBytes);
        tma_load_1d(sm + XB, gblock, kSliceBytes, bar);
      }
    }
    TA v[NLOC];
    const int* ib = idx + blk * NLOC * CB + lane;
    // node-major exchange coordinates of this thread: cell xc, component xw
    const int xc = threadIdx.x / 3, xw = threadIdx.x % 3;
    // BLN staging layout: component-major rows of KS doubles, entry k at
    // k + k / 8.  At one local index the 32 cells of a structured Q2 block sit
    // 8 list entries apart for the block's own nodes (conflict-free with the
    // skew), 4 or 2 for nodes of the previous row / layer / edge (2- to 4-way
    // conflicts remain: ncu 57k extra shared wavefronts per SM).  A plain
    // [k][comp] layout measured 16-way conflicts; an xor swizzle
    // k ^ (k >> 4 & 15) removes the conflicts but its per-entry address
    // arithmetic spills at the 168-register cap (measured 227 vs 208 us).
    constexpr int KS = KS_BLN;
    static_assert(!BLN || 3 * KS <= SMEM_DOUBLES, "node staging fits");
    static_assert(!(BLN && GSM) || 3 * KS <= XB, "node staging fits beside the geometry slice");
    // entry xc + CB j sits at xc + xc / 8 + (CB + CB / 8) j: one base register, immediate offsets
    const int xbase = xw * KS + xc + (xc >> 3);
    const int bK = BLN ? bln.cnt[blk] : 0;
    const int* bnode = BLN ? bln.node + blk * (int64_t)bln.kp : nullptr;
    if constexpr (BLN) {
      static_assert(XCH, "block-local nodes replace the node-major exchange");
      // the block's distinct node values: thread t loads entries t/3 + 32 j,
      // component t % 3 (at most NLOC rounds: 3 CB threads, <= NLOC CB
      // entries); every load of a round set is in flight together
      const int n3 = bK * 3;
      // unconditional ordered loads (clamped addresses), so that the rounds
      // of a batch are in flight together: first the node ids, then the
      // values; two batches bound the live addresses (one batch spills)
      constexpr int NB = (NLOC + 1) / 2;
#pragma unroll
      for (int j0 = 0; j0 < NLOC; j0 += NB) {
        int nd[NB];
        double val[NB];
#pragma unroll
        for (int j = 0; j < NB; ++j)
          nd[j] = j0 + j < NLOC ? ld_nc_ordered(bnode + min(xc + CB * (j0 + j), bln.kp - 1)) : -1;
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          nd[j] = j0 + j < NLOC && threadIdx.x + 96 * (j0 + j) < n3 ? nd[j] : -1;
          if (j0 + j < NLOC) val[j] = double(ld_nc_ordered(src + (int64_t)max(nd[j], 0) * 3 + xw));
        }
#pragma unroll
        for (int j = 0; j < NB; ++j)
          if (j0 + j < NLOC && nd[j] >= 0) sm[xbase + (CB + CB / 8) * (j0 + j)] = val[j];
      }
      __syncthreads();
      constexpr int NP = (NLOC + 1) / 2;
      const unsigned* bs = bln.slot + blk * (int64_t)(NP * CB) + lane;
      unsigned kk[NP];
#pragma unroll
      for (int i = 0; i < NP; ++i) kk[i] = ld_nc_ordered(bs + i * CB);
#pragma unroll
      for (int l = 0; l < NLOC; ++l) {
        const unsigned k = (l & 1) ? kk[l / 2] >> 16 : kk[l / 2] & 0xFFFFu;
        v[l] = k != 0xFFFFu ? sm[w * KS + k] : 0.0;
      }
      __syncthreads();  // phase A reuses the buffer
    } else if constexpr (XCH && XNB) {
      static_assert(!BLN && !GSM, "warp-neighbour sharing extends the plain node-major exchange");
      constexpr int NLINE = NLOC / N1;
      const int* xb = idx + blk * NLOC * CB + xc;
      {
        // node-major thread (cell xc, component xw): all indices first, then the values
        int g[NLOC], gleft[NLINE];
#pragma unroll
        for (int l = 0; l < NLOC; ++l) g[l] = __ldg(xb + l * CB);
#pragma unroll
        for (int q = 0; q < NLINE; ++q) gleft[q] = xc > 0 ? __ldg(xb + (q * N1 + N1 - 1) * CB - 1) : -2;
#pragma unroll
        for (int l = 0; l < NLOC; ++l) {
          const bool shared = l % N1 == 0 && g[l] >= 0 && gleft[l / N1] == g[l];
          smt[(l * 3 + xw) * XS + xc] =
              (g[l] >= 0 && !shared) ? TA(__ldg(src + (int64_t)g[l] * 3 + xw)) : TA(0);
        }
      }
      __syncthreads();
      {
        // component thread (w, cell lane): the first node of a shared line comes from the left cell's last node
        int gf[NLINE], gleft[NLINE];
#pragma unroll
        for (int q = 0; q < NLINE; ++q) {
          gf[q] = __ldg(ib + (q * N1) * CB);
          gleft[q] = lane > 0 ? __ldg(ib + (q * N1 + N1 - 1) * CB - 1) : -2;
        }
#pragma unroll
        for (int l = 0; l < NLOC; ++l) {
          const bool shared = l % N1 == 0 && gf[l / N1] >= 0 && gleft[l / N1] == gf[l / N1];
          v[l] = shared ? smt[((l + N1 - 1) * 3 + w) * XS + lane - 1] : smt[(l * 3 + w) * XS + lane];
        }
      }
      __syncthreads();  // phase A reuses the buffer
    } else if constexpr (XCH) {
      const int* xb = idx + blk * NLOC * CB + xc;
#pragma unroll
      for (int l = 0; l < NLOC; ++l) {
        const int g = __ldg(xb + l * CB);
        smt[(l * 3 + xw) * XS + xc] = g >= 0 ? TA(__ldg(src + (int64_t)g * 3 + xw)) : TA(0);
      }
      __syncthreads();
#pragma unroll
      for (int l = 0; l < NLOC; ++l) v[l] = smt[(l * 3 + w) * XS + lane];
      __syncthreads();  // phase A reuses the buffer
    } else {
#pragma unroll
      for (int l = 0; l < NLOC; ++l) {
        const int g = __ldcs(ib + l * CB);
        v[l] = g >= 0 ? TA(__ldg(src + (int64_t)g * 3 + w)) : TA(0);
      }
    }
    sweep_axis<0, false, TA>(tS, v);
    sweep_axis<1, false, TA>(tS, v);
    sweep_axis<2, false, TA>(tS, v);
    TA acc[NLOC];
#pragma unroll
    for (int l = 0; l < NLOC; ++l) acc[l] = 0;
    const TG* gb = geo + blk * (int64_t)NLOC * NG * CB + lane;
    const TG* eb = geo + blk * (int64_t)NE * CB + lane;
    auto e = [&](int b, int k, int a) { return double(__ldg(eb + ((b * 4 + k) * 3 + a) * CB)); };
    // GEO 2: dx/dz at (qx = w, y) = A2 + y B2 (edges along z, k = x + 2y)
    double A2[3], B2[3];
    if constexpr (GEO == 2) {
      const double x = tab.xq[w];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        A2[a] = fma(x, e(2, 1, a) - e(2, 0, a), e(2, 0, a));
        B2[a] = fma(x, e(2, 3, a) - e(2, 2, a), e(2, 2, a)) - A2[a];
      }
    }
#pragma unroll
    for (int qz = 0; qz < N1; ++qz) {
      // GEO 2: per slice dx/dy at (x = w, z) and dx/dx = A0 + y B0 at z
      double J1[3], A0[3], B0[3];
      if constexpr (GEO == 2) {
        const double x = tab.xq[w], z = tab.xq[qz];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          // edges along y: k = x + 2z;  along x: k = y + 2z
          const double lo1 = fma(x, e(1, 1, a) - e(1, 0, a), e(1, 0, a));
          const double hi1 = fma(x, e(1, 3, a) - e(1, 2, a), e(1, 2, a));
          J1[a] = fma(z, hi1 - lo1, lo1);
          const double y0 = fma(z, e(0, 2, a) - e(0, 0, a), e(0, 0, a));  // y = 0
          const double y1 = fma(z, e(0, 3, a) - e(0, 1, a), e(0, 1, a));  // y = 1
          A0[a] = y0;
          B0[a] = y1 - y0;
        }
      }
      // A: d u_w / d xhat_j at the slice's points (collocation)
#pragma unroll
      for (int s = 0; s < SLICE; ++s) {
        const int qx = s % N1, qy = s / N1;
        TA gx = 0, gy = 0, gz = 0;
#pragma unroll
        for (int r = 0; r < N1; ++r) {
          gx = fma(tDc[qx][r], v[at(r, qy, qz)], gx);
          gy = fma(tDc[qy][r], v[at(qx, r, qz)], gy);
          gz = fma(tDc[qz][r], v[at(qx, qy, r)], gz);
        }
        TA* o = gbuf + ((s * 3 + w) * 3) * CB + lane;
        o[0] = gx;
        o[CB] = gy;
        o[2 * CB] = gz;
      }
      __syncthreads();
      if constexpr (GSM) mbar_wait(bar, qz & 1);
      // B: full stress at points s = w + 3k of the slice
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int s = w + 3 * k;
        if (s < SLICE) {
          TA g[3][3];
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int j = 0; j < 3; ++j) g[c][j] = gbuf[((s * 3 + c) * 3 + j) * CB + lane];
          TA K[3][3], dv;
          if constexpr (GEO == 2) {
            // J at (qx, qy, qz) = (w, k, qz); K = J^-1 = C^T / det, dv = det w_q
            const double y = tab.xq[k];
            double J[3][3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
              J[a][0] = fma(y, B0[a], A0[a]);
              J[a][1] = J1[a];
              J[a][2] = fma(y, B2[a], A2[a]);
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
            const double rdet = __drcp_rn(det);
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
              for (int b = 0; b < 3; ++b) K[a][b] = C[b][a] * rdet;
            dv = det * (tab.w[w] * tab.w[k] * tab.w[qz]);
          } else if constexpr (GSM) {
            const TG* G = gsm + s * NG * CB + lane;
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
              for (int b = 0; b < 3; ++b) K[a][b] = TA(G[(a * 3 + b) * CB]);
            dv = TA(G[9 * CB]);
          } else {
            const TG* G = gb + (qz * SLICE + s) * NG * CB;
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
              for (int b = 0; b < 3; ++b) K[a][b] = TA(__ldcs(G + (a * 3 + b) * CB));
            dv = TA(__ldcs(G + 9 * CB));
          }
          // pg = ghat J^-1, eps = sym(pg), sigma = 2 mu eps + lam tr(eps) I, flux = sigma J^-T dv
          TA pg[3][3];
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
              TA t = 0;
#pragma unroll
              for (int j = 0; j < 3; ++j) t = fma(g[a][j], K[j][b], t);
              pg[a][b] = t;
            }
          const TA tr = pg[0][0] + pg[1][1] + pg[2][2];
          TA sig[3][3];
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) sig[a][b] = muT * (pg[a][b] + pg[b][a]) + (a == b ? lamT * tr : TA(0));
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              TA t = 0;
#pragma unroll
              for (int b = 0; b < 3; ++b) t = fma(sig[a][b], K[j][b], t);
              fbuf[((s * 3 + a) * 3 + j) * CB + lane] = t * dv;
            }
        }
      }
      __syncthreads();
      if constexpr (GSM) {
        // every thread has read this slice's geometry: refill the buffer
        if (qz + 1 < N1 && threadIdx.x == 0) {
          mbar_expect_tx(bar, kSliceBytes);
          tma_load_1d(sm + XB, gblock + (qz + 1) * SLICE * NG * CB, kSliceBytes, bar);
        }
      }
      // C: transposed collocation derivatives of this component's flux
#pragma unroll
      for (int s = 0; s < SLICE; ++s) {
        const int qx = s % N1, qy = s / N1;
        const TA* f = fbuf + ((s * 3 + w) * 3) * CB + lane;
        const TA fx = f[0], fy = f[CB], fz = f[2 * CB];
#pragma unroll
        for (int r = 0; r < N1; ++r) {
          acc[at(r, qy, qz)] = fma(tDc[qx][r], fx, acc[at(r, qy, qz)]);
          acc[at(qx, r, qz)] = fma(tDc[qy][r], fy, acc[at(qx, r, qz)]);
          acc[at(qx, qy, r)] = fma(tDc[qz][r], fz, acc[at(qx, qy, r)]);
        }
      }
      // the next slice's phase A overwrites gbuf only after every thread
      // passed the phase-B barrier above; fbuf is rewritten after the next
      // phase-A barrier, which every phase-C reader has passed
      // (GSM: the flux lives in gbuf, so phase C must finish first)
      if constexpr (GSM) {
        if (qz + 1 < N1) __syncthreads();
      }
    }
    sweep_axis<2, true, TA>(tS, acc);
    sweep_axis<1, true, TA>(tS, acc);
    sweep_axis<0, true, TA>(tS, acc);
    if constexpr (BLN) {
      if (!cellout) {
        // block-local sums in shared memory without atomics: warp w owns
        // component w of every list entry, and within one local index l the
        // 32 cells of a block hold 32 distinct nodes (checked at setup), so
        // the read-modify-write of pass l is conflict-free; passes are
        // ordered by __syncwarp.  Then one atomic per node component and block,
        // entries in list order (contiguous runs).
        __syncthreads();  // every thread is done with the phase buffers
        // re-read rather than kept live across the sweeps (the kernel sits at its register cap)
        const int n3 = ld_nc_ordered(bln.cnt + blk) * 3;
#pragma unroll
        for (int j = 0; j < NLOC; ++j)
          if (threadIdx.x + 96 * j < n3) sm[xbase + (CB + CB / 8) * j] = 0.0;
        constexpr int NP = (NLOC + 1) / 2;
        const unsigned* bs = bln.slot + blk * (int64_t)(NP * CB) + lane;
        unsigned kk[NP];
#pragma unroll
        for (int i = 0; i < NP; ++i) kk[i] = ld_nc_ordered(bs + i * CB);
        __syncthreads();
#pragma unroll
        for (int l = 0; l < NLOC; ++l) {
          const unsigned k = (l & 1) ? kk[l / 2] >> 16 : kk[l / 2] & 0xFFFFu;
          if (k != 0xFFFFu) sm[w * KS + k] += acc[l];
          __syncwarp();
        }
        int nd[NLOC];
#pragma unroll
        for (int j = 0; j < NLOC; ++j) nd[j] = ld_nc_ordered(bnode + min(xc + CB * j, bln.kp - 1));
        __syncthreads();
#pragma unroll
        for (int j = 0; j < NLOC; ++j)
          if (threadIdx.x + 96 * j < n3 && nd[j] >= 0) {
            const double a = sm[xbase + (CB + CB / 8) * j];
            atomicAdd(dst + (int64_t)nd[j] * 3 + xw, TV(kNeg ? -a : a));
          }
        return;
      }
    }
    if constexpr (XCH) {
      if (!cellout) {
        __syncthreads();  // every thread is done with the phase buffers
#pragma unroll
        for (int l = 0; l < NLOC; ++l) smt[(l * 3 + w) * XS + lane] = acc[l];
        __syncthreads();
        const int* xb = idx + blk * NLOC * CB + xc;
        if constexpr (XNB) {
          constexpr int NLINE = NLOC / N1;
          int g[NLOC], gleft[NLINE], gright[NLINE];
#pragma unroll
          for (int l = 0; l < NLOC; ++l) g[l] = __ldg(xb + l * CB);
#pragma unroll
          for (int q = 0; q < NLINE; ++q) {
            gleft[q] = xc > 0 ? __ldg(xb + (q * N1 + N1 - 1) * CB - 1) : -2;
            gright[q] = xc < CB - 1 ? __ldg(xb + (q * N1) * CB + 1) : -2;
          }
#pragma unroll
          for (int l = 0; l < NLOC; ++l) {
            TA a = smt[(l * 3 + xw) * XS + xc];
            if (l % N1 == 0 && g[l] >= 0 && gleft[l / N1] == g[l]) a += smt[((l + N1 - 1) * 3 + xw) * XS + xc - 1];
            const bool handed = l % N1 == N1 - 1 && gright[l / N1] == g[l];  // the right cell adds and scatters it
            if (g[l] >= 0 && !handed) atomicAdd(dst + (int64_t)g[l] * 3 + xw, TV(kNeg ? -a : a));
          }
          return;
        }
#pragma unroll
        for (int l = 0; l < NLOC; ++l) {
          const int g = __ldg(xb + l * CB);
          const TA a = smt[(l * 3 + xw) * XS + xc];
          if (g >= 0) atomicAdd(dst + (int64_t)g * 3 + xw, TV(kNeg ? -a : a));
        }
        return;
      }
    }
#pragma unroll
    for (int l = 0; l < NLOC; ++l) {
      const int g = __ldg(ib + l * CB);
      if (g >= 0) {
        if (cellout)  // deterministic mode: cell buffer [blk][l][comp][CB]
          cellout[((blk * NLOC + l) * 3 + w) * CB + lane] = acc[l];
        else
          atomicAdd(dst + (int64_t)g * 3 + w, TV(kNeg ? -acc[l] : acc[l]));
      }
    }
  }
};

}  // namespace nnmg
