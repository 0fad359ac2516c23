// The sum-factorised cell kernel (K1/K2) as a reusable device building block.
#pragma once

#include "nnmg_kernels.cuh"

namespace nnmg {

// NNMG_CELL_TRACE builds (diagnostic only): thread 0 of CTA 0 accumulates the
// SM cycles spent between the cell kernel's barriers, per phase
#ifdef NNMG_CELL_TRACE
__device__ unsigned long long nnmg_cell_trace[16];
#define NNMG_CT(i)                                          \
  do {                                                      \
    if (_ct_on) {                                           \
      const unsigned long long _now = clock64();            \
      _ct[(i)] = _now - _ct_last;                           \
      _ct_last = _now;                                      \
    }                                                       \
  } while (0)
#define NNMG_CT_BEGIN                                                    \
  const bool _ct_on = threadIdx.x == 0 && blockIdx.x == 0;               \
  unsigned long long _ct[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};      \
  unsigned long long _ct_last = clock64()
#define NNMG_CT_END                                                           \
  do {                                                                        \
    if (_ct_on) {                                                             \
      for (int _i = 1; _i < 12; ++_i) nnmg_cell_trace[_i] += _ct[_i];         \
      nnmg_cell_trace[14] += 1;                                               \
    }                                                                         \
  } while (0)
#else
#define NNMG_CT(i) \
  do {             \
  } while (0)
#define NNMG_CT_BEGIN \
  do {                \
  } while (0)
#define NNMG_CT_END \
  do {              \
  } while (0)
#endif

// ---------------------------------------------------------------------------
// K1/K2: the sum-factorised cell kernel.  One thread block per block of CB
// cells; gather -> interpolate to quadrature points (S sweeps) -> collocation
// gradient (Dc sweeps) -> quadrature-point physics -> transposed sweeps ->
// scatter-add.  Reproduces LaplaceOperator.apply (mfoperator.py:108-122) and
// ElasticityOperator.apply (mfoperator.py:171-202); the gradient D u is formed
// as Dc (S u), mathematically identical to the reference's D sweeps.
// ---------------------------------------------------------------------------
// SCB_ > 0: one thread group handles a sub-block of SCB_ of the CB cells of a
// block (lanes lane_off .. lane_off+SCB_-1), so a block can be spread over
// several CTAs (latency-bound coarse levels); the HBM layout keeps CB.
// reciprocal in the arithmetic type
__device__ __forceinline__ double rcp_rn(double x) { return __drcp_rn(x); }
__device__ __forceinline__ float rcp_rn(float x) { return __frcp_rn(x); }

// stored-geometry physics exists in fp64 only; the single-precision cell
// kernel recomputes its geometry (GEO 2) and never reaches this call
template <int DIM, int NCOMP, int PHYS, int CB, bool kStream, class TA>
__device__ __forceinline__ void qp_flux_any(const double* __restrict__ geo, const TA (&g)[NCOMP][DIM],
                                            TA (&f)[NCOMP][DIM], double lam, double mu) {
  if constexpr (sizeof(TA) == sizeof(double)) qp_flux<DIM, NCOMP, PHYS, CB, kStream>(geo, g, f, lam, mu);
}

// TA: the arithmetic and shared-memory type (double; float = the single-
// precision arithmetic of the mixed-precision V-cycle, GEO 2 only)
template <int DIM, int P, int NCOMP, int PHYS, int SCB_ = 0, class TA = double>
struct CellKernel {
  static constexpr int N1 = P + 1;
  static constexpr int NLOC = ipow(N1, DIM);
  static constexpr int NPEN = ipow(N1, DIM - 1);
  static constexpr int CB = cells_per_block<DIM, P, NCOMP>();
  static constexpr int SCB = SCB_ > 0 ? SCB_ : CB;
  static constexpr int NG = GeoCount<DIM, PHYS>::value;
  static constexpr int NTHREADS = NPEN * SCB;
  static constexpr int NBUF = 3;
  static constexpr size_t SMEM = size_t(NBUF) * NCOMP * NLOC * SCB * sizeof(TA);
  // geometry modes (template GEO of run / run_values):
  //   0  stored G / J^-1 streamed from HBM (L2 bulk prefetch)
  //   1  stored, the sub-block's rows staged in shared memory (LDGSTS) behind SMEM
  //   2  3D Laplace: G recomputed from the cell's 12 edge vectors (36 doubles,
  //      staged in shared memory behind SMEM) - 288 B per cell instead of
  //      NLOC*6*8 (6 KB for Q4), traded for ~60 FP64 operations per point
  static constexpr int NE = DIM * (1 << (DIM - 1)) * DIM;
  static constexpr size_t GEO_SMEM = size_t(NLOC) * NG * SCB * sizeof(double);
  static constexpr size_t EDGE_SMEM = size_t(NE) * SCB * sizeof(double);
  using PL = Pencil<DIM, N1>;

  __device__ __forceinline__ static TA& S(TA* sm, int b, int c, int pos, int lane) {
    return sm[((b * NCOMP + c) * NLOC + pos) * SCB + lane];
  }

  template <int K>
  __device__ __forceinline__ static void load(TA* sm, int b, int pen, int lane, TA (&v)[NCOMP][N1]) {
    const int base = PL::base(K, pen);
#pragma unroll
    for (int c = 0; c < NCOMP; ++c)
#pragma unroll
      for (int i = 0; i < N1; ++i) v[c][i] = S(sm, b, c, base + i * PL::stride(K), lane);
  }
  template <int K>
  __device__ __forceinline__ static void store(TA* sm, int b, int pen, int lane, const TA (&v)[NCOMP][N1]) {
    const int base = PL::base(K, pen);
#pragma unroll
    for (int c = 0; c < NCOMP; ++c)
#pragma unroll
      for (int i = 0; i < N1; ++i) S(sm, b, c, base + i * PL::stride(K), lane) = v[c][i];
  }
  __device__ __forceinline__ static void op(const TA (&M)[kMaxN1][kMaxN1], TA (&v)[NCOMP][N1], bool trans) {
#pragma unroll
    for (int c = 0; c < NCOMP; ++c) {
      TA t[N1];
      if (trans)
        sweep_t<N1>(M, v[c], t);
      else
        sweep<N1>(M, v[c], t);
#pragma unroll
      for (int i = 0; i < N1; ++i) v[c][i] = t[i];
    }
  }

  // GEO 2 receives the edge-vector table in place of the geometry pointer
  __device__ __forceinline__ static const double* edges_of(const double* p) { return p; }

  // one cell block; the NTHREADS threads tid = 0..NTHREADS-1 of a (sub)group
  // participate, `sync` synchronises exactly that group.  kNC selects the
  // read-only (non-coherent) path for the source vector, which is only legal
  // when no thread of the grid writes it during the kernel.
  // `src(i)` yields source entry i (a plain vector, or a fused expression such
  // as z + beta p inside the coarse CG).  Returns this thread's share of the
  // cell energy sum_l u_l (A_K u)_l over its x-pencil (zero-in applied), so
  // that p.Ap can be formed without waiting for the scatter to complete.
  // kRes: idx/geo point at a shared-memory copy of this block's tables
  // kNeg: scatter -A_K u (dst -= A u, used to update residuals in place)
  // global DoF indices of this thread's x-pencil nodes (-1: constrained / padding)
  template <bool kRes = false>
  __device__ __forceinline__ static void pencil_dofs(const int* __restrict__ idx, int64_t blk, int tid, int lane_off,
                                                     int (&gi)[N1]) {
    constexpr int GS = kRes ? SCB : CB;
    const int glane = kRes ? tid % SCB : lane_off + tid % SCB;
    const int base = PL::base(0, tid / SCB);
#pragma unroll
    for (int i = 0; i < N1; ++i) gi[i] = ld_geo<!kRes>(idx + (blk * NLOC + base + i) * GS + glane);
  }

  // TD: storage type of dst (double, or float in the mixed-precision
  // V-cycle); the arithmetic is fp64 either way
  template <bool kRes = false, bool kNeg = false, int GEO = 0, class Src, class Sync, class TD>
  __device__ __forceinline__ static double run(const Tables& tab, const Src& src, TD* __restrict__ dst,
                                               const int* __restrict__ idx, const double* __restrict__ geo,
                                               int64_t blk, double lam, double mu, TA* sm, int tid,
                                               Sync&& sync, int lane_off = 0, double* __restrict__ cellout = nullptr) {
    static_assert(sizeof(TA) == sizeof(double) || GEO == 2, "single-precision arithmetic: recomputed geometry only");
    // the block's geometry chunk (85% of the bytes) is consumed only in phase
    // 5: start streaming it into L2 now so it overlaps gathers and sweeps
    constexpr unsigned kGeoBytes = unsigned(NLOC) * NG * CB * sizeof(double);
    if constexpr (GEO == 2) {
      static_assert(!kRes && DIM == 3 && PHYS == kLaplace, "edge recompute: 3D Laplace apply");
      // asynchronous (LDGSTS) so the gathers below are issued right behind it
      double* es = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + SMEM);
      const double* esrc = edges_of(geo) + blk * (int64_t)NE * CB + lane_off;
      if constexpr ((SCB * sizeof(double)) % 16 == 0) {
        constexpr int CH = SCB * sizeof(double) / 16;
        for (int i = tid; i < NE * CH; i += NTHREADS)
          cp_async16(es + (i / CH) * SCB + (i % CH) * 2, esrc + (int64_t)(i / CH) * CB + (i % CH) * 2);
        cp_async_commit();
      } else {
        for (int i = tid; i < NE * SCB; i += NTHREADS) es[i] = __ldcs(esrc + (int64_t)(i / SCB) * CB + i % SCB);
      }
    } else if constexpr (GEO == 1) {
      // kGeoS: copy the sub-block's geometry rows (SCB doubles of each
      // [q][k] row) into shared memory asynchronously (LDGSTS, L2 only); it
      // lands while the gathers and sweeps run and is waited for before P5
      static_assert(!kRes && (SCB * sizeof(double)) % 16 == 0, "16-byte chunks");
      double* gs = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + SMEM);
      constexpr int CH = SCB * sizeof(double) / 16;
      constexpr int TOT = NLOC * NG * CH;
      const double* gsrc = geo + blk * (int64_t)NLOC * NG * CB + lane_off;
      for (int i = tid; i < TOT; i += NTHREADS) {
        const int row = i / CH, ch = i % CH;
        cp_async16(gs + row * SCB + ch * 2, gsrc + (int64_t)row * CB + ch * 2);
      }
      cp_async_commit();
    } else if (!kRes && lane_off == 0 && tid == 0) {
      prefetch_l2_bulk(geo + blk * (int64_t)NLOC * NG * CB, kGeoBytes);
    }
    int gi[N1];
    pencil_dofs<kRes>(idx, blk, tid, lane_off, gi);
    TA v[NCOMP][N1];
#pragma unroll
    for (int i = 0; i < N1; ++i)
#pragma unroll
      for (int c = 0; c < NCOMP; ++c) v[c][i] = gi[i] >= 0 ? TA(src((int64_t)gi[i] * NCOMP + c)) : TA(0);
    return run_values<kRes, kNeg, GEO>(tab, gi, v, dst, geo, blk, lam, mu, sm, tid, sync, lane_off, cellout);
  }

  // the cell kernel from gathered pencil values v (zero on gi < 0) onwards;
  // callers that can issue the gather early (the coarse CG) enter here
  template <bool kRes = false, bool kNeg = false, int GEO = 0, class Sync, class TD>
  __device__ __forceinline__ static double run_values(const Tables& tab, const int (&gi)[N1],
                                                      TA (&v)[NCOMP][N1], TD* __restrict__ dst,
                                                      const double* __restrict__ geo, int64_t blk, double lam,
                                                      double mu, TA* sm, int tid, Sync&& sync, int lane_off = 0,
                                                      double* __restrict__ cellout = nullptr) {
    const auto& tS = TabSel<TA>::S(tab);
    const auto& tDc = TabSel<TA>::Dc(tab);
    // lsub indexes shared memory (stride SCB); glane indexes the tables:
    // HBM layout (stride CB) or a resident shared copy of the sub-block (SCB)
    NNMG_CT_BEGIN;
    const int lsub = tid % SCB;
    const int pen = tid / SCB;
    constexpr int GS = kRes ? SCB : CB;
    const int glane = kRes ? lsub : lane_off + lsub;
    constexpr int A = 0, GX = 1, GY = 2;
    TA u0[NCOMP][N1];
    // P1: interpolate the x-pencil along x
    {
#pragma unroll
      for (int c = 0; c < NCOMP; ++c)
#pragma unroll
        for (int i = 0; i < N1; ++i) u0[c][i] = v[c][i];
      op(tS, v, false);
      store<0>(sm, A, pen, lsub, v);
    }
    sync();
    NNMG_CT(1);
    if constexpr (DIM == 3) {
      // P2: interpolate along y
      load<1>(sm, A, pen, lsub, v);
      op(tS, v, false);
      store<1>(sm, A, pen, lsub, v);
      sync();
      NNMG_CT(2);
    }
    // P3: interpolate along the last axis -> values at quadrature points
    constexpr int KL = DIM - 1;
    TA gl[NCOMP][N1];
    load<KL>(sm, A, pen, lsub, v);
    op(tS, v, false);
#pragma unroll
    for (int c = 0; c < NCOMP; ++c) sweep<N1>(tDc, v[c], gl[c]);
    store<KL>(sm, A, pen, lsub, v);
    sync();
    NNMG_CT(3);
    // P4: collocation derivatives along x (and y in 3D)
    {
      TA w[NCOMP][N1];
      load<0>(sm, A, pen, lsub, w);
      op(tDc, w, false);
      store<0>(sm, GX, pen, lsub, w);
      if constexpr (DIM == 3) {
        load<1>(sm, A, pen, lsub, w);
        op(tDc, w, false);
        store<1>(sm, GY, pen, lsub, w);
      }
    }
    if constexpr (GEO == 1 || GEO == 2) cp_async_wait_all();
    sync();
    NNMG_CT(4);
    // P5: quadrature-point physics on the last-axis pencil
    {
      const int base = PL::base(KL, pen);
      TA fl[NCOMP][N1];
      TA fx[NCOMP][N1], fy[NCOMP][N1];
      // GEO 2: the z-pencil (qx, qy) = (pen % N1, pen / N1) of the trilinear
      // map: dx/dz is constant along it, dx/dx and dx/dy are affine in z
      TA A0[3], B0[3], A1[3], B1[3], J2[3], wxy = 0;
      if constexpr (GEO == 2) {
        const double* E = reinterpret_cast<const double*>(reinterpret_cast<const char*>(sm) + SMEM) + lsub;
        auto e = [&](int b, int k, int a) { return TA(E[((b * 4 + k) * 3 + a) * SCB]); };
        const int qx = pen % N1, qy = pen / N1;
        const TA x = TA(tab.xq[qx]), y = TA(tab.xq[qy]);
        wxy = TA(tab.w[qx] * tab.w[qy]);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          // edges along b, k = (lower other axis) + 2 (higher other axis)
          J2[a] = (TA(1) - y) * fma(x, e(2, 1, a) - e(2, 0, a), e(2, 0, a)) + y * fma(x, e(2, 3, a) - e(2, 2, a), e(2, 2, a));
          A0[a] = fma(y, e(0, 1, a) - e(0, 0, a), e(0, 0, a));
          B0[a] = fma(y, e(0, 3, a) - e(0, 2, a), e(0, 2, a)) - A0[a];
          A1[a] = fma(x, e(1, 1, a) - e(1, 0, a), e(1, 0, a));
          B1[a] = fma(x, e(1, 3, a) - e(1, 2, a), e(1, 2, a)) - A1[a];
        }
      }
#pragma unroll
      for (int q = 0; q < N1; ++q) {
        const int pos = base + q * PL::stride(KL);
        TA g[NCOMP][DIM], f[NCOMP][DIM];
#pragma unroll
        for (int c = 0; c < NCOMP; ++c) {
          g[c][0] = S(sm, GX, c, pos, lsub);
          if constexpr (DIM == 3) g[c][1] = S(sm, GY, c, pos, lsub);
          g[c][DIM - 1] = gl[c][q];
        }
        if constexpr (GEO == 2) {
          // J = [A0 + z B0 | A1 + z B1 | J2]; G g = (w / det) C^T (C g), C = cofactors
          const TA z = TA(tab.xq[q]);
          TA J[3][3];
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            J[a][0] = fma(z, B0[a], A0[a]);
            J[a][1] = fma(z, B1[a], A1[a]);
            J[a][2] = J2[a];
          }
          TA C[3][3];
          C[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
          C[0][1] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
          C[0][2] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
          C[1][0] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
          C[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
          C[1][2] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
          C[2][0] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
          C[2][1] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
          C[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
          const TA det = J[0][0] * C[0][0] + J[0][1] * C[0][1] + J[0][2] * C[0][2];
          const TA sc = wxy * TA(tab.w[q]) * rcp_rn(det);
          TA h[3];
#pragma unroll
          for (int i = 0; i < 3; ++i) h[i] = sc * (C[i][0] * g[0][0] + C[i][1] * g[0][1] + C[i][2] * g[0][2]);
#pragma unroll
          for (int a = 0; a < 3; ++a) f[0][a] = C[0][a] * h[0] + C[1][a] * h[1] + C[2][a] * h[2];
        } else if constexpr (GEO == 1)
          qp_flux_any<DIM, NCOMP, PHYS, SCB, false>(reinterpret_cast<const double*>(reinterpret_cast<const char*>(sm) + SMEM) + pos * NG * SCB + lsub, g, f, lam, mu);
        else
          qp_flux_any<DIM, NCOMP, PHYS, GS, !kRes>(geo + ((blk * (int64_t)NLOC + pos) * NG) * GS + glane, g, f, lam, mu);
#pragma unroll
        for (int c = 0; c < NCOMP; ++c) {
          fx[c][q] = f[c][0];
          if constexpr (DIM == 3) fy[c][q] = f[c][1];
          fl[c][q] = f[c][DIM - 1];
        }
      }
      // last-axis derivative transpose stays in registers
#pragma unroll
      for (int c = 0; c < NCOMP; ++c) {
        TA t[N1];
        sweep_t<N1>(tDc, fl[c], t);
#pragma unroll
        for (int i = 0; i < N1; ++i) fl[c][i] = t[i];
      }
      store<KL>(sm, GX, pen, lsub, fx);
      if constexpr (DIM == 3) {
        store<KL>(sm, GY, pen, lsub, fy);
        store<KL>(sm, A, pen, lsub, fl);
      } else {
        // 2D: keep the y part in registers (v) for P7
#pragma unroll
        for (int c = 0; c < NCOMP; ++c)
#pragma unroll
          for (int i = 0; i < N1; ++i) v[c][i] = fl[c][i];
      }
    }
    sync();
    NNMG_CT(5);
    if constexpr (DIM == 3) {
      // P6: A += Dc^T fx along x
      {
        TA w[NCOMP][N1], a[NCOMP][N1];
        load<0>(sm, GX, pen, lsub, w);
        op(tDc, w, true);
        load<0>(sm, A, pen, lsub, a);
#pragma unroll
        for (int c = 0; c < NCOMP; ++c)
#pragma unroll
          for (int i = 0; i < N1; ++i) a[c][i] += w[c][i];
        store<0>(sm, A, pen, lsub, a);
      }
      sync();
      NNMG_CT(6);
      // P7: w = A + Dc^T fy along y, then S^T along y
      {
        TA w[NCOMP][N1], a[NCOMP][N1];
        load<1>(sm, GY, pen, lsub, w);
        op(tDc, w, true);
        load<1>(sm, A, pen, lsub, a);
#pragma unroll
        for (int c = 0; c < NCOMP; ++c)
#pragma unroll
          for (int i = 0; i < N1; ++i) a[c][i] += w[c][i];
        op(tS, a, true);
        store<1>(sm, A, pen, lsub, a);
      }
      sync();
      NNMG_CT(7);
      // P8: S^T along z
      load<2>(sm, A, pen, lsub, v);
      op(tS, v, true);
      store<2>(sm, A, pen, lsub, v);
      sync();
      NNMG_CT(8);
    } else {
      // 2D P6: A = Dc^T fx along x
      {
        TA w[NCOMP][N1];
        load<0>(sm, GX, pen, lsub, w);
        op(tDc, w, true);
        store<0>(sm, A, pen, lsub, w);
      }
      sync();
      NNMG_CT(9);
      // 2D P7: w = A + (y part in registers), S^T along y
      {
        TA a[NCOMP][N1];
        load<1>(sm, A, pen, lsub, a);
#pragma unroll
        for (int c = 0; c < NCOMP; ++c)
#pragma unroll
          for (int i = 0; i < N1; ++i) a[c][i] += v[c][i];
        op(tS, a, true);
        store<1>(sm, A, pen, lsub, a);
      }
      sync();
      NNMG_CT(10);
    }
    // final: S^T along x and scatter-add the x-pencil
    load<0>(sm, A, pen, lsub, v);
    op(tS, v, true);
    double energy = 0.0;
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      if (gi[i] >= 0) {
#pragma unroll
        for (int c = 0; c < NCOMP; ++c) {
          if (cellout)  // deterministic mode: cell buffer [blk][l][comp][CB]
            cellout[((blk * NLOC + PL::base(0, pen) + i) * NCOMP + c) * CB + glane] = v[c][i];
          else
            atomicAdd(dst + (int64_t)gi[i] * NCOMP + c, TD(kNeg ? -v[c][i] : v[c][i]));
          energy = fma(double(u0[c][i]), double(v[c][i]), energy);
        }
      }
    }
    NNMG_CT(11);
    NNMG_CT_END;
    return energy;
  }
};

// read-only source vector (never written during the kernel), fp64 or fp32
// storage, read as fp64
template <class T>
struct PlainSrcT {
  const T* __restrict__ s;
  __device__ __forceinline__ T operator()(int64_t i) const { return __ldg(s + i); }
};
using PlainSrc = PlainSrcT<double>;


template <class F>
inline void dispatch(int dim, int degree, int ncomp, int physics, F&& f) {
#define NNMG_CASE(D, P, NC, PH) \
  if (dim == D && degree == P && ncomp == NC && physics == PH) return f.template operator()<D, P, NC, PH>();
#define NNMG_DEG(D, P)                 \
  NNMG_CASE(D, P, 1, kLaplace)         \
  NNMG_CASE(D, P, D, kElasticity)
  NNMG_DEG(2, 1) NNMG_DEG(2, 2) NNMG_DEG(2, 3) NNMG_DEG(2, 4)
  NNMG_DEG(3, 1) NNMG_DEG(3, 2) NNMG_DEG(3, 3) NNMG_DEG(3, 4)
#undef NNMG_DEG
#undef NNMG_CASE
  throw Error{kUnsupported, "unsupported (dim, degree, components, physics) combination"};
}


}  // namespace nnmg
