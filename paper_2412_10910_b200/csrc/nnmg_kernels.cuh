// Device-side building blocks of the sum-factorised cell kernels.
//
// Layout conventions:
//   * cells are processed in blocks of CB consecutive cells; a thread block
//     of NPEN*CB threads owns one cell block, thread t = pen*CB + lane works on
//     cell `lane` of the block and on pencil `pen` (a line of N1 tensor-product
//     points along the current sweep direction);
//   * index table  idx[blk][l][CB]   int32 scalar DoF, -1 = constrained/padding;
//   * geometry     geo[blk][q][k][CB] double (k < NG per quadrature point);
//   * shared memory buffers sm[b][c][pos][CB] (cell fastest => conflict free).
// Local / quadrature position pos = i0 + N1*i1 + N1^2*i2 (x fastest) as the
// reference's local DoF order (mesh.py:20-25, mfoperator.py:58-59).
#pragma once

#include "nnmg_common.cuh"

namespace nnmg {

enum Physics : int { kLaplace = 0, kElasticity = 1 };

template <int DIM, int PHYS>
struct GeoCount {
  static constexpr int value = PHYS == kLaplace ? DIM * (DIM + 1) / 2 : DIM * DIM + 1;
};

template <int DIM, int P, int NCOMP>
__host__ __device__ constexpr int cells_per_block() {
  constexpr int N1 = P + 1;
  constexpr int NLOC = ipow(N1, DIM);
  constexpr int NPEN = ipow(N1, DIM - 1);
  return (3 * NCOMP * NLOC * 32 * 8 <= 100 * 1024 && NPEN * 32 <= 1024)   ? 32
         : (3 * NCOMP * NLOC * 16 * 8 <= 100 * 1024 && NPEN * 16 <= 1024) ? 16
                                                                            : 8;
}

template <int DIM, int N1>
struct Pencil {
  static constexpr int NLOC = ipow(N1, DIM);
  static constexpr int NPEN = ipow(N1, DIM - 1);
  // first position of pencil `pen` along direction k
  __device__ __forceinline__ static int base(int k, int pen) {
    if (DIM == 2) return k == 0 ? N1 * pen : pen;
    if (k == 0) return N1 * pen;
    if (k == 1) return (pen % N1) + N1 * N1 * (pen / N1);
    return pen;
  }
  __host__ __device__ static constexpr int stride(int k) { return k == 0 ? 1 : (k == 1 ? N1 : N1 * N1); }
};

// TMA bulk prefetch of a contiguous global range into L2 (sm_90+):
// one instruction, no registers or shared memory held.  bytes % 16 == 0.
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Ordered read-only loads: `asm volatile` keeps their issue order, so a run of
// them stays in flight together instead of being interleaved with their
// consumers (ptxas serialises long unrolled dependent-load chains otherwise)
__device__ __forceinline__ int ld_nc_ordered(const int* p) {
  int v;
  asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned ld_nc_ordered(const unsigned* p) {
  unsigned v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_nc_ordered(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_nc_ordered(const float* p) {
  float v;
  asm volatile("ld.global.nc.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}

// mbarrier + TMA 1D bulk copy (cp.async.bulk) helpers, CTA-local
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

// 16-byte asynchronous global -> shared copy (LDGSTS, cached in L2 only)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// out[q] = sum_i M[q][i] in[i]
template <int N1, class TA>
__device__ __forceinline__ void sweep(const TA (&M)[kMaxN1][kMaxN1], const TA* in, TA* out) {
#pragma unroll
  for (int q = 0; q < N1; ++q) {
    TA s = 0;
#pragma unroll
    for (int i = 0; i < N1; ++i) s = fma(M[q][i], in[i], s);
    out[q] = s;
  }
}

// out[i] = sum_q M[q][i] in[q]
template <int N1, class TA>
__device__ __forceinline__ void sweep_t(const TA (&M)[kMaxN1][kMaxN1], const TA* in, TA* out) {
#pragma unroll
  for (int i = 0; i < N1; ++i) {
    TA s = 0;
#pragma unroll
    for (int q = 0; q < N1; ++q) s = fma(M[q][i], in[q], s);
    out[i] = s;
  }
}

// streaming (evict-first) global load, or a plain load when the data was made
// resident in shared memory (generic pointer)
template <bool kStream, class T>
__device__ __forceinline__ T ld_geo(const T* p) {
  if constexpr (kStream)
    return __ldcs(p);
  else
    return *p;
}

// Quadrature-point physics.  g[c][j] = d u_c / d xhat_j at the point; returns
// the reference-coordinate flux f[c][j] that is integrated against d phi/d xhat_j.
template <int DIM, int NCOMP, int PHYS, int CB, bool kStream = true>
__device__ __forceinline__ void qp_flux(const double* __restrict__ geo, const double (&g)[NCOMP][DIM],
                                        double (&f)[NCOMP][DIM], double lam, double mu) {
#define __ldcs(p) ld_geo<kStream>(p)
  if constexpr (PHYS == kLaplace) {
    // G = J^-1 J^-T |det J| w_q, symmetric (mfoperator.py:106, 118)
    if constexpr (DIM == 3) {
      const double g00 = __ldcs(geo + 0 * CB), g01 = __ldcs(geo + 1 * CB), g02 = __ldcs(geo + 2 * CB);
      const double g11 = __ldcs(geo + 3 * CB), g12 = __ldcs(geo + 4 * CB), g22 = __ldcs(geo + 5 * CB);
      f[0][0] = g00 * g[0][0] + g01 * g[0][1] + g02 * g[0][2];
      f[0][1] = g01 * g[0][0] + g11 * g[0][1] + g12 * g[0][2];
      f[0][2] = g02 * g[0][0] + g12 * g[0][1] + g22 * g[0][2];
    } else {
      const double g00 = __ldcs(geo + 0 * CB), g01 = __ldcs(geo + 1 * CB), g11 = __ldcs(geo + 2 * CB);
      f[0][0] = g00 * g[0][0] + g01 * g[0][1];
      f[0][1] = g01 * g[0][0] + g11 * g[0][1];
    }
  } else {
    // linear elasticity (mfoperator.py:183-191): pg = ghat J^-1, eps = sym(pg),
    // sigma = 2 mu eps + lam tr(eps) I, flux = sigma J^-T |det J| w_q
    double K[DIM][DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int b = 0; b < DIM; ++b) K[a][b] = __ldcs(geo + (a * DIM + b) * CB);
    const double dv = __ldcs(geo + DIM * DIM * CB);
    double pg[DIM][DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int b = 0; b < DIM; ++b) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < DIM; ++j) s = fma(g[a][j], K[j][b], s);
        pg[a][b] = s;
      }
    double tr = 0.0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) tr += pg[a][a];
    double sig[DIM][DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int b = 0; b < DIM; ++b) sig[a][b] = mu * (pg[a][b] + pg[b][a]) + (a == b ? lam * tr : 0.0);
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int j = 0; j < DIM; ++j) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < DIM; ++b) s = fma(sig[a][b], K[j][b], s);
        f[a][j] = s * dv;
      }
  }
#undef __ldcs
}

// Lagrange basis at the Lobatto nodes evaluated at t (fespace.py:42-51); the
// reference divides by prod(node_i - node_j), here we multiply by the
// precomputed reciprocal (fp64 division is a long instruction sequence)
template <int N1>
__device__ __forceinline__ void lagrange_values(const Tables& tab, double t, double* out) {
  double d[N1];
#pragma unroll
  for (int j = 0; j < N1; ++j) d[j] = t - tab.nodes[j];
#pragma unroll
  for (int i = 0; i < N1; ++i) {
    double v = tab.rdenom[i];
#pragma unroll
    for (int j = 0; j < N1; ++j)
      if (j != i) v *= d[j];
    out[i] = v;
  }
}

}  // namespace nnmg
