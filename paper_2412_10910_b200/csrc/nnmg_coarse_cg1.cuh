// Coarse Jacobi-PCG with ONE grid barrier per iteration (Chronopoulos-Gear
// form of the reference recurrence, solvers.py:129-164, M = D^-1):
//
//   u_k = M r_k,  w_k = A u_k,  gamma_k = (r_k,u_k),  delta_k = (u_k,w_k)
//   beta_k = gamma_k/gamma_{k-1},  alpha_k = gamma_k/(delta_k - beta_k gamma_k/alpha_{k-1})
//   p_k = u_k + beta_k p_{k-1},  s_k = w_k + beta_k s_{k-1}
//   x_{k+1} = x_k + alpha_k p_k,  r_{k+1} = r_k - alpha_k s_k
//
// In exact arithmetic these are the iterates of the standard PCG (same
// alpha, beta, x_k, r_k, same stopping test ||r_k|| <= tol ||r_0||); only the
// rounding differs.  Phase k of the persistent kernel:
//   * gathers form r_k = r_{k-1} - alpha_{k-1}(w_{k-1} + beta_{k-1}s_{k-2}) and
//     u_k = M r_k on the fly, the cell kernel scatters w_k = A u_k and
//     returns the cell energies u_K.(A_K u_K) (delta_k);
//   * owners store s_{k-1}, r_k, p_{k-1}, x_k, accumulate gamma_k and ||r_k||^2,
//     set the constrained rows of w_k and zero the w buffer of phase k+1;
//   * one grid barrier, a fixed-order reduction of (gamma, delta, rr) that
//     every CTA performs identically, the convergence test and the scalars.
// r and s are double-, w triple-buffered so that no phase overwrites what
// another CTA may still gather.
#pragma once

#include "nnmg_cellkernel.cuh"

#include <cooperative_groups.h>

namespace nnmg {

struct Cg1Args {
  Tables tab;
  const int* idx;
  const double* geo;
  int64_t nblk;
  double lam, mu;
  const unsigned char* con;  // 1 on constrained rows
  const double* inv_diag;
  int64_t n;
  const double* b;
  double* x;
  double* r[2];
  double* s[2];
  double* w[3];
  double* p;
  double* part;  // [3][grid]
  int atomic_dots;  // 1: (gamma, delta, rr) accumulated by fp64 atomics into 3 rotating banks
  double reduction;
  int max_iter;
  int prefetch_owned;  // load the owners' operands before the cell phase
  const int* cdofs;    // constrained rows (elasticity's separate pass)
  int64_t ncons;
  int* status;
  unsigned long long* trace;
};

// u = M r_k with r_k = r_{k-1} - alpha (w_{k-1} + beta s_{k-2}) formed on the fly
struct Cg1Src {
  const double* r;
  const double* w;
  const double* s;
  const double* inv_diag;
  double alpha, beta;
  __device__ __forceinline__ double rk(int64_t i) const {
    const double sk = fma(beta, __ldcg(s + i), __ldcg(w + i));
    return fma(-alpha, sk, __ldcg(r + i));
  }
  __device__ __forceinline__ double operator()(int64_t i) const { return __ldg(inv_diag + i) * rk(i); }
};

// phase stamps of CTA 0: SM cycles (the host converts at the SM clock);
// cross-CTA arrival stamps: %globaltimer (ns, common to all SMs)
__device__ __forceinline__ unsigned long long cg1_timer() { return (unsigned long long)clock64(); }
__device__ __forceinline__ unsigned long long cg1_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// SPLIT CTAs share one cell block (SCB = CB / SPLIT cells each): on small
// coarse levels (fewer blocks than SMs) this spreads the cell work over more
// SMs at the price of more barrier participants.
// SPLIT == 0 ("balanced"): CTA r owns the cell range [r nc/R, (r+1) nc/R) of
// all nc = nblk CB block cells, up to 5/4 CB of them (a level with a few more
// cell blocks than SMs would otherwise give some CTAs two whole blocks).
template <int D, int P, int NC, int PH, int SPLIT>
using Cg1Kernel = CellKernel<D, P, NC, PH,
                             (SPLIT > 0 ? CellKernel<D, P, NC, PH>::CB / (SPLIT > 0 ? SPLIT : 1)
                                        : CellKernel<D, P, NC, PH>::CB + CellKernel<D, P, NC, PH>::CB / 4)>;

template <int D, int P, int NC, int PH, int SPLIT>
constexpr size_t cg1_resident_smem() {
  using CK = Cg1Kernel<D, P, NC, PH, SPLIT>;
  return CK::SMEM + size_t(CK::NLOC) * CK::NG * CK::SCB * sizeof(double) +
         ((size_t(CK::NLOC) * CK::SCB + 1) / 2) * sizeof(double);
}

// sum over the (possibly partial last) warp; lane 0 ends with the total
__device__ __forceinline__ void warp_sum3(double& a, double& b, double& c, int nth) {
  const int lane = threadIdx.x & 31;
  const int cnt = min(32, nth - int(threadIdx.x & ~31));
  const unsigned mask = cnt == 32 ? 0xffffffffu : ((1u << cnt) - 1u);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ta = __shfl_down_sync(mask, a, o);
    const double tb = __shfl_down_sync(mask, b, o);
    const double tc = __shfl_down_sync(mask, c, o);
    if (lane + o < cnt) {
      a += ta;
      b += tb;
      c += tc;
    }
  }
}

// OWW > 0: OWW dedicated owner warps (threads 0 .. 32 OWW - 1) run the owner
// updates of phase k while the cell threads (the following warps, their own
// named barrier) run the cell kernel of the same phase.  The two touch
// disjoint buffers within a phase (see the buffer rotation above), exactly as
// the owner pass of one CTA and the cell phase of another already do.
template <int D, int P, int NC, int PH, bool RES, int SPLIT, int OWW = 0>
__global__ void __launch_bounds__(Cg1Kernel<D, P, NC, PH, SPLIT>::NTHREADS + 32 * OWW) k_coarse_cg1(Cg1Args a) {
  using CK = Cg1Kernel<D, P, NC, PH, SPLIT>;
  static_assert(OWW == 0 || RES, "owner warps need the resident-table cell phase");
  constexpr int OT = 32 * OWW;                        // owner threads
  constexpr int CELLW = (CK::NTHREADS + 31) / 32 * 32;  // cell threads, warp-rounded (named barrier count)
  namespace cg = cooperative_groups;
  extern __shared__ double sm[];
  __shared__ double red[3 * 32];
  cg::grid_group grid = cg::this_grid();
  const int rank = blockIdx.x, nrank = gridDim.x;
  const int tid = threadIdx.x, nth = blockDim.x;
  const bool owner_thread = OWW == 0 || tid < OT;
  const bool cell_thread = OWW == 0 || tid >= OT;
  const int ctid = tid - OT;                        // index among the cell threads
  const int otid = OWW ? tid : tid, onth = OWW ? OT : nth;  // owner loop index / stride
  auto csync = [] __device__() {
    if constexpr (OWW > 0)
      asm volatile("bar.sync 1, %0;" ::"n"(CELLW) : "memory");
    else
      __syncthreads();
  };
  constexpr int64_t kGeoChunk = int64_t(CK::NLOC) * CK::NG * CK::SCB;
  constexpr int64_t kIdxChunk = int64_t(CK::NLOC) * CK::SCB;
  double* geo_s = sm + CK::SMEM / sizeof(double);
  int* idx_s = reinterpret_cast<int*>(geo_s + kGeoChunk);
  if constexpr (RES && SPLIT == 0) {
    // this CTA's cell range, padded to SCB with empty cells
    const int64_t ncell = a.nblk * CK::CB;
    const int64_t c0 = ncell * rank / nrank, nmine = ncell * (rank + 1) / nrank - c0;
    for (int64_t k = tid; k < kGeoChunk; k += nth) {
      const int64_t pos = k / CK::SCB, l = k % CK::SCB, c = c0 + l;
      geo_s[k] = l < nmine ? a.geo[((c / CK::CB) * CK::NLOC * CK::NG + pos) * CK::CB + c % CK::CB] : 0.0;
    }
    for (int64_t k = tid; k < kIdxChunk; k += nth) {
      const int64_t pos = k / CK::SCB, l = k % CK::SCB, c = c0 + l;
      idx_s[k] = l < nmine ? a.idx[((c / CK::CB) * CK::NLOC + pos) * CK::CB + c % CK::CB] : -1;
    }
  } else if constexpr (RES) {
    // this CTA's sub-block (lanes sub*SCB ..) of cell block rank / SPLIT
    const int64_t blk = rank / SPLIT;
    const int off = (rank % SPLIT) * CK::SCB;
    for (int64_t k = tid; k < kGeoChunk; k += nth)
      geo_s[k] = a.geo[(blk * CK::NLOC * CK::NG + k / CK::SCB) * CK::CB + off + k % CK::SCB];
    for (int64_t k = tid; k < kIdxChunk; k += nth)
      idx_s[k] = a.idx[(blk * CK::NLOC + k / CK::SCB) * CK::CB + off + k % CK::SCB];
  }
  const int64_t i0 = a.n * rank / nrank, i1 = a.n * (rank + 1) / nrank;
  unsigned long long* trace = (a.trace && rank == 0 && tid == 0) ? a.trace : nullptr;
  // state "phase -1": r_{-1} = b, w_{-1} = s_{-2} = p_{-1} = x_{-1} = 0, alpha = beta = 0
  for (int64_t i = i0 + tid; i < i1; i += nth) {
    a.r[1][i] = a.b[i];
    a.s[0][i] = 0.0;
    a.s[1][i] = 0.0;
    a.w[0][i] = 0.0;
    a.w[1][i] = 0.0;
    a.w[2][i] = 0.0;
    a.p[i] = 0.0;
    a.x[i] = 0.0;
  }
  if (a.atomic_dots && rank == 0 && tid < 12) a.part[tid] = 0.0;
  grid.sync();
  // owners' operands (final since the last barrier) are loaded right after
  // each barrier, ahead of the global reduction and the cell phase, when the
  // owned range fits KO registers per thread (always on the small levels).
  // Laplace only: measured, the live registers slow elasticity's cell phase.
  constexpr int KO = 4;
  constexpr bool kPrefetch = NC == 1;
  constexpr bool kFold = NC == 1;
  const bool fits = owner_thread && kPrefetch && a.prefetch_owned && (i1 - i0) <= KO * (int64_t)onth;
  double rp[KO], wp[KO], so[KO], di[KO], pp[KO], xx[KO];
  bool cf[KO];
  auto load_owned = [&](int k, int64_t i) {
    const double* r = a.r[(k + 1) & 1];
    const double* w = a.w[(k + 2) % 3];
    const double* s = a.s[k & 1];
#pragma unroll
    for (int j = 0; j < KO; ++j) {
      const int64_t ii = i + j * (int64_t)onth;
      if (ii < i1) {
        rp[j] = __ldcg(r + ii);
        wp[j] = __ldcg(w + ii);
        so[j] = __ldcg(s + ii);
        di[j] = a.inv_diag[ii];
        pp[j] = a.p[ii];
        xx[j] = a.x[ii];
        if constexpr (kFold) cf[j] = a.con[ii] != 0;
      }
    }
  };
  // RES: the pencil's DoFs never change, and the raw operands of the next
  // phase's gather (r_{k-1}, w_{k-1}, s_{k-2}, D^-1) are issued right after
  // the barrier too; u_k is formed from them once alpha, beta are known
  constexpr int N1 = CK::N1;
  int gi[N1];
  double gr[NC][N1], gw[NC][N1], gs[NC][N1], gd[NC][N1];
  if constexpr (RES) {
    if (cell_thread) {
      CK::template pencil_dofs<true>(idx_s, 0, ctid, 0, gi);
    } else {
#pragma unroll
      for (int i = 0; i < N1; ++i) gi[i] = -1;
    }
  }
  auto gather = [&](int k) {
    const double* r = a.r[(k + 1) & 1];
    const double* w = a.w[(k + 2) % 3];
    const double* s = a.s[k & 1];
#pragma unroll
    for (int i = 0; i < N1; ++i)
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (gi[i] >= 0) {
          const int64_t j = (int64_t)gi[i] * NC + c;
          gr[c][i] = __ldcg(r + j);
          gw[c][i] = __ldcg(w + j);
          gs[c][i] = __ldcg(s + j);
        }
  };
  if constexpr (RES) {
    // D^-1 at the pencil's DoFs never changes: loaded once, not per phase
#pragma unroll
    for (int i = 0; i < N1; ++i)
#pragma unroll
      for (int c = 0; c < NC; ++c) gd[c][i] = gi[i] >= 0 ? __ldg(a.inv_diag + (int64_t)gi[i] * NC + c) : 0.0;
    gather(0);
  }
  if (fits) load_owned(0, i0 + otid);
  double alpha = 0.0, beta = 0.0, gamma_old = 1.0, alpha_old = 1.0, target = 0.0;
  int status_it = a.max_iter, status_conv = 0, status_err = 0;
  for (int k = 0; k <= a.max_iter; ++k) {
    const int rb_prev = (k + 1) & 1, rb = k & 1;  // r_{k-1}, r_k buffers
    const int sb_old = k & 1, sb_new = (k + 1) & 1;  // s_{k-2} read, s_{k-1} written
    const int wb_prev = (k + 2) % 3, wb = k % 3, wb_next = (k + 1) % 3;
    const Cg1Src src{a.r[rb_prev], a.w[wb_prev], a.s[sb_old], a.inv_diag, alpha, beta};
    if (trace && k < 63) trace[k * 8 + 0] = cg1_timer();
    // cells: w_k = A u_k and energies
    double e = 0.0;
    if constexpr (RES) {
      double v[NC][N1];
#pragma unroll
      for (int i = 0; i < N1; ++i)
#pragma unroll
        for (int c = 0; c < NC; ++c)  // = src(gi * NC + c), bit for bit
          v[c][i] = gi[i] >= 0 ? gd[c][i] * fma(-alpha, fma(beta, gs[c][i], gw[c][i]), gr[c][i]) : 0.0;
      if (cell_thread) e = CK::template run_values<true>(a.tab, gi, v, a.w[wb], geo_s, 0, a.lam, a.mu, sm, ctid, csync);
    } else {
      for (int64_t u = rank; u < a.nblk * SPLIT; u += nrank)
        e += CK::run(a.tab, src, a.w[wb], a.idx, a.geo, u / SPLIT, a.lam, a.mu, sm, tid,
                     [] __device__() { __syncthreads(); }, int(u % SPLIT) * CK::SCB);
    }
    if (trace && k < 63) trace[k * 8 + 5] = cg1_timer();
    // constrained rows w_k[c] = u_k[c] (identity-out, energy u_c^2; no cell
    // scatters into them): Laplace folds them into the owners' pass below,
    // elasticity keeps a separate spread-out pass (measured faster there)
    if constexpr (!kFold) {
      for (int64_t q = (int64_t)rank * onth + otid; owner_thread && q < a.ncons; q += (int64_t)nrank * onth) {
        const int c = a.cdofs[q];
        const double uc = src(c);
        a.w[wb][c] = uc;
        e = fma(uc, uc, e);
      }
    }
    // owners: s_{k-1}, r_k, p_{k-1}, x_k; gamma_k, ||r_k||^2; zero w_{k+1}
    double g = 0.0, rr = 0.0;
    for (int64_t i = i0 + otid; owner_thread && i < i1; i += KO * (int64_t)onth) {
      if (!fits) load_owned(k, i);
#pragma unroll
      for (int j = 0; j < KO; ++j) {
        const int64_t ii = i + j * (int64_t)onth;
        if (ii < i1) {
          const double sk1 = fma(beta, so[j], wp[j]);    // s_{k-1}
          const double rk = fma(-alpha, sk1, rp[j]);     // r_k
          const double pk1 = fma(beta, pp[j], di[j] * rp[j]);  // p_{k-1} = u_{k-1} + beta p_{k-2}
          a.s[sb_new][ii] = sk1;
          a.r[rb][ii] = rk;
          a.p[ii] = pk1;
          a.x[ii] = fma(alpha, pk1, xx[j]);              // x_k
          a.w[wb_next][ii] = 0.0;
          const double uk = di[j] * rk;
          if (kFold && cf[j]) {
            a.w[wb][ii] = uk;
            e = fma(uk, uk, e);
          }
          g = fma(rk, uk, g);
          rr = fma(rk, rk, rr);
        }
      }
    }
    // block reduction of (gamma, delta, rr), then the single grid barrier
    if (trace && k < 63) trace[k * 8 + 7] = cg1_timer();
    warp_sum3(g, e, rr, nth);
    const int wid = tid >> 5, nw = (nth + 31) >> 5;
    __syncthreads();
    if ((tid & 31) == 0) {
      red[wid] = g;
      red[32 + wid] = e;
      red[64 + wid] = rr;
    }
    __syncthreads();
    if (tid == 0) {
      double sg = 0.0, se = 0.0, sr = 0.0;
      for (int i = 0; i < nw; ++i) {
        sg += red[i];
        se += red[32 + i];
        sr += red[64 + i];
      }
      if (a.atomic_dots) {
        // every CTA reading all per-CTA partials after the barrier is a
        // same-line hot spot in L2 (~1.2 us per iteration on 136 CTAs); one
        // fp64 RED per quantity into a rotating bank makes the read a single
        // sector.  Summation order (rounding only) varies run to run.
        double* bank = a.part + (k % 3) * 4;
        atomicAdd(bank + 0, sg);
        atomicAdd(bank + 1, se);
        atomicAdd(bank + 2, sr);
      } else {
        double* part = a.part + (k & 1) * 3 * nrank;  // alternate banks across phases
        part[rank] = sg;
        part[nrank + rank] = se;
        part[2 * nrank + rank] = sr;
      }
    }
    if (trace && k < 63) trace[k * 8 + 1] = cg1_timer();
    // per-CTA arrival times of iterations 8..15 (NNMG_COARSE_TRACE)
    if (a.trace && tid == 0 && k >= 8 && k < 16) a.trace[8 * 64 + (k - 8) * nrank + rank] = cg1_gtimer();
    grid.sync();
    if (trace && k < 63) trace[k * 8 + 2] = cg1_timer();
    // the reduced scalars are the critical path: their load goes out ahead of
    // the next phase's gather / owner prefetches (which queue many sectors)
    const double totv = (a.atomic_dots && tid < 3) ? __ldcg(a.part + (k % 3) * 4 + tid) : 0.0;
    if constexpr (RES) gather(k + 1);
    if (fits) load_owned(k + 1, i0 + otid);
    // every CTA reduces the per-CTA partials in the same fixed order
    __shared__ double tot[3];
    if (a.atomic_dots) {
      if (tid < 3) tot[tid] = totv;
      if (rank == 0 && tid == nth - 1)  // bank of phase k+2 (last read before barrier k)
        for (int j = 0; j < 3; ++j) a.part[((k + 2) % 3) * 4 + j] = 0.0;
    } else if (tid < 32) {
      const double* part = a.part + (k & 1) * 3 * nrank;
      double sg = 0.0, se = 0.0, sr = 0.0;
      for (int i = tid; i < nrank; i += 32) {
        sg += __ldcg(part + i);
        se += __ldcg(part + nrank + i);
        sr += __ldcg(part + 2 * nrank + i);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sg += __shfl_down_sync(0xffffffffu, sg, o);
        se += __shfl_down_sync(0xffffffffu, se, o);
        sr += __shfl_down_sync(0xffffffffu, sr, o);
      }
      if (tid == 0) {
        tot[0] = sg;
        tot[1] = se;
        tot[2] = sr;
      }
    }
    __syncthreads();
    const double gamma = tot[0], delta = tot[1], rrk = tot[2];
    __syncthreads();
    if (trace && k < 63) trace[k * 8 + 3] = cg1_timer();
    if (k == 0) {
      const double norm0 = sqrt(rrk);
      if (norm0 == 0.0) {
        status_it = 0;
        status_conv = 1;
        break;
      }
      target = a.reduction * norm0;
    } else if (sqrt(rrk) <= target) {
      status_it = k;
      status_conv = 1;
      break;
    }
    if (k == a.max_iter) break;
    double bk, den;
    if (k == 0) {
      bk = 0.0;
      den = delta;
    } else {
      bk = gamma / gamma_old;
      den = delta - bk * gamma / alpha_old;
    }
    if (!(den > 0.0)) {
      status_it = k + 1;
      status_err = 1;
      break;
    }
    const double ak = gamma / den;
    alpha = ak;
    beta = bk;
    alpha_old = ak;
    gamma_old = gamma;
    if (trace && k < 63) trace[k * 8 + 4] = cg1_timer();
  }
  if (rank == 0 && tid == 0) {
    a.status[0] = status_it;
    a.status[1] = status_conv;
    a.status[2] = status_err;
  }
}

}  // namespace nnmg
