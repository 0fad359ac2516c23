// K8/K10: coarsest-level solvers (replaces CoarseSolver, solvers.py:167-206).
//
// * dense: x = A^-1 b with the inverse precomputed on the host from a Cholesky
//   factorisation (n <= dense_limit), one warp per row;
// * CG-Jacobi: the reference's cg_solve(op, b, precond=inv_diag, 1e-8, 1e4)
//   (solvers.py:129-164) as ONE persistent cooperative kernel.  Per iteration
//   two grid barriers instead of four:
//     phase A  p_k = z + beta p_{k-1} is formed on the fly inside the cell
//              gather (owners also store it), Ap_k accumulates by scatter, and
//              p.Ap is summed from the per-cell energies p_K.(A_K p_K) plus
//              the constrained rows (identical to p.Ap in exact arithmetic);
//     barrier; phase B  alpha, x += alpha p, r -= alpha Ap, z = D^-1 r, r.r,
//              r.z partial sums, zero the other Ap buffer;
//     barrier; every CTA reduces the partials in the same fixed order, tests
//              ||r|| <= tol ||r0|| and forms beta.
//   Double-buffered p and Ap make the on-the-fly formulation race free.
#include "nnmg_coarse.cuh"
#include "nnmg_cellkernel.cuh"
#include "nnmg_cellreg.cuh"
#include "nnmg_coarse_cg1.cuh"

#include <algorithm>

#include <cooperative_groups.h>
#include <string>

namespace cg = cooperative_groups;

namespace nnmg {

static inline unsigned grid_for(int64_t n, int bs) { return static_cast<unsigned>((n + bs - 1) / bs); }

__global__ void k_dense_solve(const double* __restrict__ ainv, const double* __restrict__ b, double* __restrict__ x,
                              int n) {
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double s = 0.0;
  for (int j = lane; j < n; j += 32) s += ainv[(int64_t)row * n + j] * b[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) x[row] = s;
}

struct Slot;

struct CgArgs {
  Tables tab;
  const int* idx;
  const double* geo;
  int64_t nblk;
  double lam, mu;
  const int* cdofs;
  int64_t ncons;
  const double* inv_diag;
  int64_t n;
  const double* b;
  double* x;
  double *r, *z;
  double* p[2];
  double* ap[2];
  Slot* slots;   // [2][grid] barrier-with-payload banks
  Slot* result;  // [2] root-broadcast results
  int barrier;   // 0 grid.sync, 1 all-to-all, 2 root
  unsigned long long* trace;  // optional per-phase %globaltimer samples (rank 0)
  unsigned long long* solve_epoch;
  double reduction;
  int max_iter;
  int nsub;     // pencil subgroups (cell blocks) per CTA
  int* status;  // iterations, converged, error
};

// p = z + beta p_old, evaluated identically by gathers and owners; the
// operands were written by other CTAs in the previous phase: read them from L2
struct CgSrc {
  const double* z;
  const double* p_old;
  double beta;
  __device__ __forceinline__ double operator()(int64_t i) const { return fma(beta, __ldcg(p_old + i), __ldcg(z + i)); }
};

// Barrier with payload: every CTA publishes two partial sums and an epoch in
// its slot; every CTA polls all slots and sums them in one fixed order, so all
// CTAs leave with bitwise identical totals.  Two slot banks alternate so a
// slot is never overwritten before every CTA has read it.
struct Slot {
  double v[2];
  unsigned long long epoch;
  unsigned long long pad;
};

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// centralised variant: CTA 0 gathers the partials in fixed order and
// publishes one result; the other CTAs poll a single flag
__device__ __forceinline__ void exchange_root(Slot* bank, Slot* result, int rank, int nrank, unsigned long long epoch,
                                              double& a, double& b, double* sh) {
  __syncthreads();
  if (threadIdx.x == 0) {
    bank[rank].v[0] = a;
    bank[rank].v[1] = b;
    __threadfence();
    st_release(&bank[rank].epoch, epoch);
  }
  if (rank == 0 && threadIdx.x < 32) {
    double sa = 0.0, sb = 0.0;
    for (int i = threadIdx.x; i < nrank; i += 32) {
      while (ld_acquire(&bank[i].epoch) < epoch) {
      }
      sa += __ldcg(&bank[i].v[0]);
      sb += __ldcg(&bank[i].v[1]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sa += __shfl_down_sync(0xffffffffu, sa, o);
      sb += __shfl_down_sync(0xffffffffu, sb, o);
    }
    if (threadIdx.x == 0) {
      Slot* r = result + (epoch & 1);
      r->v[0] = sa;
      r->v[1] = sb;
      __threadfence();
      st_release(&r->epoch, epoch);
    }
  }
  if (threadIdx.x == 0) {
    Slot* r = result + (epoch & 1);
    while (ld_acquire(&r->epoch) < epoch) {
    }
    sh[0] = __ldcg(&r->v[0]);
    sh[1] = __ldcg(&r->v[1]);
    __threadfence();
  }
  __syncthreads();
  a = sh[0];
  b = sh[1];
}

__device__ __forceinline__ void exchange(Slot* bank, int rank, int nrank, unsigned long long epoch, double& a,
                                         double& b, double* sh) {
  __syncthreads();  // all of this CTA's writes precede the publish
  if (threadIdx.x == 0) {
    bank[rank].v[0] = a;
    bank[rank].v[1] = b;
    __threadfence();
    st_release(&bank[rank].epoch, epoch);
  }
  if (threadIdx.x < 32) {
    double sa = 0.0, sb = 0.0;
    for (int i = threadIdx.x; i < nrank; i += 32) {
      while (ld_acquire(&bank[i].epoch) < epoch) {
      }
      sa += __ldcg(&bank[i].v[0]);
      sb += __ldcg(&bank[i].v[1]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sa += __shfl_down_sync(0xffffffffu, sa, o);
      sb += __shfl_down_sync(0xffffffffu, sb, o);
    }
    if (threadIdx.x == 0) {
      sh[0] = sa;
      sh[1] = sb;
      __threadfence();
    }
  }
  __syncthreads();
  a = sh[0];
  b = sh[1];
}

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// block-wide fixed-order sum of two values; result valid in every thread
__device__ __forceinline__ void block_sum2(double& a, double& b, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (l == 0) {
    sh[2 * w] = a;
    sh[2 * w + 1] = b;
  }
  __syncthreads();
  double sa = 0.0, sb = 0.0;
  for (int i = 0; i < nw; ++i) {
    sa += sh[2 * i];
    sb += sh[2 * i + 1];
  }
  a = sa;
  b = sb;
}

// sum of part[0..n) (and part2) in one fixed order, identical in every CTA
__device__ __forceinline__ void grid_sum2(const double* part, const double* part2, int n, double& a, double& b,
                                          double* sh) {
  if (threadIdx.x < 32) {
    double sa = 0.0, sb = 0.0;
    for (int i = threadIdx.x; i < n; i += 32) {
      sa += __ldcg(part + i);
      if (part2) sb += __ldcg(part2 + i);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      sa += __shfl_down_sync(0xffffffffu, sa, o);
      sb += __shfl_down_sync(0xffffffffu, sb, o);
    }
    if (threadIdx.x == 0) {
      sh[0] = sa;
      sh[1] = sb;
    }
  }
  __syncthreads();
  a = sh[0];
  b = sh[1];
  __syncthreads();
}

// RES: one cell block per CTA whose index table and geometry stay resident in
// shared memory for the whole solve (they do not change between iterations)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// barrier + fixed-order sum of two per-CTA partials; kind 0: cooperative
// grid.sync, 1: all-to-all slot polling, 2: root gathers and broadcasts
__device__ __forceinline__ void barrier_sum(int kind, Slot* slots, Slot* result, int rank, int nrank,
                                            unsigned long long& ep, double& x, double& y, double* red) {
  ++ep;
  Slot* bank = slots + (ep & 1) * nrank;
  if (kind == 1) {
    exchange(bank, rank, nrank, ep, x, y, red);
  } else if (kind == 2) {
    exchange_root(bank, result, rank, nrank, ep, x, y, red);
  } else {
    __syncthreads();
    if (threadIdx.x == 0) {
      bank[rank].v[0] = x;
      bank[rank].v[1] = y;
    }
    cg::this_grid().sync();
    if (threadIdx.x < 32) {
      double sa = 0.0, sb = 0.0;
      for (int i = threadIdx.x; i < nrank; i += 32) {
        sa += __ldcg(&bank[i].v[0]);
        sb += __ldcg(&bank[i].v[1]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sa += __shfl_down_sync(0xffffffffu, sa, o);
        sb += __shfl_down_sync(0xffffffffu, sb, o);
      }
      if (threadIdx.x == 0) {
        red[0] = sa;
        red[1] = sb;
      }
    }
    __syncthreads();
    x = red[0];
    y = red[1];
    __syncthreads();
  }
}

// MODE 0: pencil cell kernel, tables from L2; 1: pencil, tables resident in
// shared memory (RES); 2: register-resident thread-per-cell kernel, one warp
// per cell block (Laplace, NLOC <= 27)
constexpr int kCgRegThreads = 256;

// at most max_sub() pencil subgroups per CTA.  Two only for scalar Laplace
// (measured: the halved register budget makes the elasticity / Q4 variants
// spill); more cell blocks than max_sub x SMs loop.
template <int D, int P, int NC, int PH>
__host__ __device__ constexpr int max_sub() {
  // measured (C3 coarse, 154 cell blocks): 77 CTAs x 2 subgroups shortened the
  // cell loop (5.0 -> 3.7 us) but lengthened the iteration (12.4 -> 14.4 us)
  return 1;
}

template <int D, int P, int NC, int PH, int MODE>
__global__ void __launch_bounds__(MODE == 2 ? kCgRegThreads : CellKernel<D, P, NC, PH>::NTHREADS * max_sub<D, P, NC, PH>())
    k_coarse_cg(CgArgs a) {
  using CK = CellKernel<D, P, NC, PH>;
  constexpr bool RES = MODE == 1;
  extern __shared__ double sm[];
  __shared__ double red[2 * 32 + 2];
  cg::grid_group grid = cg::this_grid();
  const int rank = blockIdx.x, nrank = gridDim.x;
  const int tid = threadIdx.x, nth = blockDim.x;
  // pencil modes: the CTA holds a.nsub independent subgroups of CK::NTHREADS
  // threads, each owning one cell block (named barriers 1..nsub), so that
  // every cell block of the level is processed in a single round
  const int sub = tid / CK::NTHREADS, stid = tid % CK::NTHREADS;
  constexpr int64_t kGeoChunk = int64_t(CK::NLOC) * CK::NG * CK::CB;
  constexpr int64_t kIdxChunk = int64_t(CK::NLOC) * CK::CB;
  constexpr size_t kSubDoubles = CK::SMEM / sizeof(double) + (RES ? kGeoChunk + (kIdxChunk + 1) / 2 : 0);
  double* sm_sub = sm + sub * kSubDoubles;
  double* geo_s = sm_sub + CK::SMEM / sizeof(double);
  int* idx_s = reinterpret_cast<int*>(geo_s + kGeoChunk);
  const int64_t my_blk = (int64_t)rank * a.nsub + sub;
  if constexpr (RES) {
    if (sub < a.nsub && my_blk < a.nblk) {
      for (int64_t k = stid; k < kGeoChunk; k += CK::NTHREADS) geo_s[k] = a.geo[my_blk * kGeoChunk + k];
      for (int64_t k = stid; k < kIdxChunk; k += CK::NTHREADS) idx_s[k] = a.idx[my_blk * kIdxChunk + k];
    }
    __syncthreads();
  }
  const int bar_id = 1 + sub;
  const int64_t i0 = a.n * rank / nrank, i1 = a.n * (rank + 1) / nrank;
  unsigned long long* trace = (a.trace && rank == 0 && tid == 0) ? a.trace : nullptr;
  unsigned long long ep = __ldcg(a.solve_epoch);  // epochs of this solve start after the last one

  double srr = 0.0, srz = 0.0;
  for (int64_t i = i0 + tid; i < i1; i += nth) {
    const double bi = a.b[i];
    const double zi = a.inv_diag[i] * bi;
    a.x[i] = 0.0;
    a.r[i] = bi;
    a.z[i] = zi;
    a.p[1][i] = 0.0;
    a.ap[1][i] = 0.0;
    a.ap[0][i] = 0.0;
    srr += bi * bi;
    srz += bi * zi;
  }
  block_sum2(srr, srz, red);
  double rr = srr, rz = srz;
  barrier_sum(a.barrier, a.slots, a.result, rank, nrank, ep, rr, rz, red + 64);
  const double norm0 = sqrt(rr);
  int status_it = 0, status_conv = 0, status_err = 0;
  if (norm0 == 0.0) {
    status_conv = 1;
  } else {
    const double target = a.reduction * norm0;
    double beta = 0.0;
    status_it = a.max_iter;
    for (int it = 1; it <= a.max_iter; ++it) {
      const int cur = it & 1, prv = cur ^ 1;
      const CgSrc src{a.z, a.p[prv], beta};
      if (trace) trace[it * 8 + 0] = gtimer();
      // phase A: Ap = A p with p formed on the fly; cell energies
      double e = 0.0;
      if constexpr (MODE == 2) {
        if constexpr (PH == kLaplace && NC == 1 && CellReg<D, P>::kSupported) {
          const int nw = nth >> 5, w = tid >> 5;
          for (int64_t blk = (int64_t)rank * nw + w; blk < a.nblk; blk += (int64_t)nrank * nw)
            e += CellReg<D, P>::template run<false, true>(a.tab, src, a.ap[cur], a.idx, a.geo, blk, tid & 31);
        }
      } else if (sub < a.nsub) {
        auto bar = [bar_id] __device__() {
          if constexpr (CK::NTHREADS % 32 == 0)
            named_sync(bar_id, CK::NTHREADS);
          else
            __syncthreads();  // nsub == 1 whenever the subgroup is not warp-aligned
        };
        if constexpr (RES) {
          if (my_blk < a.nblk) e = CK::template run<true>(a.tab, src, a.ap[cur], idx_s, geo_s, 0, a.lam, a.mu, sm_sub,
                                                          stid, bar);
        } else {
          for (int64_t blk = my_blk; blk < a.nblk; blk += (int64_t)nrank * a.nsub)
            e += CK::run(a.tab, src, a.ap[cur], a.idx, a.geo, blk, a.lam, a.mu, sm_sub, stid, bar);
        }
      }
      if (trace) trace[it * 8 + 5] = gtimer();
      // owners store p (batched: four independent L2 round trips in flight)
      for (int64_t i = i0 + tid; i < i1; i += 4 * (int64_t)nth) {
        double pv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t j = i + k * (int64_t)nth;
          if (j < i1) pv[k] = src(j);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t j = i + k * (int64_t)nth;
          if (j < i1) a.p[cur][j] = pv[k];
        }
      }
      if (trace) trace[it * 8 + 6] = gtimer();
      for (int64_t k = (int64_t)rank * nth + tid; k < a.ncons; k += (int64_t)nrank * nth) {
        const int c = a.cdofs[k];
        const double pc = src(c);
        a.ap[cur][c] = pc;
        e = fma(pc, pc, e);
      }
      if (trace) trace[it * 8 + 7] = gtimer();
      double dummy = 0.0;
      block_sum2(e, dummy, red);
      if (trace) trace[it * 8 + 1] = gtimer();
      barrier_sum(a.barrier, a.slots, a.result, rank, nrank, ep, e, dummy, red + 64);
      if (trace) trace[it * 8 + 2] = gtimer();
      const double pap = e;
      if (!(pap > 0.0)) {
        status_it = it;
        status_err = 1;
        break;
      }
      const double alpha = rz / pap;
      // phase B
      srr = 0.0;
      srz = 0.0;
      // batched by 4 so that four elements' loads are in flight per thread
      for (int64_t i = i0 + tid; i < i1; i += 4 * (int64_t)nth) {
        double xv[4], pv[4], rv[4], av[4], dv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t j = i + k * (int64_t)nth;
          if (j < i1) {
            xv[k] = a.x[j];
            pv[k] = a.p[cur][j];
            rv[k] = a.r[j];
            av[k] = __ldcg(a.ap[cur] + j);
            dv[k] = a.inv_diag[j];
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t j = i + k * (int64_t)nth;
          if (j < i1) {
            a.x[j] = xv[k] + alpha * pv[k];
            const double ri = rv[k] - alpha * av[k];
            const double zi = dv[k] * ri;
            a.r[j] = ri;
            a.z[j] = zi;
            a.ap[prv][j] = 0.0;
            srr += ri * ri;
            srz += ri * zi;
          }
        }
      }
      block_sum2(srr, srz, red);
      double rz_new = srz;
      rr = srr;
      if (trace) trace[it * 8 + 3] = gtimer();
      barrier_sum(a.barrier, a.slots, a.result, rank, nrank, ep, rr, rz_new, red + 64);
      if (trace) trace[it * 8 + 4] = gtimer();
      if (sqrt(rr) <= target) {
        status_it = it;
        status_conv = 1;
        break;
      }
      beta = rz_new / rz;
      rz = rz_new;
    }
  }
  if (rank == 0 && tid == 0) {
    a.status[0] = status_it;
    a.status[1] = status_conv;
    a.status[2] = status_err;
    *a.solve_epoch = ep;  // every CTA has read the base epoch (first exchange)
  }
}

__global__ void k_mark_rows(const int* __restrict__ rows, int64_t n, unsigned char* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) flag[rows[i]] = 1;
}

// the single-barrier kernel for the configured split / residency / owner warps
template <int D, int P, int NC, int PH, int OWW>
static void (*cg1_kernel(const Coarse& C))(Cg1Args) {
  if constexpr (OWW > 0) {
    return C.split == 0   ? k_coarse_cg1<D, P, NC, PH, true, 0, OWW>
           : C.split == 8 ? k_coarse_cg1<D, P, NC, PH, true, 8, OWW>
           : C.split == 4 ? k_coarse_cg1<D, P, NC, PH, true, 4, OWW>
           : C.split == 2 ? k_coarse_cg1<D, P, NC, PH, true, 2, OWW>
                          : k_coarse_cg1<D, P, NC, PH, true, 1, OWW>;
  } else {
    return C.split == 0   ? k_coarse_cg1<D, P, NC, PH, true, 0>
           : C.split == 8 ? k_coarse_cg1<D, P, NC, PH, true, 8>
           : C.split == 4 ? k_coarse_cg1<D, P, NC, PH, true, 4>
           : C.split == 2 ? k_coarse_cg1<D, P, NC, PH, true, 2>
           : C.mode == 1  ? k_coarse_cg1<D, P, NC, PH, true, 1>
                          : k_coarse_cg1<D, P, NC, PH, false, 1>;
  }
}

struct CgLaunch {
  Coarse& C;
  const double* b;
  double* x;
  cudaStream_t s;
  bool configure_only;
  template <int D, int P, int NC, int PH, int S>
  bool try_split(const Level& L, int nsm, int max_split) {
    using CKS = Cg1Kernel<D, P, NC, PH, S>;
    // CTAs per SM allowed for the split grid (NNMG_COARSE_CPS, default 1)
    const char* ec = getenv("NNMG_COARSE_CPS");
    const int cps = ec ? std::max(1, atoi(ec)) : 1;
    if (S > max_split || CellKernel<D, P, NC, PH>::CB % S != 0 || CKS::NTHREADS < 32 ||
        L.nblk * S > int64_t(cps) * nsm)
      return false;
    constexpr size_t ssm = cg1_resident_smem<D, P, NC, PH, S>();
    if (ssm > 200 * 1024) return false;
    auto ks = k_coarse_cg1<D, P, NC, PH, true, S>;
    NNMG_CUDA_TRY(cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
    NNMG_CUDA_TRY(cudaFuncSetAttribute(ks, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       cudaSharedmemCarveoutMaxShared));
    int ps = 0;
    NNMG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, ks, CKS::NTHREADS, ssm));
    if (ps <= 0 || L.nblk * S > int64_t(ps) * nsm) return false;
    C.split = S;
    C.mode = 1;
    C.resident = true;
    C.nsub = 1;
    C.block = CKS::NTHREADS;
    C.smem = ssm;
    C.nrank = static_cast<int>(L.nblk * S);
    return true;
  }

  // a few more cell blocks than SMs: one CTA per SM, each owning an equal
  // cell range (NNMG_COARSE_BALANCE=0 disables)
  template <int D, int P, int NC, int PH>
  bool try_balanced(const Level& L, int nsm) {
    using CKB = Cg1Kernel<D, P, NC, PH, 0>;
    const char* eb = getenv("NNMG_COARSE_BALANCE");
    if ((eb && atoi(eb) == 0) || L.nblk <= nsm || L.nblk * CKB::CB > int64_t(nsm) * CKB::SCB ||
        CKB::NTHREADS > 512)  // larger CTAs spill (register budget 64K / NTHREADS)
      return false;
    constexpr size_t bsm = cg1_resident_smem<D, P, NC, PH, 0>();
    if (bsm > 200 * 1024) return false;
    auto kb = k_coarse_cg1<D, P, NC, PH, true, 0>;
    NNMG_CUDA_TRY(cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm));
    NNMG_CUDA_TRY(cudaFuncSetAttribute(kb, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       cudaSharedmemCarveoutMaxShared));
    int ps = 0;
    NNMG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kb, CKB::NTHREADS, bsm));
    if (ps <= 0) return false;
    C.split = 0;
    C.mode = 1;
    C.resident = true;
    C.nsub = 1;
    C.block = CKB::NTHREADS;
    C.smem = bsm;
    C.nrank = nsm;
    return true;
  }

  template <int D, int P, int NC, int PH>
  void operator()() {
    using CK = CellKernel<D, P, NC, PH>;
    Level& L = *C.level;
    if (configure_only) {
      C.block = CK::NTHREADS;
      C.nsub = 1;
      int nsm = 0, dev = 0;
      NNMG_CUDA_TRY(cudaGetDevice(&dev));
      NNMG_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
      // register variant (Laplace, low order): 8 cell blocks per CTA
      C.resident = false;
      C.mode = -1;
      // measured on B200 (C2/C3 coarse): the pencil kernel spreads a cell over
      // N1^(d-1) threads and wins on this latency-bound level; the register
      // kernel only on request
      const char* ek = getenv("NNMG_COARSE_MODE");
      const bool allow_reg = ek && std::string(ek) == "2";
      if constexpr (PH == kLaplace && NC == 1 && CellReg<D, P>::kSupported) {
        if (allow_reg) {
          auto kg = k_coarse_cg<D, P, NC, PH, 2>;
          int per_sm = 0;
          NNMG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kg, kCgRegThreads, 0));
          if (per_sm > 0) {
            C.mode = 2;
            C.block = kCgRegThreads;
            C.smem = 0;
            const int64_t want = std::max<int64_t>(1, (L.nblk + kCgRegThreads / 32 - 1) / (kCgRegThreads / 32));
            C.nrank = static_cast<int>(std::min<int64_t>(want, int64_t(per_sm) * nsm));
          }
        }
      }
      // pencil modes: nsub cell blocks per CTA (named-barrier subgroups) so
      // that all cell blocks run in one round on at most one CTA per SM
      const int nsub_max = max_sub<D, P, NC, PH>();
      const int nsub = static_cast<int>(std::max<int64_t>(
          1, std::min<int64_t>(nsub_max, (L.nblk + nsm - 1) / nsm)));
      const int64_t nrank_one_round = (L.nblk + nsub - 1) / nsub;
      // resident variant: every subgroup keeps its cell block's tables in smem
      const size_t sub_res = CK::SMEM + size_t(CK::NLOC) * CK::NG * CK::CB * sizeof(double) +
                             ((size_t(CK::NLOC) * CK::CB + 1) / 2) * sizeof(double);
      const size_t res_smem = nsub * sub_res;
      if (C.mode < 0 && res_smem <= 200 * 1024 && !getenv("NNMG_COARSE_NO_RESIDENT")) {
        auto kr = k_coarse_cg<D, P, NC, PH, 1>;
        NNMG_CUDA_TRY(cudaFuncSetAttribute(kr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_smem));
        NNMG_CUDA_TRY(cudaFuncSetAttribute(kr, cudaFuncAttributePreferredSharedMemoryCarveout,
                                           cudaSharedmemCarveoutMaxShared));
        int per_sm = 0;
        NNMG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kr, nsub * CK::NTHREADS, res_smem));
        if (per_sm > 0 && nrank_one_round <= int64_t(per_sm) * nsm) {
          C.resident = true;
          C.mode = 1;
          C.smem = res_smem;
          C.nsub = nsub;
          C.block = nsub * CK::NTHREADS;
          C.nrank = static_cast<int>(nrank_one_round);
        }
      }
      if (C.mode < 0) {
        C.mode = 0;
        auto kern = k_coarse_cg<D, P, NC, PH, 0>;
        C.nsub = nsub;
        C.block = nsub * CK::NTHREADS;
        C.smem = nsub * CK::SMEM;
        NNMG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C.smem));
        NNMG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                           cudaSharedmemCarveoutMaxShared));
        int per_sm = 0;
        NNMG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C.block, C.smem));
        NNMG_REQUIRE(per_sm > 0, kCudaError, "coarse CG kernel does not fit on an SM");
        C.nrank = static_cast<int>(std::min<int64_t>(nrank_one_round, int64_t(per_sm) * nsm));
      }
      // the multi-barrier configuration, restored if the single-barrier
      // kernel turns out not to apply after splitting / owner-warp tuning
      const int s_mode = C.mode, s_block = C.block, s_nsub = C.nsub, s_nrank = C.nrank, s_split = C.split;
      const bool s_resident = C.resident;
      const size_t s_smem = C.smem;
      if (C.single_barrier && C.mode != 2) {
        auto k1 = C.mode == 1 ? k_coarse_cg1<D, P, NC, PH, true, 1> : k_coarse_cg1<D, P, NC, PH, false, 1>;
        NNMG_CUDA_TRY(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C.smem));
        NNMG_CUDA_TRY(cudaFuncSetAttribute(k1, cudaFuncAttributePreferredSharedMemoryCarveout,
                                           cudaSharedmemCarveoutMaxShared));
        int per_sm = 0;
        NNMG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1, C.block, C.smem));
        if (C.nsub != 1 || per_sm * nsm < C.nrank) C.single_barrier = false;
        // fewer cell blocks than SMs: split each block over the largest
        // number of CTAs that still fits one CTA per SM, tables resident
        // (NNMG_COARSE_SPLIT=0 disables, =k caps the split at k)
        const char* es = getenv("NNMG_COARSE_SPLIT");
        const int max_split = es ? atoi(es) : 8;
        if (C.single_barrier) {
          try_split<D, P, NC, PH, 8>(L, nsm, max_split) || try_split<D, P, NC, PH, 4>(L, nsm, max_split) ||
              try_split<D, P, NC, PH, 2>(L, nsm, max_split) || try_balanced<D, P, NC, PH>(L, nsm);
        }
        // a dedicated owner warp overlapping the owner updates with the cell
        // phase (resident tables only); NNMG_COARSE_OWNER_WARPS=0/1
        if (C.single_barrier && C.mode == 1) {
          const char* eo = getenv("NNMG_COARSE_OWNER_WARPS");
          // measured (us per iteration): C5 5.33 -> 4.63, C2 4.00 -> 3.93 with an owner
          // warp; C3 6.59 -> 8.69 (290 owned DoFs per CTA are too many for one warp)
          const int64_t owned = (L.n_dofs + C.nrank - 1) / C.nrank;
          const int want = eo ? atoi(eo) : (owned <= 5 * 32 ? 1 : 0);
          if (want > 0) {
            auto ko = cg1_kernel<D, P, NC, PH, 1>(C);
            NNMG_CUDA_TRY(cudaFuncSetAttribute(ko, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C.smem));
            NNMG_CUDA_TRY(cudaFuncSetAttribute(ko, cudaFuncAttributePreferredSharedMemoryCarveout,
                                               cudaSharedmemCarveoutMaxShared));
            int per_sm = 0;
            NNMG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ko, C.block + 32, C.smem));
            if (per_sm > 0 && int64_t(per_sm) * nsm >= C.nrank) {
              C.owner_warps = 1;
              C.block += 32;
            }
          }
        }
      }
      if (C.nrank > 256) C.single_barrier = false;  // k_coarse_cg1 reduces <= 8 partials per lane
      if (!C.single_barrier) {
        C.mode = s_mode;
        C.block = s_block;
        C.nsub = s_nsub;
        C.nrank = s_nrank;
        C.split = s_split;
        C.resident = s_resident;
        C.smem = s_smem;
        C.owner_warps = 0;
      }
      if (C.single_barrier && C.mode != 2) {
        C.con.alloc(size_t(L.n_dofs));
        C.con.zero();
        if (L.cdofs.n) {
          k_mark_rows<<<unsigned((L.cdofs.n + 255) / 256), 256>>>(L.cdofs.ptr, int64_t(L.cdofs.n), C.con.ptr);
          NNMG_CHECK_LAUNCH();
        }
      }
      C.part.alloc(4 * (2 * size_t(C.nrank) + 2));  // 2 banks of 32-byte slots + 2 result slots
      if (const char* e = getenv("NNMG_COARSE_BARRIER")) C.barrier = atoi(e);
      if (getenv("NNMG_COARSE_TRACE")) {
        C.trace.alloc(8 * 64 + 8 * size_t(C.nrank));
        C.trace.zero();
      }
      C.part.zero();
      C.epoch.alloc(1);
      C.epoch.zero();
      NNMG_CUDA_TRY(cudaDeviceSynchronize());
      return;
    }
    if (C.single_barrier && C.mode != 2) {
      Cg1Args g;
      g.tab = L.tab;
      g.idx = L.idx.ptr;
      g.geo = L.geo.ptr;
      g.nblk = L.nblk;
      g.lam = L.lam;
      g.mu = L.mu;
      g.con = C.con.ptr;
      g.cdofs = L.cdofs.ptr;
      g.ncons = static_cast<int64_t>(L.cdofs.n);
      {
        const char* e = getenv("NNMG_COARSE_PREFETCH");
        g.prefetch_owned = e ? atoi(e) : 1;
      }
      g.inv_diag = L.inv_diag.ptr;
      g.n = L.n_dofs;
      g.b = b;
      g.x = x;
      g.r[0] = C.r.ptr;
      g.r[1] = C.r.ptr + L.n_dofs;
      g.s[0] = C.s.ptr;
      g.s[1] = C.s.ptr + L.n_dofs;
      g.w[0] = C.ap.ptr;
      g.w[1] = C.ap.ptr + L.n_dofs;
      g.w[2] = C.ap.ptr + 2 * L.n_dofs;
      g.p = C.p.ptr;
      g.part = C.part.ptr;
      {
        const char* e = getenv("NNMG_COARSE_ATOMIC_DOTS");
        g.atomic_dots = e ? atoi(e) : 0;
      }
      g.reduction = C.reduction;
      g.max_iter = C.max_iter;
      g.status = C.status.ptr;
      g.trace = C.trace.n ? C.trace.ptr : nullptr;
      auto k1 = C.owner_warps ? cg1_kernel<D, P, NC, PH, 1>(C) : cg1_kernel<D, P, NC, PH, 0>(C);
      void* p1[] = {&g};
      NNMG_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k1, dim3(C.nrank), dim3(C.block), p1, C.smem, s));
      count_launch();
      return;
    }
    auto kern = C.mode == 2 ? k_coarse_cg<D, P, NC, PH, 2>
                            : (C.mode == 1 ? k_coarse_cg<D, P, NC, PH, 1> : k_coarse_cg<D, P, NC, PH, 0>);
    CgArgs a;
    a.tab = L.tab;
    a.idx = L.idx.ptr;
    a.geo = L.geo.ptr;
    a.nblk = L.nblk;
    a.lam = L.lam;
    a.mu = L.mu;
    a.cdofs = L.cdofs.ptr;
    a.ncons = static_cast<int64_t>(L.cdofs.n);
    a.inv_diag = L.inv_diag.ptr;
    a.n = L.n_dofs;
    a.b = b;
    a.x = x;
    a.r = C.r.ptr;
    a.z = C.z.ptr;
    a.p[0] = C.p.ptr;
    a.p[1] = C.p.ptr + L.n_dofs;
    a.ap[0] = C.ap.ptr;
    a.ap[1] = C.ap.ptr + L.n_dofs;
    a.slots = reinterpret_cast<Slot*>(C.part.ptr);
    a.result = reinterpret_cast<Slot*>(C.part.ptr) + 2 * C.nrank;
    a.barrier = C.barrier;
    a.trace = C.trace.n ? C.trace.ptr : nullptr;
    a.solve_epoch = reinterpret_cast<unsigned long long*>(C.epoch.ptr);
    a.reduction = C.reduction;
    a.max_iter = C.max_iter;
    a.nsub = C.nsub;
    a.status = C.status.ptr;
    void* params[] = {&a};
    NNMG_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)kern, dim3(C.nrank), dim3(C.block), params, C.smem, s));
    count_launch();
  }
};

Coarse* coarse_dense_create(Level* L, const double* inverse) {
  NNMG_REQUIRE(L && L->n_dofs <= 8192, kInvalidArgument, "dense coarse solve needs n <= 8192");
  NNMG_CUDA_TRY(cudaSetDevice(L->device));
  auto C = new Coarse();
  C->level = L;
  C->dense = true;
  C->ainv.upload(inverse, size_t(L->n_dofs) * L->n_dofs);
  C->status.alloc(3);
  C->status.zero();
  return C;
}

Coarse* coarse_cg_create(Level* L, double reduction, int max_iter) {
  NNMG_REQUIRE(L != nullptr, kInvalidArgument, "null level");
  NNMG_REQUIRE(L->diag_ready, kInvalidArgument, "level diagonal not computed");
  NNMG_CUDA_TRY(cudaSetDevice(L->device));
  auto C = new Coarse();
  try {
    C->level = L;
    C->dense = false;
    C->reduction = reduction;
    C->max_iter = max_iter;
    C->r.alloc(2 * L->n_dofs);
    C->z.alloc(L->n_dofs);
    C->p.alloc(2 * L->n_dofs);
    C->ap.alloc(3 * L->n_dofs);
    C->s.alloc(2 * L->n_dofs);
    {
      // measured (B200, same iteration counts): C2 7.05 -> 4.92, C3 13.1 ->
      // 10.5, C5 20.2 -> 18.4 us per iteration
      const char* e = getenv("NNMG_COARSE_CG1");
      C->single_barrier = e ? atoi(e) != 0 : true;
    }
    C->status.alloc(3);
    C->status.zero();
    CgLaunch f{*C, nullptr, nullptr, 0, true};
    dispatch(L->dim, L->degree, L->ncomp, L->physics, f);
  } catch (...) {
    delete C;
    throw;
  }
  return C;
}

void coarse_solve(Coarse& C, const double* b, double* x, cudaStream_t s) {
  if (C.direct) {
    coarse_direct_solve(C, b, x, s);
    return;
  }
  if (C.dense) {
    const int n = static_cast<int>(C.level->n_dofs);
    k_dense_solve<<<grid_for(n, 8), 256, 0, s>>>(C.ainv.ptr, b, x, n);
    NNMG_CHECK_LAUNCH();
    count_launch();
    return;
  }
  CgLaunch f{C, b, x, s, false};
  dispatch(C.level->dim, C.level->degree, C.level->ncomp, C.level->physics, f);
}

void coarse_status(Coarse& C, int* iterations, int* converged, int* error) {
#ifdef NNMG_CELL_TRACE
  {
    unsigned long long ct[16];
    NNMG_CUDA_TRY(cudaMemcpyFromSymbol(ct, nnmg_cell_trace, sizeof(ct)));
    fprintf(stderr, "[nnmg cell trace] calls %llu, cycles per call by phase:", ct[14]);
    for (int i = 1; i <= 11; ++i) fprintf(stderr, " P%d %.0f", i, ct[14] ? double(ct[i]) / double(ct[14]) : 0.0);
    fprintf(stderr, "\n");
  }
#endif
  if (C.direct || C.dense) {  // exact solves: no iterations
    *iterations = 0;
    *converged = 1;
    *error = 0;
    return;
  }
  int st[3];
  NNMG_CUDA_TRY(cudaMemcpy(st, C.status.ptr, sizeof(st), cudaMemcpyDeviceToHost));
  *iterations = st[0];
  *converged = st[1];
  *error = st[2];
  if (C.trace.n) {
    std::vector<unsigned long long> t(C.trace.n);
    NNMG_CUDA_TRY(cudaMemcpy(t.data(), C.trace.ptr, t.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    const int n = std::min(st[0], 63);
    double ph[4] = {0, 0, 0, 0}, sub[3] = {0, 0, 0}, tot = 0;
    int cnt = 0;
    for (int it = 2; it < n; ++it) {
      const unsigned long long* r = &t[it * 8];
      sub[0] += double(r[5] - r[0]);
      sub[1] += double(r[6] - r[5]);
      sub[2] += double(r[7] - r[6]);
      ph[0] += double(r[1] - r[0]);
      ph[1] += double(r[2] - r[1]);
      ph[2] += double(r[3] - r[2]);
      ph[3] += double(r[4] - r[3]);
      tot += double(t[(it + 1) * 8] - r[0]);
      ++cnt;
    }
    if (st[0] >= 16) {
      // arrival spread at the barrier, iterations 8..15: per-CTA lateness
      // relative to the earliest CTA, averaged
      std::vector<double> late(C.nrank, 0.0);
      for (int it = 0; it < 8; ++it) {
        const unsigned long long* r = &t[8 * 64 + size_t(it) * C.nrank];
        unsigned long long mn = r[0];
        for (int q = 0; q < C.nrank; ++q) mn = std::min(mn, r[q]);
        for (int q = 0; q < C.nrank; ++q) late[q] += double(r[q] - mn) / 8.0;
      }
      std::vector<int> order(C.nrank);
      for (int q = 0; q < C.nrank; ++q) order[q] = q;
      std::sort(order.begin(), order.end(), [&](int x, int y) { return late[x] > late[y]; });
      fprintf(stderr, "[nnmg coarse trace] barrier arrival lateness ns (slowest CTAs):");
      for (int q = 0; q < std::min(C.nrank, 8); ++q) fprintf(stderr, " %d:%.0f", order[q], late[order[q]]);
      double mean = 0;
      for (double v : late) mean += v / C.nrank;
      fprintf(stderr, " | mean %.0f, CTA0 %.0f\n", mean, late[0]);
    }
    if (cnt && C.single_barrier && C.mode != 2) {
      double q[6] = {0, 0, 0, 0, 0, 0};
      for (int it = 2; it < n; ++it) {
        const unsigned long long* r = &t[it * 8];
        q[0] += double(r[5] - r[0]);
        q[1] += double(r[7] - r[5]);
        q[2] += double(r[1] - r[7]);
        q[3] += double(r[2] - r[1]);
        q[4] += double(r[3] - r[2]);
        q[5] += double(r[4] - r[3]);
      }
      int dev = 0, khz = 0;
      NNMG_CUDA_TRY(cudaGetDevice(&dev));
      NNMG_CUDA_TRY(cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev));
      const double f = 1e6 / double(khz) / cnt;
      fprintf(stderr,
              "[nnmg coarse trace] cg1 ctas=%d threads=%d split=%d per-iteration ns (CTA 0): cells %.0f owners %.0f "
              "local-reduce %.0f barrier %.0f global-reduce %.0f scalars %.0f total %.0f\n",
              C.nrank, C.block, C.split, q[0] * f, q[1] * f, q[2] * f, q[3] * f, q[4] * f, q[5] * f,
              tot * 1e6 / double(khz) / cnt);
    } else if (cnt)
      fprintf(stderr,
              "[nnmg coarse trace] barrier=%d ctas=%d resident=%d per-iteration ns: applyA %.0f barrierA %.0f "
              "phaseB %.0f barrierB %.0f total %.0f | applyA = cells %.0f + owners %.0f + constrained %.0f + "
              "reduce\n",
              C.barrier, C.nrank, int(C.resident), ph[0] / cnt, ph[1] / cnt, ph[2] / cnt, ph[3] / cnt, tot / cnt,
              sub[0] / cnt, sub[1] / cnt, sub[2] / cnt);
  }
}

}  // namespace nnmg
