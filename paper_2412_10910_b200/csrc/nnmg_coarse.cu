// K8/K10: coarsest-level solvers (replaces CoarseSolver, solvers.py:167-206).
//
// * dense: x = A^-1 b with the inverse precomputed on the host from a Cholesky
//   factorisation (n <= dense_limit), one warp per row;
// * CG-Jacobi: the reference's cg_solve(op, b, precond=inv_diag, 1e-8, 1e4)
//   (solvers.py:129-164) as ONE persistent kernel on one thread-block cluster.
//   The matrix-free apply runs on NSUB sub-groups per CTA (named barriers), the
//   vector phases on each CTA's contiguous DoF range, dot products reduce per
//   CTA and then in fixed rank order so every CTA takes identical decisions;
//   cluster barriers separate the phases.  No host round trip per iteration.
#include "nnmg_coarse.cuh"
#include "nnmg_cellkernel.cuh"

#include <cooperative_groups.h>

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
  double *r, *z, *p, *ap;
  double* part;  // [3][nrank]
  double reduction;
  int max_iter;
  int* status;  // iterations, converged, error
  int nsub;
};

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

template <int D, int P, int NC, int PH>
__global__ void __launch_bounds__(1024) k_coarse_cg(CgArgs a) {
  using CK = CellKernel<D, P, NC, PH>;
  extern __shared__ double sm[];
  __shared__ double red[64];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = static_cast<int>(cl.block_rank()), nrank = static_cast<int>(cl.num_blocks());
  const int tid = threadIdx.x, nth = blockDim.x;
  const int64_t i0 = a.n * rank / nrank, i1 = a.n * (rank + 1) / nrank;
  double* part_rr = a.part;
  double* part_rz = a.part + nrank;
  double* part_pap = a.part + 2 * nrank;

  double srr = 0.0, srz = 0.0;
  for (int64_t i = i0 + tid; i < i1; i += nth) {
    const double bi = a.b[i];
    const double zi = a.inv_diag[i] * bi;
    a.x[i] = 0.0;
    a.r[i] = bi;
    a.z[i] = zi;
    a.p[i] = zi;
    a.ap[i] = 0.0;
    srr += bi * bi;
    srz += bi * zi;
  }
  block_sum2(srr, srz, red);
  if (tid == 0) {
    part_rr[rank] = srr;
    part_rz[rank] = srz;
  }
  cl.sync();
  double rr = 0.0, rz = 0.0;
  for (int k = 0; k < nrank; ++k) {
    rr += part_rr[k];
    rz += part_rz[k];
  }
  const double norm0 = sqrt(rr);
  if (norm0 == 0.0) {
    if (rank == 0 && tid == 0) {
      a.status[0] = 0;
      a.status[1] = 1;
      a.status[2] = 0;
    }
    return;
  }
  const double target = a.reduction * norm0;
  const int sub = tid / CK::NTHREADS, stid = tid % CK::NTHREADS;
  const size_t sub_doubles = CK::SMEM / sizeof(double);
  for (int it = 1; it <= a.max_iter; ++it) {
    // Ap = A p (zero-in / identity-out)
    if (sub < a.nsub) {
      double* smem = sm + sub * sub_doubles;
      const int bar = sub + 1;
      const int64_t stride = (int64_t)nrank * a.nsub;
      for (int64_t blk = (int64_t)rank * a.nsub + sub; blk < a.nblk; blk += stride) {
        if (a.nsub == 1)
          CK::template run<false>(a.tab, a.p, a.ap, a.idx, a.geo, blk, a.lam, a.mu, smem, stid,
                                  [] __device__() { __syncthreads(); });
        else
          CK::template run<false>(a.tab, a.p, a.ap, a.idx, a.geo, blk, a.lam, a.mu, smem, stid,
                                  [bar] __device__() { named_sync(bar, CK::NTHREADS); });
      }
    }
    for (int64_t k = (int64_t)rank * nth + tid; k < a.ncons; k += (int64_t)nrank * nth) {
      const int c = a.cdofs[k];
      a.ap[c] = a.p[c];
    }
    cl.sync();
    double spap = 0.0, dummy = 0.0;
    for (int64_t i = i0 + tid; i < i1; i += nth) spap += a.p[i] * a.ap[i];
    block_sum2(spap, dummy, red);
    if (tid == 0) part_pap[rank] = spap;
    cl.sync();
    double pap = 0.0;
    for (int k = 0; k < nrank; ++k) pap += part_pap[k];
    if (!(pap > 0.0)) {
      if (rank == 0 && tid == 0) {
        a.status[0] = it;
        a.status[1] = 0;
        a.status[2] = 1;
      }
      return;
    }
    const double alpha = rz / pap;
    srr = 0.0;
    srz = 0.0;
    for (int64_t i = i0 + tid; i < i1; i += nth) {
      a.x[i] = a.x[i] + alpha * a.p[i];
      const double ri = a.r[i] - alpha * a.ap[i];
      const double zi = a.inv_diag[i] * ri;
      a.r[i] = ri;
      a.z[i] = zi;
      a.ap[i] = 0.0;
      srr += ri * ri;
      srz += ri * zi;
    }
    block_sum2(srr, srz, red);
    if (tid == 0) {
      part_rr[rank] = srr;
      part_rz[rank] = srz;
    }
    cl.sync();
    rr = 0.0;
    double rz_new = 0.0;
    for (int k = 0; k < nrank; ++k) {
      rr += part_rr[k];
      rz_new += part_rz[k];
    }
    if (sqrt(rr) <= target) {
      if (rank == 0 && tid == 0) {
        a.status[0] = it;
        a.status[1] = 1;
        a.status[2] = 0;
      }
      return;
    }
    const double beta = rz_new / rz;
    rz = rz_new;
    for (int64_t i = i0 + tid; i < i1; i += nth) a.p[i] = a.z[i] + beta * a.p[i];
    cl.sync();
  }
  if (rank == 0 && tid == 0) {
    a.status[0] = a.max_iter;
    a.status[1] = 0;
    a.status[2] = 0;
  }
}

struct CgLaunch {
  Coarse& C;
  const double* b;
  double* x;
  cudaStream_t s;
  bool configure_only;
  template <int D, int P, int NC, int PH>
  void operator()() {
    using CK = CellKernel<D, P, NC, PH>;
    auto kern = k_coarse_cg<D, P, NC, PH>;
    Level& L = *C.level;
    if (configure_only) {
      int nsub = 1;
      if (CK::NTHREADS % 32 == 0) {
        nsub = std::max(1, std::min({15, 1024 / CK::NTHREADS, int((200 * 1024) / CK::SMEM)}));
      }
      C.nsub = nsub;
      C.block = nsub * CK::NTHREADS;
      C.smem = nsub * CK::SMEM;
      NNMG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C.smem));
      NNMG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      C.nrank = 0;
      for (int cs : {16, 8, 4, 2, 1}) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(cs);
        cfg.blockDim = dim3(C.block);
        cfg.dynamicSmemBytes = C.smem;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) == cudaSuccess && nclusters > 0) {
          C.nrank = cs;
          break;
        }
        cudaGetLastError();
      }
      NNMG_REQUIRE(C.nrank > 0, kCudaError, "no thread-block cluster configuration fits the coarse solver");
      return;
    }
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
    a.p = C.p.ptr;
    a.ap = C.ap.ptr;
    a.part = C.part.ptr;
    a.reduction = C.reduction;
    a.max_iter = C.max_iter;
    a.status = C.status.ptr;
    a.nsub = C.nsub;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C.nrank;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(C.nrank);
    cfg.blockDim = dim3(C.block);
    cfg.dynamicSmemBytes = C.smem;
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    NNMG_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a));
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
    C->r.alloc(L->n_dofs);
    C->z.alloc(L->n_dofs);
    C->p.alloc(L->n_dofs);
    C->ap.alloc(L->n_dofs);
    C->part.alloc(3 * 16);
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
  int st[3];
  NNMG_CUDA_TRY(cudaMemcpy(st, C.status.ptr, sizeof(st), cudaMemcpyDeviceToHost));
  *iterations = st[0];
  *converged = st[1];
  *error = st[2];
}

}  // namespace nnmg
