// K10b: direct coarsest-level solve for levels above the dense limit
// (a deviation from CoarseSolver's Jacobi-PCG, solvers.py:193-206, chosen where
// it is faster: see solvers.py CoarseSolver(direct=...)).
//
// x = A^-1 b on the free (unconstrained) DoFs, x = b on the constrained ones
// (zero-in / identity-out makes A block diagonal), with the SPD inverse of the
// free block stored once as packed lower-triangle 64x64 tiles, so the
// symmetric GEMV streams nf^2/2 doubles instead of n^2: an
// off-diagonal tile (I, J) serves both y_I += A_IJ x_J (row part) and
// y_J += A_IJ^T x_I (column part).  Phase 1 streams the tiles (one CTA per
// tile, 16 doubles per thread in flight, no shared-memory staging of the
// matrix) and writes per-tile 64-entry partials; phase 2 sums them per block
// row in a fixed order.  No atomics: the result is bitwise reproducible.
// HBM-bound: 8 nf^2/2 bytes per solve.
#include "nnmg_coarse.cuh"

#include <algorithm>
#include <cmath>
#include <vector>

namespace nnmg {

namespace {

constexpr int kT = 64;  // tile edge

__host__ __device__ inline int64_t tri_id(int64_t I, int64_t J) { return I * (I + 1) / 2 + J; }

__device__ inline void tri_decode(int64_t t, int& I, int& J) {
  int64_t i = static_cast<int64_t>((sqrt(8.0 * double(t) + 1.0) - 1.0) * 0.5);
  while (i * (i + 1) / 2 > t) --i;
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  I = static_cast<int>(i);
  J = static_cast<int>(t - i * (i + 1) / 2);
}

// full (lower triangle read) -> tiles; the diagonal tiles are symmetrised
// from the lower triangle, padding is zero
template <class TT>
__global__ void k_pack(const double* __restrict__ full, int64_t n, int64_t ld, TT* __restrict__ tiles, int64_t t0) {
  // full: the free-block inverse (n = number of free DoFs); this handle's tiles start at t0
  int I, J;
  tri_decode(t0 + blockIdx.x, I, J);
  TT* dst = tiles + int64_t(blockIdx.x) * kT * kT;
  for (int e = threadIdx.x; e < kT * kT; e += blockDim.x) {
    const int r = e / kT, c = e % kT;
    int64_t gr = int64_t(I) * kT + r, gc = int64_t(J) * kT + c;
    if (gc > gr) {  // upper part of a diagonal tile: mirror
      const int64_t t = gr;
      gr = gc;
      gc = t;
    }
    dst[e] = (gr < n && gc < n) ? TT(full[gr * ld + gc]) : TT(0);
  }
}

// phase 1: thread t holds elements 2(t + 256k), k < 8, of its tile, i.e. rows
// w + 8k (w = warp) and columns 2 lane, 2 lane + 1
// TT: tile storage and product type (double; float = the mixed-precision
// cycle's coarse solve: half the streamed bytes, single-precision products
// within a tile, per-tile partials and their sums in fp64)
template <class TT>
struct Tile2;
template <>
struct Tile2<double> {
  using type = double2;
};
template <>
struct Tile2<float> {
  using type = float2;
};

template <class TT>
__global__ void __launch_bounds__(256) k_symv_tiles(const TT* __restrict__ tiles, const double* __restrict__ x,
                                                    const int* __restrict__ freedofs, int64_t n,
                                                    double* __restrict__ prow, double* __restrict__ pcol, int64_t t0) {
  using double2 = typename Tile2<TT>::type;  // element pairs of the tile type
  using double_t = TT;
  __shared__ double_t xs[2][kT];
  __shared__ double2 cs[8][kT / 2];
  // tiles, prow and pcol hold this handle's tile range [t0, t0 + gridDim.x) only
  const int64_t t = blockIdx.x;
  int I, J;
  tri_decode(t0 + t, I, J);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const double2* tp = reinterpret_cast<const double2*>(tiles + t * (kT * kT));
  double2 a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = __ldcs(tp + tid + 256 * k);
  if (tid < 2 * kT) {
    const int which = tid / kT, r = tid % kT;
    const int64_t g = int64_t(which ? I : J) * kT + r;
    xs[which][r] = g < n ? double_t(__ldcg(x + freedofs[g])) : double_t(0);
  }
  __syncthreads();
  // row part: y_I[w + 8k] += sum_c A[w + 8k][c] x_J[c]
  const double_t xj0 = xs[0][2 * lane], xj1 = xs[0][2 * lane + 1];
  double_t rp[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) rp[k] = fma(a[k].x, xj0, a[k].y * xj1);
  // transposing butterfly: after it lane L holds row w + 8 k(L),
  // k(L) = 4 b4(L) + 2 b3(L) + b2(L), summed over all 64 columns
  const bool b16 = lane & 16, b8 = lane & 8, b4 = lane & 4;
  double_t r4[4], r2[2];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const double_t send = b16 ? rp[j] : rp[4 + j];
    const double_t keep = b16 ? rp[4 + j] : rp[j];
    r4[j] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const double_t send = b8 ? r4[j] : r4[2 + j];
    const double_t keep = b8 ? r4[2 + j] : r4[j];
    r2[j] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  double_t r1 = (b4 ? r2[1] : r2[0]) + __shfl_xor_sync(0xffffffffu, b4 ? r2[0] : r2[1], 4);
  r1 += __shfl_xor_sync(0xffffffffu, r1, 2);
  r1 += __shfl_xor_sync(0xffffffffu, r1, 1);
  if ((lane & 3) == 0) {
    const int k = (b16 ? 4 : 0) + (b8 ? 2 : 0) + (b4 ? 1 : 0);
    prow[t * kT + w + 8 * k] = double(r1);
  }
  if (I == J) return;  // diagonal tiles are stored whole: no column part
  // column part: y_J[c] += sum_r A[r][c] x_I[r]
  double_t c0 = 0, c1 = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double_t xi = xs[1][w + 8 * k];
    c0 = fma(a[k].x, xi, c0);
    c1 = fma(a[k].y, xi, c1);
  }
  cs[w][lane] = double2{c0, c1};
  __syncthreads();
  if (tid < kT) {
    const double_t* csd = reinterpret_cast<const double_t*>(&cs[0][0]);
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += double(csd[q * kT + tid]);
    pcol[t * kT + tid] = s;
  }
}

// phase 2: y[free[I*64 + r]] = sum_{J <= I} prow(I, J)[r] + sum_{K > I} pcol(K, I)[r];
// kRQ threads per row take every kRQ-th term, four independent loads in
// flight each, combined in a fixed order (bitwise reproducible).  Measured on
// B200 (C2, 253 block rows): 4 threads per row with one load in flight took
// 36 us for 33 MB of partials.  Blocks past nb copy the constrained entries
// (identity rows): y[c] = b[c].
constexpr int kRQ = 16;

__global__ void __launch_bounds__(kRQ * kT) k_symv_reduce(const double* __restrict__ prow,
                                                         const double* __restrict__ pcol, int nb, int64_t n,
                                                         const int* __restrict__ freedofs, const int* __restrict__ cons,
                                                         int64_t ncons, const double* __restrict__ b,
                                                         double* __restrict__ y, int64_t t0, int64_t t1, int identity) {
  // [t0, t1): the tile range of this handle (a share of the tiles when the
  // solve is split across ranks: the shares' outputs add up to the solution,
  // and exactly one share writes the identity rows, the others zeros)
  __shared__ double part[kRQ][kT];
  if (int(blockIdx.x) >= nb) {
    for (int64_t i = int64_t(blockIdx.x - nb) * blockDim.x + threadIdx.x; i < ncons;
         i += int64_t(gridDim.x - nb) * blockDim.x)
      y[cons[i]] = identity ? b[cons[i]] : 0.0;
    return;
  }
  const int I = blockIdx.x, r = threadIdx.x & (kT - 1), q = threadIdx.x >> 6;
  auto term = [&](int j) -> double {
    if (j >= nb) return 0.0;
    const int64_t t = j <= I ? tri_id(I, j) : tri_id(j, I);
    if (t < t0 || t >= t1) return 0.0;
    return j <= I ? __ldcg(prow + (t - t0) * kT + r) : __ldcg(pcol + (t - t0) * kT + r);
  };
  double s = 0.0;
  for (int j = q; j < nb; j += 4 * kRQ) {
    const double v0 = term(j), v1 = term(j + kRQ), v2 = term(j + 2 * kRQ), v3 = term(j + 3 * kRQ);
    s += (v0 + v1) + (v2 + v3);
  }
  part[q][r] = s;
  __syncthreads();
  if (q == 0) {
    const int64_t g = int64_t(I) * kT + r;
    double tot = 0.0;
#pragma unroll
    for (int k = 0; k < kRQ; ++k) tot += part[k][r];
    if (g < n) y[freedofs[g]] = tot;
  }
}

}  // namespace

Coarse* coarse_direct_create(Level* L, const double* inverse_dev, int64_t ld, bool f32, int share, int n_shares) {
  NNMG_REQUIRE(n_shares >= 1 && share >= 0 && share < n_shares, kInvalidArgument, "tile share out of range");
  NNMG_REQUIRE(L != nullptr && inverse_dev != nullptr, kInvalidArgument, "null argument");
  NNMG_CUDA_TRY(cudaSetDevice(L->device));
  // free DoFs: the complement of the level's sorted constrained list
  std::vector<int> cons(L->cdofs.n), freed;
  if (L->cdofs.n)
    NNMG_CUDA_TRY(cudaMemcpy(cons.data(), L->cdofs.ptr, cons.size() * sizeof(int), cudaMemcpyDeviceToHost));
  freed.reserve(size_t(L->n_dofs) - cons.size());
  for (int64_t i = 0, k = 0; i < L->n_dofs; ++i) {
    if (k < int64_t(cons.size()) && cons[k] == i) {
      ++k;
      continue;
    }
    freed.push_back(static_cast<int>(i));
  }
  const int64_t nf = static_cast<int64_t>(freed.size());
  NNMG_REQUIRE(ld >= nf, kInvalidArgument, "leading dimension smaller than the number of free DoFs");
  auto C = new Coarse();
  try {
    C->level = L;
    C->direct = true;
    C->nfree = nf;
    C->dfree.upload(freed);
    C->dcons.upload(cons);
    C->nb = static_cast<int>((nf + kT - 1) / kT);
    const int64_t nt_all = tri_id(C->nb, 0);
    NNMG_REQUIRE(nt_all < (int64_t(1) << 31), kInvalidArgument, "coarse level too large for the direct solve");
    // this handle's share of the tiles (equal contiguous ranges; one share = all)
    C->t0 = nt_all * share / n_shares;
    C->t1 = nt_all * (share + 1) / n_shares;
    C->identity = share == 0;
    const int64_t nt = C->t1 - C->t0;
    C->tiles_f32 = f32;
    if (f32)
      C->tiles32.alloc(size_t(nt) * kT * kT);
    else
      C->tiles.alloc(size_t(nt) * kT * kT);
    C->prow.alloc(size_t(nt) * kT);
    C->pcol.alloc(size_t(nt) * kT);
    C->status.alloc(3);
    C->status.zero();
    if (nt) {
      if (f32)
        k_pack<float><<<unsigned(nt), 256>>>(inverse_dev, nf, ld, C->tiles32.ptr, C->t0);
      else
        k_pack<double><<<unsigned(nt), 256>>>(inverse_dev, nf, ld, C->tiles.ptr, C->t0);
    }
    NNMG_CHECK_LAUNCH();
    NNMG_CUDA_TRY(cudaDeviceSynchronize());
  } catch (...) {
    delete C;
    throw;
  }
  return C;
}

void coarse_direct_solve(Coarse& C, const double* b, double* x, cudaStream_t s) {
  const int64_t nt = C.t1 - C.t0;
  const int64_t ncons = static_cast<int64_t>(C.dcons.n);
  if (nt) {
    if (C.tiles_f32)
      k_symv_tiles<float><<<unsigned(nt), 256, 0, s>>>(C.tiles32.ptr, b, C.dfree.ptr, C.nfree, C.prow.ptr, C.pcol.ptr,
                                                        C.t0);
    else
      k_symv_tiles<double><<<unsigned(nt), 256, 0, s>>>(C.tiles.ptr, b, C.dfree.ptr, C.nfree, C.prow.ptr, C.pcol.ptr,
                                                         C.t0);
    NNMG_CHECK_LAUNCH();
  }
  const unsigned extra = static_cast<unsigned>(std::min<int64_t>((ncons + kRQ * kT - 1) / (kRQ * kT), 64));
  if (C.nb + extra) {
    k_symv_reduce<<<unsigned(C.nb) + extra, kRQ * kT, 0, s>>>(C.prow.ptr, C.pcol.ptr, C.nb, C.nfree, C.dfree.ptr,
                                                          C.dcons.ptr, ncons, b, x, C.t0, C.t1, C.identity ? 1 : 0);
    NNMG_CHECK_LAUNCH();
  }
  count_launch(nt ? 2 : 1);
}

}  // namespace nnmg
