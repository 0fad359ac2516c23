// K6 prolongation, K7 restriction (deterministic, two-phase) and the GPU point
// location that builds the transfer records.
#include "nnmg_transfer.cuh"
#include "nnmg_cellkernel.cuh"
#include "nnmg_transfer_kernels.cuh"

#include <algorithm>
#include <cstdlib>
#include <cmath>

namespace nnmg {

static inline unsigned grid_for(int64_t n, int bs) { return static_cast<unsigned>((n + bs - 1) / bs); }

static constexpr int kWarps = kTransferWarps;

// ---------------------------------------------------------------------------
// TV = float: the mixed-precision V-cycle's transfers (fp32 vectors and xhat,
// fp64 arithmetic); only the default kernel variants are instantiated for it
template <class TV>
struct TransferDispatchT {
  static constexpr bool kF64 = sizeof(TV) == sizeof(double);
  Transfer& T;
  const TV* in;
  TV* out;
  int mode;  // 0 prolongate, 1 prolongate-accumulate, 2 restrict
  cudaStream_t s;
  template <int D, int P, int NC, int PH>
  void operator()() {
    constexpr int CBC = cells_per_block<D, P, NC>();
    const Level& C = *T.coarse;
    // warps (work items / cell chunks) per CTA of the prolongation and the lane restriction
    // (independent warps: one-warp CTAs retire on their own; measured on B200: C3 prolongation
    // 151.0 -> 147.5 us, restriction 176.4 -> 173.6 us; C2 (2D) prolongation 18.5 -> 24.6 us, so
    // the default is 1 in 3D and 4 in 2D; NNMG_TRANSFER_WARPS overrides)
    const int tw = (T.transfer_warps == 1 || T.transfer_warps == 2 || T.transfer_warps == 4) ? T.transfer_warps
                                                                                             : (D == 3 ? 1 : kWarps);
    const unsigned g = grid_for(T.nitems, tw);
    const TV* const xh = [&] {
      if constexpr (kF64)
        return T.xhat.ptr;
      else
        return T.xhat32.ptr;
    }();
    if (mode < 2) {
      constexpr int PPL = prolongate_ppl<D, P, NC>();
      auto kp = k_prolongate<D, P, NC, CBC, PPL, TV, TV>;
      if constexpr (kF64 && PPL == 1)
        if (T.prolong_ppl == 2) kp = k_prolongate<D, P, NC, CBC, 2>;
      // fp32 levels: single-precision arithmetic unless NNMG_MIXED_ARITH=64
      if constexpr (!kF64)
        if (T.mixed_arith32) kp = k_prolongate<D, P, NC, CBC, PPL, TV, TV, float>;
      kp<<<g, tw * 32, 0, s>>>(C.tab, in, out, mode, C.idx.ptr, T.nitems == T.ncc ? nullptr : T.item_cell.ptr,
                                   T.item_pt.ptr, T.pt_dof.ptr, xh, T.nitems);
      NNMG_CHECK_LAUNCH();
      count_launch();
    } else {
      if (T.timing) NNMG_CUDA_TRY(cudaEventRecord(T.ev[0], s));
      const int ch = T.chunk;
      const int64_t nwarps = (T.nitems + ch - 1) / ch;
      constexpr int W = StagedRestrict<D, P, NC>::WARPS;
      // two planes per lane where the 2 x INNER x NC accumulators fit in registers
      constexpr bool kPl2 = 2 * (ipow(P + 1, D) / (P + 1)) * NC <= 60 && P >= 1;
      if constexpr (ipow(P + 1, D) * NC <= 32) {
        // default: 3 points per lane and round in 3D (C3 0.176 -> 0.173 ms), 2 in 2D
        // (C2 0.022 vs 0.025 ms with 3); 4 points measured slower in both
        const int rk = T.restrict_kernel >= 0 ? T.restrict_kernel : (D == 3 ? 3 : 1);
        if constexpr (!kF64) {
          auto kl = D == 3 ? k_restrict_lane<D, P, NC, 3, TV, TV> : k_restrict_lane<D, P, NC, 1, TV, TV>;
          if (T.mixed_arith32)
            kl = D == 3 ? k_restrict_lane<D, P, NC, 3, TV, TV, float> : k_restrict_lane<D, P, NC, 1, TV, TV, float>;
          const size_t sm = tw * (T.mixed_arith32 ? restrict_lane_smem_per_warp<D, P, NC, float>()
                                                   : restrict_lane_smem_per_warp<D, P, NC, double>());
          kl<<<grid_for(nwarps, tw), tw * 32, sm, s>>>(C.tab, in, T.item_pt.ptr, T.pt_dof.ptr, xh, T.nitems, ch,
                                                      T.cellbuf.ptr);
        } else if (rk != 2) {
          auto k = rk == 0 ? k_restrict_lane<D, P, NC, 1>
                   : rk == 3 ? k_restrict_lane<D, P, NC, 3>
                             : k_restrict_lane<D, P, NC, 2>;
          k<<<grid_for(nwarps, tw), tw * 32, tw * restrict_lane_smem_per_warp<D, P, NC, double>(), s>>>(
              C.tab, in, T.item_pt.ptr, T.pt_dof.ptr, xh, T.nitems, ch, T.cellbuf.ptr);
        } else {
          k_restrict_staged<D, P, NC><<<grid_for(nwarps, W), W * 32, 0, s>>>(
              C.tab, in, T.item_pt.ptr, T.pt_dof.ptr, xh, T.nitems, ch, T.cellbuf.ptr);
        }
      } else if constexpr (ipow(P + 1, D) * NC <= 81 && kF64) {
        if (T.restrict_wide) {
          // (81 outputs: three 32-output tiles, 32 x 33 doubles per warp)
          k_restrict_lane<D, P, NC, 1><<<grid_for(nwarps, tw), tw * 32,
                                        tw * restrict_lane_smem_per_warp<D, P, NC, double>(), s>>>(
              C.tab, in, T.item_pt.ptr, T.pt_dof.ptr, xh, T.nitems, ch, T.cellbuf.ptr);
        } else if (T.restrict_pl == 2 && kPl2) {
          if constexpr (kPl2) {
            constexpr int W2 = StagedRestrict<D, P, NC, 2>::WARPS;
            k_restrict_staged<D, P, NC, TV, TV, 2><<<grid_for(nwarps, W2), W2 * 32, 0, s>>>(
                C.tab, in, T.item_pt.ptr, T.pt_dof.ptr, xh, T.nitems, ch, T.cellbuf.ptr);
          }
        } else {
          k_restrict_staged<D, P, NC><<<grid_for(nwarps, W), W * 32, 0, s>>>(
              C.tab, in, T.item_pt.ptr, T.pt_dof.ptr, xh, T.nitems, ch, T.cellbuf.ptr);
        }
      } else if (T.restrict_pl == 2 && kPl2) {
        if constexpr (kPl2) {
          constexpr int W2 = StagedRestrict<D, P, NC, 2>::WARPS;
          k_restrict_staged<D, P, NC, TV, TV, 2><<<grid_for(nwarps, W2), W2 * 32, 0, s>>>(
              C.tab, in, T.item_pt.ptr, T.pt_dof.ptr, xh, T.nitems, ch, T.cellbuf.ptr);
        }
      } else {
        bool done = false;
        if constexpr (!kF64) {
          if (T.mixed_arith32) {
            constexpr int WF = StagedRestrict<D, P, NC, 1, float>::WARPS;
            k_restrict_staged<D, P, NC, TV, TV, 1, float><<<grid_for(nwarps, WF), WF * 32, 0, s>>>(
                C.tab, in, T.item_pt.ptr, T.pt_dof.ptr, xh, T.nitems, ch, T.cellbuf.ptr);
            done = true;
          }
        }
        if (!done)
          k_restrict_staged<D, P, NC, TV, TV><<<grid_for(nwarps, W), W * 32, 0, s>>>(
              C.tab, in, T.item_pt.ptr, T.pt_dof.ptr, xh, T.nitems, ch, T.cellbuf.ptr);
      }
      NNMG_CHECK_LAUNCH();
      if (T.timing) NNMG_CUDA_TRY(cudaEventRecord(T.ev[1], s));
      k_restrict_gather<TV><<<grid_for(C.n_scalar, 256), 256, 0, s>>>(T.t_off.ptr, T.t_ent.ptr, T.cellbuf.ptr,
                                                                       C.n_scalar, NC, out);
      NNMG_CHECK_LAUNCH();
      count_launch(2);
      if (T.timing) {
        NNMG_CUDA_TRY(cudaEventRecord(T.ev[2], s));
        T.ev_eval = 0;
      }
    }
  }
};
using TransferDispatch = TransferDispatchT<double>;

Transfer* transfer_create(Level* coarse, Level* fine, int64_t npts, const int64_t* point_dofs, const int64_t* cells,
                          const double* xhat) {
  NNMG_REQUIRE(coarse && fine, kInvalidArgument, "null level handle");
  NNMG_REQUIRE(coarse->ncomp == fine->ncomp, kInvalidArgument, "component counts of the two levels must match");
  NNMG_REQUIRE(coarse->dim == fine->dim, kInvalidArgument, "levels must share the dimension");
  NNMG_REQUIRE(npts < (int64_t(1) << 31), kUnsupported, "too many transfer points");
  NNMG_CUDA_TRY(cudaSetDevice(coarse->device));
  auto T = new Transfer();
  try {
    T->coarse = coarse;
    T->fine = fine;
    T->dim = coarse->dim;
    T->pc = coarse->degree;
    T->ncomp = coarse->ncomp;
    T->npts = npts;
    T->ncc = coarse->n_cells;
    const int64_t ncc = coarse->n_cells;
    std::vector<int> start(ncc + 1, 0);
    for (int64_t i = 0; i < npts; ++i) {
      NNMG_REQUIRE(cells[i] >= 0 && cells[i] < ncc, kInvalidArgument, "owning cell out of range");
      NNMG_REQUIRE(point_dofs[i] >= 0 && point_dofs[i] < fine->n_scalar, kInvalidArgument, "point DoF out of range");
      start[cells[i] + 1] += 1;
    }
    for (int64_t c = 0; c < ncc; ++c) start[c + 1] += start[c];
    std::vector<int> fill(start.begin(), start.end() - 1);
    std::vector<int> pd(npts);
    std::vector<double> xh(size_t(npts) * T->dim);
    for (int64_t i = 0; i < npts; ++i) {
      const int k = fill[cells[i]]++;
      pd[k] = static_cast<int>(point_dofs[i]);
      for (int j = 0; j < T->dim; ++j) xh[size_t(k) * T->dim + j] = xhat[i * T->dim + j];
    }
    T->cell_start.upload(start);
    T->pt_dof.upload(pd);
    T->xhat.upload(xh);
    // work items: a coarse cell's point range split into pieces of at most
    // maxp points, so levels with few, large coarse cells (C4: ~1,400 points
    // per cell; its middle level has only 512 coarse cells) still fill the GPU.
    // Split only levels with fewer coarse cells than ~16 warps per SM
    // (measured on B200: splitting C4's fine level, 12,167 cells, costs
    // 0.437 -> 0.470 ms in the restriction)
    int nsm = 148;
    NNMG_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, coarse->device));
    int maxp = 1 << 30;
    if (ncc < int64_t(nsm) * 16) {
      const int64_t want = int64_t(nsm) * 32;  // items to aim for
      maxp = static_cast<int>(std::max<int64_t>(64, (npts + want - 1) / want));
    }
    if (const char* e = getenv("NNMG_TRANSFER_MAXP")) maxp = std::max(32, atoi(e));
    std::vector<int> ipt(1, 0), icell, ifirst(ncc + 1, 0);
    for (int64_t c = 0; c < ncc; ++c) {
      const int n = start[c + 1] - start[c];
      const int k = std::max(1, (n + maxp - 1) / maxp);
      ifirst[c] = static_cast<int>(icell.size());
      for (int j = 0; j < k; ++j) {
        icell.push_back(static_cast<int>(c));
        ipt.push_back(start[c] + static_cast<int>((int64_t(n) * (j + 1)) / k));
      }
    }
    ifirst[ncc] = static_cast<int>(icell.size());
    T->nitems = static_cast<int64_t>(icell.size());
    T->item_pt.upload(ipt);
    T->item_cell.upload(icell);
    // transposed coarse map for the restriction gather
    const int nloc = coarse->nloc;
    const int64_t nsc = coarse->n_scalar;
    std::vector<int> off(nsc + 1, 0);
    // entries (item, l) of every work item of the cells holding coarse DoF g,
    // in a fixed order (cell, local index, item): deterministic phase 2
    for (int64_t e = 0; e < ncc * nloc; ++e) {
      const int g = coarse->cell_dofs_host[e];
      if (!coarse->scalar_constrained[g]) off[g + 1] += ifirst[e / nloc + 1] - ifirst[e / nloc];
    }
    for (int64_t g = 0; g < nsc; ++g) off[g + 1] += off[g];
    NNMG_REQUIRE(int64_t(off[nsc]) < (int64_t(1) << 31) && T->nitems * nloc < (int64_t(1) << 31), kUnsupported,
                 "restriction map exceeds 2^31 entries");
    std::vector<int> pos(off.begin(), off.end() - 1);
    std::vector<int> ent(off[nsc]);
    for (int64_t e = 0; e < ncc * nloc; ++e) {
      const int g = coarse->cell_dofs_host[e];
      if (coarse->scalar_constrained[g]) continue;
      const int64_t c = e / nloc, l = e % nloc;
      for (int it = ifirst[c]; it < ifirst[c + 1]; ++it) ent[pos[g]++] = static_cast<int>(it * nloc + l);
    }
    T->t_off.upload(off);
    T->t_ent.upload(ent);
    T->cellbuf.alloc(size_t(T->nitems) * nloc * T->ncomp);
    // restriction: consecutive coarse cells per warp, so the point stream is
    // pipelined across cell boundaries; aim for >= ~4 warps per SM slot
    {
      const char* e = getenv("NNMG_RESTRICT_CHUNK");
      const int64_t target_warps = int64_t(nsm) * 16 * 4;
      int ch = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(16, T->nitems / target_warps)));
      if (e) ch = std::max(1, std::min(31, atoi(e)));
      T->chunk = ch;
      const char* pp = getenv("NNMG_PROLONG_PPL");
      T->prolong_ppl = pp ? atoi(pp) : 1;
      // NLOC*NCOMP <= 32: 0 / 1 / 3 = lane-owned with 1 / 2 / 3 points per round, 2 = staged groups,
      // unset = 3 in 3D, 1 in 2D
      const char* k = getenv("NNMG_RESTRICT_KERNEL");
      T->restrict_kernel = k ? atoi(k) : -1;
      // 32 < NLOC*NCOMP <= 81: 1 = lane-owned local vector, 0 = staged groups
      const char* w = getenv("NNMG_RESTRICT_WIDE");
      T->restrict_wide = w ? atoi(w) : 0;
      // staged groups: planes of the outermost axis per lane (1 or 2)
      const char* pl = getenv("NNMG_RESTRICT_PL");
      T->restrict_pl = pl ? atoi(pl) : 1;
      const char* ma = getenv("NNMG_MIXED_ARITH");
      T->mixed_arith32 = ma ? atoi(ma) != 64 : true;
      const char* twp = getenv("NNMG_TRANSFER_WARPS");
      T->transfer_warps = twp ? atoi(twp) : 0;  // 0: default by dimension
    }
    // fine scalar DoFs without a transfer point: zeroed by the plain prolongation
    std::vector<uint8_t> has(fine->n_scalar, 0);
    for (int64_t i = 0; i < npts; ++i) has[point_dofs[i]] = 1;
    std::vector<int> nopt;
    for (int64_t d = 0; d < fine->n_scalar; ++d)
      if (!has[d]) nopt.push_back(static_cast<int>(d));
    T->no_point.upload(nopt);
  } catch (...) {
    delete T;
    throw;
  }
  return T;
}

template <class TV>
static void prolongate_t(Transfer& T, const TV* uc, TV* uf, bool accumulate, cudaStream_t s) {
  if (T.timing) NNMG_CUDA_TRY(cudaEventRecord(T.ev[0], s));
  if (!accumulate) {
    // every point DoF is written below; only the point-less ones need zeros
    const int64_t n = int64_t(T.no_point.n) * T.ncomp;
    if (n) {
      k_zero_list<TV><<<grid_for(n, 256), 256, 0, s>>>(T.no_point.ptr, int64_t(T.no_point.n), T.ncomp, uf);
      NNMG_CHECK_LAUNCH();
      count_launch();
    }
  }
  if (T.timing) NNMG_CUDA_TRY(cudaEventRecord(T.ev[1], s));
  TransferDispatchT<TV> f{T, uc, uf, accumulate ? 1 : 0, s};
  dispatch(T.dim, T.pc, T.ncomp, T.coarse->physics, f);
  if (T.timing) {
    NNMG_CUDA_TRY(cudaEventRecord(T.ev[2], s));
    T.ev_eval = 1;
  }
}

Transfer::~Transfer() {
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
}

void transfer_set_timing(Transfer& T, bool on) {
  if (on && !T.ev[0]) {
    NNMG_CUDA_TRY(cudaSetDevice(T.coarse->device));
    for (auto& e : T.ev) NNMG_CUDA_TRY(cudaEventCreate(&e));
  }
  T.timing = on;
}

void transfer_last_timing(Transfer& T, double* evaluate_s, double* gather_scatter_s) {
  NNMG_REQUIRE(T.ev[0], kInvalidArgument, "transfer timing was never enabled");
  NNMG_CUDA_TRY(cudaEventSynchronize(T.ev[2]));
  float a = 0.f, b = 0.f;
  NNMG_CUDA_TRY(cudaEventElapsedTime(&a, T.ev[0], T.ev[1]));
  NNMG_CUDA_TRY(cudaEventElapsedTime(&b, T.ev[1], T.ev[2]));
  const double ev = (T.ev_eval == 0 ? a : b) * 1e-3, gs = (T.ev_eval == 0 ? b : a) * 1e-3;
  if (evaluate_s) *evaluate_s = ev;
  if (gather_scatter_s) *gather_scatter_s = gs;
}

void transfer_prolongate(Transfer& T, const double* uc, double* uf, bool accumulate, cudaStream_t s) {
  prolongate_t(T, uc, uf, accumulate, s);
}

void transfer_restrict(Transfer& T, const double* rf, double* rc, cudaStream_t s) {
  TransferDispatch f{T, rf, rc, 2, s};
  dispatch(T.dim, T.pc, T.ncomp, T.coarse->physics, f);
}

__global__ void k_xhat_f32(const double* __restrict__ a, float* __restrict__ b, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = float(a[i]);
}

void transfer_enable_f32(Transfer& T, cudaStream_t s) {
  if (T.xhat32.n == T.xhat.n && T.xhat32.ptr) return;
  T.xhat32.alloc(T.xhat.n);
  if (T.xhat.n) {
    k_xhat_f32<<<grid_for(int64_t(T.xhat.n), 256), 256, 0, s>>>(T.xhat.ptr, T.xhat32.ptr, int64_t(T.xhat.n));
    NNMG_CHECK_LAUNCH();
    count_launch();
  }
}

void transfer_prolongate_f32(Transfer& T, const float* uc, float* uf, bool accumulate, cudaStream_t s) {
  NNMG_REQUIRE(T.xhat32.n == T.xhat.n, kInvalidArgument, "transfer fp32 records not prepared");
  prolongate_t(T, uc, uf, accumulate, s);
}

void transfer_restrict_f32(Transfer& T, const float* rf, float* rc, cudaStream_t s) {
  NNMG_REQUIRE(T.xhat32.n == T.xhat.n, kInvalidArgument, "transfer fp32 records not prepared");
  TransferDispatchT<float> f{T, rf, rc, 2, s};
  dispatch(T.dim, T.pc, T.ncomp, T.coarse->physics, f);
}

// ---------------------------------------------------------------------------
// Point location
// ---------------------------------------------------------------------------
struct BucketGrid {
  double g0[3], h[3];
  int nb[3];
};

template <int DIM>
__device__ __forceinline__ void forward_map(const double (&X)[1 << DIM][DIM], const double* xh, double* out) {
  for (int a = 0; a < DIM; ++a) out[a] = 0.0;
  for (int v = 0; v < (1 << DIM); ++v) {
    double w = 1.0;
    for (int j = 0; j < DIM; ++j) w *= ((v >> j) & 1) ? xh[j] : 1.0 - xh[j];
    for (int a = 0; a < DIM; ++a) out[a] += w * X[v][a];
  }
}

template <int DIM>
__device__ __forceinline__ void jacobian(const double (&X)[1 << DIM][DIM], const double* xh, double (&J)[DIM][DIM]) {
  for (int a = 0; a < DIM; ++a)
    for (int b = 0; b < DIM; ++b) J[a][b] = 0.0;
  for (int v = 0; v < (1 << DIM); ++v)
    for (int b = 0; b < DIM; ++b) {
      double g = 1.0;
      for (int j = 0; j < DIM; ++j) {
        const int bit = (v >> j) & 1;
        g *= (j == b) ? (bit ? 1.0 : -1.0) : (bit ? xh[j] : 1.0 - xh[j]);
      }
      for (int a = 0; a < DIM; ++a) J[a][b] += g * X[v][a];
    }
}

template <int DIM>
__device__ __forceinline__ double norm(const double* r) {
  double s = 0.0;
  for (int a = 0; a < DIM; ++a) s += r[a] * r[a];
  return sqrt(s);
}

// LU with partial pivoting; solves J s = r (returns s in r)
template <int DIM>
__device__ __forceinline__ void lu_solve(double (&A)[DIM][DIM], double* r) {
  int piv[DIM];
  for (int k = 0; k < DIM; ++k) {
    int p = k;
    for (int i = k + 1; i < DIM; ++i)
      if (fabs(A[i][k]) > fabs(A[p][k])) p = i;
    piv[k] = p;
    if (p != k)
      for (int j = 0; j < DIM; ++j) {
        const double t = A[k][j];
        A[k][j] = A[p][j];
        A[p][j] = t;
      }
    const double rinv = 1.0 / A[k][k];
    for (int i = k + 1; i < DIM; ++i) A[i][k] *= rinv;
    for (int i = k + 1; i < DIM; ++i)
      for (int j = k + 1; j < DIM; ++j) A[i][j] -= A[i][k] * A[k][j];
  }
  for (int k = 0; k < DIM; ++k)
    if (piv[k] != k) {
      const double t = r[k];
      r[k] = r[piv[k]];
      r[piv[k]] = t;
    }
  for (int k = 0; k < DIM; ++k)
    for (int i = k + 1; i < DIM; ++i) r[i] -= r[k] * A[i][k];
  for (int j = DIM - 1; j >= 0; --j) {
    r[j] /= A[j][j];
    for (int i = 0; i < j; ++i) r[i] -= r[j] * A[i][j];
  }
}

// damped Newton inversion of one multilinear cell map (mesh.py:235-287)
template <int DIM>
__device__ bool invert_map(const double (&X)[1 << DIM][DIM], const double* x, double tol, double* xh, double* rnorm) {
  double res[DIM], f[DIM];
  for (int j = 0; j < DIM; ++j) xh[j] = 0.5;
  forward_map<DIM>(X, xh, f);
  for (int a = 0; a < DIM; ++a) res[a] = f[a] - x[a];
  double rn = norm<DIM>(res);
  bool conv = rn <= tol;
  for (int it = 0; it < 30 && !conv; ++it) {
    double J[DIM][DIM];
    jacobian<DIM>(X, xh, J);
    double det, scale = 0.0;
    if constexpr (DIM == 2)
      det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    else
      det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
            J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    for (int a = 0; a < DIM; ++a)
      for (int b = 0; b < DIM; ++b) scale = fmax(scale, fabs(J[a][b]));
    scale = (DIM == 2 ? scale * scale : scale * scale * scale) + 1e-300;
    if (fabs(det) < 1e-14 * scale) break;  // singular: failed
    double step[DIM];
    for (int a = 0; a < DIM; ++a) step[a] = res[a];
    lu_solve<DIM>(J, step);
    double nx[DIM], nr[DIM];
    for (int j = 0; j < DIM; ++j) nx[j] = xh[j] - step[j];
    forward_map<DIM>(X, nx, f);
    for (int a = 0; a < DIM; ++a) nr[a] = f[a] - x[a];
    double nn = norm<DIM>(nr);
    for (int h = 0; h < 8 && nn > rn && nn > tol; ++h) {
      for (int j = 0; j < DIM; ++j) {
        step[j] *= 0.5;
        nx[j] = xh[j] - step[j];
      }
      forward_map<DIM>(X, nx, f);
      for (int a = 0; a < DIM; ++a) nr[a] = f[a] - x[a];
      nn = norm<DIM>(nr);
    }
    for (int j = 0; j < DIM; ++j) xh[j] = nx[j];
    for (int a = 0; a < DIM; ++a) res[a] = nr[a];
    rn = nn;
    conv = nn <= tol;
  }
  *rnorm = rn;
  return conv;
}

template <int DIM>
__global__ void k_locate(const double* __restrict__ verts, const int64_t* __restrict__ cells,
                         const double* __restrict__ blo, const double* __restrict__ bhi,
                         const int* __restrict__ boff, const int* __restrict__ bcells, BucketGrid grid,
                         const double* __restrict__ pts, int64_t npts, double eps_geo, double eps_ref,
                         int64_t* __restrict__ out_cell, double* __restrict__ out_xhat, uint8_t* __restrict__ out_proj,
                         int* __restrict__ n_missing, unsigned long long* __restrict__ first_missing) {
  constexpr int NV = 1 << DIM;
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= npts) return;
  double x[DIM];
  for (int j = 0; j < DIM; ++j) x[j] = pts[p * DIM + j];
  // bucket of the point (clamped); the padded-box test below decides exactly
  int b = 0, mult = 1;
  for (int j = 0; j < DIM; ++j) {
    const double t = fmin(fmax((x[j] - grid.g0[j]) / grid.h[j], -1.0), grid.nb[j] + 1.0);
    int bj = static_cast<int>(floor(t));
    bj = max(0, min(grid.nb[j] - 1, bj));
    b += bj * mult;
    mult *= grid.nb[j];
  }
  int64_t best_cell = -1, found = -1;
  double best_dist = 0.0, best_xh[DIM], found_xh[DIM];
  {
    for (int e = boff[b]; e < boff[b + 1] && found < 0; ++e) {
      const int c = bcells[e];
      bool in = true;
      for (int j = 0; j < DIM; ++j) in = in && x[j] >= blo[(int64_t)c * DIM + j] && x[j] <= bhi[(int64_t)c * DIM + j];
      if (!in) continue;
      double X[NV][DIM];
      for (int v = 0; v < NV; ++v)
        for (int a = 0; a < DIM; ++a) X[v][a] = verts[cells[(int64_t)c * NV + v] * DIM + a];
      double diam = 0.0;
      for (int u = 0; u < NV; ++u)
        for (int v = 0; v < NV; ++v) {
          double s = 0.0;
          for (int a = 0; a < DIM; ++a) s += (X[u][a] - X[v][a]) * (X[u][a] - X[v][a]);
          diam = fmax(diam, sqrt(s));
        }
      double xh[DIM], rn;
      const bool conv = invert_map<DIM>(X, x, 1e-12 * diam, xh, &rn);
      if (!conv) continue;
      bool inside = rn <= eps_geo;
      for (int j = 0; j < DIM; ++j) inside = inside && xh[j] >= -eps_ref && xh[j] <= 1.0 + eps_ref;
      if (inside) {
        found = c;
        for (int j = 0; j < DIM; ++j) found_xh[j] = fmin(fmax(xh[j], 0.0), 1.0);
        break;
      }
      double xp[DIM], f[DIM], d[DIM];
      for (int j = 0; j < DIM; ++j) xp[j] = fmin(fmax(xh[j], 0.0), 1.0);
      forward_map<DIM>(X, xp, f);
      for (int a = 0; a < DIM; ++a) d[a] = f[a] - x[a];
      const double dist = norm<DIM>(d);
      if (best_cell < 0 || dist < best_dist) {
        best_cell = c;
        best_dist = dist;
        for (int j = 0; j < DIM; ++j) best_xh[j] = xp[j];
      }
    }
  }
  if (found >= 0) {
    out_cell[p] = found;
    for (int j = 0; j < DIM; ++j) out_xhat[p * DIM + j] = found_xh[j];
    out_proj[p] = 0;
  } else if (best_cell >= 0) {
    out_cell[p] = best_cell;
    for (int j = 0; j < DIM; ++j) out_xhat[p * DIM + j] = best_xh[j];
    out_proj[p] = 1;
  } else {
    out_cell[p] = -1;
    for (int j = 0; j < DIM; ++j) out_xhat[p * DIM + j] = nan("");
    out_proj[p] = 0;
    atomicAdd(n_missing, 1);
    atomicMin(first_missing, static_cast<unsigned long long>(p));
  }
}

LocateResult locate_points(int device, int dim, int64_t nv, const double* vertices, int64_t nc, const int64_t* cells,
                           int64_t npts, const double* points, double eps_box, double eps_geo, double eps_ref,
                           int64_t* out_cells, double* out_xhat, uint8_t* out_projected) {
  NNMG_REQUIRE(dim == 2 || dim == 3, kInvalidArgument, "dim must be 2 or 3");
  NNMG_REQUIRE(nc > 0, kInvalidArgument, "empty mesh");
  NNMG_CUDA_TRY(cudaSetDevice(device));
  LocateResult res;
  if (npts == 0) return res;
  const int NV = 1 << dim;
  // padded boxes (geosearch.py:34-37)
  std::vector<double> lo(size_t(nc) * dim), hi(size_t(nc) * dim);
  double g0[3] = {INFINITY, INFINITY, INFINITY}, g1[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t c = 0; c < nc; ++c)
    for (int j = 0; j < dim; ++j) {
      double mn = INFINITY, mx = -INFINITY;
      for (int v = 0; v < NV; ++v) {
        const int64_t vi = cells[c * NV + v];
        NNMG_REQUIRE(vi >= 0 && vi < nv, kInvalidArgument, "cell vertex index out of range");
        mn = std::min(mn, vertices[vi * dim + j]);
        mx = std::max(mx, vertices[vi * dim + j]);
      }
      lo[c * dim + j] = mn - eps_box;
      hi[c * dim + j] = mx + eps_box;
      g0[j] = std::min(g0[j], lo[c * dim + j]);
      g1[j] = std::max(g1[j], hi[c * dim + j]);
    }
  BucketGrid grid{};
  const double per_axis = std::pow(static_cast<double>(nc), 1.0 / dim);
  int64_t nbt = 1;
  for (int j = 0; j < 3; ++j) {
    if (j < dim) {
      grid.g0[j] = g0[j];
      grid.nb[j] = std::max(1, static_cast<int>(std::lround(per_axis)));
      grid.h[j] = (g1[j] - g0[j]) / grid.nb[j];
      if (!(grid.h[j] > 0.0)) grid.h[j] = 1.0;
    } else {
      grid.g0[j] = 0.0;
      grid.h[j] = 1.0;
      grid.nb[j] = 1;
    }
    nbt *= grid.nb[j];
  }
  auto range = [&](int64_t c, int j, int& a, int& b) {
    a = static_cast<int>(std::floor((lo[c * dim + j] - grid.g0[j]) / grid.h[j]));
    b = static_cast<int>(std::floor((hi[c * dim + j] - grid.g0[j]) / grid.h[j]));
    a = std::max(0, std::min(grid.nb[j] - 1, a));
    b = std::max(0, std::min(grid.nb[j] - 1, b));
  };
  std::vector<int> boff(nbt + 1, 0);
  for (int pass = 0; pass < 2; ++pass) {
    std::vector<int> fill;
    std::vector<int> bc;
    if (pass == 1) {
      for (int64_t i = 0; i < nbt; ++i) boff[i + 1] += boff[i];
      fill.assign(boff.begin(), boff.end() - 1);
      bc.resize(boff[nbt]);
    }
    for (int64_t c = 0; c < nc; ++c) {
      int a[3] = {0, 0, 0}, b[3] = {0, 0, 0};
      for (int j = 0; j < dim; ++j) range(c, j, a[j], b[j]);
      for (int k = a[2]; k <= b[2]; ++k)
        for (int jj = a[1]; jj <= b[1]; ++jj)
          for (int i = a[0]; i <= b[0]; ++i) {
            const int64_t bk = i + grid.nb[0] * (jj + int64_t(grid.nb[1]) * k);
            if (pass == 0)
              boff[bk + 1] += 1;
            else
              bc[fill[bk]++] = static_cast<int>(c);
          }
    }
    if (pass == 1) {
      // cells were appended in ascending order: each bucket list is sorted
      DevBuf<double> dv, dlo, dhi, dpts, dxh;
      DevBuf<int64_t> dcells, dout;
      DevBuf<int> dboff, dbc, dmiss;
      DevBuf<uint8_t> dproj;
      DevBuf<unsigned long long> dfirst;
      dv.upload(vertices, size_t(nv) * dim);
      dcells.upload(cells, size_t(nc) * NV);
      dlo.upload(lo);
      dhi.upload(hi);
      dboff.upload(boff);
      dbc.upload(bc);
      dpts.upload(points, size_t(npts) * dim);
      dout.alloc(npts);
      dxh.alloc(size_t(npts) * dim);
      dproj.alloc(npts);
      dmiss.alloc(1);
      dmiss.zero();
      unsigned long long init = ~0ull;
      dfirst.upload(&init, 1);
      const int bs = 128;
      if (dim == 2)
        k_locate<2><<<grid_for(npts, bs), bs>>>(dv.ptr, dcells.ptr, dlo.ptr, dhi.ptr, dboff.ptr, dbc.ptr, grid,
                                                 dpts.ptr, npts, eps_geo, eps_ref, dout.ptr, dxh.ptr, dproj.ptr,
                                                 dmiss.ptr, dfirst.ptr);
      else
        k_locate<3><<<grid_for(npts, bs), bs>>>(dv.ptr, dcells.ptr, dlo.ptr, dhi.ptr, dboff.ptr, dbc.ptr, grid,
                                                 dpts.ptr, npts, eps_geo, eps_ref, dout.ptr, dxh.ptr, dproj.ptr,
                                                 dmiss.ptr, dfirst.ptr);
      NNMG_CHECK_LAUNCH();
      count_launch();
      NNMG_CUDA_TRY(cudaMemcpy(out_cells, dout.ptr, sizeof(int64_t) * npts, cudaMemcpyDeviceToHost));
      NNMG_CUDA_TRY(cudaMemcpy(out_xhat, dxh.ptr, sizeof(double) * npts * dim, cudaMemcpyDeviceToHost));
      NNMG_CUDA_TRY(cudaMemcpy(out_projected, dproj.ptr, npts, cudaMemcpyDeviceToHost));
      unsigned long long fm = 0;
      NNMG_CUDA_TRY(cudaMemcpy(&res.n_missing, dmiss.ptr, sizeof(int), cudaMemcpyDeviceToHost));
      NNMG_CUDA_TRY(cudaMemcpy(&fm, dfirst.ptr, sizeof(fm), cudaMemcpyDeviceToHost));
      res.first_missing = res.n_missing ? static_cast<int64_t>(fm) : -1;
    }
  }
  return res;
}

}  // namespace nnmg
