// K4 geometry precompute, K1/K2 matrix-free apply, K3 diagonal.
#include "nnmg_level.cuh"
#include "nnmg_kernels.cuh"
#include "nnmg_cellkernel.cuh"
#include "nnmg_cellreg.cuh"
#include "nnmg_cellreg_elast.cuh"

#include <algorithm>
#include <cstring>

namespace nnmg {

// ---------------------------------------------------------------------------
template <bool NEG>
__global__ void k_cell_gather(const int* __restrict__ off, const int* __restrict__ ent,
                              const double* __restrict__ cellout, int64_t nsc, int ncomp, int cb,
                              double* __restrict__ dst);

// ---------------------------------------------------------------------------
// K4: per-quadrature-point geometry (mfoperator.py:28-48, 101-106, 163-169)
// J[a][b] = sum_v dW_v/dxhat_b(q) X_v[a]   (mesh.py:138-143)
// ---------------------------------------------------------------------------
template <int DIM, int PHYS>
__global__ void k_geometry(const double* __restrict__ verts, const int* __restrict__ cells,
                           int64_t n_cells, int nq1, Tables tab, int cb, double* __restrict__ geo,
                           int* __restrict__ bad) {
  constexpr int NV = 1 << DIM;
  constexpr int NG = GeoCount<DIM, PHYS>::value;
  const int nq = DIM == 2 ? nq1 * nq1 : nq1 * nq1 * nq1;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_cells * nq) return;
  const int64_t c = t / nq;
  const int q = static_cast<int>(t % nq);
  int qi[3] = {q % nq1, (q / nq1) % nq1, q / (nq1 * nq1)};
  double xh[3], wq = 1.0;
  for (int j = 0; j < DIM; ++j) {
    xh[j] = tab.xq[qi[j]];
    wq *= tab.w[qi[j]];
  }
  double J[DIM][DIM] = {};
  for (int v = 0; v < NV; ++v) {
    const double* X = verts + (int64_t)cells[c * NV + v] * DIM;
    for (int b = 0; b < DIM; ++b) {
      double gr = 1.0;
      for (int j = 0; j < DIM; ++j) {
        const int bit = (v >> j) & 1;
        if (j == b)
          gr *= bit ? 1.0 : -1.0;
        else
          gr *= bit ? xh[j] : 1.0 - xh[j];
      }
      for (int a = 0; a < DIM; ++a) J[a][b] += gr * X[a];
    }
  }
  double det, K[DIM][DIM];
  if constexpr (DIM == 2) {
    det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    K[0][0] = J[1][1] / det;
    K[0][1] = -J[0][1] / det;
    K[1][0] = -J[1][0] / det;
    K[1][1] = J[0][0] / det;
  } else {
    const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
    const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
    const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
    det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
    K[0][0] = c00 / det;
    K[1][0] = c01 / det;
    K[2][0] = c02 / det;
    K[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
    K[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
    K[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
    K[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
    K[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
    K[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
  }
  if (!(det > 0.0)) atomicOr(bad, 1);
  const int64_t blk = c / cb, lane = c % cb;
  double* out = geo + ((blk * nq + q) * NG) * cb + lane;
  if constexpr (PHYS == kLaplace) {
    int k = 0;
    for (int a = 0; a < DIM; ++a)
      for (int b = a; b < DIM; ++b) {
        double s = 0.0;
        for (int j = 0; j < DIM; ++j) s += K[a][j] * K[b][j];
        out[(k++) * cb] = s * det * wq;
      }
  } else {
    for (int a = 0; a < DIM; ++a)
      for (int b = 0; b < DIM; ++b) out[(a * DIM + b) * cb] = K[a][b];
    out[DIM * DIM * cb] = det * wq;
  }
}

template <int DIM>
__global__ void k_edges(const double* __restrict__ verts, const int* __restrict__ cells, int64_t n_cells, int cb,
                        double* __restrict__ edges);

// SPLIT CTAs per cell block (SCB = CB / SPLIT cells each): smaller CTAs get
// a larger register budget per thread (the Q4 kernel spills at CB = 32)
template <int DIM, int P, int NCOMP, int PHYS, int SPLIT, class TA = double>
using ApplyKernel = CellKernel<DIM, P, NCOMP, PHYS, CellKernel<DIM, P, NCOMP, PHYS>::CB / SPLIT, TA>;

// min resident CTAs per SM for the split variants (measured on B200: 5 gives
// C5 0.310 -> 0.279 ms, C4 0.643 -> 0.639 ms)
#ifndef NNMG_APPLY_MINB
#define NNMG_APPLY_MINB 5
#endif
// with the geometry staged in shared memory (GEOS) fewer CTAs fit per SM
#ifndef NNMG_APPLY_MINB_GEOS
#define NNMG_APPLY_MINB_GEOS 3
#endif
template <int DIM, int P, int NCOMP, int PHYS, bool NEG, int SPLIT, int GEO = 0, int MINB = 0, class TV = double,
          class TA = double>
__global__ void __launch_bounds__(ApplyKernel<DIM, P, NCOMP, PHYS, SPLIT>::NTHREADS,
                                  MINB > 0 ? MINB
                                           : (SPLIT == 1 ? 1 : (GEO == 1 ? NNMG_APPLY_MINB_GEOS : NNMG_APPLY_MINB)))
    k_apply(Tables tab, const TV* __restrict__ src, TV* __restrict__ dst, const int* __restrict__ idx,
            const double* __restrict__ geo, int64_t b0, double lam, double mu, double* __restrict__ cellout) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  TA* sm = reinterpret_cast<TA*>(sm_raw);
  using CK = ApplyKernel<DIM, P, NCOMP, PHYS, SPLIT, TA>;
  CK::template run<false, NEG, GEO>(tab, PlainSrcT<TV>{src}, dst, idx, geo, b0 + blockIdx.x / SPLIT, lam, mu, sm,
                                     threadIdx.x, [] __device__() { __syncthreads(); },
                                     int(blockIdx.x % SPLIT) * CK::SCB, cellout);
}

// ---------------------------------------------------------------------------
// K3: exact diagonal.  Thread per (cell, local DoF); sum over quadrature
// points of w gt^T G gt (Laplace, mfoperator.py:135-150) or
// dv((lam+mu) pg_a^2 + mu |pg|^2) (elasticity, mfoperator.py:219-238).
// ---------------------------------------------------------------------------
template <int DIM, int P, int NCOMP, int PHYS>
__global__ void k_diagonal(Tables tab, const int* __restrict__ idx, const double* __restrict__ geo, int64_t nblk,
                           double lam, double mu, double* __restrict__ diag, double* __restrict__ cellout) {
  using CK = CellKernel<DIM, P, NCOMP, PHYS>;
  constexpr int N1 = CK::N1, NLOC = CK::NLOC, CB = CK::CB, NG = CK::NG;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nblk * NLOC * CB) return;
  const int lane = t % CB;
  const int l = (t / CB) % NLOC;
  const int64_t blk = t / (CB * NLOC);
  const int g = idx[(blk * NLOC + l) * CB + lane];
  if (g < 0) return;
  const int li[3] = {l % N1, (l / N1) % N1, l / (N1 * N1)};
  double acc[NCOMP] = {};
  for (int q = 0; q < NLOC; ++q) {
    const int qi[3] = {q % N1, (q / N1) % N1, q / (N1 * N1)};
    double gt[DIM];
    for (int j = 0; j < DIM; ++j) {
      double s = 1.0;
      for (int k = 0; k < DIM; ++k) s *= (k == j ? tab.D[qi[k]][li[k]] : tab.S[qi[k]][li[k]]);
      gt[j] = s;
    }
    const double* G = geo + ((blk * NLOC + q) * NG) * CB + lane;
    if constexpr (PHYS == kLaplace) {
      double Gm[DIM][DIM];
      int k = 0;
      for (int a = 0; a < DIM; ++a)
        for (int b = a; b < DIM; ++b) {
          Gm[a][b] = G[(k++) * CB];
          Gm[b][a] = Gm[a][b];
        }
      double s = 0.0;
      for (int a = 0; a < DIM; ++a)
        for (int b = 0; b < DIM; ++b) s += gt[a] * Gm[a][b] * gt[b];
      acc[0] += s;
    } else {
      double pg[DIM];
      double n2 = 0.0;
      for (int b = 0; b < DIM; ++b) {
        double s = 0.0;
        for (int i = 0; i < DIM; ++i) s += gt[i] * G[(i * DIM + b) * CB];
        pg[b] = s;
        n2 += s * s;
      }
      const double dv = G[DIM * DIM * CB];
      for (int a = 0; a < NCOMP; ++a) acc[a] += dv * ((lam + mu) * pg[a] * pg[a] + mu * n2);
    }
  }
  for (int a = 0; a < NCOMP; ++a) {
    if (cellout)  // deterministic mode: summed by k_cell_gather in a fixed order
      cellout[((blk * NLOC + l) * NCOMP + a) * CB + lane] = acc[a];
    else
      atomicAdd(diag + (int64_t)g * NCOMP + a, acc[a]);
  }
}

// body load: thread per (cell, local DoF), b_l = sum_q det(J(q)) w_q prod_k S[q_k][l_k]
template <int DIM>
__global__ void k_load_vector(const double* __restrict__ verts, const int* __restrict__ cells, int64_t n_cells,
                              int n1, int cb, const int* __restrict__ idx, Tables tab, int ncomp, double f0,
                              double f1, double f2, double* __restrict__ b, double* __restrict__ cellout) {
  constexpr int NV = 1 << DIM;
  const int nloc = DIM == 2 ? n1 * n1 : n1 * n1 * n1;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_cells * nloc) return;
  const int64_t c = t / nloc;
  const int l = static_cast<int>(t % nloc);
  const int g = idx[((c / cb) * nloc + l) * cb + c % cb];
  if (g < 0) return;
  const int li[3] = {l % n1, (l / n1) % n1, l / (n1 * n1)};
  double X[NV][DIM];
  for (int v = 0; v < NV; ++v)
    for (int a = 0; a < DIM; ++a) X[v][a] = verts[(int64_t)cells[c * NV + v] * DIM + a];
  double acc = 0.0;
  for (int q = 0; q < nloc; ++q) {
    const int qi[3] = {q % n1, (q / n1) % n1, q / (n1 * n1)};
    double J[DIM][DIM] = {};
    double phi = 1.0, wq = 1.0;
    for (int j = 0; j < DIM; ++j) {
      phi *= tab.S[qi[j]][li[j]];
      wq *= tab.w[qi[j]];
    }
    for (int v = 0; v < NV; ++v)
      for (int bb = 0; bb < DIM; ++bb) {
        double gr = 1.0;
        for (int j = 0; j < DIM; ++j) {
          const int bit = (v >> j) & 1;
          gr *= (j == bb) ? (bit ? 1.0 : -1.0) : (bit ? tab.xq[qi[j]] : 1.0 - tab.xq[qi[j]]);
        }
        for (int a = 0; a < DIM; ++a) J[a][bb] += gr * X[v][a];
      }
    double det;
    if constexpr (DIM == 2)
      det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
    else
      det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
            J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    acc += det * wq * phi;
  }
  const double f[3] = {f0, f1, f2};
  for (int a = 0; a < ncomp; ++a) {
    if (cellout)  // deterministic mode
      cellout[(((c / cb) * nloc + l) * ncomp + a) * cb + c % cb] = f[a] * acc;
    else if (f[a] != 0.0)
      atomicAdd(b + (int64_t)g * ncomp + a, f[a] * acc);
  }
}

__global__ void k_copy_constrained(const int* __restrict__ cd, int64_t n, const double* __restrict__ src,
                                   double* __restrict__ dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[cd[i]] = src[cd[i]];
}

__global__ void k_set_constrained(const int* __restrict__ cd, int64_t n, double val, double* __restrict__ dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[cd[i]] = val;
}

__global__ void k_reciprocal(const double* __restrict__ a, double* __restrict__ b, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = 1.0 / a[i];
}

// ---------------------------------------------------------------------------
// dispatch
// ---------------------------------------------------------------------------
struct CbOf {
  int* out;
  template <int D, int P, int NC, int PH>
  void operator()() { *out = cells_per_block<D, P, NC>(); }
};

static int cb_of(int dim, int degree, int ncomp, int physics) {
  int cb = 0;
  CbOf f{&cb};
  dispatch(dim, degree, ncomp, physics, f);
  return cb;
}

static inline unsigned grid_for(int64_t n, int bs) { return static_cast<unsigned>((n + bs - 1) / bs); }

Level* level_create(int device, int dim, int degree, int ncomp, int physics, int64_t n_cells,
                    int64_t n_vertices, const double* vertices, const int64_t* cells, int64_t n_scalar,
                    const int64_t* cell_dofs, int64_t n_constrained, const int64_t* constrained, double lam,
                    double mu) {
  NNMG_REQUIRE(dim == 2 || dim == 3, kInvalidArgument, "dim must be 2 or 3");
  NNMG_REQUIRE(physics == kLaplace ? ncomp == 1 : ncomp == dim, kInvalidArgument,
               "Laplace needs 1 component, elasticity dim components");
  NNMG_REQUIRE(n_cells > 0, kInvalidArgument, "empty mesh");
  NNMG_REQUIRE(n_scalar * ncomp < (int64_t(1) << 31), kUnsupported, "more than 2^31 DoFs per level");
  NNMG_CUDA_TRY(cudaSetDevice(device));
  auto L = new Level();
  try {
    L->device = device;
    L->dim = dim;
    L->degree = degree;
    L->ncomp = ncomp;
    L->physics = physics;
    L->n1 = degree + 1;
    L->nloc = ipow(L->n1, dim);
    L->nq = L->nloc;
    L->ng = physics == kLaplace ? dim * (dim + 1) / 2 : dim * dim + 1;
    L->cb = cb_of(dim, degree, ncomp, physics);
    L->n_cells = n_cells;
    L->nblk = (n_cells + L->cb - 1) / L->cb;
    L->n_scalar = n_scalar;
    L->n_dofs = n_scalar * ncomp;
    L->lam = lam;
    L->mu = mu;
    L->tab = make_tables(degree);
    {
      const char* e = getenv("NNMG_APPLY_KERNEL");
      L->reg_kernel = !(e && std::string(e) == "pencil");
      const char* m = getenv("NNMG_REG_MINB");
      {
        // Q3/Q4 Laplace: G recomputed from edge vectors in the pencil apply.
        // Measured on B200 (C4, Q4): stored G 0.639 ms (split 4), recomputed
        // 0.531 ms (split 8), 0.712 (split 4), 0.876 (split 2)
        const char* rc = getenv("NNMG_APPLY_RECOMPUTE");
        L->apply_recompute = rc ? atoi(rc) != 0 : (dim == 3 && degree >= 3 && physics == kLaplace);
        const char* sp = getenv("NNMG_APPLY_SPLIT");
        // measured on B200: stored-G Q4 Laplace (C4) 0.684 -> 0.613 ms with 4,
        // Q2 elasticity pencil (C5) 0.288 -> 0.279 ms with 2
        L->apply_split = sp ? atoi(sp)
                            : (L->apply_recompute ? 8 : (dim == 3 && degree >= 4 ? 4 : (ncomp > 1 ? 2 : 1)));
        if (L->apply_split != 2 && L->apply_split != 4 && L->apply_split != 8) L->apply_split = 1;
        // Q3/Q4: geometry staged in shared memory by LDGSTS (k_apply GEOS)
        const char* gs = getenv("NNMG_APPLY_GEOS");
        // measured on B200 (C4): 0.643 ms with, 0.641 ms without: opt-in
        L->apply_geos = gs ? atoi(gs) != 0 : false;
      }
      L->reg_minb = m ? atoi(m) : 1;
      const char* fc = getenv("NNMG_FUSE_CONSTRAINED");
      L->fuse_constrained = fc ? atoi(fc) != 0 : true;
      const char* rm = getenv("NNMG_RECOMPUTE_MOD");
      L->recompute_mod = rm ? atoi(rm) : 0;
      const char* rn = getenv("NNMG_RECOMPUTE_NUM");
      L->recompute_num = rn ? atoi(rn) : 1;
      const char* rt = getenv("NNMG_REG_TMA");
      L->reg_tma = rt ? atoi(rt) != 0 : false;
      const char* er = getenv("NNMG_ELAST_RECOMPUTE");
      L->elast_recompute = er ? atoi(er) != 0 : false;
      const char* rr = getenv("NNMG_REG_RECOMPUTE");
      L->reg_recompute = rr ? atoi(rr) != 0 : false;
      const char* ex = getenv("NNMG_ELAST_XCH");
      // measured on B200 (C5 fine apply): 257 -> 222 us
      L->elast_xch = ex ? atoi(ex) != 0 : true;
      // warp-neighbour face sharing in the register Laplace apply.  Measured on
      // B200: fp32 arithmetic (mixed cycle) C3 4.66 -> 4.39 ms, C2 0.329 ->
      // 0.314 ms; fp64 2D (C2) apply 23.6 -> 21.5 us; fp64 3D (C3) apply 626
      // -> 677 us (DRAM-bound already: the extra shuffle phases only cost).
      // Default: on for the fp32 kernels and for 2D fp64, off for 3D fp64.
      const char* rw = getenv("NNMG_REG_WARPS");
      L->reg_warps = rw ? atoi(rw) : 0;  // 0: default by dimension
      const char* rw32 = getenv("NNMG_REG_WARPS32");
      L->reg_warps32 = rw32 ? atoi(rw32) : 0;
      const char* en = getenv("NNMG_ELAST_XNB");
      L->elast_xnb = en ? atoi(en) != 0 : false;
      const char* xn = getenv("NNMG_REG_XNB");
      L->reg_xnb32 = xn ? atoi(xn) != 0 : true;
      L->reg_xnb = xn ? atoi(xn) != 0 : dim == 2;
      L->reg_xnb_mode = xn ? atoi(xn) : 1;  // 2: sharing in the scatter only (fp64)
      const char* mb = getenv("NNMG_APPLY_MINB");
      L->apply_minb = mb ? atoi(mb) : 0;
      const char* ma = getenv("NNMG_MIXED_ARITH");
      L->mixed_arith32 = ma ? atoi(ma) != 64 : true;
      const char* et = getenv("NNMG_ELAST_TMA");
      L->elast_tma = et ? atoi(et) != 0 : false;
      const char* eb = getenv("NNMG_ELAST_BLN");
      L->elast_bln = eb ? atoi(eb) != 0 : false;

    }
    // constraints: the kernels support whole-node constraints (every component
    // of a scalar DoF), which is what dirichlet_constraints produces
    L->scalar_constrained.assign(n_scalar, 0);
    std::vector<int> cd(n_constrained);
    std::vector<int> per_node(n_scalar, 0);
    for (int64_t i = 0; i < n_constrained; ++i) {
      const int64_t d = constrained[i];
      NNMG_REQUIRE(d >= 0 && d < L->n_dofs, kInvalidArgument, "constrained DoF out of range");
      cd[i] = static_cast<int>(d);
      per_node[d / ncomp] += 1;
    }
    for (int64_t s = 0; s < n_scalar; ++s) {
      NNMG_REQUIRE(per_node[s] == 0 || per_node[s] == ncomp, kUnsupported,
                   "partially constrained vector nodes are not supported");
      L->scalar_constrained[s] = per_node[s] ? 1 : 0;
    }
    L->cdofs.upload(cd);
    // index table in the blocked layout
    const int nloc = L->nloc, cb = L->cb;
    std::vector<int> idx(size_t(L->nblk) * nloc * cb, -1);
    L->cell_dofs_host.resize(size_t(n_cells) * nloc);
    for (int64_t c = 0; c < n_cells; ++c) {
      const int64_t blk = c / cb, lane = c % cb;
      for (int l = 0; l < nloc; ++l) {
        const int64_t g = cell_dofs[c * nloc + l];
        NNMG_REQUIRE(g >= 0 && g < n_scalar, kInvalidArgument, "cell_dofs entry out of range");
        L->cell_dofs_host[c * nloc + l] = static_cast<int>(g);
        idx[(blk * nloc + l) * cb + lane] = L->scalar_constrained[g] ? -1 : static_cast<int>(g);
      }
    }
    L->idx.upload(idx);
    if (physics == kElasticity && dim == 3 && nloc <= 27 && L->reg_kernel && L->elast_bln) {
      // block-local node tables of the elasticity register apply
      const int nslot = nloc * cb;
      std::vector<std::vector<int>> nodes(L->nblk);
      int kmax = 0;
      for (int64_t b = 0; b < L->nblk; ++b) {
        auto& nd = nodes[b];
        nd.reserve(nslot);
        for (int sidx = 0; sidx < nslot; ++sidx) {
          const int g = idx[b * nslot + sidx];
          if (g >= 0) nd.push_back(g);
        }
        std::sort(nd.begin(), nd.end());
        nd.erase(std::unique(nd.begin(), nd.end()), nd.end());
        kmax = std::max<int>(kmax, static_cast<int>(nd.size()));
      }
      const int kp = (kmax + 31) / 32 * 32;
      L->bln_kp = kp;
      std::vector<int> bnode(size_t(L->nblk) * kp, -1), bcnt(L->nblk, 0);
      const int np = (nloc + 1) / 2;
      std::vector<unsigned> bslot(size_t(L->nblk) * np * cb, 0xFFFFFFFFu);
      bool distinct = true;  // within one local index, the cells of a block hold distinct nodes
      std::vector<uint8_t> seen;
      for (int64_t b = 0; b < L->nblk && distinct; ++b) {
        const auto& nd = nodes[b];
        bcnt[b] = static_cast<int>(nd.size());
        std::copy(nd.begin(), nd.end(), bnode.begin() + b * kp);
        for (int l = 0; l < nloc && distinct; ++l) {
          seen.assign(nd.size(), 0);
          for (int c = 0; c < cb; ++c) {
            const int g = idx[b * nslot + l * cb + c];
            if (g < 0) continue;
            const int k = static_cast<int>(std::lower_bound(nd.begin(), nd.end(), g) - nd.begin());
            unsigned& word = bslot[(b * np + l / 2) * cb + c];
            const unsigned ph = static_cast<unsigned>(k + (k >> 3));  // staging position (bln_phys)
            word = (l & 1) ? (word & 0x0000FFFFu) | (ph << 16) : (word & 0xFFFF0000u) | ph;
            if (seen[k]) distinct = false;
            seen[k] = 1;
          }
        }
      }
      if (distinct) {
        L->bln_node.upload(bnode);
        L->bln_cnt.upload(bcnt);
        L->bln_slot.upload(bslot);
      } else {
        L->elast_bln = false;  // e.g. rotated cells sharing a node at one local index: node-major exchange
      }
    }
    // geometry on the device from vertex coordinates
    NNMG_REQUIRE(n_vertices < (int64_t(1) << 31), kUnsupported, "more than 2^31 vertices");
    L->verts.upload(vertices, size_t(n_vertices) * dim);
    {
      std::vector<int> vc(size_t(n_cells) << dim);
      for (size_t i = 0; i < vc.size(); ++i) {
        NNMG_REQUIRE(cells[i] >= 0 && cells[i] < n_vertices, kInvalidArgument, "cell vertex index out of range");
        vc[i] = static_cast<int>(cells[i]);
      }
      L->vcells.upload(vc);
    }
    const double* dverts = L->verts.ptr;
    const int* dcells = L->vcells.ptr;
    L->geo.alloc(size_t(L->nblk) * L->nq * L->ng * cb);
    L->geo.zero();
    DevBuf<int> bad;
    bad.alloc(1);
    bad.zero();
    const int64_t nt = n_cells * L->nq;
    const int bs = 256;
    if (dim == 2 && physics == kLaplace)
      k_geometry<2, kLaplace><<<grid_for(nt, bs), bs>>>(dverts, dcells, n_cells, L->n1, L->tab, cb, L->geo.ptr, bad.ptr);
    else if (dim == 2)
      k_geometry<2, kElasticity><<<grid_for(nt, bs), bs>>>(dverts, dcells, n_cells, L->n1, L->tab, cb, L->geo.ptr, bad.ptr);
    else if (physics == kLaplace)
      k_geometry<3, kLaplace><<<grid_for(nt, bs), bs>>>(dverts, dcells, n_cells, L->n1, L->tab, cb, L->geo.ptr, bad.ptr);
    else
      k_geometry<3, kElasticity><<<grid_for(nt, bs), bs>>>(dverts, dcells, n_cells, L->n1, L->tab, cb, L->geo.ptr, bad.ptr);
    NNMG_CHECK_LAUNCH();
    count_launch();
    int hbad = 0;
    NNMG_CUDA_TRY(cudaMemcpy(&hbad, bad.ptr, sizeof(int), cudaMemcpyDeviceToHost));
    NNMG_REQUIRE(hbad == 0, kGeometryError, "mesh has non-positive Jacobians");
    // edge vectors for the hybrid-geometry register kernel (Laplace, low order)
    if ((physics == kLaplace && ncomp == 1 &&
         ((L->reg_kernel && (L->recompute_mod > 0 || (L->reg_recompute && dim == 3)) && L->nloc <= 27) ||
          (dim == 3 && L->apply_recompute))) ||
        (physics == kElasticity && dim == 3 && degree == 2 && L->reg_kernel && L->elast_recompute)) {
      const int ne = dim * (1 << (dim - 1)) * dim;
      L->edges.alloc(size_t(L->nblk) * ne * cb);
      L->edges.zero();
      if (dim == 2)
        k_edges<2><<<grid_for(n_cells, 256), 256>>>(dverts, dcells, n_cells, cb, L->edges.ptr);
      else
        k_edges<3><<<grid_for(n_cells, 256), 256>>>(dverts, dcells, n_cells, cb, L->edges.ptr);
      NNMG_CHECK_LAUNCH();
      count_launch();
    }
    L->diag.alloc(L->n_dofs);
    L->inv_diag.alloc(L->n_dofs);
  } catch (...) {
    delete L;
    throw;
  }
  return L;
}

// Constrained rows of the apply (mfoperator.py:114-121, zero-in / identity-out),
// fused into the cell kernels' prologue: the residual form (NEG) subtracts
// src there, the plain form copies it; cell threads never scatter to these
// rows, so there is no ordering between the two.
template <bool NEG, class TV>
__device__ __forceinline__ void constrained_rows(const int* __restrict__ cd, int64_t ncd,
                                                 const TV* __restrict__ src, TV* __restrict__ dst) {
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ncd; i += nthr) {
    const int c = cd[i];
    if constexpr (NEG)
      dst[c] -= src[c];
    else
      dst[c] = src[c];
  }
}

// one warp per cell block, one thread per cell (register-resident kernel)
// Hybrid geometry: cell blocks with blk % rmod == 0 recompute G from their
// edge vectors (288 B/cell instead of 1296 B/cell of stored G), the others
// stream the stored G; warp-uniform branch, both kinds share every SM so the
// FP64 pipe and HBM work concurrently.  rmod == 0: stored G only.
// Measured on B200 (C3): stored-G only 0.620 ms; naive recompute-only 0.700
// ms, in-kernel hybrids 0.67-0.72 ms (both paths in one kernel spill);
// sum-factorised recompute (GEO 2, 3D, k_apply_reg_rc) 0.633 ms; GEO-2
// hybrids 0.67-0.74 ms (1/4 .. 3/4 of the blocks recomputing).  Blocks with
// blk % rmod < rnum take the recompute path.  HYB is an opt-in instantiation
// (NNMG_RECOMPUTE_MOD / NNMG_RECOMPUTE_NUM) so the default kernel stays lean.
template <int D, int P, int MINB, bool NEG, bool HYB, class TV = double, class TG = double, class TA = double,
          int XNB = 0>
__global__ void __launch_bounds__(128, MINB) k_apply_reg(Tables tab, const TV* __restrict__ src, TV* __restrict__ dst,
                                                   const int* __restrict__ idx, const TG* __restrict__ geo,
                                                   int64_t b0, int64_t b1, const double* __restrict__ edges, int rmod,
                                                   int rnum, const int* __restrict__ cd, int64_t ncd,
                                                   double* __restrict__ cellout = nullptr) {
  if (ncd) constrained_rows<NEG>(cd, ncd, src, dst);
  // grid-stride over cell blocks (one pass for a full grid).  Measured on
  // B200 (profiles/r2_dual_apply_sweep.txt): persistent grids of this kernel
  // and of the recomputed-G kernel run concurrently on two streams over
  // complementary block ranges gain at most 3% on C3 (608 vs 627 us)
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t blk = b0 + blockIdx.x * wpb + (threadIdx.x >> 5); blk < b1; blk += gridDim.x * wpb) {
    if constexpr (HYB) {
      if (blk % rmod < rnum) {
        CellReg<D, P>::template run<true, false, NEG, D == 3 ? 2 : 1>(tab, PlainSrcT<TV>{src}, dst, idx, geo, blk,
                                                                      threadIdx.x & 31, edges);
        continue;
      }
    }
    CellReg<D, P>::template run<true, false, NEG, 0, TA, XNB>(tab, PlainSrcT<TV>{src}, dst, idx, geo, blk,
                                                              threadIdx.x & 31, nullptr, nullptr, cellout);
  }
}

// stored G streamed through shared memory by TMA bulk copies (3D, GEO 3)
template <int D, int P, bool NEG>
__global__ void __launch_bounds__(128, 1) k_apply_reg_tma(Tables tab, const double* __restrict__ src,
                                                         double* __restrict__ dst, const int* __restrict__ idx,
                                                         const double* __restrict__ geo, int64_t b0, int64_t b1) {
  extern __shared__ __align__(16) double dsm[];
  const int warp = threadIdx.x >> 5;
  const int64_t blk = b0 + blockIdx.x * (int64_t)(blockDim.x >> 5) + warp;
  if (blk >= b1) return;
  double* wsm = dsm + warp * (CellReg<D, P>::WARP_SMEM / sizeof(double));
  CellReg<D, P>::template run<true, false, NEG, 3>(tab, PlainSrc{src}, dst, idx, geo, blk, threadIdx.x & 31,
                                                   nullptr, wsm);
}

// fp32 geometry, the warp's whole chunk staged in shared memory by one TMA bulk copy (3D, GEO 4)
template <int D, int P>
__global__ void __launch_bounds__(128, 2) k_apply_reg_tma32(Tables tab, const float* __restrict__ src,
                                                           float* __restrict__ dst, const int* __restrict__ idx,
                                                           const float* __restrict__ geo, int64_t b0, int64_t b1,
                                                           const int* __restrict__ cd, int64_t ncd) {
  extern __shared__ __align__(128) unsigned char dsm_raw[];
  if (ncd) constrained_rows<true>(cd, ncd, src, dst);
  const int warp = threadIdx.x >> 5;
  const int64_t blk = b0 + blockIdx.x * (int64_t)(blockDim.x >> 5) + warp;
  if (blk >= b1) return;
  double* wsm = reinterpret_cast<double*>(dsm_raw + warp * ((CellReg<D, P>::WARP_SMEM32 + 127) / 128 * 128));
  CellReg<D, P>::template run<true, false, true, 4, float>(tab, PlainSrcT<float>{src}, dst, idx, geo, blk,
                                                           threadIdx.x & 31, nullptr, wsm);
}

// all blocks recompute G from edge vectors, sum-factorised along z-pencils (3D)
template <int D, int P, bool NEG>
__global__ void __launch_bounds__(128, 1) k_apply_reg_rc(Tables tab, const double* __restrict__ src,
                                                        double* __restrict__ dst, const int* __restrict__ idx,
                                                        int64_t b0, int64_t b1, const double* __restrict__ edges) {
  const int64_t wpb = blockDim.x >> 5;
  for (int64_t blk = b0 + blockIdx.x * wpb + (threadIdx.x >> 5); blk < b1; blk += gridDim.x * wpb)
  CellReg<D, P>::template run<true, false, NEG, 2>(tab, PlainSrc{src}, dst, idx, static_cast<const double*>(nullptr),
                                                   blk, threadIdx.x & 31,
                                                   edges);
}

// 3D elasticity, one thread per (cell, component): nnmg_cellreg_elast.cuh
template <int P, bool NEG, int GEO = 0, class TV = double, class TG = double, bool XCH = false, bool GSM = false,
          bool BLN = false, class TA = double, bool XNB = false>
__global__ void __launch_bounds__(96, sizeof(TA) == sizeof(float) ? 5 : 4) k_apply_reg_elast(Tables tab, const TV* __restrict__ src,
                                                        TV* __restrict__ dst, const int* __restrict__ idx,
                                                        const TG* __restrict__ geo, int64_t b0, int64_t b1,
                                                        double lam, double mu, const int* __restrict__ cd, int64_t ncd,
                                                        double* __restrict__ cellout = nullptr, BlnTables bln = {}) {
  // sized in elements of the arithmetic type: the fp32 exchange buffers take half the bytes
  __shared__ __align__(128) TA smt[CellRegElast<P>::SMEM_DOUBLES];
  double* sm = reinterpret_cast<double*>(smt);
  if (ncd) constrained_rows<NEG>(cd, ncd, src, dst);
  const int64_t blk = b0 + blockIdx.x;
  if (blk >= b1) return;
  CellRegElast<P>::template run<NEG, GEO, TV, TG, XCH, GSM, BLN, TA, XNB>(tab, src, dst, idx, geo, blk, lam, mu, sm,
                                                                          cellout, bln);
}

// per-cell edge vectors in the blocked layout [blk][(b*2^(d-1)+k)*d + a][CB]
template <int DIM>
__global__ void k_edges(const double* __restrict__ verts, const int* __restrict__ cells, int64_t n_cells, int cb,
                        double* __restrict__ edges) {
  constexpr int NV = 1 << DIM, NK = 1 << (DIM - 1), NE = DIM * NK * DIM;
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n_cells) return;
  const int64_t blk = c / cb, lane = c % cb;
  for (int b = 0; b < DIM; ++b) {
    int k = 0;
    for (int v = 0; v < NV; ++v) {
      if ((v >> b) & 1) continue;  // base vertex of an edge along b, others' bits ascending
      const int64_t v0 = cells[c * NV + v], v1 = cells[c * NV + (v | (1 << b))];
      for (int a = 0; a < DIM; ++a)
        edges[(blk * NE + (b * NK + k) * DIM + a) * cb + lane] = verts[v1 * DIM + a] - verts[v0 * DIM + a];
      ++k;
    }
  }
}

// TV = float: the mixed-precision V-cycle's apply (fp32 vectors and stored
// geometry, fp64 arithmetic); only the residual form (neg) and the default
// kernel variants are instantiated for it
template <class TV>
struct ApplyLaunchT {
  static constexpr bool kF64 = sizeof(TV) == sizeof(double);
  const Level& L;
  const TV* src;
  TV* dst;
  int64_t b0, b1;
  cudaStream_t s;
  bool neg;
  const int* cd = nullptr;  // constrained rows to fuse into the cell kernel (nullptr: caller handles them)
  double* cellout = nullptr;  // deterministic mode: cell buffer instead of atomics (fp64 only)
  int64_t ncd = 0;
  bool fused = false;       // set when the launched kernel handled them
  template <int D, int P, int NC, int PH>
  void operator()() {
    using CK = CellKernel<D, P, NC, PH>;
    if constexpr (!kF64) NNMG_REQUIRE(neg, kInvalidArgument, "fp32 apply is residual-form only");
    if constexpr (PH == kLaplace && NC == 1 && CellReg<D, P>::kSupported && !kF64) {
      if (L.reg_kernel) {
        const int64_t nb = b1 - b0;
        constexpr int kWarpsPerCta = 4;
        const unsigned g = static_cast<unsigned>((nb + kWarpsPerCta - 1) / kWarpsPerCta);
        if constexpr (D == 3) {
          if (L.mixed_arith32 && L.reg_tma) {
            constexpr size_t wsmem = (CellReg<D, P>::WARP_SMEM32 + 127) / 128 * 128;
            constexpr size_t smem = kWarpsPerCta * wsmem;
            static bool attr = false;
            if (!attr) {
              NNMG_CUDA_TRY(cudaFuncSetAttribute(k_apply_reg_tma32<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem));
              attr = true;
            }
            k_apply_reg_tma32<D, P><<<g, 32 * kWarpsPerCta, smem, s>>>(L.tab, src, dst, L.idx.ptr, L.geo32.ptr, b0, b1,
                                                                      cd, ncd);
            fused = true;
            NNMG_CHECK_LAUNCH();
            count_launch();
            return;
          }
        }
        // single-precision arithmetic (the paper's fp32 V-cycle) unless NNMG_MIXED_ARITH=64
        if (L.mixed_arith32 && L.reg_xnb32) {
          // one-warp CTAs in 3D (C3 mixed cycle 4.38 -> 4.31 ms), NNMG_REG_WARPS32 overrides
          const int wpc = (L.reg_warps32 == 1 || L.reg_warps32 == 2 || L.reg_warps32 == 4) ? L.reg_warps32
                                                                                           : (D == 3 ? 1 : 4);
          const unsigned gw = static_cast<unsigned>((nb + wpc - 1) / wpc);
          k_apply_reg<D, P, 3, true, false, float, float, float, 1><<<gw, 32 * wpc, 0, s>>>(
              L.tab, src, dst, L.idx.ptr, L.geo32.ptr, b0, b1, nullptr, 0, 1, cd, ncd, nullptr);
          fused = true;
          NNMG_CHECK_LAUNCH();
          count_launch();
          return;
        }
        auto kr = L.mixed_arith32 ? (L.reg_minb == 4 ? k_apply_reg<D, P, 4, true, false, float, float, float> : (L.reg_minb == 2 ? k_apply_reg<D, P, 2, true, false, float, float, float> : k_apply_reg<D, P, 3, true, false, float, float, float>))
                                  : k_apply_reg<D, P, 1, true, false, float, float, double>;
        kr<<<g, 32 * kWarpsPerCta, 0, s>>>(L.tab, src, dst, L.idx.ptr, L.geo32.ptr, b0, b1, nullptr, 0, 1, cd, ncd,
                                            nullptr);
        fused = true;
        NNMG_CHECK_LAUNCH();
        count_launch();
        return;
      }
    }
    if constexpr (PH == kLaplace && NC == 1 && CellReg<D, P>::kSupported && kF64) {
      if (L.reg_kernel) {
        const int64_t nb = b1 - b0;
        constexpr int kWarpsPerCta = 4;
        const unsigned g = static_cast<unsigned>((nb + kWarpsPerCta - 1) / kWarpsPerCta);
        if (cellout) {
          auto kd = neg ? k_apply_reg<D, P, 1, true, false> : k_apply_reg<D, P, 1, false, false>;
          kd<<<g, 32 * kWarpsPerCta, 0, s>>>(L.tab, src, dst, L.idx.ptr, L.geo.ptr, b0, b1, nullptr, 0, 1, cd, ncd,
                                              cellout);
          fused = true;
          NNMG_CHECK_LAUNCH();
          count_launch();
          return;
        }
        if constexpr (D == 3) {
          if (L.reg_tma) {
            constexpr size_t smem = kWarpsPerCta * CellReg<D, P>::WARP_SMEM;
            static bool attr = false;
            if (!attr) {
              NNMG_CUDA_TRY(cudaFuncSetAttribute(k_apply_reg_tma<D, P, true>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
              NNMG_CUDA_TRY(cudaFuncSetAttribute(k_apply_reg_tma<D, P, false>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
              attr = true;
            }
            auto kr = neg ? k_apply_reg_tma<D, P, true> : k_apply_reg_tma<D, P, false>;
            kr<<<g, 32 * kWarpsPerCta, smem, s>>>(L.tab, src, dst, L.idx.ptr, L.geo.ptr, b0, b1);
            NNMG_CHECK_LAUNCH();
            count_launch();
            return;
          }
          if (L.edges.ptr && L.reg_recompute) {
            auto kr = neg ? k_apply_reg_rc<D, P, true> : k_apply_reg_rc<D, P, false>;
            kr<<<g, 32 * kWarpsPerCta, 0, s>>>(L.tab, src, dst, L.idx.ptr, b0, b1, L.edges.ptr);
            NNMG_CHECK_LAUNCH();
            count_launch();
            return;
          }
        }
        if (L.reg_xnb && !(L.edges.ptr && L.recompute_mod > 0)) {
          auto kx = neg ? k_apply_reg<D, P, 1, true, false, double, double, double, 1>
                        : k_apply_reg<D, P, 1, false, false, double, double, double, 1>;
          if (L.reg_xnb_mode == 2)
            kx = neg ? k_apply_reg<D, P, 1, true, false, double, double, double, 2>
                     : k_apply_reg<D, P, 1, false, false, double, double, double, 2>;
          kx<<<g, 32 * kWarpsPerCta, 0, s>>>(L.tab, src, dst, L.idx.ptr, L.geo.ptr, b0, b1, nullptr, 0, 1, cd, ncd,
                                              nullptr);
          fused = true;
          NNMG_CHECK_LAUNCH();
          count_launch();
          return;
        }
        const bool hyb = L.edges.ptr && L.recompute_mod > 0;
        auto kr = hyb ? (neg ? k_apply_reg<D, P, 1, true, true> : k_apply_reg<D, P, 1, false, true>)
                      : (neg ? (L.reg_minb >= 3 ? k_apply_reg<D, P, 3, true, false> : k_apply_reg<D, P, 1, true, false>)
                             : (L.reg_minb >= 3 ? k_apply_reg<D, P, 3, false, false>
                                                : k_apply_reg<D, P, 1, false, false>));
        // warps (cell blocks) per CTA (NNMG_REG_WARPS): one-warp CTAs retire independently (no CTA
        // waits for its slowest warp); measured on B200: C3 apply 626.9 -> 619.4 us, cycle 7.24 ->
        // 7.16 ms with 1 instead of 4; C2 (2D) neutral.  Default 1 in 3D, 4 in 2D.
        const int wpc = (L.reg_warps == 1 || L.reg_warps == 2 || L.reg_warps == 4) ? L.reg_warps : (D == 3 ? 1 : 4);
        const unsigned gw = static_cast<unsigned>((nb + wpc - 1) / wpc);
        kr<<<gw, 32 * wpc, 0, s>>>(L.tab, src, dst, L.idx.ptr, L.geo.ptr, b0, b1, L.edges.ptr,
                                    hyb ? L.recompute_mod : 0, L.recompute_num, cd, ncd, nullptr);
        fused = true;
        NNMG_CHECK_LAUNCH();
        count_launch();
        return;
      }
    }
    if constexpr (PH == kElasticity && D == 3 && NC == 3 && CellRegElast<P>::kSupported && !kF64) {
      if (L.reg_kernel) {
        // single-precision arithmetic (the paper's fp32 V-cycle) unless NNMG_MIXED_ARITH=64
        auto kr = L.mixed_arith32 ? (L.elast_xnb ? k_apply_reg_elast<P, true, 0, float, float, true, false, false, float, true>
                                                 : k_apply_reg_elast<P, true, 0, float, float, true, false, false, float>)
                                  : k_apply_reg_elast<P, true, 0, float, float, true, false, false, double>;
        kr<<<static_cast<unsigned>(b1 - b0), 96, 0, s>>>(L.tab, src, dst, L.idx.ptr, L.geo32.ptr, b0, b1, L.lam, L.mu,
                                                          cd, ncd, nullptr, BlnTables{});
        fused = true;
        NNMG_CHECK_LAUNCH();
        count_launch();
        return;
      }
    }
    if constexpr (PH == kElasticity && D == 3 && NC == 3 && CellRegElast<P>::kSupported && kF64) {
      if (L.reg_kernel) {
        const int64_t nb = b1 - b0;
        if constexpr (P == 2) {
          if (L.edges.ptr && L.elast_recompute && !cellout) {
            auto kr = neg ? k_apply_reg_elast<P, true, 2> : k_apply_reg_elast<P, false, 2>;
            kr<<<static_cast<unsigned>(nb), 96, 0, s>>>(L.tab, src, dst, L.idx.ptr, L.edges.ptr, b0, b1, L.lam,
                                                         L.mu, nullptr, 0, nullptr, BlnTables{});
            NNMG_CHECK_LAUNCH();
            count_launch();
            return;
          }
        }
        auto kr = neg ? (L.elast_xch ? k_apply_reg_elast<P, true, 0, double, double, true>
                                     : k_apply_reg_elast<P, true>)
                      : (L.elast_xch ? k_apply_reg_elast<P, false, 0, double, double, true>
                                     : k_apply_reg_elast<P, false>);
        if (L.elast_tma && L.elast_xch)
          kr = neg ? k_apply_reg_elast<P, true, 0, double, double, true, true>
                   : k_apply_reg_elast<P, false, 0, double, double, true, true>;
        else if (L.elast_xnb && L.elast_xch && !cellout)
          kr = neg ? k_apply_reg_elast<P, true, 0, double, double, true, false, false, double, true>
                   : k_apply_reg_elast<P, false, 0, double, double, true, false, false, double, true>;
        BlnTables bln{};
        if (L.elast_bln && L.bln_node.ptr && !cellout) {
          bln = BlnTables{L.bln_node.ptr, L.bln_cnt.ptr, L.bln_slot.ptr, L.bln_kp};
          kr = L.elast_tma ? (neg ? k_apply_reg_elast<P, true, 0, double, double, true, true, true>
                                  : k_apply_reg_elast<P, false, 0, double, double, true, true, true>)
                           : (neg ? k_apply_reg_elast<P, true, 0, double, double, true, false, true>
                                  : k_apply_reg_elast<P, false, 0, double, double, true, false, true>);
        }
        kr<<<static_cast<unsigned>(nb), 96, 0, s>>>(L.tab, src, dst, L.idx.ptr, L.geo.ptr, b0, b1, L.lam, L.mu, cd,
                                                     ncd, cellout, bln);
        fused = true;
        NNMG_CHECK_LAUNCH();
        count_launch();
        return;
      }
    }
    if constexpr (!kF64) {
      // fp32 vectors: one compile-time variant per element type, the default
      // split (recomputed G for 3D Laplace Q3/Q4)
      if constexpr (D == 3 && P >= 3 && PH == kLaplace) {
        if (L.edges.ptr && L.apply_recompute) {
          // single-precision arithmetic (the paper's fp32 V-cycle) unless NNMG_MIXED_ARITH=64
          if (L.mixed_arith32) return launch<D, P, NC, PH, 8, 2, 0, float>();
          return launch<D, P, NC, PH, 8, 2>();
        }
      }
      constexpr int SP = (D == 3 && P >= 4) ? 4 : (NC > 1 ? 2 : 1);
      launch<D, P, NC, PH, SP>();
    } else {
    if constexpr (D == 3 && P >= 3 && PH == kLaplace) {
      if (L.edges.ptr && L.apply_recompute) {
        // NNMG_APPLY_MINB: min CTAs per SM of the launch bound (register cap) for the split variants
        if (L.apply_split == 8 && L.apply_minb == 6) return launch<D, P, NC, PH, 8, 2, 6>();
        if (L.apply_split == 8 && L.apply_minb == 4) return launch<D, P, NC, PH, 8, 2, 4>();
        if (L.apply_split == 4 && L.apply_minb == 3) return launch<D, P, NC, PH, 4, 2, 3>();
        if (L.apply_split == 4 && L.apply_minb == 2) return launch<D, P, NC, PH, 4, 2, 2>();
        if (L.apply_split == 8) return launch<D, P, NC, PH, 8, 2>();
        if (L.apply_split == 4) return launch<D, P, NC, PH, 4, 2>();
        if (L.apply_split == 2) return launch<D, P, NC, PH, 2, 2>();
        return launch<D, P, NC, PH, 1, 2>();
      }
    }
    if constexpr (D == 3 && P >= 3 && CK::CB % 16 == 0 && kF64) {
      if (L.apply_geos) {
        if (L.apply_split == 8) return launch<D, P, NC, PH, 8, 1>();
        if (L.apply_split == 4) return launch<D, P, NC, PH, 4, 1>();
      }
    }
    if (L.apply_split == 4) return launch<D, P, NC, PH, 4>();
    if (L.apply_split == 2) return launch<D, P, NC, PH, 2>();
    launch<D, P, NC, PH, 1>();
    }
  }
  template <int D, int P, int NC, int PH, int SPLIT, int GEO = 0, int MINB = 0, class TA = double>
  void launch() {
    using CK = ApplyKernel<D, P, NC, PH, SPLIT, TA>;
    constexpr size_t kSmem = CK::SMEM + (GEO == 1 ? CK::GEO_SMEM : (GEO == 2 ? CK::EDGE_SMEM : 0));
    // fp32 vectors: residual form only (no NEG=false instantiation)
    auto kneg = k_apply<D, P, NC, PH, true, SPLIT, GEO, MINB, TV, TA>;
    auto kpos = kneg;
    if constexpr (kF64) kpos = k_apply<D, P, NC, PH, false, SPLIT, GEO, MINB, TV, TA>;
    auto kern = neg ? kneg : kpos;
    const double* gsrc = GEO == 2 ? L.edges.ptr : L.geo.ptr;
    static bool attr = false;
    if (!attr) {
      NNMG_CUDA_TRY(cudaFuncSetAttribute(kneg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
      NNMG_CUDA_TRY(cudaFuncSetAttribute(kpos, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
      attr = true;
    }
    const int64_t nb = (b1 - b0) * SPLIT;
    constexpr int64_t kMaxGrid = (0x7fffffff / SPLIT) * SPLIT;
    for (int64_t off = 0; off < nb; off += kMaxGrid) {
      const unsigned g = static_cast<unsigned>(std::min<int64_t>(nb - off, kMaxGrid));
      kern<<<g, CK::NTHREADS, kSmem, s>>>(L.tab, src, dst, L.idx.ptr, gsrc, b0 + off / SPLIT, L.lam, L.mu, cellout);
      NNMG_CHECK_LAUNCH();
      count_launch();
    }
  }
};

using ApplyLaunch = ApplyLaunchT<double>;

void launch_apply_cells(const Level& L, const double* src, double* dst, int64_t b0, int64_t b1, cudaStream_t s,
                        bool negate) {
  if (b1 <= b0) return;
  ApplyLaunch f{L, src, dst, b0, b1, s, negate};
  dispatch(L.dim, L.degree, L.ncomp, L.physics, f);
}

// all cells plus the constrained rows; returns false when the rows are left to the caller
// deterministic mode, phase 2: per scalar DoF the sum of its cell-buffer
// slots in ascending slot order (a fixed order: results are bitwise
// reproducible); NEG: dst -= sum (residual form), else dst = sum
template <bool NEG>
__global__ void k_cell_gather(const int* __restrict__ off, const int* __restrict__ ent,
                              const double* __restrict__ cellout, int64_t nsc, int ncomp, int cb,
                              double* __restrict__ dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nsc * ncomp) return;
  const int64_t g = i / ncomp;
  const int c = static_cast<int>(i % ncomp);
  const int e0 = off[g], e1 = off[g + 1];
  if (e0 == e1) return;  // constrained: handled by the cell kernel's prologue
  double sum = 0.0;
  for (int e = e0; e < e1; ++e) sum += cellout[ent[e] + int64_t(c) * cb];
  dst[i] = NEG ? dst[i] - sum : sum;
}

template <class TV>
static bool launch_apply_all(const Level& L, const TV* src, TV* dst, cudaStream_t s, bool negate) {
  if (L.nblk <= 0) return false;
  ApplyLaunchT<TV> f{L, src, dst, 0, L.nblk, s, negate};
  if constexpr (sizeof(TV) == sizeof(double)) {
    if (L.deterministic) {
      f.cellout = L.cellout.ptr;
      f.cd = L.cdofs.ptr;
      f.ncd = static_cast<int64_t>(L.cdofs.n);
      dispatch(L.dim, L.degree, L.ncomp, L.physics, f);
      const int64_t nt = L.n_scalar * L.ncomp;
      if (negate)
        k_cell_gather<true><<<grid_for(nt, 256), 256, 0, s>>>(L.det_off.ptr, L.det_ent.ptr, L.cellout.ptr,
                                                               L.n_scalar, L.ncomp, L.cb, dst);
      else
        k_cell_gather<false><<<grid_for(nt, 256), 256, 0, s>>>(L.det_off.ptr, L.det_ent.ptr, L.cellout.ptr,
                                                                L.n_scalar, L.ncomp, L.cb, dst);
      NNMG_CHECK_LAUNCH();
      count_launch();
      return f.fused && f.ncd == static_cast<int64_t>(L.cdofs.n);
    }
  }
  if (L.fuse_constrained) {
    f.cd = L.cdofs.ptr;
    f.ncd = static_cast<int64_t>(L.cdofs.n);
  }
  dispatch(L.dim, L.degree, L.ncomp, L.physics, f);
  return f.fused && f.ncd == static_cast<int64_t>(L.cdofs.n);
}

template <class TV>
__global__ void k_sub_constrained(const int* __restrict__ cd, int64_t n, const TV* __restrict__ src,
                                  TV* __restrict__ dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[cd[i]] -= src[cd[i]];
}

// fp32 residual-form apply of the mixed-precision V-cycle: dst -= A src with
// fp32 vectors and stored geometry (level_enable_f32), fp64 arithmetic
void level_apply_sub_f32(Level& L, const float* src, float* dst, cudaStream_t s) {
  NNMG_REQUIRE(L.f32_ready, kInvalidArgument, "level fp32 data not prepared");
  NNMG_REQUIRE(src != dst, kInvalidArgument, "apply needs distinct source and destination");
  const bool fused = launch_apply_all(L, src, dst, s, true);
  const int64_t n = static_cast<int64_t>(L.cdofs.n);
  if (n && !fused) {
    k_sub_constrained<float><<<grid_for(n, 256), 256, 0, s>>>(L.cdofs.ptr, n, src, dst);
    NNMG_CHECK_LAUNCH();
    count_launch();
  }
}

__global__ void k_to_f32(const double* __restrict__ a, float* __restrict__ b, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = float(a[i]);
}

// [.. q][k][cb] doubles -> [.. q][k/2][cb][2] floats (ng even)
__global__ void k_to_f32_paired(const double* __restrict__ a, float* __restrict__ b, int64_t n, int ng, int cb) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t lane = i % cb, k = (i / cb) % ng, row = i / (int64_t(cb) * ng);  // row = blk * nq + q
  b[((row * (ng / 2) + k / 2) * cb + lane) * 2 + (k & 1)] = float(a[i]);
}

void level_enable_f32(Level& L, cudaStream_t s) {
  if (L.f32_ready) return;
  NNMG_REQUIRE(L.diag_ready, kInvalidArgument, "level diagonal not computed");
  L.geo32.alloc(L.geo.n);
  L.inv_diag32.alloc(L.inv_diag.n);
  // the register Laplace apply reads 3D fp32 geometry as float2 pairs (CellReg::kPairedGeo)
  const bool paired = L.physics == kLaplace && L.dim == 3 && L.reg_kernel && L.nloc <= 27 && L.ng % 2 == 0;
  if (L.geo.n) {
    if (paired)
      k_to_f32_paired<<<grid_for(int64_t(L.geo.n), 256), 256, 0, s>>>(L.geo.ptr, L.geo32.ptr, int64_t(L.geo.n), L.ng,
                                                                      L.cb);
    else
      k_to_f32<<<grid_for(int64_t(L.geo.n), 256), 256, 0, s>>>(L.geo.ptr, L.geo32.ptr, int64_t(L.geo.n));
  }
  NNMG_CHECK_LAUNCH();
  if (L.inv_diag.n)
    k_to_f32<<<grid_for(int64_t(L.inv_diag.n), 256), 256, 0, s>>>(L.inv_diag.ptr, L.inv_diag32.ptr,
                                                                   int64_t(L.inv_diag.n));
  NNMG_CHECK_LAUNCH();
  count_launch(2);
  L.f32_ready = true;
}

void level_apply_sub(Level& L, const double* src, double* dst, cudaStream_t s) {
  NNMG_REQUIRE(src != dst, kInvalidArgument, "apply needs distinct source and destination");
  const bool fused = launch_apply_all(L, src, dst, s, true);
  const int64_t n = static_cast<int64_t>(L.cdofs.n);
  if (n && !fused) {
    k_sub_constrained<double><<<grid_for(n, 256), 256, 0, s>>>(L.cdofs.ptr, n, src, dst);
    NNMG_CHECK_LAUNCH();
    count_launch();
  }
}

void launch_copy_constrained(const Level& L, const double* src, double* dst, cudaStream_t s) {
  const int64_t n = static_cast<int64_t>(L.cdofs.n);
  if (!n) return;
  k_copy_constrained<<<grid_for(n, 256), 256, 0, s>>>(L.cdofs.ptr, n, src, dst);
  NNMG_CHECK_LAUNCH();
  count_launch();
}

void level_load_vector(Level& L, const double* f, double* b, cudaStream_t s) {
  NNMG_CUDA_TRY(cudaMemsetAsync(b, 0, sizeof(double) * L.n_dofs, s));
  const double f0 = f[0], f1 = L.ncomp > 1 ? f[1] : 0.0, f2 = L.ncomp > 2 ? f[2] : 0.0;
  const int64_t nt = L.n_cells * L.nloc;
  double* co = L.deterministic ? L.cellout.ptr : nullptr;
  if (L.dim == 2)
    k_load_vector<2><<<grid_for(nt, 128), 128, 0, s>>>(L.verts.ptr, L.vcells.ptr, L.n_cells, L.n1, L.cb, L.idx.ptr,
                                                      L.tab, L.ncomp, f0, f1, f2, b, co);
  else
    k_load_vector<3><<<grid_for(nt, 128), 128, 0, s>>>(L.verts.ptr, L.vcells.ptr, L.n_cells, L.n1, L.cb, L.idx.ptr,
                                                      L.tab, L.ncomp, f0, f1, f2, b, co);
  NNMG_CHECK_LAUNCH();
  count_launch();
  if (co) {
    const int64_t n = L.n_scalar * L.ncomp;
    k_cell_gather<false><<<grid_for(n, 256), 256, 0, s>>>(L.det_off.ptr, L.det_ent.ptr, co, L.n_scalar, L.ncomp,
                                                           L.cb, b);
    NNMG_CHECK_LAUNCH();
    count_launch();
  }
}

void level_apply(Level& L, const double* src, double* dst, cudaStream_t s) {
  NNMG_REQUIRE(src != dst, kInvalidArgument, "apply needs distinct source and destination");
  NNMG_CUDA_TRY(cudaMemsetAsync(dst, 0, sizeof(double) * L.n_dofs, s));
  if (!launch_apply_all(L, src, dst, s, false)) launch_copy_constrained(L, src, dst, s);
}

// Partial applies for the distributed levels: the interior
// cell blocks run while the ghost import is in flight on another stream, the
// boundary blocks after it.  begin: dst = 0 and identity-out on the constrained
// rows; cells: dst += sum over the cell blocks [b0, b1) (free rows only).
// negate: the residual form dst -= A src (begin subtracts src on the
// constrained rows and does not zero dst).
void level_apply_begin(Level& L, const double* src, double* dst, bool negate, cudaStream_t s) {
  NNMG_REQUIRE(src != dst, kInvalidArgument, "apply needs distinct source and destination");
  if (negate) {
    // residual form dst -= A src: identity-out rows subtract src
    const int64_t n = static_cast<int64_t>(L.cdofs.n);
    if (n) {
      k_sub_constrained<double><<<grid_for(n, 256), 256, 0, s>>>(L.cdofs.ptr, n, src, dst);
      NNMG_CHECK_LAUNCH();
      count_launch();
    }
    return;
  }
  NNMG_CUDA_TRY(cudaMemsetAsync(dst, 0, sizeof(double) * L.n_dofs, s));
  launch_copy_constrained(L, src, dst, s);
}

void level_apply_cells(Level& L, const double* src, double* dst, int64_t b0, int64_t b1, bool negate,
                       cudaStream_t s) {
  NNMG_REQUIRE(src != dst, kInvalidArgument, "apply needs distinct source and destination");
  NNMG_REQUIRE(0 <= b0 && b0 <= b1 && b1 <= L.nblk, kInvalidArgument, "cell block range out of bounds");
  NNMG_REQUIRE(!L.deterministic, kUnsupported, "partial applies are not available in deterministic mode");
  launch_apply_cells(L, src, dst, b0, b1, s, negate);
}

struct DiagLaunch {
  Level& L;
  cudaStream_t s;
  template <int D, int P, int NC, int PH>
  void operator()() {
    using CK = CellKernel<D, P, NC, PH>;
    const int64_t nt = L.nblk * CK::NLOC * CK::CB;
    double* co = L.deterministic ? L.cellout.ptr : nullptr;
    k_diagonal<D, P, NC, PH><<<grid_for(nt, 128), 128, 0, s>>>(L.tab, L.idx.ptr, L.geo.ptr, L.nblk, L.lam, L.mu,
                                                                L.diag.ptr, co);
    NNMG_CHECK_LAUNCH();
    count_launch();
    if (co) {
      const int64_t n = L.n_scalar * L.ncomp;
      k_cell_gather<false><<<grid_for(n, 256), 256, 0, s>>>(L.det_off.ptr, L.det_ent.ptr, co, L.n_scalar, L.ncomp,
                                                             L.cb, L.diag.ptr);
      NNMG_CHECK_LAUNCH();
      count_launch();
    }
  }
};

// deterministic mode (SURVEY §7 hard part 1, mfoperator.py:88-90): the apply,
// diagonal and load-vector kernels write per-cell results to a cell buffer in
// the idx layout and k_cell_gather sums each DoF's slots in a fixed order;
// bitwise reproducible, at the cost of the buffer round trip
// (8 B x NLOC x NCOMP per cell written + read, 4 B per slot of index)
void level_set_deterministic(Level& L, bool on) {
  if (!on) {
    L.deterministic = false;
    L.cellout.release();
    L.det_off.release();
    L.det_ent.release();
    return;
  }
  if (L.deterministic) return;
  const int nloc = L.nloc, cb = L.cb, nc = L.ncomp;
  const int64_t nslot = L.nblk * nloc * nc * cb;
  NNMG_REQUIRE(nslot < (int64_t(1) << 31), kUnsupported, "level too large for the deterministic cell buffer");
  std::vector<int> off(L.n_scalar + 1, 0);
  for (int64_t c = 0; c < L.n_cells; ++c)
    for (int l = 0; l < nloc; ++l) {
      const int g = L.cell_dofs_host[c * nloc + l];
      if (!L.scalar_constrained[g]) off[g + 1] += 1;
    }
  for (int64_t g = 0; g < L.n_scalar; ++g) off[g + 1] += off[g];
  std::vector<int> ent(off[L.n_scalar]);
  std::vector<int> pos(off.begin(), off.end() - 1);
  for (int64_t c = 0; c < L.n_cells; ++c) {
    const int64_t blk = c / cb, lane = c % cb;
    for (int l = 0; l < nloc; ++l) {
      const int g = L.cell_dofs_host[c * nloc + l];
      if (!L.scalar_constrained[g]) ent[pos[g]++] = static_cast<int>((blk * nloc + l) * nc * cb + lane);
    }
  }
  L.det_off.upload(off);
  L.det_ent.upload(ent);
  L.cellout.alloc(size_t(nslot));
  L.cellout.zero();
  L.deterministic = true;
}

void level_compute_diagonal(Level& L, cudaStream_t s) {
  L.diag.zero(s);
  DiagLaunch f{L, s};
  dispatch(L.dim, L.degree, L.ncomp, L.physics, f);
  const int64_t n = static_cast<int64_t>(L.cdofs.n);
  if (n) {
    k_set_constrained<<<grid_for(n, 256), 256, 0, s>>>(L.cdofs.ptr, n, 1.0, L.diag.ptr);
    NNMG_CHECK_LAUNCH();
    count_launch();
  }
  k_reciprocal<<<grid_for(L.n_dofs, 256), 256, 0, s>>>(L.diag.ptr, L.inv_diag.ptr, L.n_dofs);
  NNMG_CHECK_LAUNCH();
  count_launch();
  L.diag_ready = true;
}

}  // namespace nnmg
