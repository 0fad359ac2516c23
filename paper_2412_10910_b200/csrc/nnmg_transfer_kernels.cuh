// K6 prolongation and K7 restriction kernels (non-nested transfer).
//
// Records are grouped by owning coarse cell (CSR cell_start / pt_dof / xhat),
// one warp per coarse cell.  See DESIGN.md "Transfers".
//
// FP64 instruction count decides these kernels on B200 (ncu: FP64 pipe 42-55%
// busy while DRAM is far from peak), so the per-point arithmetic is kept at the
// minimum of the tensor-product form:
//   * 1D Lagrange values by prefix/suffix products without the 1/denom factors
//     (3 N1 - 5 ops per axis), which are applied per local DoF once per cell;
//   * restriction weights factorised (v X2[i2]) X1[i1] X0[i0]: N1^d FMAs plus
//     N1 + N1^2 products instead of 2 N1^d products;
//   * cell-end reductions through shared memory in a fixed order instead of a
//     butterfly per output (5 shuffles per output).
#pragma once

#include "nnmg_kernels.cuh"

namespace nnmg {

static constexpr int kTransferWarps = 4;  // coarse cells (one per warp) per thread block

// Unnormalised values prod_{j!=i} (t - node_j) (3 N1 - 5 ops per axis; the
// end nodes are exactly 0 and 1, nnmg_common.cu).  The 1/denom factors are
// per local DoF, so the kernels apply their tensor product once per cell
// (staged coarse values, cell-end sums) instead of once per point.
template <int N1, class TA = double>
__device__ __forceinline__ void lagrange_un(const Tables& tab, TA t, TA (&out)[N1]) {
  if constexpr (N1 == 1) {
    out[0] = TA(1);
  } else {
    TA d[N1];
    d[0] = t;
#pragma unroll
    for (int j = 1; j < N1 - 1; ++j) d[j] = t - TabSel<TA>::nodes(tab)[j];
    d[N1 - 1] = t - TA(1);
    TA suf[N1];
    suf[N1 - 1] = d[N1 - 1];
#pragma unroll
    for (int j = N1 - 2; j >= 1; --j) suf[j] = d[j] * suf[j + 1];
    out[0] = suf[1];
    TA pre = d[0];
#pragma unroll
    for (int i = 1; i < N1 - 1; ++i) {
      out[i] = pre * suf[i + 1];
      pre *= d[i];
    }
    out[N1 - 1] = pre;
  }
}

// prod_j 1/denom[l_j] of local point l (x fastest)
template <int DIM, int N1, class TA = double>
__device__ __forceinline__ TA lagrange_norm(const Tables& tab, int l) {
  TA r = TabSel<TA>::rdenom(tab)[l % N1];
#pragma unroll
  for (int j = 1; j < DIM; ++j) {
    l /= N1;
    r *= TabSel<TA>::rdenom(tab)[l % N1];
  }
  return r;
}

// ---------------------------------------------------------------------------
// K6: u_f[pt] (+)= sum_l u_c[gather[pt,l]] prod_j phi_{l_j}(xhat_j)
// (transfer.py:31-44, 87-102).  The cell's coarse values are staged once in
// shared memory and broadcast; each lane evaluates PPL points per round.  The
// records of the next round are loaded before the current round's arithmetic.
// Contraction order x, y, z as transfer.py:93-95.
// ---------------------------------------------------------------------------
template <int DIM, int N1, class TA = double>
__device__ __forceinline__ TA contract(const TA* __restrict__ U, const TA (&X)[DIM][N1]) {
  if constexpr (DIM == 2) {
    TA val = 0;
#pragma unroll
    for (int i1 = 0; i1 < N1; ++i1) {
      TA s = 0;
#pragma unroll
      for (int i0 = 0; i0 < N1; ++i0) s = fma(U[i0 + N1 * i1], X[0][i0], s);
      val = fma(s, X[1][i1], val);
    }
    return val;
  } else {
    TA val = 0;
#pragma unroll
    for (int i2 = 0; i2 < N1; ++i2) {
      TA s2 = 0;
#pragma unroll
      for (int i1 = 0; i1 < N1; ++i1) {
        TA s = 0;
#pragma unroll
        for (int i0 = 0; i0 < N1; ++i0) s = fma(U[i0 + N1 * i1 + N1 * N1 * i2], X[0][i0], s);
        s2 = fma(s, X[1][i1], s2);
      }
      val = fma(s2, X[2][i2], val);
    }
    return val;
  }
}

// points per lane per round: two (each staged coarse value read from shared
// memory serves both); measured on B200: C3 0.251 -> 0.195 ms, C4 (Q4) 0.365
// -> 0.314 ms, C5 (3 components, 126 registers) 0.047 -> 0.045 ms
template <int DIM, int PC, int NCOMP>
__host__ __device__ constexpr int prolongate_ppl() {
  return 2;
}

// TV / TX: storage types of the vectors and of xhat (double, or float in the
// mixed-precision V-cycle); TA: the arithmetic type (float = the paper's
// single-precision V-cycle; fp64 arithmetic on fp32 storage pays F2F
// conversions on every record: the fp32 restriction measured 206 us against
// 159 us in fp64 on C3)
template <int DIM, int PC, int NCOMP, int CBC, int PPL, class TV = double, class TX = double, class TA = double>
__global__ void __launch_bounds__(kTransferWarps * 32, PPL > 1 && (PC >= 3 || NCOMP > 1) ? 4 : 6)
    k_prolongate(Tables tab, const TV* __restrict__ uc, TV* __restrict__ uf, int accumulate,
                 const int* __restrict__ cidx, const int* __restrict__ item_cell, const int* __restrict__ item_pt,
                 const int* __restrict__ pt_dof, const TX* __restrict__ xhat, int64_t nitems) {
  constexpr int N1 = PC + 1;
  constexpr int NLOC = ipow(N1, DIM);
  __shared__ TA su[kTransferWarps][NCOMP * NLOC];
  // blockDim.x / 32 <= kTransferWarps warps per CTA (independent: one work item each)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t item = blockIdx.x * (int64_t)(blockDim.x >> 5) + warp;
  if (item >= nitems) return;
  // item_cell == nullptr: one item per cell (saves a dependent load)
  const int64_t cell = item_cell ? (int64_t)item_cell[item] : item;
  const int64_t blk = cell / CBC, cl = cell % CBC;
  const int p0 = item_pt[item], p1 = item_pt[item + 1];
  constexpr int STEP = 32 * PPL;
  // first round's records are in flight while the coarse values are staged
  int dd[PPL];
  TA xt[PPL][DIM];
  auto load = [&](int base) {
#pragma unroll
    for (int k = 0; k < PPL; ++k) {
      const int p = base + 32 * k + lane;
      const bool ok = p < p1;
      dd[k] = ok ? __ldcs(pt_dof + p) : -1;
#pragma unroll
      for (int j = 0; j < DIM; ++j) xt[k][j] = ok ? TA(__ldcs(xhat + (int64_t)p * DIM + j)) : TA(0.5);
    }
  };
  load(p0);
  for (int l = lane; l < NLOC; l += 32) {
    const int g = cidx[(blk * NLOC + l) * CBC + cl];
#pragma unroll
    for (int c = 0; c < NCOMP; ++c)
      su[warp][c * NLOC + l] = g >= 0 ? TA(uc[(int64_t)g * NCOMP + c]) * lagrange_norm<DIM, N1, TA>(tab, l) : TA(0);
  }
  __syncwarp();
  for (int base = p0; base < p1; base += STEP) {
    int cd[PPL];
    TA X[PPL][DIM][N1];
#pragma unroll
    for (int k = 0; k < PPL; ++k) {
      cd[k] = dd[k];
#pragma unroll
      for (int j = 0; j < DIM; ++j) lagrange_un<N1, TA>(tab, xt[k][j], X[k][j]);
    }
    if (base + STEP < p1) load(base + STEP);
#pragma unroll
    for (int c = 0; c < NCOMP; ++c) {
      const TA* U = su[warp] + c * NLOC;
#pragma unroll
      for (int k = 0; k < PPL; ++k) {
        const TA a = contract<DIM, N1, TA>(U, X[k]);
        if (cd[k] >= 0) {
          TV* o = uf + (int64_t)cd[k] * NCOMP + c;
          *o = TV(accumulate ? TA(*o) + a : a);
        }
      }
    }
  }
}

// zero the fine DoFs that carry no transfer point (constrained): the
// non-accumulating prolongation writes every other entry
template <class TV>
__global__ void k_zero_list(const int* __restrict__ list, int64_t n, int ncomp, TV* __restrict__ uf) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n * ncomp) uf[(int64_t)list[i / ncomp] * ncomp + i % ncomp] = TV(0);
}

// ---------------------------------------------------------------------------
// K7 phase 1: per owning coarse cell the local vector
//   R_l = sum_pt r_f[pt] W_l(pt),  W = phi_{l2}(z) phi_{l1}(y) phi_{l0}(x)
// (transfer.py:104-109, 115).  Deterministic, no atomics.
//
// A warp owns a chunk of consecutive coarse cells and streams their points in
// rounds that never straddle a cell.  The gather r_f[pt_dof[p]] is a
// dependent load chain, so the stream is software-pipelined ACROSS cells: the
// records (pt_dof, xhat) of round k+2 and the values of round k+1 are in
// flight while round k is evaluated.  (With ~160 points per coarse cell, a
// per-cell pipeline spends most of its time in the cell_start -> records ->
// values latency chain at each cell start.)
// ---------------------------------------------------------------------------

// Round state machine over the cells [c0, c0+nch) of a chunk (nch <= 31).
// Lane i holds cell_start[c0+i]; rounds of RS points; empty cells are skipped
// (their outputs are zero-filled separately).  Warp-uniform.
struct CellRounds {
  int cs, nch;
  __device__ __forceinline__ int start(int i) const { return __shfl_sync(0xffffffffu, cs, i); }
  __device__ __forceinline__ void skip(int& ci, int base) const {
    while (ci < nch && base >= start(ci + 1)) ++ci;
  }
  __device__ __forceinline__ void first(int& ci, int& base) const {
    ci = 0;
    base = start(0);
    skip(ci, base);
  }
  __device__ __forceinline__ void next(int& ci, int& base, int rs) const {
    if (ci >= nch) return;
    base += rs;
    const int e = start(ci + 1);
    if (base >= e) {
      base = e;
      ++ci;
      skip(ci, base);
    }
  }
  __device__ __forceinline__ int end(int ci) const { return start(ci < nch ? ci + 1 : nch); }
};

__device__ __forceinline__ void zero_empty_cells(const CellRounds& R, int64_t c0, int nout, int lane,
                                                 double* __restrict__ cellbuf) {
  const int a = R.start(lane < R.nch ? lane : R.nch), b = R.start(lane < R.nch ? lane + 1 : R.nch);
  if (lane < R.nch && a == b)
    for (int o = 0; o < nout; ++o) cellbuf[(c0 + lane) * nout + o] = 0.0;
}

// per-lane point records of one round: point p = base + k*stride + off
template <int DIM, int NCOMP, int PPR, class TA = double>
struct PointRec {
  int d[PPR];
  TA x[PPR][DIM];
  template <class TX>
  __device__ __forceinline__ void load(const int* __restrict__ pt_dof, const TX* __restrict__ xhat, int base,
                                       int end, int stride, int off, bool live) {
#pragma unroll
    for (int k = 0; k < PPR; ++k) {
      const int p = base + k * stride + off;
      const bool ok = live && p < end;
      d[k] = ok ? __ldcs(pt_dof + p) : -1;
#pragma unroll
      for (int j = 0; j < DIM; ++j) x[k][j] = ok ? TA(__ldcs(xhat + (int64_t)p * DIM + j)) : TA(0.5);
    }
  }
  template <class TV>
  __device__ __forceinline__ void values(const TV* __restrict__ rf, TA (&v)[PPR][NCOMP]) const {
#pragma unroll
    for (int k = 0; k < PPR; ++k)
#pragma unroll
      for (int c = 0; c < NCOMP; ++c) v[k][c] = d[k] >= 0 ? TA(rf[(int64_t)d[k] * NCOMP + c]) : TA(0);
  }
};

// The pipelined round loop shared by the restriction kernels.  body(rec_x, v)
// evaluates the current round; flush(ci) is called after the last round of
// chunk cell ci.
template <int DIM, int NCOMP, int PPR, class TA = double, class TX, class TV, class Body, class Flush>
__device__ __forceinline__ void stream_rounds(const CellRounds& R, const int* __restrict__ pt_dof,
                                              const TX* __restrict__ xhat, const TV* __restrict__ rf,
                                              int stride, int off, bool live, Body&& body, Flush&& flush) {
  constexpr int RS_K = PPR;
  const int rs = RS_K * stride;
  int ciA, bA;
  R.first(ciA, bA);
  int ciB = ciA, bB = bA;
  R.next(ciB, bB, rs);
  int ciC = ciB, bC = bB;
  R.next(ciC, bC, rs);
  PointRec<DIM, NCOMP, PPR, TA> rA, rB, rC;
  rA.load(pt_dof, xhat, bA, R.end(ciA), stride, off, live && ciA < R.nch);
  rB.load(pt_dof, xhat, bB, R.end(ciB), stride, off, live && ciB < R.nch);
  TA vA[PPR][NCOMP], vB[PPR][NCOMP];
  rA.values(rf, vA);
  while (ciA < R.nch) {
    rB.values(rf, vB);
    rC.load(pt_dof, xhat, bC, R.end(ciC), stride, off, live && ciC < R.nch);
    body(rA.x, vA);
    if (ciB != ciA) flush(ciA);
    ciA = ciB;
    ciB = ciC;
    bB = bC;
    R.next(ciC, bC, rs);
    rA = rB;
    rB = rC;
#pragma unroll
    for (int k = 0; k < PPR; ++k)
#pragma unroll
      for (int c = 0; c < NCOMP; ++c) vA[k][c] = vB[k][c];
  }
}

// dynamic shared memory of k_restrict_lane per warp
template <int DIM, int PC, int NCOMP, class TA>
constexpr size_t restrict_lane_smem_per_warp() {
  constexpr int NOUT = ipow(PC + 1, DIM) * NCOMP;
  constexpr int TW = NOUT < 32 ? NOUT : 32;
  return size_t(32) * (TW | 1) * sizeof(TA);
}

// A lane owns a point and the full local vector in registers (NLOC*NCOMP <=
// 32: Q1/Q2 scalar, 2D vector; up to 81 with NNMG_RESTRICT_WIDE: 3D Q2
// elasticity, Q3 scalar); a cell's lanes are combined through shared memory
// at the cell end, 32 outputs at a time, lane l ending with output l of a tile.
template <int DIM, int PC, int NCOMP, int PPR, class TV = double, class TX = double, class TA = double>
__global__ void __launch_bounds__(kTransferWarps * 32)
    k_restrict_lane(Tables tab, const TV* __restrict__ rf, const int* __restrict__ cell_start,
                    const int* __restrict__ pt_dof, const TX* __restrict__ xhat, int64_t ncc, int chunk,
                    double* __restrict__ cellbuf) {
  constexpr int N1 = PC + 1;
  constexpr int NLOC = ipow(N1, DIM);
  constexpr int NOUT = NLOC * NCOMP;
  static_assert(NOUT <= 81, "lane-owned local vector");
  // blockDim.x / 32 <= kTransferWarps independent warps per CTA; the reduction
  // buffer is dynamic shared memory, 32 * RS elements per warp (lane_smem_bytes)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c0 = (blockIdx.x * (int64_t)(blockDim.x >> 5) + warp) * chunk;
  if (c0 >= ncc) return;
  const int nch = (int)(ncc - c0 < chunk ? ncc - c0 : chunk);
  const CellRounds R{cell_start[c0 + min(lane, nch)], nch};
  zero_empty_cells(R, c0, NOUT, lane, cellbuf);
  // cell-end reduction through shared memory: 32 lanes x (up to 32) partials
  // per tile (odd row stride: conflict-free both ways), then lane l sums
  // column l over the 32 lanes in a fixed order.  ~2 NOUT + 32 instructions
  // per lane and tile instead of the transposing shuffle reduction's ~15 per
  // value (64-bit selects and shuffles, wrapped in warp-sync because the
  // flush is conditional).
  constexpr int TW = NOUT < 32 ? NOUT : 32;
  constexpr int RS = TW | 1;
  extern __shared__ __align__(16) unsigned char lane_smem[];
  TA* rw = reinterpret_cast<TA*>(lane_smem) + warp * (32 * RS);
  TA acc[NOUT];
#pragma unroll
  for (int o = 0; o < NOUT; ++o) acc[o] = 0;
  stream_rounds<DIM, NCOMP, PPR, TA>(
      R, pt_dof, xhat, rf, 32, lane, true,
      [&](const TA (&xs)[PPR][DIM], const TA (&vs)[PPR][NCOMP]) {
#pragma unroll
        for (int k = 0; k < PPR; ++k) {
          TA X[DIM][N1];
#pragma unroll
          for (int j = 0; j < DIM; ++j) lagrange_un<N1, TA>(tab, xs[k][j], X[j]);
#pragma unroll
          for (int c = 0; c < NCOMP; ++c) {
            if constexpr (DIM == 3) {
#pragma unroll
              for (int i2 = 0; i2 < N1; ++i2) {
                const TA a = vs[k][c] * X[2][i2];
#pragma unroll
                for (int i1 = 0; i1 < N1; ++i1) {
                  const TA b = a * X[1][i1];
#pragma unroll
                  for (int i0 = 0; i0 < N1; ++i0) {
                    const int o = (i0 + N1 * (i1 + N1 * i2)) * NCOMP + c;
                    acc[o] = fma(b, X[0][i0], acc[o]);
                  }
                }
              }
            } else {
#pragma unroll
              for (int i1 = 0; i1 < N1; ++i1) {
                const TA b = vs[k][c] * X[1][i1];
#pragma unroll
                for (int i0 = 0; i0 < N1; ++i0) {
                  const int o = (i0 + N1 * i1) * NCOMP + c;
                  acc[o] = fma(b, X[0][i0], acc[o]);
                }
              }
            }
          }
        }
      },
      [&](int ci) {
#pragma unroll
        for (int t0 = 0; t0 < NOUT; t0 += TW) {
#pragma unroll
          for (int j = 0; j < TW; ++j)
            if (t0 + j < NOUT) {
              rw[lane * RS + j] = acc[t0 + j];
              acc[t0 + j] = 0;
            }
          __syncwarp();
          const int o = t0 + lane;
          if (lane < TW && o < NOUT) {
            TA r = 0;
#pragma unroll
            for (int sl = 0; sl < 32; ++sl) r += rw[sl * RS + lane];
            cellbuf[(c0 + ci) * NOUT + o] = double(r * lagrange_norm<DIM, N1, TA>(tab, o / NCOMP));
          }
          __syncwarp();
        }
      });
}

// NLOC*NCOMP > 32 (3D Q2 elasticity, Q3/Q4 scalar).  Rounds of P = SLOTS*SUB
// points (SLOTS = 32/N1): every lane loads one point and evaluates its full 1D
// tables (prefix/suffix products, once per point) into a shared staging
// buffer; then, in SUB sub-rounds, the N1 lanes of a slot share a staged point
// and lane g accumulates the outermost-axis plane l_last = g of the local
// vector (all components) in registers.  Slots are combined in shared memory
// in a fixed order at each cell end.
// PL = planes of the outermost axis per lane: a slot of G = ceil(N1 / PL) lanes
// shares a staged point, and each 16-byte table read then feeds PL x INNER
// FMAs per component.  ncu (r2, C4, PL = 1): 6.2 shared-memory wavefronts per
// point, the L1 data pipe 87% busy and the FP64 pipe 47%: the restriction is
// bound by its table reads, so PL = 2 (10 points instead of 6 per sub-round
// for Q4, the same reads) trades idle lanes of the last slot lane for
// 40% fewer reads per point.
template <int DIM, int PC, int NCOMP, int PL = 1, class TA = double>
struct StagedRestrict {
  static constexpr int N1 = PC + 1;
  static constexpr int NLOC = ipow(N1, DIM);
  static constexpr int NOUT = NLOC * NCOMP;
  static constexpr int G = (N1 + PL - 1) / PL;
  static constexpr int SLOTS = 32 / G;
  static constexpr int SUB = 32 / SLOTS;
  static constexpr int P = SLOTS * SUB;  // points per round
  static constexpr int INNER = NLOC / N1;
  static constexpr int PLANE = INNER * NCOMP;
  // staged record of a point: X0 at 0, X1 at A (16-byte aligned pairs, read
  // as double2), X_last at OZ, values at OV; stride REC = 2 mod 16 doubles so
  // the slots' 16-byte reads fall in distinct bank quads
  static constexpr int A = (N1 + 1) & ~1;
  static constexpr int OZ = DIM == 3 ? A + N1 : A;
  static constexpr int OV = OZ + N1;
  static constexpr int REC0 = OV + NCOMP;
  static constexpr int REC = ((REC0 - 2 + 15) / 16) * 16 + 2;
  // per-warp buffer in elements of the arithmetic type (even: keeps the
  // 2-element alignment).  The cell-end reduction buffer [SLOTS][N1][PLANE]
  // aliases the two staging buffers: at a cell end both are dead (the round's
  // sub-rounds are over, the next round has not staged yet), so a warp needs
  // max(staging, reduction) instead of their sum (C5: 15.1 -> 8.6 KB) and more
  // warps fit per SM.
  static constexpr int STAGE_ELEMS = 2 * P * REC;
  static constexpr int RED_ELEMS = SLOTS * N1 * PLANE;
  // measured on B200: C5 (vector Q2, latency-bound) restriction 68.0 -> 65.8 us with the alias,
  // C4 (scalar Q4, bound by its table reads) 437 -> 442 us: aliased for vector fields only
  static constexpr bool kAlias = NCOMP > 1;
  static constexpr int WARP_DOUBLES =
      ((kAlias ? (STAGE_ELEMS > RED_ELEMS ? STAGE_ELEMS : RED_ELEMS) : STAGE_ELEMS + RED_ELEMS) + 1) & ~1;
  // (a launch bound of 5 CTAs per SM on top, 96 registers with spills: C4 437 -> 584 us, C5 68 -> 89 us)
  static constexpr int WARP_BYTES = WARP_DOUBLES * int(sizeof(TA));
  static constexpr int WARPS = (48 * 1024) / WARP_BYTES >= kTransferWarps
                                   ? kTransferWarps
                                   : ((48 * 1024) / WARP_BYTES >= 1 ? (48 * 1024) / WARP_BYTES : 1);
};

// two consecutive staged table entries in one load (16 bytes in fp64, 8 in fp32)
template <class TA>
struct Pair2;
template <>
struct Pair2<double> {
  using type = double2;
};
template <>
struct Pair2<float> {
  using type = float2;
};

template <int DIM, int PC, int NCOMP, class TV = double, class TX = double, int PL = 1, class TA = double>
__global__ void __launch_bounds__(StagedRestrict<DIM, PC, NCOMP, PL, TA>::WARPS * 32)
    k_restrict_staged(Tables tab, const TV* __restrict__ rf, const int* __restrict__ cell_start,
                      const int* __restrict__ pt_dof, const TX* __restrict__ xhat, int64_t ncc, int chunk,
                      double* __restrict__ cellbuf) {
  using K = StagedRestrict<DIM, PC, NCOMP, PL, TA>;
  using V2 = typename Pair2<TA>::type;
  constexpr int N1 = K::N1, G = K::G, SLOTS = K::SLOTS, SUB = K::SUB, P = K::P, INNER = K::INNER,
                PLANE = K::PLANE, REC = K::REC, NOUT = K::NOUT;
  __shared__ __align__(16) TA smem[K::WARPS][K::WARP_DOUBLES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c0 = (blockIdx.x * (int64_t)K::WARPS + warp) * chunk;
  if (c0 >= ncc) return;
  const int nch = (int)(ncc - c0 < chunk ? ncc - c0 : chunk);
  TA* stage = smem[warp];  // [2][P][REC]
  TA* red = smem[warp] + (K::kAlias ? 0 : K::STAGE_ELEMS);  // [SLOTS][N1][PLANE]; kAlias: over the staging buffers
  const CellRounds R{cell_start[c0 + min(lane, nch)], nch};
  zero_empty_cells(R, c0, NOUT, lane, cellbuf);
  const int slot = lane / G, g = lane % G;
  const bool grp = slot < SLOTS;
  TA acc[PL][INNER][NCOMP];
#pragma unroll
  for (int p = 0; p < PL; ++p)
#pragma unroll
    for (int i = 0; i < INNER; ++i)
#pragma unroll
      for (int c = 0; c < NCOMP; ++c) acc[p][i][c] = 0;
  int buf = 0;
  stream_rounds<DIM, NCOMP, 1, TA>(
      R, pt_dof, xhat, rf, P, lane, lane < P,
      [&](const TA (&xs)[1][DIM], const TA (&vs)[1][NCOMP]) {
        // stage this lane's point: 1D tables and values
        TA* st = stage + buf * P * REC;
        if (lane < P) {
          TA X[N1];
#pragma unroll
          for (int j = 0; j < DIM; ++j) {
            lagrange_un<N1, TA>(tab, xs[0][j], X);
#pragma unroll
            for (int i = 0; i < N1; ++i) st[lane * REC + (j == 0 ? 0 : (j == DIM - 1 ? K::OZ : K::A)) + i] = X[i];
          }
#pragma unroll
          for (int c = 0; c < NCOMP; ++c) st[lane * REC + K::OV + c] = vs[0][c];
        }
        __syncwarp();
        if (grp) {
#pragma unroll 1
          for (int s = 0; s < SUB; ++s) {
            const TA* q = st + (s * SLOTS + slot) * REC;
            TA X0[K::A], X1[DIM == 3 ? K::A : 1];
#pragma unroll
            for (int i = 0; i < K::A; i += 2) {
              const V2 t = *reinterpret_cast<const V2*>(q + i);
              X0[i] = t.x;
              X0[i + 1] = t.y;
            }
            if constexpr (DIM == 3) {
#pragma unroll
              for (int i = 0; i < K::A; i += 2) {
                const V2 t = *reinterpret_cast<const V2*>(q + K::A + i);
                X1[i] = t.x;
                X1[i + 1] = t.y;
              }
            }
            // this lane's planes g PL .. g PL + PL - 1 (a plane past N1 - 1 adds zeros)
            TA z[PL];
#pragma unroll
            for (int p = 0; p < PL; ++p) z[p] = g * PL + p < N1 ? q[K::OZ + g * PL + p] : TA(0);
#pragma unroll
            for (int c = 0; c < NCOMP; ++c) {
              const TA v = q[K::OV + c];
#pragma unroll
              for (int p = 0; p < PL; ++p) {
                const TA a = v * z[p];
                if constexpr (DIM == 3) {
#pragma unroll
                  for (int i1 = 0; i1 < N1; ++i1) {
                    const TA b = a * X1[i1];
#pragma unroll
                    for (int i0 = 0; i0 < N1; ++i0)
                      acc[p][i0 + N1 * i1][c] = fma(b, X0[i0], acc[p][i0 + N1 * i1][c]);
                  }
                } else {
#pragma unroll
                  for (int i0 = 0; i0 < N1; ++i0) acc[p][i0][c] = fma(a, X0[i0], acc[p][i0][c]);
                }
              }
            }
          }
        }
        buf ^= 1;  // the next round writes the other buffer: one barrier per round
      },
      [&](int ci) {
        if constexpr (K::kAlias) __syncwarp();  // every lane is done with the staged round: its buffers become the reduction buffer
        if (grp) {
#pragma unroll
          for (int p = 0; p < PL; ++p)
            if (g * PL + p < N1) {
#pragma unroll
              for (int i = 0; i < INNER; ++i)
#pragma unroll
                for (int c = 0; c < NCOMP; ++c) red[((slot * N1 + g * PL + p) * INNER + i) * NCOMP + c] = acc[p][i][c];
            }
#pragma unroll
          for (int p = 0; p < PL; ++p)
#pragma unroll
            for (int i = 0; i < INNER; ++i)
#pragma unroll
              for (int c = 0; c < NCOMP; ++c) acc[p][i][c] = 0;
        }
        __syncwarp();
        // output o = l * NCOMP + c with l = plane * INNER + i: slot sum in fixed order
        for (int o = lane; o < NOUT; o += 32) {
          const int plane = o / PLANE, k = o % PLANE;
          TA sum = 0;
#pragma unroll
          for (int sl = 0; sl < SLOTS; ++sl) sum += red[(sl * N1 + plane) * PLANE + k];
          cellbuf[(c0 + ci) * NOUT + o] = double(sum * lagrange_norm<DIM, N1, TA>(tab, o / NCOMP));
        }
        __syncwarp();
      });
}

// K7 phase 2: r_c[g] = sum over the (cell, l) slots holding g, fixed order
template <class TV>
__global__ void k_restrict_gather(const int* __restrict__ t_off, const int* __restrict__ t_ent,
                                  const double* __restrict__ cellbuf, int64_t nsc, int ncomp, TV* __restrict__ rc) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= nsc) return;
  const int e0 = t_off[g], e1 = t_off[g + 1];
  for (int c = 0; c < ncomp; ++c) {
    double s = 0.0;
    for (int e = e0; e < e1; ++e) s += cellbuf[(int64_t)t_ent[e] * ncomp + c];
    rc[g * ncomp + c] = TV(s);
  }
}

}  // namespace nnmg
