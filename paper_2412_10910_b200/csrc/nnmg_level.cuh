// Level handle: the device-resident state of one multigrid level
// (replaces the reference _OperatorBase + LaplaceOperator / ElasticityOperator,
// mfoperator.py:25-252).
#pragma once

#include "nnmg_common.cuh"

namespace nnmg {

struct Level {
  int device = 0;
  int dim = 0, degree = 0, ncomp = 1, physics = 0;
  int n1 = 0, nloc = 0, nq = 0, ng = 0, cb = 32;
  int64_t n_cells = 0, nblk = 0, n_scalar = 0, n_dofs = 0;
  double lam = 0.0, mu = 0.0;
  Tables tab{};
  DevBuf<int> idx;       // [nblk][nloc][cb], -1 = constrained or padding
  DevBuf<double> geo;    // [nblk][nq][ng][cb]
  DevBuf<int> cdofs;     // constrained full DoFs, sorted
  DevBuf<double> verts;  // vertex coordinates (n_vertices, dim)
  DevBuf<int> vcells;    // cell vertices (n_cells, 2^dim)
  DevBuf<double> diag;   // cached exact diagonal (constrained = 1)
  DevBuf<double> inv_diag;
  bool diag_ready = false;
  bool reg_kernel = true;  // register-resident thread-per-cell apply where supported
  int apply_minb = 0;      // launch bound (min CTAs/SM) of the recomputed-G pencil apply (0: default 5)
  int apply_split = 1;     // CTAs per cell block of the pencil apply kernel (1, 2, 4, 8)
  bool apply_geos = false; // pencil apply: geometry staged in shared memory (Q3/Q4)
  bool apply_recompute = false; // pencil apply: G recomputed from edge vectors (3D Laplace Q3/Q4)
  bool reg_recompute = false;   // register apply: G recomputed from edge vectors (3D Laplace Q1/Q2)
  bool elast_recompute = false; // elasticity register apply (3D Q2): J^-1, |det J| from edge vectors
  // elasticity register apply, block-local nodes (BLN): per cell block the
  // sorted distinct free nodes and each slot's position in that list; the
  // block's node values are gathered once (contiguous runs) and each node
  // component gets ONE atomic per block
  bool elast_bln = false;
  int bln_kp = 0;                 // padded node-list length per block
  DevBuf<int> bln_node, bln_cnt;  // [nblk][kp] global scalar node (-1 pad), [nblk] count
  DevBuf<unsigned> bln_slot;      // [nblk][(nloc+1)/2][cb] staging positions (CellRegElast::bln_phys) of two local points per word, 0xFFFF = constrained / padding
  bool elast_xnb = false;       // elasticity register apply: x-adjacent cells share their face nodes (with elast_xch)
  bool elast_tma = false;       // elasticity register apply: geometry slices staged in shared memory by TMA
  bool elast_xch = true;        // elasticity register apply: node-major gather/scatter via shared memory
  bool reg_xnb = false;         // fp64 register apply: x-adjacent cells of a warp share their face nodes (shuffles instead of gathers / atomics)
  int reg_warps = 0;            // fp64 register apply: warps (cell blocks) per CTA (0: 1 in 3D, 4 in 2D)
  int reg_warps32 = 0;          // the same for the fp32-arithmetic apply (0: 1 in 3D, 4 in 2D)
  int reg_xnb_mode = 1;         // 1: gather and scatter, 2: scatter only
  bool reg_xnb32 = true;        // the same in the fp32-arithmetic apply of the mixed-precision cycle
  bool reg_tma = false;         // register apply (3D): G streamed through shared memory by TMA bulk copies
  bool fuse_constrained = true;  // register kernels handle the constrained rows in their prologue
  int reg_minb = 1;        // min CTAs/SM launch bound of that kernel (4 caps registers at 128: spills)
  int recompute_mod = 0;   // hybrid geometry: blocks with blk % mod < num recompute G (0 = off)
  int recompute_num = 1;
  DevBuf<double> edges;    // [nblk][d*2^(d-1)*d][cb] cell edge vectors (hybrid geometry)
  // mixed-precision V-cycle (level_enable_f32): fp32 copies of the stored
  // geometry and of the inverse diagonal
  DevBuf<float> geo32, inv_diag32;
  bool f32_ready = false;
  bool mixed_arith32 = true;  // fp32 levels: single-precision arithmetic in the register apply (false: fp64 arithmetic on fp32 storage)
  // deterministic mode (level_set_deterministic): cell buffer [nblk][nloc][ncomp][cb]
  // and, per scalar DoF, its slots in a fixed order (CSR)
  bool deterministic = false;
  DevBuf<double> cellout;
  DevBuf<int> det_off, det_ent;
  std::vector<int> cell_dofs_host;  // plain (nc, nloc) copy for transfer setup
  std::vector<uint8_t> scalar_constrained;  // per scalar DoF
};

Level* level_create(int device, int dim, int degree, int ncomp, int physics, int64_t n_cells,
                    int64_t n_vertices, const double* vertices, const int64_t* cells,
                    int64_t n_scalar, const int64_t* cell_dofs, int64_t n_constrained,
                    const int64_t* constrained, double lam, double mu);

// v = A u with zero-in / identity-out constraint convention (mfoperator.py:108-122)
void level_apply(Level& L, const double* src, double* dst, cudaStream_t s);
// partial applies (distributed levels): zero + constrained rows, then cell-block ranges
void level_apply_begin(Level& L, const double* src, double* dst, bool negate, cudaStream_t s);
void level_apply_cells(Level& L, const double* src, double* dst, int64_t b0, int64_t b1, bool negate,
                       cudaStream_t s);
// exact diagonal, constrained = 1 (mfoperator.py:92-95, 135-150, 219-238)
void level_compute_diagonal(Level& L, cudaStream_t s);

// b = (f, phi_i) for a constant per-component body load f[ncomp]; constrained
// entries 0 (body-load part of assemble_rhs, mfoperator.py:313-355)
void level_load_vector(Level& L, const double* f, double* b, cudaStream_t s);

// launch the raw cell kernel (no zeroing, no constraint fix-up) over cell blocks [b0, b1)
void launch_apply_cells(const Level& L, const double* src, double* dst, int64_t b0, int64_t b1,
                        cudaStream_t s, bool negate = false);
// dst -= A src (constrained rows: dst[c] -= src[c]); no zeroing pass
void level_apply_sub(Level& L, const double* src, double* dst, cudaStream_t s);
void launch_copy_constrained(const Level& L, const double* src, double* dst, cudaStream_t s);
// mixed-precision V-cycle: fp32 copies of geometry / inverse diagonal, and the
// residual-form apply on fp32 vectors (fp64 arithmetic)
void level_enable_f32(Level& L, cudaStream_t s);
// fixed-order (atomic-free) summation of cell contributions in apply /
// diagonal / load vector: bitwise reproducible results
void level_set_deterministic(Level& L, bool on);
void level_apply_sub_f32(Level& L, const float* src, float* dst, cudaStream_t s);

}  // namespace nnmg
