#pragma once

#include "nnmg_level.cuh"

namespace nnmg {

struct Coarse {
  Level* level = nullptr;
  bool dense = false;
  DevBuf<double> ainv;  // dense inverse (row-major)
  double reduction = 1e-8;
  int max_iter = 10000;
  DevBuf<double> r, z, p, ap, part, s;
  bool single_barrier = false;  // Chronopoulos-Gear form, one grid barrier per iteration
  DevBuf<unsigned char> con;  // constrained-row flags (single-barrier kernel)
  DevBuf<unsigned long long> epoch;  // last barrier epoch used (persists across solves)
  DevBuf<int> status;  // iterations, converged, error
  int nrank = 1, nsub = 1, block = 0;
  int split = 1;  // CTAs per cell block (single-barrier kernel); 0: balanced cell ranges
  bool resident = false;  // cell-block tables kept in shared memory
  int mode = 0;           // 0 pencil, 1 pencil resident, 2 register kernel
  int owner_warps = 0;    // single-barrier kernel: dedicated owner warps (overlap owner updates with cells)
  int barrier = 0;        // 0 grid.sync, 1 all-to-all slots, 2 root broadcast (NNMG_COARSE_BARRIER)
  DevBuf<unsigned long long> trace;  // NNMG_COARSE_TRACE: per-phase timestamps of CTA 0
  size_t smem = 0;
  // direct path: packed lower-triangle 64x64 tiles of the SPD inverse of
  // the free-DoF block
  bool direct = false;
  int64_t nfree = 0;
  DevBuf<int> dfree, dcons;      // free DoFs (ascending), constrained DoFs
  int nb = 0;                    // 64-row blocks of free DoFs
  DevBuf<double> tiles;          // [nb(nb+1)/2][64][64], tile (I, J <= I) at I(I+1)/2 + J
  bool tiles_f32 = false;        // fp32 tiles (the mixed-precision cycle's coarse solve)
  DevBuf<float> tiles32;
  DevBuf<double> prow, pcol;     // per-tile partial products (rows of I / columns of J)
  int64_t t0 = 0, t1 = 0;        // this handle's tile range (a share of the tiles when split across ranks)
  bool identity = true;          // this share writes the identity (constrained) rows
};

Coarse* coarse_dense_create(Level* L, const double* inverse);
Coarse* coarse_cg_create(Level* L, double reduction, int max_iter);
// direct path: inverse_dev (nf x nf row-major, leading dimension ld, device
// memory): the inverse of the free-DoF block (free DoFs ascending, the
// complement of the level's constrained list), read in its lower triangle
// only and packed into symmetric tiles
// share / n_shares: this handle streams an equal contiguous share of the tiles
// (cell-partitioned runs: the shares' outputs are summed by an all-reduce)
Coarse* coarse_direct_create(Level* L, const double* inverse_dev, int64_t ld, bool f32 = false, int share = 0,
                             int n_shares = 1);
void coarse_direct_solve(Coarse& C, const double* b, double* x, cudaStream_t s);
void coarse_solve(Coarse& C, const double* b, double* x, cudaStream_t s);
void coarse_status(Coarse& C, int* iterations, int* converged, int* error);

}  // namespace nnmg
