#pragma once

#include "nnmg_coarse.cuh"
#include "nnmg_level.cuh"
#include "nnmg_transfer.cuh"

#include <memory>

namespace nnmg {

// residual_out: one more residual-form apply after the last step leaves
// b - A x in work[0, n) (the recurrence keeps r = b - A (x - d)).
// t != nullptr: work[0, n) already holds b - A x on entry and the sweep
// starts from x + t (x0 == x, t added in the first vector kernel).
void smoother_sweep(Level& L, double lam_max, double lam_min, int degree, const double* b, const double* x0,
                    double* x, double* work, cudaStream_t s, bool residual_out = false,
                    const double* t = nullptr);

struct VCycle {
  std::vector<Level*> levels;        // coarsest first
  std::vector<Transfer*> transfers;  // transfers[l-1] connects l-1 -> l
  Coarse* coarse = nullptr;
  Coarse* coarse32 = nullptr;  // optional coarse solver of the mixed-precision cycle (fp32 inverse tiles)
  std::vector<double> lam_max, lam_min;
  std::vector<int> degree;
  int m1 = 1, m2 = 1;
  // per level: right-hand side and correction (coarse levels), residual, smoother work
  std::vector<DevBuf<double>> f, x, r, work;
  bool use_graph = false;
  // mixed precision (vcycle_set_precision(32)): fp32 level vectors above the
  // coarsest level, fp64 coarse solve through cf/cx
  bool mixed = false;
  std::vector<DevBuf<float>> f32, x32, r32, work32;
  DevBuf<double> cf, cx;
  bool smoother_residual = true;  // residual after pre-smoothing from the smoother's recurrence (no b copy)
  bool post_from_residual = true; // first post-smoothing sweep starts from that residual (no b copy)
  struct Graph {
    const double* f;
    double* x;
    cudaStream_t s;
    cudaGraphExec_t exec;
    uint64_t last_use;
  };
  std::vector<Graph> graphs;  // small LRU keyed by (f, x, stream)
  uint64_t clock = 0;
  int64_t kernels_per_cycle = 0;
  ~VCycle();
};

VCycle* vcycle_create(int n_levels, Level* const* levels, Transfer* const* transfers, Coarse* coarse,
                      const double* lam_max, const double* lam_min, const int* degree, int m1, int m2);
void vcycle_run(VCycle& V, const double* f, double* x, cudaStream_t s);
// 64: the fp64 cycle (default); 32: the mixed-precision cycle (fp32 storage
// of vectors / geometry / transfer records on levels >= 1, fp64 arithmetic,
// fp64 coarse solve); input and output stay fp64
void vcycle_set_precision(VCycle& V, int bits);
// coarse solver used by the mixed-precision cycle instead of V.coarse (nullptr: the same); drops captured graphs
void vcycle_set_mixed_coarse(VCycle& V, Coarse* coarse);
int64_t vcycle_kernels(VCycle& V);

}  // namespace nnmg
