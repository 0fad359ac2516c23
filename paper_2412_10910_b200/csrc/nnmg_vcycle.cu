// Chebyshev-Jacobi smoother sweep and the V-cycle executor
// (replaces ChebyshevJacobi._sweep, solvers.py:88-108, and
// MultigridHierarchy._v, multigrid.py:83-113), optionally replayed as one
// CUDA graph so a whole cycle costs one launch.
#include "nnmg_vcycle.cuh"
#include "nnmg_vector.cuh"

#include <algorithm>
#include <cstdlib>

namespace nnmg {

void smoother_sweep(Level& L, double lam_max, double lam_min, int degree, const double* b, const double* x0,
                    double* x, double* work, cudaStream_t s, bool residual_out, const double* t) {
  NNMG_REQUIRE(L.diag_ready, kInvalidArgument, "level diagonal not computed");
  const int64_t n = L.n_dofs;
  double* r = work;
  double* d = work + n;
  const double theta = (lam_max + lam_min) / 2.0;
  const double delta = (lam_max - lam_min) / 2.0;
  const double sigma = theta / delta;
  // residual form: the apply scatters -A(.) straight into r (no zeroing pass,
  // no separate A d vector); same recurrence as solvers.py:94-107
  if (t != nullptr) {
    // work[0, n) holds f - A x: r = f - A (x + t), x = (x + t) + d
    level_apply_sub(L, t, r, s);
    cheb_init_add(n, t, L.inv_diag.ptr, theta, r, d, x, s);
  } else if (x0 == nullptr) {
    // x = d is folded into the first update when there is one
    cheb_init(n, b, nullptr, L.inv_diag.ptr, theta, r, d, degree > 1 ? nullptr : x, s);
  } else {
    NNMG_CUDA_TRY(cudaMemcpyAsync(r, b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    level_apply_sub(L, x0, r, s);
    cheb_init(n, b, x0, L.inv_diag.ptr, theta, r, d, x, s);
  }
  double rho_old = 1.0 / sigma;
  for (int k = 0; k < degree - 1; ++k) {
    level_apply_sub(L, d, r, s);
    const double rho = 1.0 / (2.0 * sigma - rho_old);
    cheb_update(n, L.inv_diag.ptr, rho * rho_old, 2.0 * rho / delta, r, d, x, s,
                k == 0 && x0 == nullptr && t == nullptr);
    rho_old = rho;
  }
  if (residual_out) level_apply_sub(L, d, r, s);
}

// the same sweep on fp32 vectors (mixed-precision V-cycle, fp64 arithmetic)
static void smoother_sweep_f32(Level& L, double lam_max, double lam_min, int degree, const float* b, const float* x0,
                               float* x, float* work, cudaStream_t s, bool residual_out, const float* t) {
  const int64_t n = L.n_dofs;
  float* r = work;
  float* d = work + ((n + 3) & ~int64_t(3));  // 16-byte aligned: the float4 vector kernels
  const float* idg = L.inv_diag32.ptr;
  const double theta = (lam_max + lam_min) / 2.0;
  const double delta = (lam_max - lam_min) / 2.0;
  const double sigma = theta / delta;
  if (t != nullptr) {
    level_apply_sub_f32(L, t, r, s);
    cheb_init_add(n, t, idg, theta, r, d, x, s);
  } else if (x0 == nullptr) {
    cheb_init(n, b, static_cast<const float*>(nullptr), idg, theta, r, d, degree > 1 ? nullptr : x, s);
  } else {
    NNMG_CUDA_TRY(cudaMemcpyAsync(r, b, sizeof(float) * n, cudaMemcpyDeviceToDevice, s));
    level_apply_sub_f32(L, x0, r, s);
    cheb_init(n, b, x0, idg, theta, r, d, x, s);
  }
  double rho_old = 1.0 / sigma;
  for (int k = 0; k < degree - 1; ++k) {
    level_apply_sub_f32(L, d, r, s);
    const double rho = 1.0 / (2.0 * sigma - rho_old);
    cheb_update(n, idg, rho * rho_old, 2.0 * rho / delta, r, d, x, s, k == 0 && x0 == nullptr && t == nullptr);
    rho_old = rho;
  }
  if (residual_out) level_apply_sub_f32(L, d, r, s);
}

VCycle::~VCycle() {
  for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
}

VCycle* vcycle_create(int n_levels, Level* const* levels, Transfer* const* transfers, Coarse* coarse,
                      const double* lam_max, const double* lam_min, const int* degree, int m1, int m2) {
  NNMG_REQUIRE(n_levels >= 1, kInvalidArgument, "need at least one level");
  NNMG_REQUIRE(coarse && coarse->level == levels[0], kInvalidArgument, "coarse solver must own level 0");
  auto V = new VCycle();
  try {
    V->m1 = m1;
    V->m2 = m2;
    if (const char* e = getenv("NNMG_SMOOTHER_RESIDUAL")) V->smoother_residual = atoi(e) != 0;
    if (const char* e = getenv("NNMG_POST_FROM_RESIDUAL")) V->post_from_residual = atoi(e) != 0;
    for (int l = 0; l < n_levels; ++l) {
      NNMG_REQUIRE(levels[l] != nullptr, kInvalidArgument, "null level");
      V->levels.push_back(levels[l]);
      V->lam_max.push_back(lam_max[l]);
      V->lam_min.push_back(lam_min[l]);
      V->degree.push_back(degree[l]);
      if (l > 0) {
        Transfer* T = transfers[l - 1];
        NNMG_REQUIRE(T && T->coarse == levels[l - 1] && T->fine == levels[l], kInvalidArgument,
                     "transfer " + std::to_string(l - 1) + " does not connect levels " + std::to_string(l - 1) +
                         " and " + std::to_string(l));
        NNMG_REQUIRE(levels[l]->diag_ready, kInvalidArgument, "level diagonal not computed");
        V->transfers.push_back(T);
      }
    }
    V->coarse = coarse;
    V->f.resize(n_levels);
    V->x.resize(n_levels);
    V->r.resize(n_levels);
    V->work.resize(n_levels);
    for (int l = 0; l < n_levels; ++l) {
      const int64_t n = levels[l]->n_dofs;
      if (l < n_levels - 1) {
        V->f[l].alloc(n);
        V->x[l].alloc(n);
      }
      V->r[l].alloc(n);
      V->work[l].alloc(3 * n);
    }
  } catch (...) {
    delete V;
    throw;
  }
  return V;
}

static void cycle(VCycle& V, int l, const double* f, double* x, cudaStream_t s) {
  if (l == 0) {
    coarse_solve(*V.coarse, f, x, s);
    return;
  }
  Level& L = *V.levels[l];
  Transfer& T = *V.transfers[l - 1];
  double* w = V.work[l].ptr;
  // the residual f - A x (multigrid.py:101) costs one apply either way; taken
  // from the last sweep's recurrence it needs no copy of f (same apply count)
  const bool rec = V.smoother_residual && V.m1 > 0;
  for (int k = 0; k < V.m1; ++k)
    smoother_sweep(L, V.lam_max[l], V.lam_min[l], V.degree[l], f, k == 0 ? nullptr : x, x, w, s,
                   rec && k == V.m1 - 1);
  if (V.m1 == 0) NNMG_CUDA_TRY(cudaMemsetAsync(x, 0, sizeof(double) * L.n_dofs, s));
  double* r = rec ? w : V.r[l].ptr;
  if (!rec) {
    NNMG_CUDA_TRY(cudaMemcpyAsync(r, f, sizeof(double) * L.n_dofs, cudaMemcpyDeviceToDevice, s));
    level_apply_sub(L, x, r, s);
  }
  transfer_restrict(T, r, V.f[l - 1].ptr, s);
  cycle(V, l - 1, V.f[l - 1].ptr, V.x[l - 1].ptr, s);
  if (rec && V.m2 > 0 && V.post_from_residual) {
    // the first post-smoothing sweep starts from the residual still in w:
    // f - A (x + P e_c) = (f - A x) - A (P e_c), no copy of f; the
    // correction is added inside the sweep's first vector kernel
    double* t = V.r[l].ptr;
    transfer_prolongate(T, V.x[l - 1].ptr, t, false, s);
    smoother_sweep(L, V.lam_max[l], V.lam_min[l], V.degree[l], f, x, x, w, s, false, t);
    for (int k = 1; k < V.m2; ++k) smoother_sweep(L, V.lam_max[l], V.lam_min[l], V.degree[l], f, x, x, w, s);
  } else {
    transfer_prolongate(T, V.x[l - 1].ptr, x, true, s);
    for (int k = 0; k < V.m2; ++k) smoother_sweep(L, V.lam_max[l], V.lam_min[l], V.degree[l], f, x, x, w, s);
  }
}

// mixed-precision cycle (the paper's fp32 V-cycle inside fp64 CG,
// PAPER.md:392): fp32 vectors, geometry and transfer records on every level
// above the coarsest; the coarse solve stays fp64 (converted in and out)
static void cycle32(VCycle& V, int l, const float* f, float* x, cudaStream_t s) {
  if (l == 0) {
    const int64_t n0 = V.levels[0]->n_dofs;
    convert(n0, f, V.cf.ptr, s);
    coarse_solve(V.coarse32 ? *V.coarse32 : *V.coarse, V.cf.ptr, V.cx.ptr, s);
    convert(n0, V.cx.ptr, x, s);
    return;
  }
  Level& L = *V.levels[l];
  Transfer& T = *V.transfers[l - 1];
  float* w = V.work32[l].ptr;
  // residual from the smoother recurrence, post-smoothing from that residual
  for (int k = 0; k < V.m1; ++k)
    smoother_sweep_f32(L, V.lam_max[l], V.lam_min[l], V.degree[l], f, k == 0 ? nullptr : x, x, w, s,
                       k == V.m1 - 1, nullptr);
  float* r = w;
  if (V.m1 == 0) {
    NNMG_CUDA_TRY(cudaMemsetAsync(x, 0, sizeof(float) * L.n_dofs, s));
    NNMG_CUDA_TRY(cudaMemcpyAsync(r, f, sizeof(float) * L.n_dofs, cudaMemcpyDeviceToDevice, s));
  }
  transfer_restrict_f32(T, r, V.f32[l - 1].ptr, s);
  cycle32(V, l - 1, V.f32[l - 1].ptr, V.x32[l - 1].ptr, s);
  if (V.m2 > 0) {
    float* t = V.r32[l].ptr;
    transfer_prolongate_f32(T, V.x32[l - 1].ptr, t, false, s);
    smoother_sweep_f32(L, V.lam_max[l], V.lam_min[l], V.degree[l], f, x, x, w, s, false, t);
    for (int k = 1; k < V.m2; ++k)
      smoother_sweep_f32(L, V.lam_max[l], V.lam_min[l], V.degree[l], f, x, x, w, s, false, nullptr);
  } else {
    transfer_prolongate_f32(T, V.x32[l - 1].ptr, x, true, s);
  }
}

static void run_cycle(VCycle& V, const double* f, double* x, cudaStream_t s) {
  const int top = static_cast<int>(V.levels.size()) - 1;
  if (!V.mixed || top == 0) {
    cycle(V, top, f, x, s);
    return;
  }
  const int64_t n = V.levels[top]->n_dofs;
  convert(n, f, V.f32[top].ptr, s);
  cycle32(V, top, V.f32[top].ptr, V.x32[top].ptr, s);
  convert(n, V.x32[top].ptr, x, s);
}

void vcycle_set_mixed_coarse(VCycle& V, Coarse* coarse) {
  NNMG_REQUIRE(coarse == nullptr || coarse->level == V.levels[0], kInvalidArgument,
               "coarse solver belongs to another level");
  if (coarse == V.coarse32) return;
  for (auto& g : V.graphs) cudaGraphExecDestroy(g.exec);
  V.graphs.clear();
  V.coarse32 = coarse;
}

void vcycle_set_precision(VCycle& V, int bits) {
  NNMG_REQUIRE(bits == 64 || bits == 32, kInvalidArgument, "precision must be 64 or 32 bits");
  const bool mixed = bits == 32;
  if (mixed == V.mixed) return;
  for (auto& g : V.graphs) cudaGraphExecDestroy(g.exec);
  V.graphs.clear();
  V.kernels_per_cycle = 0;
  V.mixed = mixed;
  if (!mixed || !V.f32.empty()) return;
  const int nl = static_cast<int>(V.levels.size());
  V.f32.resize(nl);
  V.x32.resize(nl);
  V.r32.resize(nl);
  V.work32.resize(nl);
  for (int l = 0; l < nl; ++l) {
    const int64_t n = V.levels[l]->n_dofs;
    V.f32[l].alloc(n);
    V.x32[l].alloc(n);
    if (l > 0) {
      level_enable_f32(*V.levels[l], 0);
      transfer_enable_f32(*V.transfers[l - 1], 0);
      V.r32[l].alloc(n);
      V.work32[l].alloc(3 * ((n + 3) & ~int64_t(3)));
    }
  }
  V.cf.alloc(V.levels[0]->n_dofs);
  V.cx.alloc(V.levels[0]->n_dofs);
  NNMG_CUDA_TRY(cudaDeviceSynchronize());
}

void vcycle_run(VCycle& V, const double* f, double* x, cudaStream_t s) {
  if (!V.use_graph) {
    run_cycle(V, f, x, s);
    return;
  }
  NNMG_REQUIRE(s != nullptr, kInvalidArgument, "graph replay needs a non-default stream");
  V.clock += 1;
  VCycle::Graph* hit = nullptr;
  for (auto& g : V.graphs)
    if (g.f == f && g.x == x && g.s == s) hit = &g;
  if (!hit) {
    constexpr size_t kMaxGraphs = 4;
    if (V.graphs.size() >= kMaxGraphs) {
      auto oldest = std::min_element(V.graphs.begin(), V.graphs.end(),
                                     [](const VCycle::Graph& a, const VCycle::Graph& b) { return a.last_use < b.last_use; });
      cudaGraphExecDestroy(oldest->exec);
      V.graphs.erase(oldest);
    }
    cudaGraph_t g = nullptr;
    const uint64_t c0 = launch_count();
    NNMG_CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    try {
      run_cycle(V, f, x, s);
    } catch (...) {
      cudaStreamEndCapture(s, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    NNMG_CUDA_TRY(cudaStreamEndCapture(s, &g));
    V.kernels_per_cycle = static_cast<int64_t>(launch_count() - c0);
    // capture records launches without executing them
    count_launch(-static_cast<int>(V.kernels_per_cycle));
    cudaGraphExec_t exec = nullptr;
    cudaError_t e = cudaGraphInstantiate(&exec, g, 0);
    cudaGraphDestroy(g);
    NNMG_CUDA_TRY(e);
    V.graphs.push_back(VCycle::Graph{f, x, s, exec, 0});
    hit = &V.graphs.back();
  }
  hit->last_use = V.clock;
  NNMG_CUDA_TRY(cudaGraphLaunch(hit->exec, s));
  count_launch(static_cast<int>(V.kernels_per_cycle));
}

int64_t vcycle_kernels(VCycle& V) {
  if (V.kernels_per_cycle > 0) return V.kernels_per_cycle;
  return -1;
}

}  // namespace nnmg
