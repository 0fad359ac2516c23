// extern "C" boundary of libnnmg_cuda.so (declared in include/nnmg_cuda.h).
#include "../../include/nnmg_cuda.h"
#include "nnmg_coarse.cuh"
#include "nnmg_level.cuh"
#include "nnmg_transfer.cuh"
#include "nnmg_vcycle.cuh"
#include "nnmg_vector.cuh"

#include <exception>

using namespace nnmg;

namespace {

template <class F>
int guard(F&& f) {
  try {
    f();
    return kOk;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.status;
  } catch (const std::exception& e) {
    set_error(e.what());
    return kCudaError;
  } catch (...) {
    set_error("unknown error");
    return kCudaError;
  }
}

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline Level* LV(nnmg_level_t h) { return reinterpret_cast<Level*>(h); }
inline Transfer* TR(nnmg_transfer_t h) { return reinterpret_cast<Transfer*>(h); }
inline Coarse* CO(nnmg_coarse_t h) { return reinterpret_cast<Coarse*>(h); }
inline VCycle* VC(nnmg_vcycle_t h) { return reinterpret_cast<VCycle*>(h); }

#define REQUIRE_HANDLE(h) NNMG_REQUIRE((h) != nullptr, kInvalidArgument, "null handle")

}  // namespace

extern "C" {

int nnmg_abi_version(void) { return 1; }
const char* nnmg_last_error(void) { return last_error(); }
uint64_t nnmg_launch_count(void) { return launch_count(); }

int nnmg_measure_fp64_peak(int device, double* tflops) {
  return guard([&] {
    NNMG_REQUIRE(tflops, kInvalidArgument, "null argument");
    *tflops = measure_fp64_peak(device);
  });
}

int nnmg_level_create(int device, int dim, int degree, int n_components, int physics, int64_t n_cells,
                      int64_t n_vertices, const double* vertices_host, const int64_t* cells_host,
                      int64_t n_scalar_dofs, const int64_t* cell_dofs_host, int64_t n_constrained,
                      const int64_t* constrained_host, double lambda, double mu, nnmg_level_t* out) {
  return guard([&] {
    NNMG_REQUIRE(out && vertices_host && cells_host && cell_dofs_host, kInvalidArgument, "null argument");
    NNMG_REQUIRE(n_constrained == 0 || constrained_host, kInvalidArgument, "null constraint list");
    *out = reinterpret_cast<nnmg_level_t>(level_create(device, dim, degree, n_components, physics, n_cells,
                                                       n_vertices, vertices_host, cells_host, n_scalar_dofs,
                                                       cell_dofs_host, n_constrained, constrained_host, lambda, mu));
  });
}

int nnmg_level_destroy(nnmg_level_t level) {
  return guard([&] { delete LV(level); });
}

int nnmg_level_info(nnmg_level_t level, int64_t* n_dofs, int64_t* n_cells, int* cells_per_block,
                    int64_t* geometry_bytes, int64_t* index_bytes) {
  return guard([&] {
    REQUIRE_HANDLE(level);
    Level* L = LV(level);
    if (n_dofs) *n_dofs = L->n_dofs;
    if (n_cells) *n_cells = L->n_cells;
    if (cells_per_block) *cells_per_block = L->cb;
    if (geometry_bytes) *geometry_bytes = static_cast<int64_t>(L->geo.n * sizeof(double));
    if (index_bytes) *index_bytes = static_cast<int64_t>(L->idx.n * sizeof(int));
  });
}

int nnmg_level_apply(nnmg_level_t level, const double* src, double* dst, void* stream) {
  return guard([&] {
    REQUIRE_HANDLE(level);
    level_apply(*LV(level), src, dst, S(stream));
  });
}

int nnmg_level_apply_begin(nnmg_level_t level, const double* src, double* dst, int negate, void* stream) {
  return guard([&] {
    REQUIRE_HANDLE(level);
    level_apply_begin(*LV(level), src, dst, negate != 0, S(stream));
  });
}

int nnmg_level_apply_cells(nnmg_level_t level, const double* src, double* dst, int64_t block0, int64_t block1,
                           int negate, void* stream) {
  return guard([&] {
    REQUIRE_HANDLE(level);
    level_apply_cells(*LV(level), src, dst, block0, block1, negate != 0, S(stream));
  });
}

int nnmg_level_residual(nnmg_level_t level, const double* f, const double* x, double* r, void* stream) {
  return guard([&] {
    REQUIRE_HANDLE(level);
    NNMG_REQUIRE(r != f && r != x, kInvalidArgument, "residual output must not alias f or x");
    NNMG_CUDA_TRY(cudaMemcpyAsync(r, f, sizeof(double) * LV(level)->n_dofs, cudaMemcpyDeviceToDevice, S(stream)));
    level_apply_sub(*LV(level), x, r, S(stream));
  });
}

int nnmg_level_compute_diagonal(nnmg_level_t level, void* stream) {
  return guard([&] {
    REQUIRE_HANDLE(level);
    level_compute_diagonal(*LV(level), S(stream));
  });
}

int nnmg_level_diagonal(nnmg_level_t level, double* diag_dev, void* stream) {
  return guard([&] {
    REQUIRE_HANDLE(level);
    Level* L = LV(level);
    if (!L->diag_ready) level_compute_diagonal(*L, S(stream));
    NNMG_CUDA_TRY(cudaMemcpyAsync(diag_dev, L->diag.ptr, sizeof(double) * L->n_dofs, cudaMemcpyDeviceToDevice,
                                  S(stream)));
  });
}

int nnmg_level_load_vector(nnmg_level_t level, const double* f_host, double* b_dev, void* stream) {
  return guard([&] {
    REQUIRE_HANDLE(level);
    NNMG_REQUIRE(f_host && b_dev, kInvalidArgument, "null argument");
    level_load_vector(*LV(level), f_host, b_dev, S(stream));
  });
}

int nnmg_smoother_sweep(nnmg_level_t level, double lam_max, double lam_min, int degree, const double* b_dev,
                        const double* x0_dev, double* x_dev, double* work_dev, void* stream) {
  return guard([&] {
    REQUIRE_HANDLE(level);
    NNMG_REQUIRE(degree >= 1, kInvalidArgument, "Chebyshev degree must be >= 1");
    smoother_sweep(*LV(level), lam_max, lam_min, degree, b_dev, x0_dev, x_dev, work_dev, S(stream));
  });
}

int nnmg_cheb_start(int64_t n, const double* b, const double* ax, const double* x0, const double* inv_diag,
                    double theta, double* r, double* d, double* x, void* stream) {
  return guard([&] { cheb_start(n, b, ax, x0, inv_diag, theta, r, d, x, S(stream)); });
}

int nnmg_cheb_start_t(int64_t n, const double* t, const double* x0, const double* inv_diag, double theta,
                      const double* r, double* d, double* x, void* stream) {
  return guard([&] {
    NNMG_REQUIRE(n >= 0 && (n == 0 || (t && x0 && inv_diag && r && d && x)), kInvalidArgument, "null vector");
    cheb_start_t(n, t, x0, inv_diag, theta, r, d, x, S(stream));
  });
}

int nnmg_cheb_step(int64_t n, const double* ad, const double* inv_diag, double c1, double c2, double* r, double* d,
                   double* x, void* stream) {
  return guard([&] { cheb_step(n, ad, inv_diag, c1, c2, r, d, x, S(stream)); });
}

int nnmg_dot_workspace(void) { return static_cast<int>(dot_workspace_doubles()); }

int nnmg_dot2(int64_t n, const double* a, const double* b, const double* c, const double* d, double* out,
              double* work, void* stream) {
  return guard([&] { dot2(n, a, b, c, d, out, work, S(stream)); });
}

int nnmg_axpby(int64_t n, double alpha, const double* x, double beta, double* y, void* stream) {
  return guard([&] { axpby(n, alpha, x, beta, y, S(stream)); });
}

int nnmg_sub(int64_t n, const double* a, const double* b, double* out, void* stream) {
  return guard([&] { sub(n, a, b, out, S(stream)); });
}

int nnmg_mul(int64_t n, const double* a, const double* b, double* out, void* stream) {
  return guard([&] { mul(n, a, b, out, S(stream)); });
}

int nnmg_cg_update(int64_t n, double alpha, const double* p, const double* ap, double* x, double* r, void* stream) {
  return guard([&] { cg_update(n, alpha, p, ap, x, r, S(stream)); });
}

int nnmg_transfer_create(nnmg_level_t coarse, nnmg_level_t fine, int64_t n_points, const int64_t* point_dofs,
                         const int64_t* cells, const double* xhat, nnmg_transfer_t* out) {
  return guard([&] {
    REQUIRE_HANDLE(coarse);
    REQUIRE_HANDLE(fine);
    NNMG_REQUIRE(out && (n_points == 0 || (point_dofs && cells && xhat)), kInvalidArgument, "null argument");
    *out = reinterpret_cast<nnmg_transfer_t>(transfer_create(LV(coarse), LV(fine), n_points, point_dofs, cells, xhat));
  });
}

int nnmg_transfer_destroy(nnmg_transfer_t transfer) {
  return guard([&] { delete TR(transfer); });
}

int nnmg_transfer_prolongate(nnmg_transfer_t transfer, const double* uc, double* uf, int accumulate, void* stream) {
  return guard([&] {
    REQUIRE_HANDLE(transfer);
    transfer_prolongate(*TR(transfer), uc, uf, accumulate != 0, S(stream));
  });
}

int nnmg_transfer_set_timing(nnmg_transfer_t transfer, int enable) {
  return guard([&] {
    REQUIRE_HANDLE(transfer);
    transfer_set_timing(*TR(transfer), enable != 0);
  });
}

int nnmg_transfer_last_timing(nnmg_transfer_t transfer, double* evaluate_s, double* gather_scatter_s) {
  return guard([&] {
    REQUIRE_HANDLE(transfer);
    transfer_last_timing(*TR(transfer), evaluate_s, gather_scatter_s);
  });
}

int nnmg_transfer_restrict(nnmg_transfer_t transfer, const double* rf, double* rc, void* stream) {
  return guard([&] {
    REQUIRE_HANDLE(transfer);
    transfer_restrict(*TR(transfer), rf, rc, S(stream));
  });
}

int nnmg_locate_points(int device, int dim, int64_t n_vertices, const double* vertices, int64_t n_cells,
                       const int64_t* cells, int64_t n_points, const double* points, double eps_box, double eps_geo,
                       double eps_ref, int64_t* cells_out, double* xhat_out, uint8_t* projected_out,
                       int64_t* n_failed, int64_t* first_failed) {
  return guard([&] {
    NNMG_REQUIRE(vertices && cells && (n_points == 0 || (points && cells_out && xhat_out && projected_out)),
                 kInvalidArgument, "null argument");
    LocateResult r = locate_points(device, dim, n_vertices, vertices, n_cells, cells, n_points, points, eps_box,
                                   eps_geo, eps_ref, cells_out, xhat_out, projected_out);
    if (n_failed) *n_failed = r.n_missing;
    if (first_failed) *first_failed = r.first_missing;
    NNMG_REQUIRE(r.n_missing == 0, kSearchError,
                 "points outside padded domain: " + std::to_string(r.n_missing) + " point(s), first index " +
                     std::to_string(r.first_missing));
  });
}

int nnmg_coarse_dense_create(nnmg_level_t level, const double* inverse, nnmg_coarse_t* out) {
  return guard([&] {
    REQUIRE_HANDLE(level);
    NNMG_REQUIRE(out && inverse, kInvalidArgument, "null argument");
    *out = reinterpret_cast<nnmg_coarse_t>(coarse_dense_create(LV(level), inverse));
  });
}

int nnmg_coarse_cg_create(nnmg_level_t level, double reduction, int max_iter, nnmg_coarse_t* out) {
  return guard([&] {
    REQUIRE_HANDLE(level);
    NNMG_REQUIRE(out, kInvalidArgument, "null argument");
    *out = reinterpret_cast<nnmg_coarse_t>(coarse_cg_create(LV(level), reduction, max_iter));
  });
}

int nnmg_coarse_direct_create(nnmg_level_t level, const double* inverse_dev, int64_t ld, nnmg_coarse_t* out) {
  return guard([&] {
    REQUIRE_HANDLE(level);
    NNMG_REQUIRE(out && inverse_dev, kInvalidArgument, "null argument");
    *out = reinterpret_cast<nnmg_coarse_t>(coarse_direct_create(LV(level), inverse_dev, ld));
  });
}

int nnmg_coarse_direct_create_share(nnmg_level_t level, const double* inverse_dev, int64_t ld, int share, int n_shares,
                                    nnmg_coarse_t* out) {
  return guard([&] {
    REQUIRE_HANDLE(level);
    NNMG_REQUIRE(out && inverse_dev, kInvalidArgument, "null argument");
    *out = reinterpret_cast<nnmg_coarse_t>(coarse_direct_create(LV(level), inverse_dev, ld, false, share, n_shares));
  });
}

int nnmg_coarse_direct_create_f32(nnmg_level_t level, const double* inverse_dev, int64_t ld, nnmg_coarse_t* out) {
  return guard([&] {
    REQUIRE_HANDLE(level);
    NNMG_REQUIRE(out && inverse_dev, kInvalidArgument, "null argument");
    *out = reinterpret_cast<nnmg_coarse_t>(coarse_direct_create(LV(level), inverse_dev, ld, true));
  });
}

int nnmg_coarse_destroy(nnmg_coarse_t coarse) {
  return guard([&] { delete CO(coarse); });
}

int nnmg_coarse_solve(nnmg_coarse_t coarse, const double* b, double* x, void* stream) {
  return guard([&] {
    REQUIRE_HANDLE(coarse);
    coarse_solve(*CO(coarse), b, x, S(stream));
  });
}

int nnmg_coarse_status(nnmg_coarse_t coarse, int* iterations, int* converged, int* indefinite) {
  return guard([&] {
    REQUIRE_HANDLE(coarse);
    int it = 0, cv = 0, er = 0;
    coarse_status(*CO(coarse), &it, &cv, &er);
    if (iterations) *iterations = it;
    if (converged) *converged = cv;
    if (indefinite) *indefinite = er;
  });
}

int nnmg_coarse_info(nnmg_coarse_t coarse, int* cluster_ctas, int* threads_per_cta, int* subgroups) {
  return guard([&] {
    REQUIRE_HANDLE(coarse);
    Coarse* C = CO(coarse);
    if (cluster_ctas) *cluster_ctas = (C->dense || C->direct) ? 0 : C->nrank;
    if (threads_per_cta) *threads_per_cta = C->block;
    if (subgroups) *subgroups = C->nsub;
  });
}

int nnmg_vcycle_create(int n_levels, const nnmg_level_t* levels, const nnmg_transfer_t* transfers,
                       nnmg_coarse_t coarse, const double* lam_max, const double* lam_min, const int* cheb_degree,
                       int m1, int m2, nnmg_vcycle_t* out) {
  return guard([&] {
    NNMG_REQUIRE(out && levels && lam_max && lam_min && cheb_degree, kInvalidArgument, "null argument");
    std::vector<Level*> lv(n_levels);
    std::vector<Transfer*> tr(n_levels > 0 ? n_levels - 1 : 0);
    for (int i = 0; i < n_levels; ++i) lv[i] = LV(levels[i]);
    for (int i = 0; i + 1 < n_levels; ++i) tr[i] = TR(transfers[i]);
    *out = reinterpret_cast<nnmg_vcycle_t>(
        vcycle_create(n_levels, lv.data(), tr.data(), CO(coarse), lam_max, lam_min, cheb_degree, m1, m2));
  });
}

int nnmg_vcycle_destroy(nnmg_vcycle_t vcycle) {
  return guard([&] { delete VC(vcycle); });
}

int nnmg_vcycle_run(nnmg_vcycle_t vcycle, const double* f, double* x, void* stream) {
  return guard([&] {
    REQUIRE_HANDLE(vcycle);
    vcycle_run(*VC(vcycle), f, x, S(stream));
  });
}

int nnmg_halo_pack(int64_t n, const int64_t* idx, const double* src, double* dst, void* stream) {
  return guard([&] {
    NNMG_REQUIRE(n == 0 || (idx && src && dst), kInvalidArgument, "null argument");
    gather_idx(n, idx, src, dst, S(stream));
  });
}

int nnmg_halo_unpack(int64_t n, const int64_t* idx, const double* src, double* dst, int add, void* stream) {
  return guard([&] {
    NNMG_REQUIRE(n == 0 || (idx && src && dst), kInvalidArgument, "null argument");
    scatter_idx(n, idx, src, dst, add != 0, S(stream));
  });
}

int nnmg_level_set_deterministic(nnmg_level_t level, int enable) {
  return guard([&] {
    REQUIRE_HANDLE(level);
    level_set_deterministic(*LV(level), enable != 0);
  });
}

int nnmg_vcycle_set_precision(nnmg_vcycle_t vcycle, int bits) {
  return guard([&] {
    REQUIRE_HANDLE(vcycle);
    vcycle_set_precision(*VC(vcycle), bits);
  });
}

int nnmg_vcycle_set_mixed_coarse(nnmg_vcycle_t vcycle, nnmg_coarse_t coarse) {
  return guard([&] {
    REQUIRE_HANDLE(vcycle);
    vcycle_set_mixed_coarse(*VC(vcycle), CO(coarse));
  });
}

int nnmg_vcycle_use_graph(nnmg_vcycle_t vcycle, int enable) {
  return guard([&] {
    REQUIRE_HANDLE(vcycle);
    VC(vcycle)->use_graph = enable != 0;
  });
}

int nnmg_vcycle_kernels_per_cycle(nnmg_vcycle_t vcycle, int64_t* n) {
  return guard([&] {
    REQUIRE_HANDLE(vcycle);
    *n = vcycle_kernels(*VC(vcycle));
  });
}

}  // extern "C"
