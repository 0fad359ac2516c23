/*
 * nnmg_cuda.h - C ABI of libnnmg_cuda.so, the B200 (sm_100a) fp64 hot path of the
 * matrix-free non-nested multigrid method (arXiv 2412.10910).
 *
 * The reference (`/root/reference/pkg/src/nnmg`, pure Python/NumPy) has no FFI:
 * its hot path is a set of duck-typed Python protocols.  Each entry point below
 * names the reference interface it replaces (file:line).  The Python package
 * `paper_2412_10910_b200` binds this header with ctypes and keeps the
 * reference's class/method names on top of it; INTEGRATION.md shows the binding
 * a maintainer of the reference would add.
 *
 * Conventions
 *   - every function returns 0 on success, otherwise a status code
 *       1 invalid argument (-> ValueError)      2 CUDA error (-> RuntimeError)
 *       3 unsupported configuration             4 non-positive Jacobian
 *       5 point location failure (GeosearchError)
 *       6 indefinite operator (IndefiniteOperatorError)
 *     and nnmg_last_error() returns the thread's last message;
 *   - `host` pointers are read during the call only; `dev` pointers are device
 *     memory owned by the caller (e.g. torch tensors' data_ptr());
 *   - vectors are float64, length n_dofs, components interleaved fastest
 *     (reference fespace.py:104-131); index inputs are int64 like NumPy's;
 *   - work is enqueued on `stream` (a cudaStream_t, NULL = legacy default
 *     stream); nothing on the apply/transfer/smoother/coarse paths allocates
 *     or synchronises;
 *   - handles are bound to the device given at creation and are not
 *     thread-safe.
 */
#ifndef NNMG_CUDA_H_
#define NNMG_CUDA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nnmg_level_s* nnmg_level_t;
typedef struct nnmg_transfer_s* nnmg_transfer_t;
typedef struct nnmg_coarse_s* nnmg_coarse_t;
typedef struct nnmg_vcycle_s* nnmg_vcycle_t;

#define NNMG_PHYSICS_LAPLACE 0
#define NNMG_PHYSICS_ELASTICITY 1

/* ---- library ----------------------------------------------------------- */
int nnmg_abi_version(void);
const char* nnmg_last_error(void);
/* number of kernels this library has launched so far (process-wide) */
uint64_t nnmg_launch_count(void);
/* measured DFMA throughput of `device` in TFLOP/s (synchronises; the FP64
 * roofline denominator bench.py reports - not on any hot path) */
int nnmg_measure_fp64_peak(int device, double* tflops);

/* ---- levels: replaces _OperatorBase.__init__ (mfoperator.py:28-48),
 *      LaplaceOperator.__init__ (mfoperator.py:101-106) and
 *      ElasticityOperator.__init__ (mfoperator.py:163-169).
 * vertices_host (n_vertices, dim) f64; cells_host (n_cells, 2^dim) int64 with
 * the reference's local vertex order (mesh.py:5-7); cell_dofs_host
 * (n_cells, (degree+1)^dim) int64 scalar DoFs (fespace.py:137-163);
 * constrained_host: sorted constrained full DoFs (fespace.py:74-101, all
 * components of a constrained node).  The per-quadrature-point geometry is
 * computed on the device.  physics: NNMG_PHYSICS_*; lambda/mu for elasticity. */
int nnmg_level_create(int device, int dim, int degree, int n_components, int physics, int64_t n_cells,
                      int64_t n_vertices, const double* vertices_host, const int64_t* cells_host,
                      int64_t n_scalar_dofs, const int64_t* cell_dofs_host, int64_t n_constrained,
                      const int64_t* constrained_host, double lambda, double mu, nnmg_level_t* out);
int nnmg_level_destroy(nnmg_level_t level);
/* sizes and the stored bytes of the geometry and index streams */
int nnmg_level_info(nnmg_level_t level, int64_t* n_dofs, int64_t* n_cells, int* cells_per_block,
                    int64_t* geometry_bytes, int64_t* index_bytes);
/* dst_dev = A src_dev, zero-in/identity-out on constrained DoFs
 * replaces LaplaceOperator.apply (mfoperator.py:108-122) and
 * ElasticityOperator.apply (mfoperator.py:171-202) */
int nnmg_level_apply(nnmg_level_t level, const double* src_dev, double* dst_dev, void* stream);
/* the same apply in pieces, for the distributed levels (overlap
 * interior cells with the ghost exchange).  begin: dst = 0 plus identity-out on
 * the constrained rows; cells: dst += contributions of the cell blocks
 * [block0, block1) (blocks of `cells_per_block` consecutive cells, see
 * nnmg_level_info) to the free rows.  begin + cells(0, n_blocks) == apply.
 * negate != 0: the residual form dst -= A src of the smoother and the
 * V-cycle residual (solvers.py:97, 102; multigrid.py:97): begin subtracts src
 * on the constrained rows and leaves the rest of dst alone, cells subtracts.
 * Not available in deterministic mode (status 3). */
int nnmg_level_apply_begin(nnmg_level_t level, const double* src_dev, double* dst_dev, int negate, void* stream);
int nnmg_level_apply_cells(nnmg_level_t level, const double* src_dev, double* dst_dev, int64_t block0,
                           int64_t block1, int negate, void* stream);
/* r_dev = f_dev - A x_dev   (multigrid.py:97) */
int nnmg_level_residual(nnmg_level_t level, const double* f_dev, const double* x_dev, double* r_dev, void* stream);
/* compute/cache the exact diagonal and its inverse; copy it out
 * replaces _compute_diagonal / diagonal() (mfoperator.py:92-95, 135-150, 219-238) */
int nnmg_level_compute_diagonal(nnmg_level_t level, void* stream);
int nnmg_level_diagonal(nnmg_level_t level, double* diag_dev, void* stream);

/* deterministic mode (enable != 0): the apply, residual, diagonal and load
 * vector sum each DoF's cell contributions in a fixed order (per-cell buffer
 * + gather) instead of fp64 atomics, like the reference's serial bincount
 * scatter (mfoperator.py:88-90): bitwise reproducible results at the cost of
 * the buffer round trip.  Set before the diagonal is computed. */
int nnmg_level_set_deterministic(nnmg_level_t level, int enable);

/* b_dev = (f, phi_i) for a constant body load f_host[n_components],
 * constrained entries 0 (body-load part of assemble_rhs, mfoperator.py:313-355) */
int nnmg_level_load_vector(nnmg_level_t level, const double* f_host, double* b_dev, void* stream);

/* ---- Chebyshev-Jacobi smoother: replaces ChebyshevJacobi._sweep / smooth
 * (solvers.py:88-114).  One degree-k pass; x0_dev may be NULL (zero initial
 * guess).  work_dev: 3 * n_dofs doubles of scratch. */
int nnmg_smoother_sweep(nnmg_level_t level, double lam_max, double lam_min, int degree, const double* b_dev,
                        const double* x0_dev, double* x_dev, double* work_dev, void* stream);

/* fused Chebyshev vector updates for externally applied operators (the
 * distributed smoother): start  r = b - Ax (ax may be NULL: r = b; b may be
 * NULL: r already holds the residual), d = inv_diag*r/theta, x = x0 + d (x0
 * may be NULL);  step  r -= Ad (ad may be NULL: the apply already subtracted
 * it in place), d = c1 d + c2 inv_diag r, x += d   (solvers.py:94-107) */
int nnmg_cheb_start(int64_t n, const double* b, const double* ax, const double* x0, const double* inv_diag,
                    double theta, double* r, double* d, double* x, void* stream);
/* first post-smoothing sweep right after the prolongation (multigrid.py:107-111):
 * r already holds b - A (x0 + t); d = inv_diag*r/theta, x = (x0 + t) + d */
int nnmg_cheb_start_t(int64_t n, const double* t, const double* x0, const double* inv_diag, double theta,
                      const double* r, double* d, double* x, void* stream);
int nnmg_cheb_step(int64_t n, const double* ad, const double* inv_diag, double c1, double c2, double* r, double* d,
                   double* x, void* stream);

/* ---- vector kernels used by cg_solve (solvers.py:129-164) ---------------- */
/* out_dev[0] = a.b, out_dev[1] = c.d (c may be NULL); deterministic.
 * work_dev: nnmg_dot_workspace() doubles */
int nnmg_dot_workspace(void);
int nnmg_dot2(int64_t n, const double* a, const double* b, const double* c, const double* d, double* out_dev,
              double* work_dev, void* stream);
int nnmg_axpby(int64_t n, double alpha, const double* x, double beta, double* y, void* stream);
int nnmg_sub(int64_t n, const double* a, const double* b, double* out, void* stream);
int nnmg_mul(int64_t n, const double* a, const double* b, double* out, void* stream);
int nnmg_cg_update(int64_t n, double alpha, const double* p, const double* ap, double* x, double* r, void* stream);

/* ---- halo exchange of the distributed levels: pack
 * dst[i] = src[idx[i]] into a send buffer, unpack dst[idx[i]] = src[i]
 * (add = 0, ghost import) or dst[idx[i]] += src[i] (add != 0, export of ghost
 * partial sums); idx entries distinct within one call; device pointers */
int nnmg_halo_pack(int64_t n, const int64_t* idx, const double* src, double* dst, void* stream);
int nnmg_halo_unpack(int64_t n, const int64_t* idx, const double* src, double* dst, int add, void* stream);

/* ---- non-nested transfer: replaces TwoLevelTransferNonNested
 * (transfer.py:61-124).  point_dofs_host: fine scalar DoFs not fully
 * constrained (transfer.py:72-73); cells_host/xhat_host: owning coarse cell and
 * reference coordinates (transfer.py:79-82).  The records are regrouped by
 * owning cell on the device. */
int nnmg_transfer_create(nnmg_level_t coarse, nnmg_level_t fine, int64_t n_points, const int64_t* point_dofs_host,
                         const int64_t* cells_host, const double* xhat_host, nnmg_transfer_t* out);
int nnmg_transfer_destroy(nnmg_transfer_t transfer);
/* uf = P uc, or uf += P uc when accumulate != 0 (prolongate, transfer.py:31-44, 87-102) */
int nnmg_transfer_prolongate(nnmg_transfer_t transfer, const double* uc_dev, double* uf_dev, int accumulate,
                             void* stream);
/* rc = P^T rf, deterministic (restrict, transfer.py:46-58, 104-124) */
int nnmg_transfer_restrict(nnmg_transfer_t transfer, const double* rf_dev, double* rc_dev, void* stream);
/* per-phase timing rows: replaces timings["evaluate"] / timings["gather_scatter"]
 * (transfer.py:29, 100-101, 122-123).  While enabled, prolongate / restrict
 * record CUDA events around the point-evaluation kernel ("evaluate") and around
 * the zero-fill of point-less DoFs / the fixed-order coarse gather
 * ("gather_scatter"); last_timing synchronises on the last call and returns
 * seconds.  Leave it off for calls inside a CUDA-graph capture. */
int nnmg_transfer_set_timing(nnmg_transfer_t transfer, int enable);
int nnmg_transfer_last_timing(nnmg_transfer_t transfer, double* evaluate_s, double* gather_scatter_s);

/* ---- point location: replaces locate_points (geosearch.py:163-227) with its
 * tie-break and projection rules.  Outputs are host arrays of n_points.
 * Returns 5 if a point has no converged candidate; *n_failed/*first_failed
 * report them. */
int nnmg_locate_points(int device, int dim, int64_t n_vertices, const double* vertices_host, int64_t n_cells,
                       const int64_t* cells_host, int64_t n_points, const double* points_host, double eps_box,
                       double eps_geo, double eps_ref, int64_t* cells_out, double* xhat_out,
                       uint8_t* projected_out, int64_t* n_failed, int64_t* first_failed);

/* ---- coarsest-level solver: replaces CoarseSolver (solvers.py:167-206) ---- */
/* dense path: inverse_host (n x n, row-major) of the SPD coarse matrix */
int nnmg_coarse_dense_create(nnmg_level_t level, const double* inverse_host, nnmg_coarse_t* out);
/* Jacobi-PCG path (the reference's CoarseSolver above the dense limit) as one
 * persistent cooperative kernel over the whole GPU (one CTA per SM or per
 * cell-block piece, Chronopoulos-Gear form with one grid barrier per
 * iteration, fixed-order dot products) */
int nnmg_coarse_cg_create(nnmg_level_t level, double reduction, int max_iter, nnmg_coarse_t* out);
/* direct path for levels above the dense limit (a documented deviation: an
 * exact solve where the reference iterates to a 1e-8 reduction; selected by
 * CoarseSolver(direct=...) where it is faster): x = A_ff^-1 b on the free
 * DoFs, x = b on the constrained ones.  inverse_dev is A_ff^-1 (nf x nf, free
 * DoFs ascending = the complement of the level's constrained list) in DEVICE
 * memory, row-major with leading dimension ld; only its lower triangle is
 * read.  The library packs it into symmetric 64x64 tiles (nf^2/2 doubles
 * streamed per solve, no atomics: bitwise reproducible). */
int nnmg_coarse_direct_create(nnmg_level_t level, const double* inverse_dev, int64_t ld, nnmg_coarse_t* out);
/* one share of the same solve for cell-partitioned runs: this
 * handle packs and streams the tiles [nt share / n_shares, nt (share+1) / n_shares)
 * only; the outputs of all shares add up to the solution (share 0 also
 * writes the identity rows, the others zeros), so the ranks all-reduce x. */
int nnmg_coarse_direct_create_share(nnmg_level_t level, const double* inverse_dev, int64_t ld, int share,
                                    int n_shares, nnmg_coarse_t* out);
/* the same with the tiles stored in fp32 (half the streamed bytes;
 * single-precision products within a tile, fp64 partial sums): the coarse
 * solver of the mixed-precision cycle, see nnmg_vcycle_set_mixed_coarse */
int nnmg_coarse_direct_create_f32(nnmg_level_t level, const double* inverse_dev, int64_t ld, nnmg_coarse_t* out);
int nnmg_coarse_destroy(nnmg_coarse_t coarse);
int nnmg_coarse_solve(nnmg_coarse_t coarse, const double* b_dev, double* x_dev, void* stream);
/* iterations / converged / indefinite flag of the last CG solve (synchronises) */
int nnmg_coarse_status(nnmg_coarse_t coarse, int* iterations, int* converged, int* indefinite);
int nnmg_coarse_info(nnmg_coarse_t coarse, int* cluster_ctas, int* threads_per_cta, int* subgroups);

/* ---- V-cycle executor: replaces MultigridHierarchy._v (multigrid.py:83-113)
 * levels[0] is the coarsest; transfers[i] connects levels i and i+1; one
 * Chebyshev degree and (lam_max, lam_min) per level (index 0 unused); m1/m2
 * pre/post sweeps.  The whole cycle can be captured into a CUDA graph. */
int nnmg_vcycle_create(int n_levels, const nnmg_level_t* levels, const nnmg_transfer_t* transfers,
                       nnmg_coarse_t coarse, const double* lam_max, const double* lam_min, const int* cheb_degree,
                       int m1, int m2, nnmg_vcycle_t* out);
int nnmg_vcycle_destroy(nnmg_vcycle_t vcycle);
/* x_dev = V-cycle(f_dev) on the finest level (MultigridHierarchy.precondition) */
int nnmg_vcycle_run(nnmg_vcycle_t vcycle, const double* f_dev, double* x_dev, void* stream);
/* 64 (default): the fp64 cycle.  32: the mixed-precision cycle of the paper
 * (the V-cycle in single precision inside double-precision CG):
 * level vectors, stored geometry, inverse diagonals and transfer reference
 * coordinates in fp32 on every level above the coarsest, single-precision
 * arithmetic in the cell applies and the transfers (environment
 * NNMG_MIXED_ARITH=64: fp64 arithmetic on the fp32 storage), fp64 coarse
 * vectors; f_dev / x_dev stay fp64.  Parity is by outer CG iteration count. */
int nnmg_vcycle_set_precision(nnmg_vcycle_t vcycle, int bits);
/* coarse solver the mixed-precision cycle uses instead of the fp64 cycle's
 * (NULL: the same one); the caller keeps it alive while it is attached */
int nnmg_vcycle_set_mixed_coarse(nnmg_vcycle_t vcycle, nnmg_coarse_t coarse);
/* capture the cycle for (f_dev, x_dev) into a CUDA graph and replay it on run */
int nnmg_vcycle_use_graph(nnmg_vcycle_t vcycle, int enable);
/* number of kernels one cycle launches (for graph replays) */
int nnmg_vcycle_kernels_per_cycle(nnmg_vcycle_t vcycle, int64_t* n);

#ifdef __cplusplus
}
#endif

#endif /* NNMG_CUDA_H_ */
