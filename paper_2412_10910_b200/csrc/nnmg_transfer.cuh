// Non-nested transfer handle (replaces TwoLevelTransferNonNested,
// transfer.py:61-124) and the GPU point location that builds its records
// (replaces geosearch.locate_points, geosearch.py:163-227).
#pragma once

#include "nnmg_level.cuh"

namespace nnmg {

struct Transfer {
  Level* coarse = nullptr;
  Level* fine = nullptr;
  int dim = 0, pc = 0, ncomp = 1;
  int64_t npts = 0, ncc = 0;
  int chunk = 1;            // coarse cells per warp in the restriction
  int restrict_kernel = -1;  // variant for NLOC*NCOMP <= 32 (see transfer_create; -1: by dimension)
  int restrict_wide = 0;    // 32 < NLOC*NCOMP <= 81: lane-owned local vector instead of staged groups
  int transfer_warps = 0;   // warps (work items / cell chunks) per CTA of the prolongation and the lane restriction (0: 1 in 3D, 4 in 2D)
  bool mixed_arith32 = true;  // fp32 vectors: single-precision arithmetic in the transfer kernels
  int restrict_pl = 1;      // staged restriction: planes of the outermost axis per lane (1, 2)
  int prolong_ppl = 1;      // 2: two points per lane also where one is the default
  DevBuf<int> cell_start;   // [ncc+1] CSR of points by owning coarse cell
  int64_t nitems = 0;       // work items: pieces of a cell's point range (<= NNMG_TRANSFER_MAXP points)
  DevBuf<int> item_pt;      // [nitems+1] point range of each item
  DevBuf<int> item_cell;    // [nitems] owning coarse cell of each item
  DevBuf<int> pt_dof;       // [npts] fine scalar DoF (sorted by cell, then point order)
  DevBuf<double> xhat;      // [npts][dim]
  DevBuf<float> xhat32;     // fp32 copy for the mixed-precision V-cycle (transfer_enable_f32)
  DevBuf<double> cellbuf;   // [nitems][nloc][ncomp] restriction partial local vectors
  DevBuf<int> t_off, t_ent; // coarse DoF -> (cell*nloc + l) entries, fixed order
  DevBuf<int> no_point;     // fine scalar DoFs without a point (zero in P u_c)
  // per-phase timing rows (the reference's timings["evaluate"] /
  // ["gather_scatter"], transfer.py:29, 100-101, 122-123): events around the
  // point-evaluation kernel and around the zero-fill / fixed-order gather;
  // off on the V-cycle path (events cannot be recorded into a graph capture)
  bool timing = false;
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  int ev_eval = 0;          // the evaluation kernel ran between ev[ev_eval] and ev[ev_eval + 1]
  ~Transfer();
};

Transfer* transfer_create(Level* coarse, Level* fine, int64_t npts, const int64_t* point_dofs, const int64_t* cells,
                          const double* xhat);
// u_f = P u_c (accumulate: u_f += P u_c) with symmetric constraint masking (transfer.py:31-44, 87-102)
void transfer_prolongate(Transfer& T, const double* uc, double* uf, bool accumulate, cudaStream_t s);
// r_c = P^T r_f, deterministic two-phase segmented reduction (transfer.py:46-58, 104-124)
void transfer_restrict(Transfer& T, const double* rf, double* rc, cudaStream_t s);
// enable / read the per-phase timers of the last prolongate / restrict call
// (seconds; synchronises on the call's last event)
void transfer_set_timing(Transfer& T, bool on);
void transfer_last_timing(Transfer& T, double* evaluate_s, double* gather_scatter_s);
// mixed-precision V-cycle: fp32 xhat copy, fp32 vectors (fp64 arithmetic)
void transfer_enable_f32(Transfer& T, cudaStream_t s);
void transfer_prolongate_f32(Transfer& T, const float* uc, float* uf, bool accumulate, cudaStream_t s);
void transfer_restrict_f32(Transfer& T, const float* rf, float* rc, cudaStream_t s);

struct LocateResult {
  int n_missing = 0;       // points with no candidate / no converged candidate
  int64_t first_missing = -1;
};

// GPU point location with the reference's semantics: candidates = cells whose
// eps_box-padded bounding box contains the point; damped Newton inversion
// (mesh.py:235-287); first containing candidate in ascending cell order wins;
// otherwise the converged candidate whose clamped image is nearest (ties to the
// lowest cell) and the point is flagged projected.
LocateResult locate_points(int device, int dim, int64_t nv, const double* vertices, int64_t nc, const int64_t* cells,
                           int64_t npts, const double* points, double eps_box, double eps_geo, double eps_ref,
                           int64_t* out_cells, double* out_xhat, uint8_t* out_projected);

}  // namespace nnmg
