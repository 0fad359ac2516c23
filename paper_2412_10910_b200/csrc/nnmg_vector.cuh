#pragma once

#include "nnmg_common.cuh"

namespace nnmg {

size_t dot_workspace_doubles();
// out[0] = a.b, out[1] = c.d (if c != nullptr); deterministic; out on device
void dot2(int64_t n, const double* a, const double* b, const double* c, const double* d, double* out, double* work,
          cudaStream_t s);
void cheb_start(int64_t n, const double* b, const double* ax, const double* x0, const double* inv_diag, double theta,
                double* r, double* d, double* x, cudaStream_t s);
void cheb_start_t(int64_t n, const double* t, const double* x0, const double* inv_diag, double theta,
                  const double* r, double* d, double* x, cudaStream_t s);
void cheb_step(int64_t n, const double* ad, const double* inv_diag, double c1, double c2, double* r, double* d,
               double* x, cudaStream_t s);
void cheb_init_add(int64_t n, const double* t, const double* inv_diag, double theta, const double* r, double* d,
                   double* x, cudaStream_t s);
void cheb_init(int64_t n, const double* b, const double* x0, const double* inv_diag, double theta, double* r,
               double* d, double* x, cudaStream_t s);
void cheb_update(int64_t n, const double* inv_diag, double c1, double c2, const double* r, double* d, double* x,
                 cudaStream_t s, bool x_is_d = false);
// fp32 storage, fp64 arithmetic (mixed-precision V-cycle)
void cheb_init_add(int64_t n, const float* t, const float* inv_diag, double theta, const float* r, float* d, float* x,
                   cudaStream_t s);
void cheb_init(int64_t n, const float* b, const float* x0, const float* inv_diag, double theta, float* r, float* d,
               float* x, cudaStream_t s);
void cheb_update(int64_t n, const float* inv_diag, double c1, double c2, const float* r, float* d, float* x,
                 cudaStream_t s, bool x_is_d = false);
// halo pack (dst[i] = src[idx[i]]) and unpack (dst[idx[i]] (+)= src[i])
void gather_idx(int64_t n, const int64_t* idx, const double* src, double* dst, cudaStream_t s);
void scatter_idx(int64_t n, const int64_t* idx, const double* src, double* dst, bool add, cudaStream_t s);
void convert(int64_t n, const double* a, float* b, cudaStream_t s);
void convert(int64_t n, const float* a, double* b, cudaStream_t s);
void axpby(int64_t n, double alpha, const double* x, double beta, double* y, cudaStream_t s);
void sub(int64_t n, const double* a, const double* b, double* out, cudaStream_t s);
void mul(int64_t n, const double* a, const double* b, double* out, cudaStream_t s);
void cg_update(int64_t n, double alpha, const double* p, const double* ap, double* x, double* r, cudaStream_t s);

// DFMA throughput of the device in TFLOP/s (roofline denominator for FP64-bound kernels)
double measure_fp64_peak(int device);

}  // namespace nnmg
