// K5/K8 vector kernels: fused Chebyshev-Jacobi updates (solvers.py:88-108),
// CG updates (solvers.py:129-164) and deterministic two-stage dot products.
#include "nnmg_vector.cuh"

#include <algorithm>

namespace nnmg {

static constexpr int kBS = 256;
static inline unsigned grid_for(int64_t n) { return static_cast<unsigned>((n + kBS - 1) / kBS); }

// r = b - Ax (or b); d = inv_diag*r/theta; x = x0 + d (or d)       (solvers.py:94-100)
__global__ void k_cheb_start(int64_t n, const double* b, const double* __restrict__ ax,
                             const double* x0, const double* __restrict__ inv_diag, double theta,
                             double* r, double* __restrict__ d, double* x) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  // b == nullptr: r already holds the residual (the in-place form r -= A x0)
  const double ri = b ? (ax ? b[i] - ax[i] : b[i]) : r[i];
  const double di = inv_diag[i] * ri / theta;
  if (b) r[i] = ri;
  d[i] = di;
  x[i] = x0 ? x0[i] + di : di;
}

// r already holds b - A (x0 + t): d = inv_diag*r/theta; x = (x0 + t) + d (the first
// post-smoothing sweep right after the prolongation, multigrid.py:107-111)
__global__ void k_cheb_start_t(int64_t n, const double* __restrict__ t, const double* x0,
                               const double* __restrict__ inv_diag, double theta, const double* __restrict__ r,
                               double* __restrict__ d, double* x) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double di = inv_diag[i] * r[i] / theta;
  d[i] = di;
  x[i] = (x0[i] + t[i]) + di;
}

// r -= Ad; z = inv_diag r; d = c1 d + c2 z; x += d                 (solvers.py:101-107)
__global__ void k_cheb_step(int64_t n, const double* __restrict__ ad, const double* __restrict__ inv_diag,
                            double c1, double c2, double* __restrict__ r, double* __restrict__ d,
                            double* __restrict__ x) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  // ad == nullptr: the apply already subtracted A d from r in place
  const double ri = ad ? r[i] - ad[i] : r[i];
  const double z = inv_diag[i] * ri;
  const double di = c1 * d[i] + c2 * z;
  if (ad) r[i] = ri;
  d[i] = di;
  x[i] += di;
}

// fp32 vectors, four entries per thread (16-byte loads / stores; one entry
// per thread moves 128 bytes per warp instruction and measured 4.7 TB/s on
// C3 against 6.9 TB/s for the fp64 kernel).  Single-precision arithmetic.
// Thread i < n4 handles entries 4 i .. 4 i + 3, the first n - 4 n4 threads
// also one tail entry.  All pointers 16-byte aligned (checked by the caller).
__device__ __forceinline__ float4 ld4(const float* p, int64_t i) { return reinterpret_cast<const float4*>(p)[i]; }
__device__ __forceinline__ void st4(float* p, int64_t i, float4 v) { reinterpret_cast<float4*>(p)[i] = v; }

__global__ void k_cheb_update_f4(int64_t n4, int64_t n, const float* __restrict__ inv_diag, float c1, float c2,
                                 const float* __restrict__ r, float* __restrict__ d, float* __restrict__ x,
                                 int x_is_d) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  auto one = [&](float di_old, float id, float ri, float xi, float& dn, float& xn) {
    dn = c1 * di_old + c2 * (id * ri);
    xn = (x_is_d ? di_old : xi) + dn;
  };
  if (i < n4) {
    const float4 id = ld4(inv_diag, i), rr = ld4(r, i), dd = ld4(d, i);
    float4 xx = x_is_d ? dd : ld4(x, i);
    float4 dn, xn;
    one(dd.x, id.x, rr.x, xx.x, dn.x, xn.x);
    one(dd.y, id.y, rr.y, xx.y, dn.y, xn.y);
    one(dd.z, id.z, rr.z, xx.z, dn.z, xn.z);
    one(dd.w, id.w, rr.w, xx.w, dn.w, xn.w);
    st4(d, i, dn);
    st4(x, i, xn);
  }
  const int64_t j = 4 * n4 + i;
  if (i < n - 4 * n4) {
    const float dold = d[j];
    float dn, xn;
    one(dold, inv_diag[j], r[j], x_is_d ? dold : x[j], dn, xn);
    d[j] = dn;
    x[j] = xn;
  }
}

// x0 == nullptr: r = b, d = inv_diag b / theta, x = d (if x); else r holds b - A x0: d = inv_diag r / theta, x = x0 + d
__global__ void k_cheb_init_f4(int64_t n4, int64_t n, const float* __restrict__ b, const float* x0,
                               const float* __restrict__ inv_diag, float rtheta, float* __restrict__ r,
                               float* __restrict__ d, float* x) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n4) {
    const float4 id = ld4(inv_diag, i);
    float4 ri;
    if (x0) {
      ri = ld4(r, i);
    } else {
      ri = ld4(b, i);
      st4(r, i, ri);
    }
    const float4 di = make_float4(id.x * ri.x * rtheta, id.y * ri.y * rtheta, id.z * ri.z * rtheta,
                                  id.w * ri.w * rtheta);
    st4(d, i, di);
    if (x) {
      if (x0) {
        const float4 xo = ld4(x0, i);
        st4(x, i, make_float4(xo.x + di.x, xo.y + di.y, xo.z + di.z, xo.w + di.w));
      } else {
        st4(x, i, di);
      }
    }
  }
  const int64_t j = 4 * n4 + i;
  if (i < n - 4 * n4) {
    float ri;
    if (x0) {
      ri = r[j];
    } else {
      ri = b[j];
      r[j] = ri;
    }
    const float di = inv_diag[j] * ri * rtheta;
    d[j] = di;
    if (x) x[j] = x0 ? x0[j] + di : di;
  }
}

// r holds f - A (x + t): d = inv_diag r / theta, x = (x + t) + d
__global__ void k_cheb_init_add_f4(int64_t n4, int64_t n, const float* __restrict__ t,
                                   const float* __restrict__ inv_diag, float rtheta, const float* __restrict__ r,
                                   float* __restrict__ d, float* __restrict__ x) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n4) {
    const float4 id = ld4(inv_diag, i), ri = ld4(r, i), tt = ld4(t, i), xx = ld4(x, i);
    const float4 di = make_float4(id.x * ri.x * rtheta, id.y * ri.y * rtheta, id.z * ri.z * rtheta,
                                  id.w * ri.w * rtheta);
    st4(d, i, di);
    st4(x, i, make_float4((xx.x + tt.x) + di.x, (xx.y + tt.y) + di.y, (xx.z + tt.z) + di.z, (xx.w + tt.w) + di.w));
  }
  const int64_t j = 4 * n4 + i;
  if (i < n - 4 * n4) {
    const float di = inv_diag[j] * r[j] * rtheta;
    d[j] = di;
    x[j] = (x[j] + t[j]) + di;
  }
}

static inline bool aligned16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
// NNMG_MIXED_ARITH=64 keeps the scalar kernels (fp64 arithmetic on the fp32 storage)
static bool vec_f32() {
  static const bool on = [] {
    const char* e = getenv("NNMG_MIXED_ARITH");
    return !(e && atoi(e) == 64);
  }();
  return on;
}

// In-place residual form: the apply scatters -A d straight into r.
// x0 == nullptr: r = b, d = inv_diag*b/theta, x = d
// otherwise r already holds b - A x0: d = inv_diag*r/theta, x = x0 + d
// T: vector storage (double; float in the mixed-precision V-cycle, fp64
// arithmetic on fp32 storage)
template <class T>
__global__ void k_cheb_init(int64_t n, const T* __restrict__ b, const T* x0, const T* __restrict__ inv_diag,
                            double theta, T* __restrict__ r, T* __restrict__ d, T* x) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ri;
  if (x0) {
    ri = r[i];
  } else {
    ri = b[i];
    r[i] = T(ri);
  }
  const double di = double(inv_diag[i]) * ri / theta;
  d[i] = T(di);
  if (x) x[i] = T(x0 ? double(x0[i]) + di : di);  // x == nullptr: x = d is left to the first update
}

// post-smoothing start from the pre-smoothing residual: r already holds
// f - A (x + t) (t = the prolongated correction, not yet added to x):
// d = inv_diag*r/theta; x = (x + t) + d, the same roundings as x += t
// followed by k_cheb_init
template <class T>
__global__ void k_cheb_init_add(int64_t n, const T* __restrict__ t, const T* __restrict__ inv_diag, double theta,
                                const T* __restrict__ r, T* __restrict__ d, T* __restrict__ x) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double di = double(inv_diag[i]) * double(r[i]) / theta;
  d[i] = T(di);
  if constexpr (sizeof(T) == sizeof(double))
    x[i] = (x[i] + t[i]) + di;
  else
    x[i] = T((double(x[i]) + double(t[i])) + di);
}

template <class T>
void cheb_init_add_t(int64_t n, const T* t, const T* inv_diag, double theta, const T* r, T* d, T* x, cudaStream_t s) {
  if (!n) return;
  k_cheb_init_add<T><<<grid_for(n), kBS, 0, s>>>(n, t, inv_diag, theta, r, d, x);
  NNMG_CHECK_LAUNCH();
  count_launch();
}
void cheb_init_add(int64_t n, const double* t, const double* inv_diag, double theta, const double* r, double* d,
                   double* x, cudaStream_t s) {
  cheb_init_add_t(n, t, inv_diag, theta, r, d, x, s);
}
void cheb_init_add(int64_t n, const float* t, const float* inv_diag, double theta, const float* r, float* d,
                   float* x, cudaStream_t s) {
  if (n && vec_f32() && aligned16(t) && aligned16(inv_diag) && aligned16(r) && aligned16(d) && aligned16(x)) {
    const int64_t n4 = n / 4;
    k_cheb_init_add_f4<<<grid_for(n4 + 1), kBS, 0, s>>>(n4, n, t, inv_diag, float(1.0 / theta), r, d, x);
    NNMG_CHECK_LAUNCH();
    count_launch();
    return;
  }
  cheb_init_add_t(n, t, inv_diag, theta, r, d, x, s);
}

// r already holds r - A d: d = c1 d + c2 inv_diag r; x += d
// (x_is_d: x was never written and equals the old d, so x = d_old + d_new:
// the same rounding, one vector read and one write fewer)
template <class T>
__global__ void k_cheb_update(int64_t n, const T* __restrict__ inv_diag, double c1, double c2,
                              const T* __restrict__ r, T* __restrict__ d, T* __restrict__ x, int x_is_d) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double dold = d[i];
  const double di = c1 * dold + c2 * (double(inv_diag[i]) * double(r[i]));
  d[i] = T(di);
  x[i] = T((x_is_d ? dold : double(x[i])) + di);
}

template <class T>
void cheb_init_t(int64_t n, const T* b, const T* x0, const T* inv_diag, double theta, T* r, T* d, T* x,
                 cudaStream_t s) {
  if (!n) return;
  k_cheb_init<T><<<grid_for(n), kBS, 0, s>>>(n, b, x0, inv_diag, theta, r, d, x);
  NNMG_CHECK_LAUNCH();
  count_launch();
}
void cheb_init(int64_t n, const double* b, const double* x0, const double* inv_diag, double theta, double* r,
               double* d, double* x, cudaStream_t s) {
  cheb_init_t(n, b, x0, inv_diag, theta, r, d, x, s);
}
void cheb_init(int64_t n, const float* b, const float* x0, const float* inv_diag, double theta, float* r, float* d,
               float* x, cudaStream_t s) {
  if (n && vec_f32() && aligned16(b) && aligned16(x0) && aligned16(inv_diag) && aligned16(r) && aligned16(d) &&
      aligned16(x)) {
    const int64_t n4 = n / 4;
    k_cheb_init_f4<<<grid_for(n4 + 1), kBS, 0, s>>>(n4, n, b, x0, inv_diag, float(1.0 / theta), r, d, x);
    NNMG_CHECK_LAUNCH();
    count_launch();
    return;
  }
  cheb_init_t(n, b, x0, inv_diag, theta, r, d, x, s);
}

template <class T>
void cheb_update_t(int64_t n, const T* inv_diag, double c1, double c2, const T* r, T* d, T* x, cudaStream_t s,
                   bool x_is_d) {
  if (!n) return;
  k_cheb_update<T><<<grid_for(n), kBS, 0, s>>>(n, inv_diag, c1, c2, r, d, x, x_is_d ? 1 : 0);
  NNMG_CHECK_LAUNCH();
  count_launch();
}
void cheb_update(int64_t n, const double* inv_diag, double c1, double c2, const double* r, double* d, double* x,
                 cudaStream_t s, bool x_is_d) {
  cheb_update_t(n, inv_diag, c1, c2, r, d, x, s, x_is_d);
}
void cheb_update(int64_t n, const float* inv_diag, double c1, double c2, const float* r, float* d, float* x,
                 cudaStream_t s, bool x_is_d) {
  if (n && vec_f32() && aligned16(inv_diag) && aligned16(r) && aligned16(d) && aligned16(x)) {
    const int64_t n4 = n / 4;
    k_cheb_update_f4<<<grid_for(n4 + 1), kBS, 0, s>>>(n4, n, inv_diag, float(c1), float(c2), r, d, x, x_is_d ? 1 : 0);
    NNMG_CHECK_LAUNCH();
    count_launch();
    return;
  }
  cheb_update_t(n, inv_diag, c1, c2, r, d, x, s, x_is_d);
}

// K9 halo pack / unpack of the distributed levels: pack the
// listed entries of a local vector into a contiguous send buffer, unpack a
// receive buffer into the listed entries (copy for ghost import, add for the
// export of ghost partial sums).  The indices of one list are distinct, so
// the unpack has no write conflicts; lists of different peers are applied in
// a fixed peer order by the caller.
__global__ void k_gather_idx(int64_t n, const int64_t* __restrict__ idx, const double* __restrict__ src,
                             double* __restrict__ dst) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[idx[i]];
}
__global__ void k_scatter_idx(int64_t n, const int64_t* __restrict__ idx, const double* __restrict__ src,
                              double* __restrict__ dst, int add) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t j = idx[i];
  dst[j] = add ? dst[j] + src[i] : src[i];
}
void gather_idx(int64_t n, const int64_t* idx, const double* src, double* dst, cudaStream_t s) {
  if (!n) return;
  k_gather_idx<<<grid_for(n), kBS, 0, s>>>(n, idx, src, dst);
  NNMG_CHECK_LAUNCH();
  count_launch();
}
void scatter_idx(int64_t n, const int64_t* idx, const double* src, double* dst, bool add, cudaStream_t s) {
  if (!n) return;
  k_scatter_idx<<<grid_for(n), kBS, 0, s>>>(n, idx, src, dst, add ? 1 : 0);
  NNMG_CHECK_LAUNCH();
  count_launch();
}

// precision conversion at the mixed-precision V-cycle's boundaries
template <class A, class B>
__global__ void k_convert(int64_t n, const A* __restrict__ a, B* __restrict__ b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) b[i] = B(a[i]);
}
template <class A, class B>
void convert_t(int64_t n, const A* a, B* b, cudaStream_t s) {
  if (!n) return;
  k_convert<A, B><<<grid_for(n), kBS, 0, s>>>(n, a, b);
  NNMG_CHECK_LAUNCH();
  count_launch();
}
// four entries per thread (16-byte accesses on the fp32 side, 2 x 16 on the fp64 side)
__global__ void k_convert_d2f4(int64_t n4, int64_t n, const double* __restrict__ a, float* __restrict__ b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n4) {
    const double2 lo = reinterpret_cast<const double2*>(a)[2 * i], hi = reinterpret_cast<const double2*>(a)[2 * i + 1];
    reinterpret_cast<float4*>(b)[i] = make_float4(float(lo.x), float(lo.y), float(hi.x), float(hi.y));
  }
  if (i < n - 4 * n4) b[4 * n4 + i] = float(a[4 * n4 + i]);
}
__global__ void k_convert_f2d4(int64_t n4, int64_t n, const float* __restrict__ a, double* __restrict__ b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n4) {
    const float4 v = reinterpret_cast<const float4*>(a)[i];
    reinterpret_cast<double2*>(b)[2 * i] = make_double2(double(v.x), double(v.y));
    reinterpret_cast<double2*>(b)[2 * i + 1] = make_double2(double(v.z), double(v.w));
  }
  if (i < n - 4 * n4) b[4 * n4 + i] = double(a[4 * n4 + i]);
}
void convert(int64_t n, const double* a, float* b, cudaStream_t s) {
  if (n && aligned16(a) && aligned16(b)) {
    k_convert_d2f4<<<grid_for(n / 4 + 1), kBS, 0, s>>>(n / 4, n, a, b);
    NNMG_CHECK_LAUNCH();
    count_launch();
    return;
  }
  convert_t(n, a, b, s);
}
void convert(int64_t n, const float* a, double* b, cudaStream_t s) {
  if (n && aligned16(a) && aligned16(b)) {
    k_convert_f2d4<<<grid_for(n / 4 + 1), kBS, 0, s>>>(n / 4, n, a, b);
    NNMG_CHECK_LAUNCH();
    count_launch();
    return;
  }
  convert_t(n, a, b, s);
}

// y = alpha*x + beta*y  (general axpby; beta==0 ignores y's content)
__global__ void k_axpby(int64_t n, double alpha, const double* __restrict__ x, double beta, double* __restrict__ y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  y[i] = beta == 0.0 ? alpha * x[i] : alpha * x[i] + beta * y[i];
}

// out = a - b
__global__ void k_sub(int64_t n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] - b[i];
}

// out = a * b
__global__ void k_mul(int64_t n, const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] * b[i];
}

// x += alpha p; r -= alpha ap                                      (solvers.py:153-154)
__global__ void k_cg_update(int64_t n, double alpha, const double* __restrict__ p, const double* __restrict__ ap,
                            double* __restrict__ x, double* __restrict__ r) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  x[i] = x[i] + alpha * p[i];
  r[i] = r[i] - alpha * ap[i];
}

// ---------------------------------------------------------------------------
// deterministic dots: fixed grid, fixed per-thread order, fixed tree.
// ---------------------------------------------------------------------------
static constexpr int kDotBlocks = 296;

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += sh[i];
  __syncthreads();
  return s;
}

__global__ void k_dot_partial(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                              const double* __restrict__ c, const double* __restrict__ d, double* __restrict__ part) {
  __shared__ double sh[32];
  double s0 = 0.0, s1 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    s0 += a[i] * b[i];
    if (c) s1 += c[i] * d[i];
  }
  s0 = block_sum(s0, sh);
  s1 = c ? block_sum(s1, sh) : 0.0;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s0;
    part[gridDim.x + blockIdx.x] = s1;
  }
}

__global__ void k_dot_final(const double* __restrict__ part, int nb, double* __restrict__ out, int two) {
  __shared__ double sh[32];
  double s0 = 0.0, s1 = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    s0 += part[i];
    s1 += part[nb + i];
  }
  s0 = block_sum(s0, sh);
  s1 = two ? block_sum(s1, sh) : 0.0;
  if (threadIdx.x == 0) {
    out[0] = s0;
    if (two) out[1] = s1;
  }
}

size_t dot_workspace_doubles() { return 2 * kDotBlocks; }

void dot2(int64_t n, const double* a, const double* b, const double* c, const double* d, double* out,
          double* work, cudaStream_t s) {
  k_dot_partial<<<kDotBlocks, kBS, 0, s>>>(n, a, b, c, d, work);
  NNMG_CHECK_LAUNCH();
  k_dot_final<<<1, kBS, 0, s>>>(work, kDotBlocks, out, c ? 1 : 0);
  NNMG_CHECK_LAUNCH();
  count_launch(2);
}

void cheb_start(int64_t n, const double* b, const double* ax, const double* x0, const double* inv_diag, double theta,
                double* r, double* d, double* x, cudaStream_t s) {
  if (!n) return;
  k_cheb_start<<<grid_for(n), kBS, 0, s>>>(n, b, ax, x0, inv_diag, theta, r, d, x);
  NNMG_CHECK_LAUNCH();
  count_launch();
}

void cheb_start_t(int64_t n, const double* t, const double* x0, const double* inv_diag, double theta,
                  const double* r, double* d, double* x, cudaStream_t s) {
  if (!n) return;
  k_cheb_start_t<<<grid_for(n), kBS, 0, s>>>(n, t, x0, inv_diag, theta, r, d, x);
  NNMG_CHECK_LAUNCH();
  count_launch();
}

void cheb_step(int64_t n, const double* ad, const double* inv_diag, double c1, double c2, double* r, double* d,
               double* x, cudaStream_t s) {
  if (!n) return;
  k_cheb_step<<<grid_for(n), kBS, 0, s>>>(n, ad, inv_diag, c1, c2, r, d, x);
  NNMG_CHECK_LAUNCH();
  count_launch();
}

void axpby(int64_t n, double alpha, const double* x, double beta, double* y, cudaStream_t s) {
  if (!n) return;
  k_axpby<<<grid_for(n), kBS, 0, s>>>(n, alpha, x, beta, y);
  NNMG_CHECK_LAUNCH();
  count_launch();
}

void sub(int64_t n, const double* a, const double* b, double* out, cudaStream_t s) {
  if (!n) return;
  k_sub<<<grid_for(n), kBS, 0, s>>>(n, a, b, out);
  NNMG_CHECK_LAUNCH();
  count_launch();
}

void mul(int64_t n, const double* a, const double* b, double* out, cudaStream_t s) {
  if (!n) return;
  k_mul<<<grid_for(n), kBS, 0, s>>>(n, a, b, out);
  NNMG_CHECK_LAUNCH();
  count_launch();
}

void cg_update(int64_t n, double alpha, const double* p, const double* ap, double* x, double* r, cudaStream_t s) {
  if (!n) return;
  k_cg_update<<<grid_for(n), kBS, 0, s>>>(n, alpha, p, ap, x, r);
  NNMG_CHECK_LAUNCH();
  count_launch();
}

}  // namespace nnmg

// ---------------------------------------------------------------------------
// FP64 roofline denominator: dependent-chain-free DFMA throughput (8
// independent chains per thread, 16 warps per SM), timed with CUDA events.
// MEASURED_PEAKS.json carries no FP64 figure; bench.py reports this one.
// ---------------------------------------------------------------------------
namespace nnmg {

__global__ void k_dfma_probe(double* out, int iters, double b, double c) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

// FP64 tensor-core probe (mma.sync m8n8k4 f64, SASS DMMA): 4 independent
// accumulator chains per warp.  DMMA and DFMA share one FP64 budget on B200
// (profiles/r1_dmma_probe.txt); the larger of the two is the FP64 roof.
__global__ void k_dmma_probe(double* out, int iters) {
  double acc[4][2] = {};
  const double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[j][0]), "+d"(acc[j][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += acc[j][0] + acc[j][1];
  if (s == 12345.678) out[0] = s;
}

static double time_dmma(int sms, double* out) {
  const int threads = 256, blocks = sms * 8, iters = 4096;
  cudaEvent_t e0, e1;
  NNMG_CUDA_TRY(cudaEventCreate(&e0));
  NNMG_CUDA_TRY(cudaEventCreate(&e1));
  k_dmma_probe<<<blocks, threads>>>(out, 16);
  NNMG_CUDA_TRY(cudaEventRecord(e0));
  k_dmma_probe<<<blocks, threads>>>(out, iters);
  NNMG_CUDA_TRY(cudaEventRecord(e1));
  NNMG_CUDA_TRY(cudaEventSynchronize(e1));
  NNMG_CHECK_LAUNCH();
  count_launch(2);
  float ms = 0.f;
  NNMG_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double warps = double(blocks) * threads / 32;
  return warps * iters * 4 * (8.0 * 8 * 4 * 2) / (ms * 1e-3) / 1e12;
}

double measure_fp64_peak(int device) {
  NNMG_CUDA_TRY(cudaSetDevice(device));
  int sms = 0;
  NNMG_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  DevBuf<double> out;
  out.alloc(1);
  const int threads = 512, blocks = sms * 4, iters = 4096;
  cudaEvent_t e0, e1;
  NNMG_CUDA_TRY(cudaEventCreate(&e0));
  NNMG_CUDA_TRY(cudaEventCreate(&e1));
  k_dfma_probe<<<blocks, threads>>>(out.ptr, 64, 0.999, 1e-3);  // warm-up
  NNMG_CUDA_TRY(cudaEventRecord(e0));
  k_dfma_probe<<<blocks, threads>>>(out.ptr, iters, 0.999, 1e-3);
  NNMG_CUDA_TRY(cudaEventRecord(e1));
  NNMG_CUDA_TRY(cudaEventSynchronize(e1));
  NNMG_CHECK_LAUNCH();
  count_launch(2);
  float ms = 0.f;
  NNMG_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double flops = 2.0 * 8.0 * iters * double(threads) * blocks;
  const double dfma = flops / (ms * 1e-3) / 1e12;
  return std::max(dfma, time_dmma(sms, out.ptr));
}

}  // namespace nnmg
