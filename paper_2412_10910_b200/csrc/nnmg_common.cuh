// Shared infrastructure for libnnmg_cuda: error reporting, launch counting,
// owned device buffers and compile-time helpers.  sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

namespace nnmg {

// ---------------------------------------------------------------------------
// error state (thread-local message, int status codes mapped in Python)
// ---------------------------------------------------------------------------
enum Status : int {
  kOk = 0,
  kInvalidArgument = 1,  // -> ValueError
  kCudaError = 2,        // -> RuntimeError
  kUnsupported = 3,      // -> NotImplementedError
  kGeometryError = 4,    // -> ValueError (non-positive Jacobian)
  kSearchError = 5,      // -> GeosearchError
  kIndefinite = 6,       // -> IndefiniteOperatorError
};

void set_error(const std::string& msg);
const char* last_error();

struct Error {
  int status;
  std::string msg;
};

#define NNMG_CUDA_TRY(expr)                                                       \
  do {                                                                            \
    cudaError_t _e = (expr);                                                      \
    if (_e != cudaSuccess) {                                                      \
      throw ::nnmg::Error{::nnmg::kCudaError,                                      \
                          std::string(#expr) + ": " + cudaGetErrorString(_e)};    \
    }                                                                             \
  } while (0)

#define NNMG_CHECK_LAUNCH() NNMG_CUDA_TRY(cudaGetLastError())

#define NNMG_REQUIRE(cond, status, msg)                                           \
  do {                                                                            \
    if (!(cond)) throw ::nnmg::Error{(status), (msg)};                            \
  } while (0)

// number of kernels launched by this library (process-wide), so the bench can
// report how many of our kernels ran inside the timed region
void count_launch(int n = 1);
uint64_t launch_count();

// ---------------------------------------------------------------------------
// device buffer owned by a handle
// ---------------------------------------------------------------------------
template <class T>
struct DevBuf {
  T* ptr = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), n(o.n) {
    o.ptr = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      ptr = o.ptr;
      n = o.n;
      o.ptr = nullptr;
      o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void release() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) NNMG_CUDA_TRY(cudaMalloc(&ptr, count * sizeof(T)));
  }
  void upload(const T* host, size_t count) {
    alloc(count);
    if (count) NNMG_CUDA_TRY(cudaMemcpy(ptr, host, count * sizeof(T), cudaMemcpyHostToDevice));
  }
  void upload(const std::vector<T>& v) { upload(v.data(), v.size()); }
  void zero(cudaStream_t s = 0) {
    if (n) NNMG_CUDA_TRY(cudaMemsetAsync(ptr, 0, n * sizeof(T), s));
  }
};

// ---------------------------------------------------------------------------
// compile-time helpers
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }

constexpr int kMaxDegree = 4;
constexpr int kMaxN1 = kMaxDegree + 1;

// 1D tables of the degree-p Lagrange basis on Gauss-Lobatto nodes evaluated at
// the (p+1)-point Gauss-Legendre rule on [0,1] (reference fespace.py:11-71,
// mfoperator.py:33-37).  Stored at max size; kernels read the leading n1 x n1.
struct Tables {
  int n1;
  double S[kMaxN1][kMaxN1];   // S[q][i]  = phi_i(x_q)
  double D[kMaxN1][kMaxN1];   // D[q][i]  = phi_i'(x_q)
  double Dc[kMaxN1][kMaxN1];  // Dc[q][r] = l_r'(x_q), collocation derivative on the Gauss points
  double w[kMaxN1];           // Gauss weights on [0,1]
  double xq[kMaxN1];          // Gauss points on [0,1]
  double nodes[kMaxN1];       // Lobatto nodes on [0,1]
  double denom[kMaxN1];       // prod_{j!=i} (node_i - node_j)
  double rdenom[kMaxN1];      // 1 / denom (multiplications instead of fp64 divisions)
  // fp32 copies for the single-precision arithmetic of the mixed-precision V-cycle
  float S32[kMaxN1][kMaxN1];
  float Dc32[kMaxN1][kMaxN1];
  float nodes32[kMaxN1];
  float rdenom32[kMaxN1];
};

// sweep matrices in the arithmetic type TA
template <class TA>
struct TabSel;
template <>
struct TabSel<double> {
  __host__ __device__ static const double (&S(const Tables& t))[kMaxN1][kMaxN1] { return t.S; }
  __host__ __device__ static const double (&Dc(const Tables& t))[kMaxN1][kMaxN1] { return t.Dc; }
  __host__ __device__ static const double (&nodes(const Tables& t))[kMaxN1] { return t.nodes; }
  __host__ __device__ static const double (&rdenom(const Tables& t))[kMaxN1] { return t.rdenom; }
};
template <>
struct TabSel<float> {
  __host__ __device__ static const float (&S(const Tables& t))[kMaxN1][kMaxN1] { return t.S32; }
  __host__ __device__ static const float (&Dc(const Tables& t))[kMaxN1][kMaxN1] { return t.Dc32; }
  __host__ __device__ static const float (&nodes(const Tables& t))[kMaxN1] { return t.nodes32; }
  __host__ __device__ static const float (&rdenom(const Tables& t))[kMaxN1] { return t.rdenom32; }
};

Tables make_tables(int degree);

}  // namespace nnmg
