// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput on sm_100a, alone and
// concurrently with DFMA work in the same kernel: does the FP64 tensor path add
// throughput on top of the FP64 FMA pipe?   nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <int MODE>  // 0 DMMA only, 1 DFMA only, 2 both
__global__ void k(double* out, int iters) {
  double acc[4][2] = {};
  double f[8];
  for (int i = 0; i < 8; ++i) f[i] = threadIdx.x * 1e-3 + i;
  const double a = 1.0 + threadIdx.x * 1e-6, b = 0.999;
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1) {
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma(acc[j], a, b);
    }
    if (MODE != 0) {
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] = fma(f[j], 0.999, 1e-3);
    }
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) s += acc[j][0] + acc[j][1];
  for (int j = 0; j < 8; ++j) s += f[j];
  if (s == 1234.5) out[0] = s;
}

template <int MODE>
double run(int sms) {
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 4096, threads = 256, blocks = sms * 8;
  k<MODE><<<blocks, threads>>>(out, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  const double warps = double(blocks) * threads / 32;
  const double dmma_flops = MODE != 1 ? warps * iters * 4 * (8.0 * 8 * 4 * 2) : 0.0;
  const double dfma_flops = MODE != 0 ? double(blocks) * threads * iters * 8 * 2 : 0.0;
  printf("mode %d: %.3f ms  DMMA %.1f TF/s  DFMA %.1f TF/s  total %.1f TF/s\n", MODE, ms,
         dmma_flops / ms / 1e9, dfma_flops / ms / 1e9, (dmma_flops + dfma_flops) / ms / 1e9);
  return ms;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>(sms);
  run<1>(sms);
  run<2>(sms);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
