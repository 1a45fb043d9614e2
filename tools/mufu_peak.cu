// MUFU (XU pipe) throughput on this B200 ("measure it, do not assume it"):
// every SM, 1024 threads, 8 independent ex2.approx.ftz / lg2.approx.ftz chains per thread.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/mufu_peak tools/mufu_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool EX2>
__global__ void __launch_bounds__(1024) k_mufu(float* out, int iters) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = 0.001f * (threadIdx.x + k);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (EX2)
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[k]));
      else
        asm volatile("lg2.approx.ftz.f32 %0, %0;" : "+f"(x[k]));
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.f) out[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 4096);
  const int iters = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int which = 0; which < 2; ++which) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (which == 0) k_mufu<true><<<sms * 2, 1024>>>(out, iters);
      else k_mufu<false><<<sms * 2, 1024>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)sms * 2 * 1024 * 8 * iters;
      if (rep == 1)
        printf("{\"op\": \"%s\", \"ops_per_s\": %.4e, \"per_sm_per_clk_at_1965MHz\": %.2f, \"ms\": %.3f}\n",
               which == 0 ? "ex2.approx.ftz.f32" : "lg2.approx.ftz.f32", ops / (ms * 1e-3),
               ops / (ms * 1e-3) / sms / 1.965e9, ms);
    }
  }
  return 0;
}
