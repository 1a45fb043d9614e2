// pcie_probe.cu — host<->device transfer rates on the GPU box: copy engine (1 and 4
// streams) vs SM-driven zero-copy loads/stores of mapped pinned host memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/pcie_probe.cu -o tools/pcie_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void zc_read(const float4* __restrict__ h, float4* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    d[i] = h[i];
}
__global__ void zc_write(const float4* __restrict__ d, float4* __restrict__ h, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    h[i] = d[i];
}

int main() {
  cudaStream_t s[4];
  for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (size_t bytes : {(size_t)1228800, (size_t)64 << 20}) {
    float *h, *h2, *d;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    cudaHostAlloc(&h2, bytes, cudaHostAllocMapped);
    cudaMalloc(&d, bytes);
    for (size_t i = 0; i < bytes / 4; ++i) h[i] = (float)i;
    const int reps = bytes < (8 << 20) ? 200 : 10;
    auto timeit = [&](const char* name, auto fn) {
      for (int w = 0; w < 3; ++w) fn();
      cudaDeviceSynchronize();
      cudaEventRecord(e0, s[0]);
      for (int r = 0; r < reps; ++r) fn();
      for (int k = 1; k < 4; ++k) {
        cudaEvent_t ev;
        cudaEventCreate(&ev);
        cudaEventRecord(ev, s[k]);
        cudaStreamWaitEvent(s[0], ev, 0);
      }
      cudaEventRecord(e1, s[0]);
      cudaDeviceSynchronize();
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%8zu B  %-28s %8.1f us  %6.1f GB/s  (%s)\n", bytes, name, ms * 1e3 / reps,
             bytes / (ms * 1e-3 / reps) / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    timeit("H2D memcpy 1 stream", [&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s[0]); });
    timeit("D2H memcpy 1 stream", [&] { cudaMemcpyAsync(h2, d, bytes, cudaMemcpyDeviceToHost, s[0]); });
    timeit("H2D memcpy 4 streams", [&] {
      for (int k = 0; k < 4; ++k)
        cudaMemcpyAsync((char*)d + k * bytes / 4, (char*)h + k * bytes / 4, bytes / 4,
                        cudaMemcpyHostToDevice, s[k]);
    });
    timeit("H2D+D2H memcpy 2 streams", [&] {
      cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s[0]);
      cudaMemcpyAsync(h2, d, bytes, cudaMemcpyDeviceToHost, s[1]);
    });
    for (int g : {148, 592, 2368}) {
      char nm[64];
      snprintf(nm, 64, "zero-copy read grid %d", g);
      timeit(nm, [&] { zc_read<<<g, 256, 0, s[0]>>>((const float4*)h, (float4*)d, bytes / 16); });
      snprintf(nm, 64, "zero-copy write grid %d", g);
      timeit(nm, [&] { zc_write<<<g, 256, 0, s[0]>>>((const float4*)d, (float4*)h2, bytes / 16); });
    }
    cudaFreeHost(h);
    cudaFreeHost(h2);
    cudaFree(d);
  }
  return 0;
}
