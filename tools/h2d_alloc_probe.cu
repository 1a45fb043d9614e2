// h2d_alloc_probe.cu — H2D / D2H rate of a 1.2 MB (cfg2) payload vs how the pinned host
// buffer was allocated (flags, block size, offset), to choose ts_host_alloc's strategy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/h2d_alloc_probe.cu -o tools/h2d_alloc_probe
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
#include <sys/mman.h>

static float time_copy(void* dst, const void* src, size_t n, cudaMemcpyKind k, cudaStream_t s) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 5; ++w) cudaMemcpyAsync(dst, src, n, k, s);
  cudaEventRecord(e0, s);
  const int reps = 200;
  for (int r = 0; r < reps; ++r) cudaMemcpyAsync(dst, src, n, k, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1000.f / reps;
}

int main() {
  const size_t n = 1228800;
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  void* d;
  cudaMalloc(&d, n);
  struct F { const char* name; unsigned flags; } fl[] = {
      {"Default", cudaHostAllocDefault}, {"Portable", cudaHostAllocPortable},
      {"Mapped", cudaHostAllocMapped}, {"Portable|Mapped", cudaHostAllocPortable | cudaHostAllocMapped},
      {"WriteCombined", cudaHostAllocWriteCombined}};
  for (int rep = 0; rep < 2; ++rep)
    for (auto& f : fl)
      for (size_t blk : {n, (size_t)4 << 20, (size_t)32 << 20, (size_t)256 << 20}) {
        void* h = nullptr;
        if (cudaHostAlloc(&h, blk, f.flags) != cudaSuccess) { printf("alloc fail\n"); continue; }
        memset(h, 1, blk);
        const float a = time_copy(d, h, n, cudaMemcpyHostToDevice, s);
        const float b = time_copy(h, d, n, cudaMemcpyDeviceToHost, s);
        printf("rep %d %-16s block %4zu MB: H2D %6.1f us (%5.1f GB/s)  D2H %6.1f us (%5.1f GB/s)\n", rep, f.name,
               blk >> 20, a, n / a / 1e3, b, n / b / 1e3);
        cudaFreeHost(h);
      }
  // malloc + cudaHostRegister, and mmap + register
  for (size_t blk : {n, (size_t)32 << 20}) {
    void* h = aligned_alloc(4096, (blk + 4095) / 4096 * 4096);
    memset(h, 1, blk);
    cudaHostRegister(h, blk, cudaHostRegisterDefault);
    const float a = time_copy(d, h, n, cudaMemcpyHostToDevice, s);
    const float b = time_copy(h, d, n, cudaMemcpyDeviceToHost, s);
    printf("aligned_alloc+register block %4zu MB: H2D %6.1f us (%5.1f GB/s)  D2H %6.1f us (%5.1f GB/s)\n",
           blk >> 20, a, n / a / 1e3, b, n / b / 1e3);
    cudaHostUnregister(h);
    free(h);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
