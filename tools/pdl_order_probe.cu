// pdl_order_probe.cu — does stream order survive a PDL secondary that never waits?  A primary
// kernel triggers its dependents at once, spins ~200 us, then writes a flag; the secondary
// (programmatic stream serialization, no griddepcontrol.wait) exits at once; then a D2H copy
// of the flag and an event.  Prints whether the copy saw the primary's write (debug tool).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/pdl_order_probe tools/pdl_order_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void primary(int* flag, long long spin) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const long long t0 = clock64();
  while (clock64() - t0 < spin) {}
  if (threadIdx.x == 0) *flag = 1;
}
__global__ void secondary(int* out, int wait) {
  if (wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) *out = 2;
}
int main() {
  int *flag, *out, h[2];
  cudaMalloc(&flag, 4); cudaMalloc(&out, 4);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int wait = 0; wait < 2; ++wait)
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemsetAsync(flag, 0, 4, st); cudaMemsetAsync(out, 0, 4, st);
      primary<<<1, 32, 0, st>>>(flag, 400000);
      cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(1); cfg.blockDim = dim3(32); cfg.stream = st;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, secondary, out, wait);
      cudaMemcpyAsync(&h[0], flag, 4, cudaMemcpyDeviceToHost, st);
      cudaMemcpyAsync(&h[1], out, 4, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      printf("secondary waits=%d: copy after the secondary saw primary flag=%d, secondary out=%d  %s\n", wait, h[0], h[1],
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
