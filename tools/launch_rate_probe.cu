// launch_rate_probe.cu — the floor of back-to-back kernel launches in a CUDA graph: empty
// kernels of 32 CTAs x 256 threads (cfg2's grid), with and without programmatic dependent
// launch, and with a 5 us body, per launch (debug tool).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/launch_rate_probe tools/launch_rate_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void body(long long spin, int trigger) {
  extern __shared__ float smem_probe[];
  if (trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (spin < 0) smem_probe[threadIdx.x] = 0.f;  // (never: keeps the dynamic smem alive)
  const long long t0 = clock64();
  while (clock64() - t0 < spin) {}
}
// a body holding ~120 live registers (a stand-in for fb_tiny's 122)
__global__ void __launch_bounds__(256, 2) body_regs(long long spin, int trigger) {
  if (trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  float r[100];
#pragma unroll
  for (int i = 0; i < 100; ++i) r[i] = (float)(clock() + i);
  const long long t0 = clock64();
  while (clock64() - t0 < spin) {
#pragma unroll
    for (int i = 0; i < 100; ++i) r[i] = r[i] * 1.0001f + r[(i + 1) % 100];
  }
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 100; ++i) acc += r[i];
  if (acc == 12345.f) asm volatile("trap;");
}
int main() {
  {
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, body_regs);
    printf("body_regs: %d registers\n", fa.numRegs);
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    for (long long spin : {0LL, 10000LL}) {
      const int K = 2000;
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
      for (int k = 0; k < K; ++k) {
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(32); cfg.blockDim = dim3(256); cfg.stream = st;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, body_regs, spin, 1);
      }
      cudaStreamEndCapture(st, &g); cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("regs kernel, spin %lld, pdl=1: %.3f us per launch (%s)\n", spin, ms * 1000.f / K,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaFuncSetAttribute(body, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (size_t smem : {(size_t)0, (size_t)48 * 1024, (size_t)92 * 1024})
  for (long long spin : {0LL, 10000LL})
    for (int pdl = 0; pdl < 2; ++pdl) {
      const int K = 2000;
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
      for (int k = 0; k < K; ++k) {
        cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(32); cfg.blockDim = dim3(256); cfg.stream = st;
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = pdl;
        cudaLaunchKernelEx(&cfg, body, spin, pdl);
      }
      cudaStreamEndCapture(st, &g);
      cudaGraphInstantiate(&ge, g, 0);
      cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("smem %zu KB, spin %lld cycles, pdl=%d: %.3f us per launch (%s)\n", smem >> 10, spin, pdl, ms * 1000.f / K,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
