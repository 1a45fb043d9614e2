// Per-step latency of the small-kernel sweep with 1 warp vs 16 warps per CTA (debug tool).
#include <cstdio>
#include "../paper_2002_00876_b200/csrc/fb_small.cu"
using namespace tsb;
__device__ long long g_t[4];
template <int NT>
__global__ void k(int Eb) {
  extern __shared__ __align__(16) float sm[];
  constexpr int CT = 20, TT = CT * CT;
  float* X = sm; float* EX = X + Eb * TT; float* RS = EX + Eb * TT; float* Tm = RS + Eb * CT;
  float* lS = Tm + Eb; float* vec = lS + Eb + 4; float* pb = vec + (Eb + 1) * 32 + 4;
  pb = (float*)(((uintptr_t)pb + 15) & ~15);
  for (int q = threadIdx.x; q < Eb * TT; q += NT) { X[q] = -((q * 7) % 13) * 0.3f; EX[q] = ex2(X[q]); }
  for (int q = threadIdx.x; q < Eb * CT; q += NT) RS[q] = 3.f;
  for (int q = threadIdx.x; q < Eb; q += NT) Tm[q] = 0.f;
  __syncthreads();
  if (threadIdx.x < 32) {
    double O;
    long long t0 = clock64();
    sweep<true, CT>(X, EX, RS, vec, lS, Tm, Eb, 20, threadIdx.x, &O, pb);
    long long t1 = clock64();
    if (threadIdx.x == 0) { g_t[0] = t1 - t0; g_t[1] = (long long)O; }
  }
  __syncthreads();
}
int main() {
  int Eb = 24; size_t smem = 200 * 1024;
  cudaFuncSetAttribute(k<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long long t[4];
  for (int rep = 0; rep < 2; ++rep) {
    k<32><<<1, 32, smem>>>(Eb); cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(t, g_t, sizeof(t)); printf("1 warp  : %.1f cycles/step\n", (double)t[0] / Eb);
    k<512><<<1, 512, smem>>>(Eb); cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(t, g_t, sizeof(t)); printf("16 warps: %.1f cycles/step\n", (double)t[0] / Eb);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
