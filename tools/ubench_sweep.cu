// Per-step latency of the real tiny_sweep (tiny.cuh) in isolation vs inside fb_tiny (debug).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Iinclude -o tools/ubench_sweep tools/ubench_sweep.cu
#include <cstdio>
#include "../paper_2002_00876_b200/csrc/fb_tiny.cu"
using namespace tsb;
__device__ long long g_c[8];
template <int NREC>
__global__ void __launch_bounds__(384, 1) k(int Eb) {
  extern __shared__ __align__(16) float sm[];
  constexpr int C = 20, RS = tiny_rs(C), TB = (C + 1) * RS;
  float* X = sm;                    // [Eb][TB]
  float* V = X + Eb * TB;           // [Eb+1][32] x 2 (fwd, bwd)
  float* H = V + 2 * (Eb + 1) * 32;
  float* cf = H + 2 * (Eb + 1) * 32;
  float* Tm = cf + Eb + 4;
  uint64_t* nb = reinterpret_cast<uint64_t*>(Tm + Eb + 4);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int q = tid; q < Eb * TB; q += 384) X[q] = 0.02f + 0.001f * (q % 13);
  for (int q = tid; q < Eb; q += 384) Tm[q] = 0.f;
  for (int q = tid; q < 2 * (Eb + 1); q += 384) mbar_init(&nb[q], 1);
  fence_mbar_init();
  __syncthreads();
  const float ones0 = lane < C ? 1.f : (lane == C ? (float)C : 0.f);
  if (warp == 2) {
    long long t0 = clock64();
    tiny_sweep<true, C>(X, X, Tm, V, H, cf, nb, Eb, lane, ones0);
    long long t1 = clock64();
    if (lane == 0) g_c[NREC] = t1 - t0;
  } else if (NREC == 2 && warp == 3) {
    tiny_sweep<false, C>(X, X, Tm, V + (Eb + 1) * 32, H + (Eb + 1) * 32, nullptr, nb + Eb + 1, Eb, lane, ones0);
  }
}
int main() {
  const int Eb = 24;
  const int smem = (Eb * 21 * 20 + 4 * (Eb + 1) * 32 + 2 * Eb + 16) * 4 + 2 * (Eb + 1) * 8 + 64;
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int r = 0; r < 3; ++r) { k<1><<<1, 384, smem>>>(Eb); k<2><<<1, 384, smem>>>(Eb); }
  cudaDeviceSynchronize();
  long long c[8];
  cudaMemcpyFromSymbol(c, g_c, sizeof(c));
  printf("tiny_sweep fwd alone: %.1f cycles/step\n", (double)c[1] / Eb);
  printf("tiny_sweep fwd with bwd concurrently: %.1f cycles/step\n", (double)c[2] / Eb);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
