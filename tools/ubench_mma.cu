// Latency of the cluster scan's pieces on one CTA, plain launch vs cluster launch (debug tool).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -Iinclude -o tools/ubench_mma tools/ubench_mma.cu
#include <cstdio>
#include "../paper_2002_00876_b200/csrc/fb_tiny.cu"
#include "../paper_2002_00876_b200/csrc/fb_cscan.cu"
using namespace tsb;
__device__ long long g_c[16];
__device__ float g_s[512];
template <int C>
__global__ void k_chain(int it) {
  constexpr int MB = cs_mb(C);
  __shared__ __align__(16) float sm[4 * MB + 64];
  for (int q = threadIdx.x; q < 4 * MB; q += blockDim.x) sm[q] = 0.01f * (q % 17) + 0.001f;
  for (int q = 0; q < 4; ++q) if (threadIdx.x == 0) *reinterpret_cast<double*>(sm + q * MB + MB - 4) = 0.5;
  __syncthreads();
  float acc = 0.f;
  long long t0 = clock64();
  for (int i = 0; i < it; ++i) {
    double A;
    acc += cs_chain<true, C>(sm, 0, 3, sm + 4 * MB, threadIdx.x & 31, &A);
    acc += (float)A;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) g_c[0] = t1 - t0;
  g_s[threadIdx.x] = acc;
}
template <int C, int W>
__global__ void k_rows(int it) {  // the summary row chains over 6 tiles, 12 warps
  constexpr int MB = cs_mb(C), TS = 2 * MB;
  extern __shared__ __align__(16) float sm[];
  float* EXF = sm;
  float* msg = sm + 6 * TS;
  float* vb = msg + 2 * MB;
  for (int q = threadIdx.x; q < 6 * TS; q += blockDim.x) sm[q] = 0.05f * (q % 17) + 0.01f;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int bad = 0;
  long long t0 = clock64();
  for (int i = 0; i < it; ++i)
    bad |= __syncthreads_or(cs_summary_rows<C, TS, W>(EXF, msg, msg + MB, vb + 32 * 8 * warp, 6, warp, lane));
  long long t1 = clock64();
  if (threadIdx.x == 0) g_c[1] = t1 - t0;
  g_s[threadIdx.x] = msg[threadIdx.x] + bad;
}
template <typename K, typename... Args>
void launch(K k, int grid, int block, int smem, int cluster, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = cluster > 1 ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, args...);
  cudaDeviceSynchronize();
}
int main() {
  const int it = 64;
  long long c[16];
  const int rs = (6 * 2 * cs_mb(20) + 2 * cs_mb(20) + 12 * 8 * 32) * 4;
  cudaFuncSetAttribute(k_rows<20, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_rows<20, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int cl : {1, 4}) {
    for (int sm : {rs, 190 * 1024}) {
      launch(k_chain<20>, cl, 32, 0, cl, it);
      cudaMemcpyFromSymbol(c, g_c, sizeof(c));
      printf("cluster=%d: chain of 3 steps: %.1f cyc\n", cl, (double)c[0] / it);
      launch(k_rows<20, 4>, cl, 384, sm, cl, it);
      cudaMemcpyFromSymbol(c, g_c, sizeof(c));
      printf("cluster=%d smem=%d: row chains W=4 (6 steps): %.1f cyc\n", cl, sm, (double)c[1] / it);
      launch(k_rows<20, 12>, cl, 384, sm, cl, it);
      cudaMemcpyFromSymbol(c, g_c, sizeof(c));
      printf("cluster=%d smem=%d: row chains W=12 (6 steps): %.1f cyc\n", cl, sm, (double)c[1] / it);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
