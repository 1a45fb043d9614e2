// Latency microbenchmarks on the B200 (debug tool): one warp, dependent chains.
#include <cstdio>

__device__ long long g_out[16];
__device__ float g_sink[64];

__global__ void k_lds(int iters) {
  __shared__ float s[64];
  int lane = threadIdx.x;
  s[lane] = 0.f;
  s[lane + 32] = 0.f;
  __syncwarp();
  int idx = lane;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) idx = __float_as_int(s[idx & 63]) + lane;  // dependent LDS
  long long t1 = clock64();
  if (lane == 0) g_out[0] = (t1 - t0);
  g_sink[lane] = idx;
}

__global__ void k_sts_sync_lds(int iters) {
  __shared__ float s[64];
  int lane = threadIdx.x;
  float v = lane;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    s[(i & 1) * 32 + lane] = v;
    __syncwarp();
    float4 q = *reinterpret_cast<float4*>(s + (i & 1) * 32);
    v = q.x + q.y + 1.f;
  }
  long long t1 = clock64();
  if (lane == 0) g_out[1] = (t1 - t0);
  g_sink[lane] = v;
}

__global__ void k_shfl(int iters) {
  int lane = threadIdx.x;
  float v = lane;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = __shfl_sync(0xffffffffu, v, (lane + 1) & 31) + 1.f;
  long long t1 = clock64();
  if (lane == 0) g_out[2] = (t1 - t0);
  g_sink[lane] = v;
}

__global__ void k_mufu(int iters) {
  int lane = threadIdx.x;
  float v = lane + 1.f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    float y;
    asm volatile("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v));
    v = y + 2.f;
  }
  long long t1 = clock64();
  if (lane == 0) g_out[3] = (t1 - t0);
  g_sink[lane] = v;
}

__global__ void k_dadd(int iters) {
  int lane = threadIdx.x;
  double v = lane;
  float f = lane * 0.5f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v += (double)f * 0.69;
  long long t1 = clock64();
  if (lane == 0) g_out[4] = (t1 - t0);
  g_sink[lane] = (float)v;
}

__global__ void k_ffma(int iters) {
  int lane = threadIdx.x;
  float v = lane;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) v = fmaf(v, 0.999f, 0.5f);
  long long t1 = clock64();
  if (lane == 0) g_out[5] = (t1 - t0);
  g_sink[lane] = v;
}

__global__ void k_vote(int iters) {
  int lane = threadIdx.x;
  float v = lane;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (__any_sync(0xffffffffu, v < -1.f)) v = 0.f;
    v = v + 1.f;
  }
  long long t1 = clock64();
  if (lane == 0) g_out[6] = (t1 - t0);
  g_sink[lane] = v;
}

int main() {
  const int it = 1000;
  k_lds<<<1, 32>>>(it);
  k_sts_sync_lds<<<1, 32>>>(it);
  k_shfl<<<1, 32>>>(it);
  k_mufu<<<1, 32>>>(it);
  k_dadd<<<1, 32>>>(it);
  k_ffma<<<1, 32>>>(it);
  k_vote<<<1, 32>>>(it);
  cudaDeviceSynchronize();
  long long o[16];
  cudaMemcpyFromSymbol(o, g_out, sizeof(o));
  const char* n[] = {"LDS dep", "STS+syncwarp+LDS128", "SHFL dep", "MUFU.LG2 dep", "DADD dep",
                     "FFMA dep", "VOTE+FADD"};
  for (int k = 0; k < 7; ++k) printf("%-22s %.1f cycles/iter\n", n[k], (double)o[k] / it);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
