// Dissect the per-step latency (debug tool).
#include <cstdio>
#include "../paper_2002_00876_b200/csrc/common.cuh"
using namespace tsb;
__device__ long long g_t[8];
__device__ float g_sink[32];
template <int V>
__global__ void k(int Eb) {
  extern __shared__ __align__(16) float sm[];
  constexpr int CT = 20, TT = CT * CT;
  float* EX = sm; float* RS = EX + Eb * TT; float* vec = RS + Eb * CT; float* pbuf = vec + (Eb + 1) * 32;
  for (int q = threadIdx.x; q < Eb * TT; q += 32) EX[q] = 0.5f + (q % 7) * 0.01f;
  for (int q = threadIdx.x; q < Eb * CT; q += 32) RS[q] = 3.f;
  __syncwarp();
  const int lane = threadIdx.x, jj = lane < CT ? lane : 0;
  float p = lane < 20 ? 0.05f : 0.f;
  long long t0 = clock64();
  for (int t = 0; t < Eb; ++t) {
    const float* Mt = EX + t * TT + jj;
    const float* Wt = RS + t * CT;
    float mv[CT];
#pragma unroll
    for (int i = 0; i < CT; ++i) mv[i] = Mt[i * CT];
    float* pb = pbuf + (t & 1) * 32;
    pb[lane] = p;
    __syncwarp();
    float sa[4] = {0, 0, 0, 0}, Sa[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < CT; i += 4) {
      const float4 q = *reinterpret_cast<const float4*>(pb + i);
      const float4 w = *reinterpret_cast<const float4*>(Wt + i);
      sa[0] = fmaf(q.x, mv[i], sa[0]); sa[1] = fmaf(q.y, mv[i + 1], sa[1]);
      sa[2] = fmaf(q.z, mv[i + 2], sa[2]); sa[3] = fmaf(q.w, mv[i + 3], sa[3]);
      Sa[0] = fmaf(q.x, w.x, Sa[0]); Sa[1] = fmaf(q.y, w.y, Sa[1]);
      Sa[2] = fmaf(q.z, w.z, Sa[2]); Sa[3] = fmaf(q.w, w.w, Sa[3]);
    }
    const float s = (sa[0] + sa[1]) + (sa[2] + sa[3]);
    const float S = (Sa[0] + Sa[1]) + (Sa[2] + Sa[3]);
    float np;
    if (V == 0) np = s * (1.f / S);
    if (V == 1) np = __fdividef(s, S);
    if (V >= 2) {
      np = __fdividef(s, S);
      float nh = lg2(s) - lg2(S);
      if (V >= 3) {
        if (__any_sync(0xffffffffu, !(s >= kGate))) nh = 0.f;
      }
      if (V >= 4) vec[(t + 1) * 32 + lane] = nh;
      else np += nh * 1e-30f;
    }
    p = np;
  }
  long long t1 = clock64();
  if (lane == 0) g_t[V] = t1 - t0;
  g_sink[lane] = p;
}
// pipelined: M column and W for step t+1 loaded into registers during step t
__global__ void kp(int Eb) {
  extern __shared__ __align__(16) float sm[];
  constexpr int CT = 20, TT = CT * CT;
  float* EX = sm; float* RS = EX + Eb * TT; float* vec = RS + Eb * CT; float* pbuf = vec + (Eb + 1) * 32;
  for (int q = threadIdx.x; q < Eb * TT; q += 32) EX[q] = 0.5f + (q % 7) * 0.01f;
  for (int q = threadIdx.x; q < Eb * CT; q += 32) RS[q] = 3.f;
  __syncwarp();
  const int lane = threadIdx.x, jj = lane < CT ? lane : 0;
  float p = lane < 20 ? 0.05f : 0.f;
  float mv[CT], wv[CT];
#pragma unroll
  for (int i = 0; i < CT; ++i) { mv[i] = EX[jj + i * CT]; wv[i] = RS[i]; }
  long long t0 = clock64();
  for (int t = 0; t < Eb; ++t) {
    float* pb = pbuf + (t & 1) * 32;
    pb[lane] = p;
    __syncwarp();
    float pv[CT];
#pragma unroll
    for (int i = 0; i < CT; i += 4) {
      const float4 q = *reinterpret_cast<const float4*>(pb + i);
      pv[i] = q.x; pv[i + 1] = q.y; pv[i + 2] = q.z; pv[i + 3] = q.w;
    }
    const int tn = (t + 1 < Eb) ? t + 1 : t;
    float mn[CT], wn[CT];
#pragma unroll
    for (int i = 0; i < CT; ++i) { mn[i] = EX[tn * TT + jj + i * CT]; }
#pragma unroll
    for (int i = 0; i < CT; i += 4) {
      const float4 w = *reinterpret_cast<const float4*>(RS + tn * CT + i);
      wn[i] = w.x; wn[i + 1] = w.y; wn[i + 2] = w.z; wn[i + 3] = w.w;
    }
    float sa[4] = {0, 0, 0, 0}, Sa[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < CT; i += 4) {
      sa[0] = fmaf(pv[i], mv[i], sa[0]); sa[1] = fmaf(pv[i + 1], mv[i + 1], sa[1]);
      sa[2] = fmaf(pv[i + 2], mv[i + 2], sa[2]); sa[3] = fmaf(pv[i + 3], mv[i + 3], sa[3]);
      Sa[0] = fmaf(pv[i], wv[i], Sa[0]); Sa[1] = fmaf(pv[i + 1], wv[i + 1], Sa[1]);
      Sa[2] = fmaf(pv[i + 2], wv[i + 2], Sa[2]); Sa[3] = fmaf(pv[i + 3], wv[i + 3], Sa[3]);
    }
    const float s = (sa[0] + sa[1]) + (sa[2] + sa[3]);
    const float S = (Sa[0] + Sa[1]) + (Sa[2] + Sa[3]);
    float np = __fdividef(s, S);
    float nh = lg2(s) - lg2(S);
    if (__any_sync(0xffffffffu, !(s >= kGate))) nh = 0.f;
    vec[(t + 1) * 32 + lane] = nh;
    p = np;
#pragma unroll
    for (int i = 0; i < CT; ++i) { mv[i] = mn[i]; wv[i] = wn[i]; }
  }
  long long t1 = clock64();
  if (lane == 0) g_t[5] = t1 - t0;
  g_sink[lane] = p;
}
int main() {
  int Eb = 64; size_t smem = 200 * 1024;
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) {
    k<0><<<1, 32, smem>>>(Eb); k<1><<<1, 32, smem>>>(Eb); k<2><<<1, 32, smem>>>(Eb);
    k<3><<<1, 32, smem>>>(Eb); k<4><<<1, 32, smem>>>(Eb); kp<<<1, 32, smem>>>(Eb);
    cudaDeviceSynchronize();
  }
  long long t[8]; cudaMemcpyFromSymbol(t, g_t, sizeof(t));
  const char* n[] = {"dot + 1/S", "dot + fdividef", "+lg2 x2", "+vote", "+store", "pipelined"};
  for (int v = 0; v < 6; ++v) printf("%-16s %.1f cycles/step\n", n[v], (double)t[v] / Eb);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
