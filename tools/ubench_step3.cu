// Dissect the per-step latency of the sum-normalised sweep (debug tool).
#include <cstdio>
__device__ long long g_t[8];
__device__ float g_sink[32];
template <int V>
__global__ void k(int steps) {
  __shared__ __align__(16) float pbuf[64];
  __shared__ __align__(16) float EX[16 * 400];
  __shared__ __align__(16) float RS[16 * 20];
  const int lane = threadIdx.x;
  for (int q = lane; q < 16 * 400; q += 32) EX[q] = 0.5f + (q % 7) * 0.01f;
  for (int q = lane; q < 16 * 20; q += 32) RS[q] = 3.f;
  __syncwarp();
  float p = lane < 20 ? 0.05f : 0.f;
  long long t0 = clock64();
  for (int t = 0; t < steps; ++t) {
    float* pb = pbuf + (t & 1) * 32;
    pb[lane] = p;
    __syncwarp();
    float q[20];
#pragma unroll
    for (int i = 0; i < 20; i += 4) {
      const float4 v = *reinterpret_cast<const float4*>(pb + i);
      q[i] = v.x; q[i + 1] = v.y; q[i + 2] = v.z; q[i + 3] = v.w;
    }
    if (V == 0) {  // smem round trip + sum tree only
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < 20; ++i) s += q[i];
      p = s * 0.05f;
    } else {
      const float* Mt = EX + (t & 15) * 400 + (lane < 20 ? lane : 0);
      float sa[4] = {0, 0, 0, 0};
#pragma unroll
      for (int i = 0; i < 20; ++i) sa[i & 3] = fmaf(q[i], Mt[i * 20], sa[i & 3]);
      const float s = (sa[0] + sa[1]) + (sa[2] + sa[3]);
      if (V == 1) {
        p = s * 0.05f;
      } else {
        const float* Wt = RS + (t & 15) * 20;
        float Sa[4] = {0, 0, 0, 0};
#pragma unroll
        for (int i = 0; i < 20; ++i) Sa[i & 3] = fmaf(q[i], Wt[i], Sa[i & 3]);
        const float S = (Sa[0] + Sa[1]) + (Sa[2] + Sa[3]);
        if (V == 2) p = s * (1.f / S);
        if (V == 3) p = __fdividef(s, S);
        if (V == 4) {
          float r;
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(S));
          p = s * r;
        }
        if (V == 5) {  // transposed M: lane reads its contiguous column with LDS.128
          const float* MT = EX + (t & 15) * 400 + (lane < 20 ? lane : 0) * 20;
          float sb[4] = {0, 0, 0, 0};
#pragma unroll
          for (int i = 0; i < 20; i += 4) {
            const float4 m = *reinterpret_cast<const float4*>(MT + i);
            sb[0] = fmaf(q[i], m.x, sb[0]); sb[1] = fmaf(q[i + 1], m.y, sb[1]);
            sb[2] = fmaf(q[i + 2], m.z, sb[2]); sb[3] = fmaf(q[i + 3], m.w, sb[3]);
          }
          const float s2 = (sb[0] + sb[1]) + (sb[2] + sb[3]);
          float Sb[4] = {0, 0, 0, 0};
#pragma unroll
          for (int i = 0; i < 20; i += 4) {
            const float4 w = *reinterpret_cast<const float4*>(Wt + i);
            Sb[0] = fmaf(q[i], w.x, Sb[0]); Sb[1] = fmaf(q[i + 1], w.y, Sb[1]);
            Sb[2] = fmaf(q[i + 2], w.z, Sb[2]); Sb[3] = fmaf(q[i + 3], w.w, Sb[3]);
          }
          const float S2 = (Sb[0] + Sb[1]) + (Sb[2] + Sb[3]);
          float r;
          asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(S2));
          p = s2 * r;
        }
      }
    }
  }
  long long t1 = clock64();
  if (lane == 0) g_t[V] = t1 - t0;
  g_sink[lane] = p;
}
int main() {
  const int steps = 256;
  for (int rep = 0; rep < 2; ++rep) {
    k<0><<<1, 32>>>(steps); k<1><<<1, 32>>>(steps); k<2><<<1, 32>>>(steps);
    k<3><<<1, 32>>>(steps); k<4><<<1, 32>>>(steps); k<5><<<1, 32>>>(steps);
    cudaDeviceSynchronize();
  }
  long long t[8];
  cudaMemcpyFromSymbol(t, g_t, sizeof(t));
  const char* n[] = {"smem roundtrip+sum", "+dot (20 LDS, 20 FFMA)", "+rowsum dot, 1/S",
                     "fdividef", "rcp.approx", "transposed M, LDS.128"};
  for (int v = 0; v < 6; ++v) printf("%-26s %.1f cycles/step\n", n[v], (double)t[v] / steps);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
