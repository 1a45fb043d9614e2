// Per-step latency of the fb_tiny recursion loop, dissected (debug tool).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Iinclude -o tools/ubench_rec tools/ubench_rec.cu
// One recursion warp (warp 2 of a 384-thread CTA) runs STEPS steps of u_{t+1} = (u_t EX_t) / U_t
// over 24 cyclically reused 20x20 tiles; template flags switch parts of the loop off.
#include <cstdio>

#include "../paper_2002_00876_b200/csrc/common.cuh"
using namespace tsb;

__device__ long long g_cyc[64];
__device__ float g_sink[32];

constexpr int C = 20, RS = 20, TB = (C + 1) * RS, NT = 24, STEPS = 240;

__device__ __forceinline__ float rcpa(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// VOTE: one-step-late any() gate vote; PUB: mbarrier arrive per step; PRE: next row prefetched
// into registers; SLEEPERS: other warps poll an mbarrier with nanosleep meanwhile
template <bool VOTE, bool PUB, bool PRE, bool SLEEPERS, int VID, bool TWO = false, bool STG = false, int SL = 0>
__global__ void __launch_bounds__(384, 1) k() {
  extern __shared__ __align__(16) float sm[];
  float* X = sm;                    // [NT][TB]
  float* V = X + NT * TB;           // [STEPS+1][32]
  uint64_t* nb = reinterpret_cast<uint64_t*>(V + 2 * (STEPS + 1) * 32);  // [STEPS+1]
  uint64_t* stop = nb + 2 * (STEPS + 1);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int q = tid; q < NT * TB; q += 384) X[q] = 0.02f + 0.001f * (q % 13);
  for (int q = tid; q < 2 * (STEPS + 1) + 1; q += 384) mbar_init(&nb[q], 1);
  fence_mbar_init();
  __syncthreads();
  if (warp == 2 || (TWO && warp == 3)) {
    const bool act = lane < C, live = lane <= C;
    const int row = live ? lane : 0;
    V[(warp == 3 ? (STEPS + 1) * 32 : 0) + lane] = act ? 1.f : (lane == C ? (float)C : 0.f);
    __syncwarp();
    float m[C], mn[C];
    const float* mp = X + row * RS;
    const float* u = V + (warp == 3 ? (STEPS + 1) * 32 : 0);
    uint64_t* np = nb + (warp == 3 ? STEPS + 1 : 0);
#pragma unroll
    for (int q = 0; q < C / 4; ++q) {
      const float4 w = *reinterpret_cast<const float4*>(mp + 4 * q);
      m[4 * q] = w.x; m[4 * q + 1] = w.y; m[4 * q + 2] = w.z; m[4 * q + 3] = w.w;
    }
    bool prev_bad = false;
    long long t0 = clock64();
    int tile = 0;
    for (int k = 0; k < STEPS; ++k) {
      float4 x[C / 4];
#pragma unroll
      for (int q = 0; q < C / 4; ++q) x[q] = *reinterpret_cast<const float4*>(u + 4 * q);
      const float U = u[C];
      if (VOTE && k > 0) {
        if (__any_sync(0xffffffffu, prev_bad)) break;
      }
      if (PUB && k > 0 && lane == 0) mbar_arrive(np);
      const int ntile = tile + 1 == NT ? 0 : tile + 1;
      if (PRE) {
        const float* mq = X + ntile * TB + row * RS;
#pragma unroll
        for (int q = 0; q < C / 4; ++q) {
          const float4 w = *reinterpret_cast<const float4*>(mq + 4 * q);
          mn[4 * q] = w.x; mn[4 * q + 1] = w.y; mn[4 * q + 2] = w.z; mn[4 * q + 3] = w.w;
        }
      } else {
        const float* mq = X + tile * TB + row * RS;
#pragma unroll
        for (int q = 0; q < C / 4; ++q) {
          const float4 w = *reinterpret_cast<const float4*>(mq + 4 * q);
          m[4 * q] = w.x; m[4 * q + 1] = w.y; m[4 * q + 2] = w.z; m[4 * q + 3] = w.w;
        }
      }
      const float r = rcpa(U);
      float sa[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int q = 0; q < C / 4; ++q) {
        sa[0] = fmaf(x[q].x, m[4 * q], sa[0]);
        sa[1] = fmaf(x[q].y, m[4 * q + 1], sa[1]);
        sa[2] = fmaf(x[q].z, m[4 * q + 2], sa[2]);
        sa[3] = fmaf(x[q].w, m[4 * q + 3], sa[3]);
      }
      const float un = ((sa[0] + sa[1]) + (sa[2] + sa[3])) * r;
      const_cast<float*>(u)[32 + lane] = live ? un : 0.f;
      prev_bad = live && !(un >= kGate);
      if (PRE) {
#pragma unroll
        for (int i = 0; i < C; ++i) m[i] = mn[i];
      }
      u += 32;
      np += 1;
      tile = ntile;
#ifdef NOSTG
#else
      if (STG && lane == 0 && blockIdx.x == 0 && k < 64) g_cyc[32 + (k & 31)] = clock64();
#endif
      __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0 && warp == 2) {
      g_cyc[VID] = t1 - t0;
      mbar_arrive(stop);
    }
    g_sink[lane] = u[lane];
  } else if (SLEEPERS) {
    if (SL == 0) mbar_wait_sleep(stop, 0, 64);
    if (SL == 1) mbar_wait_sleep(&nb[12 + (warp % 10)], 0, 64);
    if (SL == 2) mbar_wait(&nb[12 + (warp % 10)], 0);
    if (SL == 3) mbar_wait_sleep(&nb[200], 0, 64);
  }
}

template <bool VOTE, bool PUB, bool PRE, bool SLEEPERS, int VID, bool TWO = false, bool STG = false, int SL = 0>
void run() {
  const int smem = (NT * TB + 2 * (STEPS + 1) * 32) * 4 + (2 * STEPS + 8) * 8;
  cudaFuncSetAttribute(k<VOTE, PUB, PRE, SLEEPERS, VID, TWO, STG, SL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int r = 0; r < 3; ++r) k<VOTE, PUB, PRE, SLEEPERS, VID, TWO, STG, SL><<<1, 384, smem>>>();
}

int main() {
  run<true, true, true, true, 0>();
  run<true, true, true, false, 1>();
  run<false, true, true, false, 2>();
  run<false, false, true, false, 3>();
  run<false, false, false, false, 4>();
  run<true, false, true, false, 5>();
  run<false, false, true, true, 6>();
  run<true, true, true, false, 7, true>();
  run<true, true, true, true, 8, true>();
  run<true, true, true, true, 9, true, true>();
  run<true, true, true, true, 10, true, false, 1>();
  run<true, true, true, true, 11, true, false, 2>();
  run<true, true, true, true, 12, true, false, 3>();
  cudaDeviceSynchronize();
  long long c[64];
  cudaMemcpyFromSymbol(c, g_cyc, sizeof(c));
  const char* nm[] = {"fb_tiny loop (vote+pub+pre) + sleepers", "vote+pub+pre", "pub+pre", "pre only",
                      "no prefetch", "vote+pre", "pre + sleepers", "2 rec warps (vote+pub+pre)", "2 rec warps + sleepers", "2 rec + sleepers + per-step STG", "2 rec + sleepers on node bars", "2 rec + try_wait waiters on node bars", "2 rec + sleepers on far bar"};
  for (int v = 0; v < 13; ++v) printf("%-42s %.1f cycles/step\n", nm[v], (double)c[v] / STEPS);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
