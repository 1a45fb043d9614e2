// Phase timing harness for fb_tiny_kernel (debug tool; build with -DTS_PHASE_TIMING):
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DTS_PHASE_TIMING -Iinclude \
//        -o tools/phase_tiny tools/phase_tiny.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2002_00876_b200/csrc/fb_tiny.cu"
using namespace tsb;
int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 32, N = argc > 2 ? atoi(argv[2]) : 25,
            C = argc > 3 ? atoi(argv[3]) : 20, E = N - 1;
  size_t n = (size_t)B * E * C * C;
  std::vector<float> h(n);
  for (size_t k = 0; k < n; ++k) h[k] = (float)((k * 2654435761u) % 1000) / 250.f - 2.f;
  float *pot, *marg, *logz; uint32_t* flags;
  cudaMalloc(&pot, n * 4); cudaMalloc(&marg, n * 4); cudaMalloc(&logz, B * 4); cudaMalloc(&flags, B * 4);
  cudaMemcpy(pot, h.data(), n * 4, cudaMemcpyHostToDevice);
  SmallArgs a{pot, nullptr, B, N, C, marg, logz, flags};
  for (int it = 0; it < 5; ++it) launch_tiny(a, 0);
  cudaDeviceSynchronize();
  static long long ph[1024][8];
  cudaMemcpyFromSymbol(ph, g_tiny_phase, sizeof(ph));
  const char* nm[] = {"start", "loaded", "prepass", "fwd", "bwd", "sweeps", "marg"};
  for (int c = 0; c < 3; ++c) {
    printf("cta %d:", c);
    for (int k = 1; k < 7; ++k) printf(" %s=%lld", nm[k], ph[c][k] - ph[c][0]);
    printf("\n");
  }
  static long long wp[4][16][8];
  cudaMemcpyFromSymbol(wp, g_tiny_wp, sizeof(wp));
  for (int w = 0; w < 16; ++w)
    printf("cta0 warp %2d: start=%lld maxed=%lld stored=%lld summed=%lld marg=%lld\n", w, wp[0][w][0] - ph[0][0],
           wp[0][w][3] - ph[0][0], wp[0][w][4] - ph[0][0], wp[0][w][5] - ph[0][0], wp[0][w][2] - ph[0][0]);
  static long long ed[64][4];
  cudaMemcpyFromSymbol(ed, g_tiny_edge, sizeof(ed));
  for (int t = 0; t < E && t < 64; ++t)
    printf("edge %2d: ready=%lld sum=+%lld stored=+%lld\n", t, ed[t][0] - ph[0][0], ed[t][1] - ed[t][0],
           ed[t][2] - ed[t][1]);
  long long st[2][64];
  cudaMemcpyFromSymbol(st, g_tiny_steps, sizeof(st));
  printf("fwd step deltas:");
  for (int k = 1; k < E && k < 64; ++k) printf(" %lld", st[0][k] - st[0][k - 1]);
  printf("\nbwd step deltas:");
  for (int k = 1; k < E && k < 64; ++k) printf(" %lld", st[1][k] - st[1][k - 1]);
  printf("\n");
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 200; ++it) launch_tiny(a, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("avg per launch (back-to-back eager, warm L2): %.2f us  err=%s\n", ms * 5.f,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
