// Phase timing harness for fb_small_kernel (debug tool, not part of the product path).
// nvcc -DTS_PHASE_TIMING -Iinclude -Ipaper_2002_00876_b200/csrc ... tools/phase_small.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2002_00876_b200/csrc/fb_small.cu"
using namespace tsb;
int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 32, N = 25, C = 20, E = N - 1;
  size_t n = (size_t)B * E * C * C;
  std::vector<float> h(n);
  for (size_t k = 0; k < n; ++k) h[k] = (float)((k * 2654435761u) % 1000) / 250.f - 2.f;
  float *pot, *marg, *logz; uint32_t* flags;
  cudaMalloc(&pot, n * 4); cudaMalloc(&marg, n * 4); cudaMalloc(&logz, B * 4); cudaMalloc(&flags, B * 4);
  cudaMemcpy(pot, h.data(), n * 4, cudaMemcpyHostToDevice);
  SmallArgs a{pot, nullptr, B, N, C, marg, logz, flags};
  for (int it = 0; it < 5; ++it) launch_small(a, 0);
  cudaDeviceSynchronize();
  long long ph[1024][8];
  cudaMemcpyFromSymbol(ph, g_phase, sizeof(ph));
  const char* names[] = {"start", "loaded", "prepass", "fwd_done", "bwd_done", "sweeps_bar", "Ln", "marg_end"};
  for (int b = 0; b < 3; ++b) {
    printf("cta %d:", b);
    for (int k = 1; k < 8; ++k) printf(" %s=%lld", names[k], ph[b][k] - ph[b][0]);
    printf("\n");
  }
  long long st[2][64];
  cudaMemcpyFromSymbol(st, g_steps, sizeof(st));
  printf("fwd step deltas:");
  for (int k = 1; k < 24; ++k) printf(" %lld", st[0][k] - st[0][k - 1]);
  printf("\nbwd step deltas:");
  for (int k = 1; k < 24; ++k) printf(" %lld", st[1][k] - st[1][k - 1]);
  printf("\n");
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 100; ++it) launch_small(a, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("avg per launch (back-to-back, warm L2): %.2f us\n", ms * 10.f);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
