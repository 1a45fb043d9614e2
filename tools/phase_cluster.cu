// Phase timing harness for fb_cluster_kernel (debug tool; build with -DTS_PHASE_TIMING).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2002_00876_b200/csrc/fb_cluster.cu"
using namespace tsb;
int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 32, G = argc > 2 ? atoi(argv[2]) : 4;
  const int N = 25, C = 20, E = N - 1;
  size_t n = (size_t)B * E * C * C;
  std::vector<float> h(n);
  for (size_t k = 0; k < n; ++k) h[k] = (float)((k * 2654435761u) % 1000) / 250.f - 2.f;
  float *pot, *marg, *logz; uint32_t* flags;
  cudaMalloc(&pot, n * 4); cudaMalloc(&marg, n * 4); cudaMalloc(&logz, B * 4); cudaMalloc(&flags, B * 4);
  cudaMemcpy(pot, h.data(), n * 4, cudaMemcpyHostToDevice);
  SmallArgs a{pot, nullptr, B, N, C, marg, logz, flags};
  for (int it = 0; it < 5; ++it) launch_cluster(a, G, 0);
  cudaDeviceSynchronize();
  static long long ph[4096][10];
  cudaMemcpyFromSymbol(ph, g_cl_phase, sizeof(ph));
  const char* nm[] = {"start", "loaded", "prepass", "summary", "csync1", "exchange", "sweeps", "marg"};
  for (int c = 0; c < G; ++c) {
    printf("cta %d:", c);
    for (int k = 1; k < 8; ++k) printf(" %s=%lld", nm[k], ph[c][k] - ph[c][0]);
    printf("\n");
  }
  long long st[4][64];
  cudaMemcpyFromSymbol(st, g_cl_steps, sizeof(st));
  printf("summary step: t_done_w0 / after_bar:");
  for (int k = 0; k < 6; ++k) printf(" %lld/%lld", st[0][k] - ph[0][2], st[1][k] - ph[0][2]);
  printf("\n");
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 100; ++it) launch_cluster(a, G, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("G=%d avg per launch (back-to-back, warm L2): %.2f us  err=%s\n", G, ms * 10.f,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
