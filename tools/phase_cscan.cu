// Phase timing harness for fb_cscan_kernel (debug tool; build with -DTS_PHASE_TIMING):
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DTS_PHASE_TIMING -DTS_PHASE_NOSTEPS \
//        -Iinclude -o tools/phase_cscan tools/phase_cscan.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2002_00876_b200/csrc/fb_tiny.cu"
#include "../paper_2002_00876_b200/csrc/fb_cscan.cu"
using namespace tsb;
int main(int argc, char** argv) {
  const int B = argc > 1 ? atoi(argv[1]) : 32, N = argc > 2 ? atoi(argv[2]) : 25,
            C = argc > 3 ? atoi(argv[3]) : 20, G = argc > 4 ? atoi(argv[4]) : 4, E = N - 1;
  size_t n = (size_t)B * E * C * C;
  std::vector<float> h(n);
  for (size_t k = 0; k < n; ++k) h[k] = (float)((k * 2654435761u) % 1000) / 250.f - 2.f;
  float *pot, *marg, *logz; uint32_t* flags;
  cudaMalloc(&pot, n * 4); cudaMalloc(&marg, n * 4); cudaMalloc(&logz, B * 4); cudaMalloc(&flags, B * 4);
  cudaMemcpy(pot, h.data(), n * 4, cudaMemcpyHostToDevice);
  SmallArgs a{pot, nullptr, B, N, C, marg, logz, flags};
  for (int it = 0; it < 5; ++it) launch_cscan(a, G, 0);
  cudaDeviceSynchronize();
  printf("launch: %s\n", cudaGetErrorString(cudaGetLastError()));
  static long long ph[64][16];
#ifdef TS_PHASE_TIMING
  cudaMemcpyFromSymbol(ph, g_cs_phase, sizeof(ph));
#endif
  const char* nm[] = {"start", "prepass", "tree", "csync", "xrecv", "fchain", "fsweep", "bchain", "bsweep", "end"};
  for (int c = 0; c < 2 * G && c < 64; ++c) {
    printf("cta %d:", c);
    for (int k = 1; k < 10; ++k) printf(" %s=%lld", nm[k], ph[c][k] - ph[c][0]);

    printf("\n");
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 200; ++it) launch_cscan(a, G, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("avg per launch (back-to-back eager, warm L2): %.2f us  err=%s\n", ms * 5.f,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
