// Phase timing harness for summary_tc_kernel (debug tool; build with -DTS_TC_TIMING):
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DTS_TC_TIMING -Iinclude \
//        -o tools/phase_tc tools/phase_tc.cu
// One chunk of L edges, C = 128: per-step stamps of the MMA issuer, epilogue and producer.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2002_00876_b200/csrc/scan_tc.cu"
using namespace tsb;
int main(int argc, char** argv) {
  const int L = argc > 1 ? atoi(argv[1]) : 64, C = 128, NCTA = argc > 2 ? atoi(argv[2]) : 1;
  const int64_t N = L + 1, E = L;
  size_t n = (size_t)NCTA * E * C * C;
  std::vector<float> h(n);
  for (size_t k = 0; k < n; ++k) h[k] = (float)((k * 2654435761u) % 1000) / 250.f - 2.f;
  float *pot, *mat; double* off; uint8_t* ident; uint32_t *cflag, *wflags;
  cudaMalloc(&pot, n * 4); cudaMalloc(&mat, (size_t)NCTA * C * C * 4); cudaMalloc(&off, NCTA * C * 8);
  cudaMalloc(&ident, NCTA); cudaMalloc(&cflag, NCTA * 4); cudaMalloc(&wflags, NCTA * 4);
  cudaMemcpy(pot, h.data(), n * 4, cudaMemcpyHostToDevice);
  ScanArgs a{};
  a.pot = pot; a.lengths = nullptr; a.B = NCTA; a.N = N; a.C = C; a.L = L; a.P = 1; a.Ppad = 1;
  a.nodes = 1; a.H = 0; a.mat = mat; a.off = off; a.ident = ident; a.cflag = cflag; a.wflags = wflags;
  if (getenv("TC1")) set_tc_summary(1);
  {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, summary_tc_kernel<3, 128>);
    printf("summary_tc<3,128>: regs %d, maxThreadsPerBlock %d, local %zu B, static smem %zu\n", fa.numRegs,
           fa.maxThreadsPerBlock, fa.localSizeBytes, fa.sharedSizeBytes);
  }
  for (int it = 0; it < 3; ++it) { cudaError_t le = launch_summary_tc(a, 0); if (le != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(le)); }
  cudaDeviceSynchronize();
  static long long t[64][8];
#ifdef TS_TC_TIMING
  cudaMemcpyFromSymbol(t, g_tc_t, sizeof(t));
#endif
  printf("u: Await | Aready | issued | Dready | sum | Wready | Awritten | prodB(u)   (rel. to Await of u)\n");
  for (int u = 0; u < 20 && u < L; ++u) {
    printf("%2d:", u);
    for (int k = 1; k < 8; ++k) printf(" %7lld", t[u][k] - t[u][0]);
    if (u > 0) printf("   step=%lld", t[u][0] - t[u - 1][0]);
    printf("\n");
  }
  static long long pp[64][6];
#ifdef TS_TC_TIMING
  cudaMemcpyFromSymbol(pp, g_tc_p, sizeof(pp));
#endif
  printf("producer warp 0 (rel. to MMA issuer t0 of the same u): staged | pass1 | Bfree | pass2\n");
  for (int u = 0; u < 20 && u < L; ++u)
    printf("%2d: %7lld %7lld %7lld %7lld | loopdone %7lld fenced %7lld\n", u, pp[u][0] - t[u][0], pp[u][1] - t[u][0], pp[u][2] - t[u][0], pp[u][3] - t[u][0], pp[u][4] - t[u][0], pp[u][5] - t[u][0]);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int it = 0; it < 5; ++it) launch_summary_tc(a, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("L=%d CTAs=%d: %.2f us per launch, %.3f us per step  err=%s\n", L, NCTA, ms * 200.f,
         ms * 200.f / L, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
