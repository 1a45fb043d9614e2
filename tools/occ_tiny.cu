// occ_tiny.cu — residency of overlapped fb_tiny calls (debug; build with -DTINY_OCC_TRACE):
// a graph of K cfg2 calls on rotating buffers (early mode), per-CTA smid / start / end from
// %globaltimer; prints the period, the CTA lifetime and the co-resident CTAs per SM and calls.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DTINY_OCC_TRACE -Iinclude -o tools/occ_tiny tools/occ_tiny.cu
#include <algorithm>
#include <cstdio>
#include <map>
#include <vector>
#include "../paper_2002_00876_b200/csrc/fb_tiny.cu"
using namespace tsb;
int main() {
  const int B = 32, N = 25, C = 20, E = N - 1, R = 160, K = 1000;
  const size_t n = (size_t)B * E * C * C;
  std::vector<float> h(n);
  for (size_t k = 0; k < n; ++k) h[k] = (float)((k * 2654435761u) % 1000) / 250.f - 2.f;
  std::vector<float*> pot(R), marg(R), logz(R); std::vector<uint32_t*> flags(R);
  for (int r = 0; r < R; ++r) {
    cudaMalloc(&pot[r], n * 4); cudaMalloc(&marg[r], n * 4); cudaMalloc(&logz[r], B * 4); cudaMalloc(&flags[r], B * 4);
    cudaMemcpy(pot[r], h.data(), n * 4, cudaMemcpyHostToDevice);
  }
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  auto call = [&](int k) {
    SmallArgs a{}; const int r = k % R;
    a.pot = pot[r]; a.B = B; a.N = N; a.C = C; a.marg = marg[r]; a.logz = logz[r]; a.flags = flags[r];
    launch_tiny(a, st);
  };
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int k = 0; k < K; ++k) call(k);
  cudaStreamEndCapture(st, &g); cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
  unsigned long long zero = 0; cudaMemcpyToSymbol(g_occ_idx, &zero, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cnt; cudaMemcpyFromSymbol(&cnt, g_occ_idx, 8);
  std::vector<unsigned long long> rec((size_t)cnt * 5);
  cudaMemcpyFromSymbol(rec.data(), g_occ_rec, rec.size() * 8);
  printf("%.3f us per call, %llu CTA records (%s)\n", ms * 1000.f / K, cnt, cudaGetErrorString(cudaGetLastError()));
  double life = 0, pre = 0, body = 0, tail = 0; unsigned long long tmin = ~0ull, tmax = 0;
  std::vector<std::pair<unsigned long long, int>> ev;  // (time, +1/-1) per SM and overall
  std::map<int, std::vector<std::pair<unsigned long long, int>>> per_sm;
  for (unsigned long long i = 0; i < cnt; ++i) {
    const int sm = (int)rec[5 * i]; const auto t0 = rec[5 * i + 1], t1 = rec[5 * i + 2];
    pre += (double)(rec[5 * i + 3] - t0); body += (double)(rec[5 * i + 4] - rec[5 * i + 3]);
    tail += (double)(t1 - rec[5 * i + 4]);
    life += (double)(t1 - t0); tmin = std::min(tmin, t0); tmax = std::max(tmax, t1);
    ev.push_back({t0, 1}); ev.push_back({t1, -1});
    per_sm[sm].push_back({t0, 1}); per_sm[sm].push_back({t1, -1});
  }
  std::sort(ev.begin(), ev.end());
  int cur = 0, mx = 0; double area = 0; unsigned long long last = ev.empty() ? 0 : ev[0].first;
  for (auto& e : ev) { area += (double)cur * (e.first - last); last = e.first; cur += e.second; mx = std::max(mx, cur); }
  int mx_sm = 0;
  for (auto& kv : per_sm) {
    auto v = kv.second; std::sort(v.begin(), v.end()); int c = 0;
    for (auto& e : v) { c += e.second; mx_sm = std::max(mx_sm, c); }
  }
  printf("mean CTA lifetime %.2f us (prologue + prepass %.2f, recursions + marginals %.2f, tail %.2f), "
         "mean resident CTAs %.1f (max %d), max per SM %d, SMs used %zu\n",
         life / cnt / 1e3, pre / cnt / 1e3, body / cnt / 1e3, tail / cnt / 1e3, area / (double)(tmax - tmin), mx,
         mx_sm, per_sm.size());
  return 0;
}
