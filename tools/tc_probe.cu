// tc_probe.cu — standalone check of the tcgen05 kind::tf32 building blocks used by the
// tensor-core chunk-summary kernel (csrc/tc.cuh): A (128 x 128) staged in TMEM as tf32
// hi/lo columns, B (128 x 128) in shared memory in the MN-major no-swizzle canonical
// layout, D = A.B accumulated in TMEM (1 pass and the 3xTF32 split), read back with
// tcgen05.ld.  Compared with an fp64 host product.  Also times a chain of products.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2002_00876_b200/csrc \
//        tools/tc_probe.cu -o /tmp/tc_probe
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "tc.cuh"

using namespace tsb;

constexpr int M = 128, NN = 128, K = 128;

__device__ __forceinline__ uint32_t b_off_bytes(int k, int n) {
  // K-major canonical (no swizzle): 8 n-rows x 16 B (4 k's) core matrices, k-groups at
  // LBO = 128 B, n-groups at SBO = (K/4)*128 = 4096 B  (tf32 MN-major B is a no-op)
  return (uint32_t)((n >> 3) * 4096 + (k >> 2) * 128 + (n & 7) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ uint32_t a_off_bytes(int m, int k) {
  // K-major canonical (no swizzle): 8 m-rows x 16 B core matrices (128 B), k-groups at
  // LBO = 128 B, m-groups at SBO = (K/4) * 128 B
  return (uint32_t)((m >> 3) * (K / 4) * 128 + (k >> 2) * 128 + (m & 7) * 16 + (k & 3) * 4);
}

__global__ void __launch_bounds__(128) probe_kernel(const float* A, const float* B, float* D1,
                                                    float* D3, int reps, long long* cycles,
                                                    float* Dss) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* Bhi = smem;
  uint8_t* Blo = smem + K * NN * 4;
  uint8_t* As = smem + 2 * K * NN * 4;
  for (int q = threadIdx.x; q < M * K; q += 128)
    *reinterpret_cast<float*>(As + a_off_bytes(q / K, q % K)) = A[q];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  if (warp == 0) tc::tmem_alloc<512>(&tbase);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  for (int q = tid; q < K * NN; q += 128) {
    const int k = q / NN, n = q % NN;
    float hi, lo;
    tc::split_tf32(B[q], hi, lo);
    *reinterpret_cast<float*>(Bhi + b_off_bytes(k, n)) = hi;
    *reinterpret_cast<float*>(Blo + b_off_bytes(k, n)) = lo;
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tbase;
  const uint32_t lane_base = (uint32_t)(32 * warp) << 16;
  const uint32_t cD = 0, cAh = 128, cAl = 256, cD3 = 384;
  // A row tid -> TMEM lane tid, columns cAh.. (hi), cAl.. (lo)
  for (int c0 = 0; c0 < K; c0 += 32) {
    uint32_t vh[32], vl[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      float hi, lo;
      tc::split_tf32(A[tid * K + c0 + c], hi, lo);
      vh[c] = __float_as_uint(hi);
      vl[c] = __float_as_uint(lo);
    }
    tc::st32(tm + lane_base + cAh + c0, vh);
    tc::st32(tm + lane_base + cAl + c0, vl);
  }
  tc::wait_st();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  {  // roundtrip check: A_hi row back from TMEM
    uint32_t v[32];
    tc::ld32(tm + lane_base + cAh, v);
    if (tid == 0 || tid == 1 || tid == 33)
      printf("tid %d tbase %u: A_hi[%d][0..3] via TMEM = %f %f %f %f (A = %f %f %f %f)\n", tid, tm, tid,
             __uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]),
             __uint_as_float(v[3]), A[tid * K], A[tid * K + 1], A[tid * K + 2], A[tid * K + 3]);
  }
  constexpr uint32_t idesc = tc::idesc_tf32(M, NN, 0, 0);
  if (tid == 0) {
    for (int s = 0; s < K / 8; ++s) {
      const uint64_t ad = tc::smem_desc(As + s * 256, 128, (K / 4) * 128);
      const uint64_t bd = tc::smem_desc(Bhi + s * 256, 128, 4096);
      tc::mma_tf32_ss(tm + 0, ad, bd, idesc, s > 0);
    }
    tc::commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc::fence_after();
  for (int c0 = 0; c0 < NN; c0 += 32) {
    uint32_t v[32];
    tc::ld32(tm + lane_base + c0, v);
    tc::wait_ld();
#pragma unroll
    for (int c = 0; c < 32; ++c) Dss[tid * NN + c0 + c] = __uint_as_float(v[c]);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  long long t0 = clock64();
  if (tid == 0) {
    for (int r = 0; r < reps; ++r) {
      for (int s = 0; s < K / 8; ++s) {
        const uint64_t bh = tc::smem_desc(Bhi + s * 256, 128, 4096);
        tc::mma_tf32_ts(tm + cD, tm + cAh + 8 * s, bh, idesc, s > 0);
      }
      for (int s = 0; s < K / 8; ++s) {
        const uint64_t bh = tc::smem_desc(Bhi + s * 256, 128, 4096);
        const uint64_t bl = tc::smem_desc(Blo + s * 256, 128, 4096);
        tc::mma_tf32_ts(tm + cD3, tm + cAh + 8 * s, bh, idesc, s > 0);
        tc::mma_tf32_ts(tm + cD3, tm + cAh + 8 * s, bl, idesc, 1);
        tc::mma_tf32_ts(tm + cD3, tm + cAl + 8 * s, bh, idesc, 1);
      }
    }
    tc::commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 1);
  tc::fence_after();
  long long t1 = clock64();
  if (tid == 0) *cycles = t1 - t0;
  for (int c0 = 0; c0 < NN; c0 += 32) {
    uint32_t v[32], w[32];
    tc::ld32(tm + lane_base + cD + c0, v);
    tc::ld32(tm + lane_base + cD3 + c0, w);
    tc::wait_ld();
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      D1[tid * NN + c0 + c] = __uint_as_float(v[c]);
      D3[tid * NN + c0 + c] = __uint_as_float(w[c]);
    }
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_dealloc<512>(tm);
}

static float *dA, *dB, *d1, *d3, *dss;
static long long* dc;

static void run(const std::vector<float>& A, const std::vector<float>& B, std::vector<float>& h1,
                std::vector<float>& h3, std::vector<float>& hs, int reps, long long* cyc) {
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 3 * K * NN * 4;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<<<1, 128, smem>>>(dA, dB, d1, d3, reps, dc, dss);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("CUDA error %s\n", cudaGetErrorString(e));
    exit(1);
  }
  h1.resize(M * NN);
  h3.resize(M * NN);
  hs.resize(M * NN);
  cudaMemcpy(h1.data(), d1, h1.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(h3.data(), d3, h3.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hs.data(), dss, hs.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(cyc, dc, 8, cudaMemcpyDeviceToHost);
}

int main() {
  cudaMalloc(&dA, M * K * 4);
  cudaMalloc(&dB, K * NN * 4);
  cudaMalloc(&d1, M * NN * 4);
  cudaMalloc(&d3, M * NN * 4);
  cudaMalloc(&dss, M * NN * 4);
  cudaMalloc(&dc, 8);
  std::vector<float> A(M * K), B(K * NN), h1, h3, hs;
  long long cyc;
  // structured: A = I, B = k (then n): D should equal B
  for (int mode = 0; mode < 2; ++mode) {
    for (int m = 0; m < M; ++m)
      for (int k = 0; k < K; ++k) A[m * K + k] = (m == k) ? 1.f : 0.f;
    for (int k = 0; k < K; ++k)
      for (int n = 0; n < NN; ++n) B[k * NN + n] = mode == 0 ? (float)k : (float)n;
    run(A, B, h1, h3, hs, 1, &cyc);
    printf("A=I, B=%s: D_ts[m][n] for m,n in {0,1,2,8,9,127}:\n", mode ? "n" : "k");
    for (int m : {0, 1, 2, 8, 9, 127}) {
      printf("  m=%3d ts:", m);
      for (int n : {0, 1, 2, 8, 9, 127}) printf(" %6.1f", h1[m * NN + n]);
      printf("   ss:");
      for (int n : {0, 1, 2, 8, 9, 127}) printf(" %6.1f", hs[m * NN + n]);
      printf("\n");
    }
  }
  srand(1);
  for (auto& x : A) x = expf(-8.f * rand() / (float)RAND_MAX);
  for (auto& x : B) x = expf(-8.f * rand() / (float)RAND_MAX);
  for (int reps : {1, 64}) {
    run(A, B, h1, h3, hs, reps, &cyc);
    double e1 = 0, e3 = 0, es = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < NN; ++n) {
        double r = 0;
        for (int k = 0; k < K; ++k) r += (double)A[m * K + k] * B[k * NN + n];
        e1 = fmax(e1, fabs(h1[m * NN + n] - r) / r);
        e3 = fmax(e3, fabs(h3[m * NN + n] - r) / r);
        es = fmax(es, fabs(hs[m * NN + n] - r) / r);
      }
    printf("reps %d: max rel err ts-1xTF32 %.3e  ts-3xTF32 %.3e  ss-1x %.3e | %lld cycles = %.1f "
           "cycles per 128^3 tf32 MMA-product (4 products per rep)\n",
           reps, e1, e3, es, cyc, (double)cyc / (4.0 * reps));
  }
  return 0;
}
