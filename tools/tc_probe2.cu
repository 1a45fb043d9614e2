// tc_probe2.cu — find a working tcgen05 kind::tf32 / kind::f16 configuration (diagnostic).
// D is pre-filled with 7.0 via tcgen05.st; the MMA accumulates (enable-input-d = 1) so a
// no-op MMA leaves 7.0 and a working one gives 7 + (A.B).  A = I, B[k][n] = k + n/256.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "tc.cuh"

using namespace tsb;
constexpr int M = 128, NN = 128, K = 128;

__device__ __forceinline__ uint32_t kmaj(int r, int k, int esz, int kdim) {
  // K-major, no swizzle: core matrix 8 rows x 16 B; k-groups (16 B) at LBO = 128 B;
  // 8-row groups at SBO = (kdim*esz/16)*128 B
  const int kpg = 16 / esz;  // elements per 16 B
  return (uint32_t)((r >> 3) * (kdim / kpg) * 128 + (k / kpg) * 128 + (r & 7) * 16 + (k % kpg) * esz);
}

__global__ void probe(int variant, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  const bool bf16 = (variant & 1);
  const bool mbit23 = (variant & 2);
  const bool bmn = (variant & 4);
  const bool masked_form = (variant & 8);
  uint8_t* As = smem;
  uint8_t* Bs = smem + 64 * 1024;
  const int esz = bf16 ? 2 : 4;
  for (int q = tid; q < M * K; q += 128) {
    const int m = q / K, k = q % K;
    const float a = (m == k) ? 1.f : 0.f;
    if (bf16)
      *reinterpret_cast<__nv_bfloat16*>(As + kmaj(m, k, 2, K)) = __float2bfloat16(a);
    else
      *reinterpret_cast<float*>(As + kmaj(m, k, 4, K)) = a;
  }
  for (int q = tid; q < K * NN; q += 128) {
    const int k = q / NN, n = q % NN;
    const float b = (float)k + (float)n / 256.f;  // exact in tf32/bf16? (bf16: approx)
    uint32_t off;
    if (bmn) {
      const int npg = 16 / esz;
      off = (uint32_t)((n / npg) * 128 + (k >> 3) * (NN / npg) * 128 + (k & 7) * 16 + (n % npg) * esz);
    } else {
      off = kmaj(n, k, esz, K);
    }
    if (bf16)
      *reinterpret_cast<__nv_bfloat16*>(Bs + off) = __float2bfloat16(b);
    else
      *reinterpret_cast<float*>(Bs + off) = b;
  }
  if (warp == 0) tc::tmem_alloc<256>(&tbase);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = tbase, lb = (uint32_t)(32 * warp) << 16;
  {
    uint32_t v[32];
    for (int c = 0; c < 32; ++c) v[c] = __float_as_uint(7.f);
    for (int c0 = 0; c0 < NN; c0 += 32) tc::st32(tm + lb + c0, v);
    tc::wait_st();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  uint32_t idesc = (1u << 4) | ((bf16 ? 1u : 2u) << 7) | ((bf16 ? 1u : 2u) << 10) |
                   ((bmn ? 1u : 0u) << 16) | ((uint32_t)(NN >> 3) << 17);
  idesc |= mbit23 ? ((uint32_t)(M >> 4) << 23) : ((uint32_t)(M >> 4) << 24);
  const int kstep = bf16 ? 16 : 8;  // 32 bytes of K per instruction
  if (tid == 0) {
    for (int s = 0; s < K / kstep; ++s) {
      const uint64_t ad = tc::smem_desc(As + s * 256, 128, (K * esz / 16) * 128);
      const uint64_t bd = bmn ? tc::smem_desc(Bs + s * (NN * esz / 16) * 128, (NN * esz / 16) * 128, 128)
                              : tc::smem_desc(Bs + s * 256, 128, (K * esz / 16) * 128);
      if (masked_form) {
        if (bf16)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n\t}\n" ::"r"(tm),
              "l"(ad), "l"(bd), "r"(idesc), "r"(1), "r"(0));
        else
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, {%5, %5, %5, %5}, p;\n\t}\n" ::"r"(tm),
              "l"(ad), "l"(bd), "r"(idesc), "r"(1), "r"(0));
      } else {
        if (bf16)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm), "l"(ad),
              "l"(bd), "r"(idesc), "r"(1));
        else
          tc::mma_tf32_ss(tm, ad, bd, idesc, 1);
      }
    }
    tc::commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc::fence_after();
  for (int c0 = 0; c0 < NN; c0 += 32) {
    uint32_t v[32];
    tc::ld32(tm + lb + c0, v);
    for (int c = 0; c < 32; ++c) out[tid * NN + c0 + c] = __uint_as_float(v[c]);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) tc::tmem_dealloc<256>(tm);
}

int main() {
  float* d;
  cudaMalloc(&d, M * NN * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  std::vector<float> h(M * NN);
  for (int v = 0; v < 16; ++v) {
    cudaMemset(d, 0, M * NN * 4);
    probe<<<1, 128, 160 * 1024>>>(v, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h.data(), d, M * NN * 4, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < NN; ++n) {
        const double ref = 7.0 + m + n / 256.0;
        err = fmax(err, fabs(h[m * NN + n] - ref));
      }
    printf("variant %2d (bf16=%d mbit23=%d b_mn=%d maskform=%d): %s  D[0][0..2]=%g %g %g D[5][3]=%g "
           "D[127][127]=%g  maxerr %.3g\n",
           v, v & 1, (v >> 1) & 1, (v >> 2) & 1, (v >> 3) & 1, cudaGetErrorString(e), h[0], h[1], h[2],
           h[5 * NN + 3], h[127 * NN + 127], err);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
