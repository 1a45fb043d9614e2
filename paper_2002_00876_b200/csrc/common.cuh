// common.cuh — shared device helpers for the sm_100a linear-chain CRF kernels.
//
// Numerics (DESIGN.md §4 "Numerics"): the log semiring runs in base 2 —
// x = (l - ref) * log2(e) after an exact re-centring subtraction in natural units,
// ex2.approx.ftz / lg2.approx on the MUFU pipe, fp64 accumulation of the per-step
// offsets.  Max-plus (Viterbi) runs on the raw fp32 values (exact on dyadic inputs).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "ts_b200.h"

namespace tsb {

// One-time opt-in of kernel `kern` to `bytes` of dynamic shared memory, per DEVICE: the
// attribute is device state, so bit d of `mask` (one mask per kernel instantiation) records
// that device d has it.  Devices >= 64 (none exist on one node) re-apply it every launch.
template <typename K>
inline cudaError_t smem_optin_once(K kern, std::atomic<uint64_t>& mask, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = (dev >= 0 && dev < 64) ? (1ull << dev) : 0;
  if (bit && (mask.load(std::memory_order_acquire) & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && bit) mask.fetch_or(bit, std::memory_order_release);
  return e;
}

constexpr float kLog2e = 1.4426950408889634f;
constexpr double kLn2 = 0.69314718055994530942;

__device__ __forceinline__ float neg_inf() { return __int_as_float(0xff800000); }
__device__ __forceinline__ float pos_inf() { return __int_as_float(0x7f800000); }
__device__ __forceinline__ float qnan() { return __int_as_float(0x7fffffff); }

// MUFU exp2 / log2 (approximate, flush-to-zero).  ex2(-inf) = 0, lg2(0) = -inf.
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Underflow gate: a linear-space partial sum below 2^-60 means the
// fast exp-shifted dot product may have lost significant terms to flush-to-zero;
// the column/row is then recomputed exactly in log space.
constexpr float kGate = 8.673617379884035e-19f;  // 2^-60

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ unsigned warp_or(unsigned v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// log2(sum 2^v) over a warp, stable (max-shifted); -inf if all -inf.
__device__ __forceinline__ float warp_lse2(float v) {
  float m = warp_max(v);
  float e = (m == neg_inf()) ? 0.f : ex2(v - m);
  float s = warp_sum(e);
  return (m == neg_inf()) ? neg_inf() : m + lg2(s);
}

// ---- cp.async (LDGSTS) staging ------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
// wait until at most n (runtime, clamped to [0,7]) committed groups are pending
__device__ __forceinline__ void cp_async_wait_dyn(int n) {
  switch (n <= 0 ? 0 : (n >= 7 ? 7 : n)) {
    case 0: cp_async_wait<0>(); break;
    case 1: cp_async_wait<1>(); break;
    case 2: cp_async_wait<2>(); break;
    case 3: cp_async_wait<3>(); break;
    case 4: cp_async_wait<4>(); break;
    case 5: cp_async_wait<5>(); break;
    case 6: cp_async_wait<6>(); break;
    default: cp_async_wait<7>(); break;
  }
}

// ---- TMA bulk copies + mbarriers (1-D cp.async.bulk, no tensor map) ----------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n fence.proxy.async.shared::cta;" ::: "memory");
}
// arm `bar` for `bytes` of async-proxy transactions (one arrival) and issue one bulk copy
// global -> shared of `bytes` (16-byte aligned, multiple of 16) completing on `bar`.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  const uint32_t b = smem_u32(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t b = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
  } while (!done);
}
// mbarrier wait for consumers that expect to wait long: back off with __nanosleep so the
// spinning warps leave issue slots and the MIO pipe to the producers.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity, unsigned ns) {
  const uint32_t b = smem_u32(bar);
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
    if (done) break;
    __nanosleep(ns);
  }
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// bulk copy completing on `bar` without arriving (the arrival is a separate expect_tx)
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// cluster-scope variants (DSMEM): address of the same smem object in CTA `rank`
__device__ __forceinline__ uint32_t mapa_u32(const void* p, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_f32(const float* local_ptr, int rank, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(mapa_u32(local_ptr, rank)), "f"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* local_bar, int rank) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                   mapa_u32(local_bar, rank))
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t b = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
  } while (!done);
}
// named barrier over `n` threads (id 1..15; id 0 is __syncthreads)
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// ---- misc -------------------------------------------------------------------------------
__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Row stride (floats) of a C x C tile staged in shared memory: C+4 when rows can be
// moved in 16-byte pieces (conflict-free float4 row reads by thread-per-row sweeps),
// otherwise an odd stride (conflict-free scalar column/row reads).
__host__ __device__ __forceinline__ int tile_stride(int C, bool vec4) {
  return vec4 ? C + 4 : ((C & 1) ? C : C + 1);
}

// Stage one C x C tile (global, row-major, contiguous) into smem rows of `stride` floats.
// All `nthreads` threads participate; completion via cp.async groups.
__device__ __forceinline__ void stage_tile(float* dst, const float* __restrict__ src, int C,
                                           int stride, bool vec4, int tid, int nthreads) {
  if (vec4) {
    const int q = C >> 2;  // float4 per row
    const int n = C * q;
    for (int k = tid; k < n; k += nthreads) {
      int r = k / q, c4 = k - r * q;
      cp_async16(dst + r * stride + 4 * c4, src + (int64_t)r * C + 4 * c4);
    }
  } else {
    const int n = C * C;
    for (int k = tid; k < n; k += nthreads) {
      int r = k / C, c = k - r * C;
      cp_async4(dst + r * stride + c, src + k);
    }
  }
}

// Per-sequence length with validation (reading R10).  Returns len or -1 if bad.
__device__ __forceinline__ int64_t seq_len(const int32_t* __restrict__ lengths, int64_t b,
                                           int64_t N) {
  if (!lengths) return N;
  int64_t l = lengths[b];
  return (l >= 1 && l <= N) ? l : -1;
}

}  // namespace tsb
