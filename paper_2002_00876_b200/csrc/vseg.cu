// vseg.cu — time-sharded Viterbi (SURVEY §8(e), cfg5-shaped chains split in time across
// ranks): the max-plus form of the §6(a) scan applied across devices.
//
// Rank r owns the contiguous edges of every sequence; its local chain has nodes
// [s_r, s_r + E_r] (the last node is the first node of rank r+1).
//
//  1. summary   S_r[m][j] = max over local label paths from label m at the first local node
//               to label j at the last one of their score (the max-plus product
//               l_{s_r} (x) ... (x) l_{s_r+E_r-1}, Table 2 'Max' P:200): C independent max-plus
//               forward recursions started from the unit vectors e_m (0 at m, -inf elsewhere),
//               R of them per CTA sharing each staged tile.
//  2. combine   (after the all-gather of the S_q, identical on every rank, fixed order)
//               delta_in = 0 (x) S_0 (x) ... (x) S_{r-1}  (this segment's boundary vector),
//               final = delta_in (x) S_r (x) ... (x) S_{G-1}, A* = max final, z_E = its smallest
//               argmax (reading R5).
//  3. local forward from delta_in with first-index backpointers (viterbi_fwd_kernel), then
//     maps[j] = the label at the first local node reached by backtracking from label j at the
//     last local node (C independent walks through the staged backpointer rows).
//  4. (after the all-gather of the maps) end label e_r = maps_{r+1}[ ... maps_{G-1}[z_E] ],
//     then the local backtrack from e_r (backtrack_kernel).
// With dyadic inputs every max-plus sum is exact in fp32, so delta_in equals
// the serial recursion's delta at that node bit for bit, the backpointers (smallest index
// on ties) are the serial ones and the path is the unsharded path exactly.
#include <atomic>

#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

namespace {
constexpr int kVsR = 4;  // start labels (summary rows) per CTA

__device__ __forceinline__ float max_nan2(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
}  // namespace

// grid (B, ceil(C / R)), NT = C rounded up to 32 threads; thread j owns column j.
__global__ void __launch_bounds__(128) vseg_summary_kernel(VsegArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int C = (int)a.C;
  const int64_t E = a.N - 1, CC = (int64_t)C * C;
  const int64_t b = blockIdx.x;
  const int m0 = blockIdx.y * kVsR;
  const int tid = threadIdx.x, NT = blockDim.x;
  const bool act = tid < C;
  float* ring = sm;                            // [2][CC]
  float* dl = ring + 2 * ((CC + 3) & ~3);      // [2][R][NT]
  const float* potb = a.pot + b * E * CC;
  const bool v4 = (C % 4) == 0 && (reinterpret_cast<uintptr_t>(potb) & 15) == 0;
  auto stage = [&](int64_t t) {
    if (t < E) {
      float* dst = ring + (t & 1) * ((CC + 3) & ~3);
      const float* src = potb + t * CC;
      if (v4) {
        for (int64_t q = tid; q < CC / 4; q += NT) cp_async16(dst + 4 * q, src + 4 * q);
      } else {
        for (int64_t q = tid; q < CC; q += NT) cp_async4(dst + q, src + q);
      }
    }
    cp_async_commit();
  };
  for (int r = 0; r < kVsR; ++r) dl[r * NT + tid] = (act && tid == m0 + r) ? 0.f : neg_inf();
  stage(0);
  int buf = 0;
  for (int64_t t = 0; t < E; ++t) {
    stage(t + 1);
    cp_async_wait<1>();
    __syncthreads();
    const float* tile = ring + (t & 1) * ((CC + 3) & ~3);
    const float* d = dl + buf * kVsR * NT;
    float best[kVsR];
#pragma unroll
    for (int r = 0; r < kVsR; ++r) best[r] = neg_inf();
    if (act) {
#pragma unroll 4
      for (int i = 0; i < C; ++i) {
        const float v = tile[i * C + tid];
#pragma unroll
        for (int r = 0; r < kVsR; ++r) best[r] = max_nan2(best[r], d[r * NT + i] + v);
      }
    }
    float* dn = dl + (buf ^ 1) * kVsR * NT;
#pragma unroll
    for (int r = 0; r < kVsR; ++r) dn[r * NT + tid] = act ? best[r] : neg_inf();
    buf ^= 1;
    __syncthreads();
  }
  cp_async_wait<0>();
  if (act)
    for (int r = 0; r < kVsR; ++r)
      if (m0 + r < C) a.summary[(b * C + m0 + r) * C + tid] = dl[buf * kVsR * NT + r * NT + tid];
}

// One CTA per sequence: the fixed-order max-plus chain over the gathered summaries.
__global__ void __launch_bounds__(256) vseg_combine_kernel(VsegArgs a) {
  __shared__ float v[2][256];
  __shared__ float rv[8];
  __shared__ int ri[8];
  const int C = (int)a.C;
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const bool act = tid < C;
  int cur = 0;
  v[0][tid] = act ? 0.f : neg_inf();
  __syncthreads();
  for (int q = 0; q < a.world; ++q) {
    if (q == a.rank && act) a.delta_in[b * C + tid] = v[cur][tid];
    const float* S = a.all_summ + ((int64_t)q * a.B + b) * C * C;
    float best = neg_inf();
    if (act)
      for (int i = 0; i < C; ++i) best = max_nan2(best, v[cur][i] + S[(int64_t)i * C + tid]);
    v[cur ^ 1][tid] = act ? best : neg_inf();
    cur ^= 1;
    __syncthreads();
  }
  // A* and the smallest argmax; NaN anywhere -> NONFINITE
  float x = act ? v[cur][tid] : neg_inf();
  int idx = act ? tid : 0x7fffffff;
  float bad = x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ox = __shfl_xor_sync(0xffffffffu, x, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    bad = max_nan2(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    if (ox > x || (ox == x && oi < idx)) {
      x = ox;
      idx = oi;
    }
  }
  __shared__ float rb[8];
  if (lane == 0) {
    rv[w] = x;
    ri[w] = idx;
    rb[w] = bad;
  }
  __syncthreads();
  if (tid == 0) {
    float bv = rv[0], bb = rb[0];
    int bi = ri[0];
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      if (rv[k] > bv || (rv[k] == bv && ri[k] < bi)) {
        bv = rv[k];
        bi = ri[k];
      }
      bb = max_nan2(bb, rb[k]);
    }
    uint32_t fl = 0;
    if (bb != bb || bb == pos_inf()) {
      fl = TS_F_NONFINITE;
      bv = qnan();
      bi = -1;
    } else if (bv == neg_inf()) {
      fl = TS_F_EMPTY;
      bi = -1;
    }
    a.score[b] = bv;
    a.zglob[b] = bi;
    if (a.flags) a.flags[b] = fl;
  }
}

// One CTA per sequence, thread j walks back from label j through the local backpointers,
// staged in SMEM in chunks of kRows rows.
__global__ void __launch_bounds__(256) vseg_maps_kernel(VsegArgs a) {
  constexpr int kRows = 128;
  __shared__ uint8_t rows[kRows * 256];
  const int C = (int)a.C;
  const int64_t E = a.N - 1, b = blockIdx.x;
  const int tid = threadIdx.x;
  const uint8_t* bpb = a.bp + b * E * C;
  int z = tid;
  for (int64_t hi = E; hi > 0; hi -= kRows) {
    const int64_t lo = hi - kRows > 0 ? hi - kRows : 0;
    const int n = (int)(hi - lo);
    __syncthreads();
    for (int q = tid; q < n * C; q += blockDim.x) rows[q] = bpb[lo * C + q];
    __syncthreads();
    if (tid < C)
      for (int r = n - 1; r >= 0; --r) z = rows[r * C + z];
  }
  if (tid < C) a.maps[b * C + tid] = z;
}

// e_r = maps_{r+1}[ ... maps_{G-1}[z_E] ]  (-1 when the distribution is empty / flagged)
__global__ void vseg_endlabel_kernel(VsegArgs a) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  int e = a.zglob[b];
  for (int q = a.world - 1; q > a.rank && e >= 0; --q)
    e = a.all_maps[((int64_t)q * a.B + b) * a.C + e];
  a.zend[b] = e;
}

// ---- launchers ---------------------------------------------------------------------------
cudaError_t launch_vseg_summary(const VsegArgs& a, cudaStream_t st) {
  static std::atomic<uint32_t> attr{0};
  const int C = (int)a.C;
  const int NT = ((C + 31) / 32) * 32;
  const size_t smem = (2 * (((size_t)C * C + 3) & ~(size_t)3) + 2 * kVsR * NT) * sizeof(float);
  int dev = 0;
  cudaGetDevice(&dev);
  const uint32_t bit = 1u << (dev & 31);
  if (!(attr.load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(vseg_summary_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr.fetch_or(bit);
  }
  vseg_summary_kernel<<<dim3((unsigned)a.B, (unsigned)((C + kVsR - 1) / kVsR)), NT, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_vseg_combine(const VsegArgs& a, cudaStream_t st) {
  vseg_combine_kernel<<<(unsigned)a.B, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_vseg_maps(const VsegArgs& a, cudaStream_t st) {
  vseg_maps_kernel<<<(unsigned)a.B, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_vseg_endlabel(const VsegArgs& a, cudaStream_t st) {
  vseg_endlabel_kernel<<<(unsigned)((a.B + 127) / 128), 128, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace tsb
