// viterbi.cu — max-plus forward with backpointers, backtrack, and the argmax indicator.
//
// PAPER.md P:160 / P:265 (Max semiring, Table 2), reading R5:
//   delta_0 = 0;  delta_{t+1}[j] = max_i (delta_t[i] + l_t[i][j]);
//   bp_t[j] = the smallest i attaining the max (strict '>' while scanning i upward);
//   z_E = smallest argmax_j delta_E[j];  z_t = bp_t[z_{t+1}];  score = delta_E[z_E].
// fp32 adds of dyadic inputs are exact, so delta equals the fp64 oracle bit-for-bit.
// One CTA per sequence; column j is owned by SL = 8/4/2/1 consecutive lanes (C * SL <= 256),
// lane s scanning rows i = s (mod SL) in two interleaved compare chains; the SL partial
// (max, first index) pairs are merged by shuffles at the end of each tile (smaller index on
// ties: reading R5).  Tiles stream through a cp.async ring of row blocks (a 256 x 256 tile
// is 256 KB, larger than SMEM).
#include <atomic>

#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

namespace {
__device__ __forceinline__ float max_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
// lanes per column: the largest power of two <= 8 with C * SL <= 256
inline int vit_lanes(int64_t C) {
  int SL = 8;
  while (SL > 1 && C * SL > 256) SL >>= 1;
  return SL;
}
inline int vit_threads(int64_t C) { return (int)(((C * vit_lanes(C) + 31) / 32) * 32); }
inline int vit_rows(int64_t C) { return C <= 128 ? (int)C : 32; }
}  // namespace

size_t vit_smem_bytes(int64_t C, int stages, int rows_per_stage) {
  const int NT = vit_threads(C);
  const size_t stage = (((size_t)rows_per_stage * C) + 3) & ~(size_t)3;
  return (stages * stage + 2 * NT + 3 * (NT / 32) + 8) * sizeof(float);
}

template <bool VEC4>
__global__ void __launch_bounds__(256) viterbi_fwd_kernel(VitArgs a, int S, int RB) {
  extern __shared__ __align__(16) float sm[];
  const int C = (int)a.C;
  const int64_t N = a.N, E = N - 1, CC = (int64_t)C * C;
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int NT = blockDim.x, NW = NT >> 5;
  const int SF = ((RB * C) + 3) & ~3;
  float* ring = sm;
  float* dl = ring + (size_t)S * SF;  // [2][NT]
  float* redv = dl + 2 * NT;          // [2*NW]: per-warp best value, per-warp NaN probe
  int* redi = reinterpret_cast<int*>(redv + 2 * NW);  // [NW]

  const int64_t len = seq_len(a.lengths, b, N);
  if (len < 0) {
    if (tid == 0) {
      a.zend[b] = -1;
      a.score[b] = qnan();
      if (a.logz) a.logz[b] = qnan();
      if (a.flags) a.flags[b] = TS_F_BADLEN;
    }
    return;
  }
  const int64_t Eb = len - 1;
  const int nblk = (C + RB - 1) / RB;
  const int64_t G = Eb * nblk;
  const float* potb = a.pot + b * E * CC;
  const bool act = tid < C;                       // label-indexed work (delta, final arg-max)
  int SL = 8;
  while (SL > 1 && C * SL > 256) SL >>= 1;
  const int col = tid / SL, sl = tid - col * SL;  // the step loop: SL lanes per column
  const bool actc = col < C;

  auto issue = [&](int64_t g) {
    if (g < G) {
      const int64_t t = g / nblk;
      const int blk = (int)(g - t * nblk);
      const int r0 = blk * RB, nr = min(RB, C - r0);
      float* dst = ring + (size_t)(g % S) * SF;
      const float* src = potb + t * CC + (int64_t)r0 * C;
      const int n = nr * C;
      if (VEC4) {
        for (int q = tid; q < (n >> 2); q += NT) cp_async16(dst + 4 * q, src + 4 * q);
      } else {
        for (int q = tid; q < n; q += NT) cp_async4(dst + q, src + q);
      }
    }
    cp_async_commit();
  };

  for (int u = 0; u < S - 1; ++u) issue(u);
  dl[tid] = act ? (a.delta_in ? a.delta_in[b * C + tid] : 0.f) : neg_inf();
  float best = neg_inf(), chk = neg_inf();
  int arg = 0;
  int buf = 0;
  for (int64_t g = 0; g < G; ++g) {
    cp_async_wait_dyn(S - 2);
    __syncthreads();
    issue(g + S - 1);
    const int64_t t = g / nblk;
    const int blk = (int)(g - t * nblk);
    const int r0 = blk * RB, nr = min(RB, C - r0);
    const float* tile = ring + (size_t)(g % S) * SF;
    const float* d = dl + buf * NT + r0;
    if (actc) {
      // two interleaved row streams (independent compare chains), merged with the
      // smallest-index rule on ties (reading R5)
      float best1 = neg_inf();
      int arg1 = 0x7fffffff;
      int r = sl;
#pragma unroll 2
      for (; r + SL < nr; r += 2 * SL) {
        const float v0 = d[r] + tile[r * C + col];
        const float v1 = d[r + SL] + tile[(r + SL) * C + col];
        chk = max_nan(chk, max_nan(v0, v1));
        if (v0 > best) {
          best = v0;
          arg = r0 + r;
        }
        if (v1 > best1) {
          best1 = v1;
          arg1 = r0 + r + SL;
        }
      }
      if (r < nr) {
        const float v0 = d[r] + tile[r * C + col];
        chk = max_nan(chk, v0);
        if (v0 > best) {
          best = v0;
          arg = r0 + r;
        }
      }
      if (best1 > best || (best1 == best && arg1 < arg)) {
        best = best1;
        arg = arg1;
      }
    }
    if (blk == nblk - 1) {
      for (int o = 1; o < SL; o <<= 1) {  // merge the SL lanes of the column
        const float ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
        chk = max_nan(chk, __shfl_xor_sync(0xffffffffu, chk, o));
        if (ov > best || (ov == best && oa < arg)) {
          best = ov;
          arg = oa;
        }
      }
      const float nd = (chk != chk) ? qnan() : best;
      if (actc && sl == 0) {
        dl[(buf ^ 1) * NT + col] = nd;
        a.bp[(b * E + t) * C + col] = (uint8_t)arg;
      }
      best = neg_inf();
      chk = neg_inf();
      arg = 0;
      buf ^= 1;
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  // final argmax: smallest j attaining the max (NaN poisons)
  float v = act ? dl[buf * NT + tid] : neg_inf();
  int idx = act ? tid : 0x7fffffff;
  float bad = v;  // NaN propagates through max_nan
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    bad = max_nan(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    if (ov > v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
  if (lane == 0) {
    redv[w] = v;
    redi[w] = idx;
    redv[NW + w] = bad;
  }
  __syncthreads();
  if (tid == 0) {
    float bv = redv[0];
    int bi = redi[0];
    float bb = redv[NW];
    for (int q = 1; q < NW; ++q) {
      if (redv[q] > bv || (redv[q] == bv && redi[q] < bi)) {
        bv = redv[q];
        bi = redi[q];
      }
      bb = max_nan(bb, redv[NW + q]);
    }
    uint32_t fl = 0;
    float sc = bv;
    int z = bi;
    if (bb != bb || bb == pos_inf()) {
      fl = TS_F_NONFINITE;
      sc = qnan();
      z = -1;
    } else if (bv == neg_inf()) {
      fl = TS_F_EMPTY;
      z = -1;
    }
    a.zend[b] = z;
    a.score[b] = sc;
    if (a.logz) a.logz[b] = sc;
    if (a.flags) a.flags[b] = fl;
  }
}

// One warp per sequence: backpointer rows are staged in SMEM in chunks of kBtRows rows
// (double-buffered 1-D bulk copies when C % 16 == 0, else a cooperative copy) while lane 0
// walks the previous chunk back serially; the path is written with coalesced stores.
constexpr int kBtRows = 128;
constexpr size_t kBtSmem = 2 * kBtRows * 256 + kBtRows * 4 + 32;
__global__ void __launch_bounds__(32) backtrack_kernel(VitArgs a) {
  extern __shared__ __align__(128) uint8_t bsm[];
  const int C = (int)a.C;
  const int64_t N = a.N, E = N - 1;
  const int64_t b = blockIdx.x;
  const int lane = threadIdx.x;
  int32_t* pb = a.path ? a.path + b * N : nullptr;
  const int64_t len = seq_len(a.lengths, b, N);
  const int32_t z_end = a.zend[b];
  if (len < 0 || z_end < 0) {
    if (pb)
      for (int64_t n = lane; n < N; n += 32) pb[n] = -1;
    return;
  }
  const int64_t Eb = len - 1;
  if (pb)
    for (int64_t n = Eb + 1 + lane; n < N; n += 32) pb[n] = -1;
  uint8_t* buf[2] = {bsm, bsm + kBtRows * 256};
  int32_t* zs = reinterpret_cast<int32_t*>(bsm + 2 * kBtRows * 256);
  uint64_t* bar = reinterpret_cast<uint64_t*>(bsm + 2 * kBtRows * 256 + kBtRows * 4);
  const uint8_t* bpb = a.bp + b * E * C;
  const bool bulk = (C & 15) == 0 && ((reinterpret_cast<uintptr_t>(bpb)) & 15) == 0;
  const int64_t nchunk = (Eb + kBtRows - 1) / kBtRows;  // chunk k: rows [lo_k, hi_k), from the top
  auto lo_of = [&](int64_t k) { const int64_t hi = Eb - k * kBtRows; return hi - kBtRows > 0 ? hi - kBtRows : 0; };
  auto hi_of = [&](int64_t k) { return Eb - k * kBtRows; };
  if (bulk) {
    if (lane == 0) {
      mbar_init(&bar[0], 1);
      mbar_init(&bar[1], 1);
      fence_mbar_init();
      for (int64_t k = 0; k < 2 && k < nchunk; ++k) {
        const int64_t lo = lo_of(k), n = hi_of(k) - lo;
        bulk_load(buf[k & 1], bpb + lo * C, (uint32_t)(n * C), &bar[k & 1]);
      }
    }
    __syncwarp();
  }
  int z = z_end;
  if (lane == 0 && pb) pb[Eb] = z;
  for (int64_t k = 0; k < nchunk; ++k) {
    const int64_t lo = lo_of(k), hi = hi_of(k);
    const int nrow = (int)(hi - lo);
    uint8_t* rows = buf[k & 1];
    if (bulk) {
      mbar_wait(&bar[k & 1], (uint32_t)((k >> 1) & 1));
    } else {
      const uint8_t* src = bpb + lo * C;
      for (int q = lane; q < nrow * C; q += 32) rows[q] = src[q];
      __syncwarp();
    }
    if (lane == 0) {
      for (int r = nrow - 1; r >= 0; --r) {
        z = rows[r * C + z];
        zs[r] = z;
      }
    }
    __syncwarp();
    if (bulk && lane == 0 && k + 2 < nchunk) {  // refill this buffer with chunk k+2
      const int64_t lo2 = lo_of(k + 2), n2 = hi_of(k + 2) - lo2;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic reads before async writes
      bulk_load(rows, bpb + lo2 * C, (uint32_t)(n2 * C), &bar[k & 1]);
    }
    z = __shfl_sync(0xffffffffu, z, 0);
    if (pb)
      for (int r = lane; r < nrow; r += 32) pb[lo + r] = zs[r];
    __syncwarp();
  }
}

// Indicator d(A*)/d(l): one-hot (z_t, z_{t+1}) per used edge, zeros elsewhere.
__global__ void __launch_bounds__(256) indicator_kernel(VitArgs a) {
  const int C = (int)a.C;
  const int64_t N = a.N, E = N - 1, CC = (int64_t)C * C;
  const int64_t b = blockIdx.y;
  const int64_t t = blockIdx.x;
  if (t >= E) return;
  float* m = a.marg + (b * E + t) * CC;
  const int32_t* pb = a.path + b * N;
  const int zi = pb[t], zj = pb[t + 1];
  const int64_t hot = (zi >= 0 && zj >= 0) ? (int64_t)zi * C + zj : -1;
  for (int64_t q = threadIdx.x; q < CC; q += blockDim.x) m[q] = (q == hot) ? 1.f : 0.f;
}

cudaError_t launch_vit1(const VitArgs& a, cudaStream_t st);

namespace {
std::atomic<uint64_t> g_attr_vit{0};
template <typename K>
cudaError_t set_smem(K kern, int bit) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t m = 1ull << ((dev & 15) * 4 + bit);
  if (g_attr_vit.load() & m) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) g_attr_vit.fetch_or(m);
  return e;
}
}  // namespace

cudaError_t launch_viterbi(const VitArgs& a, cudaStream_t st, int* launches, int vsplit) {
  cudaError_t e;
  if (vsplit >= 0 && vit2_ok(a) && !a.delta_in) {
    if ((e = launch_vit2(a, vsplit, st)) != cudaSuccess) return e;
  } else {
    if ((e = launch_vit1(a, st)) != cudaSuccess) return e;
  }
  int n = 1;
  if (a.path) {
    if ((e = set_smem(backtrack_kernel, 2)) != cudaSuccess) return e;
    backtrack_kernel<<<(unsigned)a.B, 32, kBtSmem, st>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++n;
  }
  if (a.marg && a.N > 1) {
    indicator_kernel<<<dim3((unsigned)(a.N - 1), (unsigned)a.B), 256, 0, st>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++n;
  }
  if (launches) *launches = n;
  return cudaSuccess;
}

cudaError_t launch_indicator(const VitArgs& a, cudaStream_t st) {
  if (!(a.marg && a.N > 1)) return cudaSuccess;
  indicator_kernel<<<dim3((unsigned)(a.N - 1), (unsigned)a.B), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_backtrack(const VitArgs& a, cudaStream_t st) {
  cudaError_t e = set_smem(backtrack_kernel, 2);
  if (e != cudaSuccess) return e;
  backtrack_kernel<<<(unsigned)a.B, 32, kBtSmem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_vit1(const VitArgs& a, cudaStream_t st) {
  const int C = (int)a.C;
  const int RB = vit_rows(C);
  const size_t stage = (((size_t)RB * C) + 3) & ~(size_t)3;
  // stages sized for occupancy: ceil(B / #SMs) CTAs should be resident per SM (up to 4)
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t per_sm = (a.B + sms - 1) / sms;
  per_sm = per_sm < 1 ? 1 : (per_sm > 4 ? 4 : per_sm);
  int S = (int)(((200 * 1024) / per_sm) / (stage * 4));
  S = S < 2 ? 2 : (S > 8 ? 8 : S);
  const bool vec4 = (C % 4) == 0 && (reinterpret_cast<uintptr_t>(a.pot) & 15) == 0;
  const size_t smem = vit_smem_bytes(C, S, RB);
  cudaError_t e;
  if (vec4) {
    if ((e = set_smem(viterbi_fwd_kernel<true>, 0)) != cudaSuccess) return e;
    viterbi_fwd_kernel<true><<<(unsigned)a.B, vit_threads(C), smem, st>>>(a, S, RB);
  } else {
    if ((e = set_smem(viterbi_fwd_kernel<false>, 1)) != cudaSuccess) return e;
    viterbi_fwd_kernel<false><<<(unsigned)a.B, vit_threads(C), smem, st>>>(a, S, RB);
  }
  return cudaGetLastError();
}

}  // namespace tsb
