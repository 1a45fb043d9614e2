// vchunk.cu — single-GPU time-chunked Viterbi (SURVEY §8(a) a7 "the chunked variant takes
// boundary delta from max-plus a2/a3/a4"; the Max semiring of Table 2, on the scan of
// §6(a)).  Each sequence's E_b edges are cut into P chunks of L edges; chunk k of
// sequence b is the "virtual segment" s = b P + k, edges [k L, k L + n_s), n_s = clamp(E_b - k L,
// 0, L) (chunks past the sequence are empty: identity summary, identity map).
//
//  1. summary   S_s[m][j] = the max-plus product of the chunk's edges (best chunk-local path
//               score from label m at its first node to label j at its last): C independent
//               max-plus recursions from the unit vectors, R per CTA sharing each staged tile
//               (the row-chain form of vseg.cu's summary).
//  2. combine   one CTA per sequence, the fixed-order max-plus vector chain over its chunks:
//               delta_in[s] = 0 (x) S_{b,0} (x) ... (x) S_{b,k-1}, A* = max of the final vector,
//               z_E = its smallest argmax (reading R5); NaN / +inf -> NONFINITE, -inf -> EMPTY.
//  3. forward   one CTA per chunk from delta_in[s] with first-index backpointers (the serial
//               recursion of P:265 restarted at the chunk boundary).
//  4. maps      one CTA per chunk: maps[s][j] = the chunk's first-node label reached by
//               backtracking from label j at its last node.
//  5. end labels one thread per sequence: e_{P-1} = z_E, e_{k-1} = maps[s_k][e_k]; nodes past
//               the sequence (and every node of a flagged one) get -1.
//  6. backtrack one warp per chunk from e_k over its backpointer rows.
// With inputs whose partial path sums are exact in fp32 (the dyadic generator)
// every max-plus sum is exact in any association order, so delta_in equals the serial delta at
// that node bit for bit, the chunk backpointers are the serial ones, and the path is the serial
// path exactly (tests/test_vchunk_gpu.py checks L in {1, 7, 64, E} against the oracle).
#include <atomic>

#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

namespace {
constexpr int kVcR = 4;  // summary rows (start labels) per CTA

__device__ __forceinline__ float max_nan3(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// chunk geometry of virtual segment s
struct Chunk {
  int64_t b, k, t0, n;  // sequence, chunk index, first edge, edge count (0: empty)
  bool valid;           // the sequence has a valid length
};
__device__ __forceinline__ Chunk chunk_of(const VChunkArgs& a, int64_t s) {
  Chunk c;
  c.b = s / a.P;
  c.k = s - c.b * a.P;
  const int64_t len = seq_len(a.lengths, c.b, a.N);
  c.valid = len >= 1;
  const int64_t Eb = c.valid ? len - 1 : 0;
  c.t0 = c.k * a.L;
  const int64_t rem = Eb - c.t0;
  c.n = rem <= 0 ? 0 : (rem < a.L ? rem : a.L);
  return c;
}
}  // namespace

// grid (B P, ceil(C / R)), NT = C rounded up to 32 threads; thread j owns column j.
__global__ void __launch_bounds__(256) vch_summary_kernel(VChunkArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int C = (int)a.C;
  const int64_t E = a.N - 1, CC = (int64_t)C * C;
  const int64_t s = blockIdx.x;
  const Chunk ch = chunk_of(a, s);
  const int m0 = blockIdx.y * kVcR;
  const int tid = threadIdx.x, NT = blockDim.x;
  const bool act = tid < C;
  float* ring = sm;                        // [2][CC]
  float* dl = ring + 2 * ((CC + 3) & ~3);  // [2][R][NT]
  const float* potc = a.pot + (ch.b * E + ch.t0) * CC;
  const bool v4 = (C % 4) == 0 && (reinterpret_cast<uintptr_t>(potc) & 15) == 0;
  auto stage = [&](int64_t t) {
    if (t < ch.n) {
      float* dst = ring + (t & 1) * ((CC + 3) & ~3);
      const float* src = potc + t * CC;
      if (v4) {
        for (int64_t q = tid; q < CC / 4; q += NT) cp_async16(dst + 4 * q, src + 4 * q);
      } else {
        for (int64_t q = tid; q < CC; q += NT) cp_async4(dst + q, src + q);
      }
    }
    cp_async_commit();
  };
  for (int r = 0; r < kVcR; ++r) dl[r * NT + tid] = (act && tid == m0 + r) ? 0.f : neg_inf();
  stage(0);
  int buf = 0;
  for (int64_t t = 0; t < ch.n; ++t) {
    stage(t + 1);
    cp_async_wait<1>();
    __syncthreads();
    const float* tile = ring + (t & 1) * ((CC + 3) & ~3);
    const float* d = dl + buf * kVcR * NT;
    float best[kVcR];
#pragma unroll
    for (int r = 0; r < kVcR; ++r) best[r] = neg_inf();
    if (act) {
#pragma unroll 4
      for (int i = 0; i < C; ++i) {
        const float v = tile[i * C + tid];
#pragma unroll
        for (int r = 0; r < kVcR; ++r) best[r] = max_nan3(best[r], d[r * NT + i] + v);
      }
    }
    float* dn = dl + (buf ^ 1) * kVcR * NT;
#pragma unroll
    for (int r = 0; r < kVcR; ++r) dn[r * NT + tid] = act ? best[r] : neg_inf();
    buf ^= 1;
    __syncthreads();
  }
  cp_async_wait<0>();
  if (act)
    for (int r = 0; r < kVcR; ++r)
      if (m0 + r < C) a.summ[(s * C + m0 + r) * C + tid] = dl[buf * kVcR * NT + r * NT + tid];
}

// Register-blocked max-plus chunk summary for C % 16 == 0 (C <= 128): one CTA per chunk holds
// the running product S = X_0 (x) ... (x) X_{t-1} (C x C, row-major in shared memory) and
// multiplies it by the next tile, S'[m][j] = max_i S[m][i] + X[i][j]; thread (tr, tc) owns an
// 8 x 8 output block, strided so that shared-memory reads are conflict-free (T = C / 8, T^2
// threads; S rows padded by 4 floats).
// Tiles are staged pair-interleaved, XP[i/2][j] = (X[i][j], X[i+1][j]), so that one packed
// FADD2 forms the two terms of an i-pair and one FMNMX3.NaN folds both into the running max:
// one instruction per term, NaN / +inf propagate into the summary (the combine flags them).
// The next tile is loaded into registers while the current one is multiplied.
__device__ __forceinline__ uint64_t add_f32x2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ float max3_nan(float a, float b, float c) {
  float r;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

template <int C>
__global__ void __launch_bounds__((C / 8) * (C / 8), 1) vch_summary_mm_kernel(VChunkArgs a) {
  constexpr int T = C / 8, NT = T * T, CC = C * C;
  constexpr int SP = C + 4;         // padded S row: the warp's T-row groups land on distinct banks
  constexpr int PER = CC / NT;      // tile elements loaded per thread per step (64 at C = 128)
  constexpr int GRP = PER / 8;      // (row pair, 4 columns) groups per thread
  extern __shared__ __align__(16) float sm[];
  float* S = sm;                    // [C][SP]
  float2* XP = reinterpret_cast<float2*>(sm + C * SP);  // [2][C/2][C]
  const int64_t E = a.N - 1;
  const int64_t s = blockIdx.x;
  const Chunk ch = chunk_of(a, s);
  const int tid = threadIdx.x, tr = tid / T, tc = tid - (tid / T) * T;
  const float* potc = a.pot + (ch.b * E + ch.t0) * (int64_t)CC;
  // identity start
  for (int q = tid; q < CC; q += NT) S[(q / C) * SP + q % C] = ((q / C) == (q % C)) ? 0.f : neg_inf();
  // group g of this thread: row pair rp = (tid + NT g) / (C / 4), column quad cq
  float4 nx[GRP][2];
  auto load = [&](int64_t t) {
    const float* tile = potc + t * CC;
#pragma unroll
    for (int g = 0; g < GRP; ++g) {
      const int idx = tid + NT * g, rp = idx / (C / 4), cq = idx - rp * (C / 4);
      nx[g][0] = *reinterpret_cast<const float4*>(tile + (2 * rp) * C + 4 * cq);
      nx[g][1] = *reinterpret_cast<const float4*>(tile + (2 * rp + 1) * C + 4 * cq);
    }
  };
  auto store = [&](int buf) {
    float2* xp = XP + buf * (C / 2) * C;
#pragma unroll
    for (int g = 0; g < GRP; ++g) {
      const int idx = tid + NT * g, rp = idx / (C / 4), cq = idx - rp * (C / 4);
      float4* dst = reinterpret_cast<float4*>(xp + rp * C + 4 * cq);
      dst[0] = make_float4(nx[g][0].x, nx[g][1].x, nx[g][0].y, nx[g][1].y);
      dst[1] = make_float4(nx[g][0].z, nx[g][1].z, nx[g][0].w, nx[g][1].w);
    }
  };
  if (ch.n > 0) {
    load(0);
    store(0);
  }
  // thread (tr, tc) owns rows tr + T r and columns 2 tc + 2 T m + e (r < 8, m < 4, e < 2):
  // a warp's column loads are T contiguous 16-byte float4s, its row loads 32 / T distinct
  // padded rows in distinct banks
  for (int64_t t = 0; t < ch.n; ++t) {
    __syncthreads();  // S and XP[t & 1] ready
    if (t + 1 < ch.n) load(t + 1);
    const float2* xp = XP + (t & 1) * (C / 2) * C + 2 * tc;
    const float* srow = S + tr * SP;
    float acc[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = neg_inf();
#pragma unroll 2
    for (int ip = 0; ip < C / 2; ++ip) {
      uint64_t av[8], bv[8];
#pragma unroll
      for (int r = 0; r < 8; ++r)
        av[r] = *reinterpret_cast<const uint64_t*>(srow + (T * r) * SP + 2 * ip);
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const float4 q = *reinterpret_cast<const float4*>(xp + ip * C + 2 * T * m);
        bv[2 * m] = (uint64_t)__float_as_uint(q.x) | ((uint64_t)__float_as_uint(q.y) << 32);
        bv[2 * m + 1] = (uint64_t)__float_as_uint(q.z) | ((uint64_t)__float_as_uint(q.w) << 32);
      }
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint64_t sum = add_f32x2(av[r], bv[c]);
          acc[r][c] = max3_nan(acc[r][c], __uint_as_float((uint32_t)sum),
                               __uint_as_float((uint32_t)(sum >> 32)));
        }
    }
    __syncthreads();  // every read of S and XP[t & 1] done
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int m = 0; m < 4; ++m)
        *reinterpret_cast<float2*>(S + (tr + T * r) * SP + 2 * tc + 2 * T * m) =
            make_float2(acc[r][2 * m], acc[r][2 * m + 1]);
    if (t + 1 < ch.n) store((int)((t + 1) & 1));
  }
  __syncthreads();
  float* out = a.summ + s * (int64_t)CC;
  for (int q = tid; q < CC / 4; q += NT) {
    const int i = (4 * q) / C, j = 4 * q - i * C;
    reinterpret_cast<float4*>(out)[q] = *reinterpret_cast<const float4*>(S + i * SP + j);
  }
}

// One CTA (256 threads) per sequence: delta_in of every chunk, A*, z_E, flags.
__global__ void __launch_bounds__(256) vch_combine_kernel(VChunkArgs a) {
  __shared__ float v[2][256];
  __shared__ float rv[8], rb[8];
  __shared__ int ri[8];
  const int C = (int)a.C;
  const int64_t b = blockIdx.x, P = a.P;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const bool act = tid < C;
  const int64_t len = seq_len(a.lengths, b, a.N);
  if (len < 1) {
    if (tid == 0) {
      a.score[b] = qnan();
      if (a.logz) a.logz[b] = qnan();
      a.zglob[b] = -1;
      if (a.flags) a.flags[b] = TS_F_BADLEN;
    }
    return;
  }
  int cur = 0;
  v[0][tid] = act ? 0.f : neg_inf();
  __syncthreads();
  for (int64_t k = 0; k < P; ++k) {
    const int64_t s = b * P + k;
    if (act) a.din[s * C + tid] = v[cur][tid];
    const float* S = a.summ + s * C * C;
    float best = neg_inf();
    if (act)
      for (int i = 0; i < C; ++i) best = max_nan3(best, v[cur][i] + S[(int64_t)i * C + tid]);
    v[cur ^ 1][tid] = act ? best : neg_inf();
    cur ^= 1;
    __syncthreads();
  }
  float x = act ? v[cur][tid] : neg_inf();
  int idx = act ? tid : 0x7fffffff;
  float bad = x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ox = __shfl_xor_sync(0xffffffffu, x, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    bad = max_nan3(bad, __shfl_xor_sync(0xffffffffu, bad, o));
    if (ox > x || (ox == x && oi < idx)) {
      x = ox;
      idx = oi;
    }
  }
  if (lane == 0) {
    rv[w] = x;
    ri[w] = idx;
    rb[w] = bad;
  }
  __syncthreads();
  if (tid == 0) {
    float bv = rv[0], bb = rb[0];
    int bi = ri[0];
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q) {
      if (rv[q] > bv || (rv[q] == bv && ri[q] < bi)) {
        bv = rv[q];
        bi = ri[q];
      }
      bb = max_nan3(bb, rb[q]);
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
    if (a.logz) a.logz[b] = bv;
    a.zglob[b] = bi;
    if (a.flags) a.flags[b] = fl;
  }
}

// One CTA per chunk: the max-plus recursion from delta_in with first-index backpointers.
__global__ void __launch_bounds__(256) vch_forward_kernel(VChunkArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int C = (int)a.C;
  const int64_t E = a.N - 1, CC = (int64_t)C * C;
  const int64_t s = blockIdx.x;
  const Chunk ch = chunk_of(a, s);
  if (ch.n == 0) return;
  const int tid = threadIdx.x, NT = blockDim.x;
  const bool act = tid < C;
  float* ring = sm;                        // [2][CC]
  float* dl = ring + 2 * ((CC + 3) & ~3);  // [2][NT]
  const float* potc = a.pot + (ch.b * E + ch.t0) * CC;
  uint8_t* bpc = a.bp + (ch.b * E + ch.t0) * C;
  const bool v4 = (C % 4) == 0 && (reinterpret_cast<uintptr_t>(potc) & 15) == 0;
  auto stage = [&](int64_t t) {
    if (t < ch.n) {
      float* dst = ring + (t & 1) * ((CC + 3) & ~3);
      const float* src = potc + t * CC;
      if (v4) {
        for (int64_t q = tid; q < CC / 4; q += NT) cp_async16(dst + 4 * q, src + 4 * q);
      } else {
        for (int64_t q = tid; q < CC; q += NT) cp_async4(dst + q, src + q);
      }
    }
    cp_async_commit();
  };
  dl[tid] = act ? a.din[s * C + tid] : neg_inf();
  stage(0);
  int buf = 0;
  for (int64_t t = 0; t < ch.n; ++t) {
    stage(t + 1);
    cp_async_wait<1>();
    __syncthreads();
    const float* tile = ring + (t & 1) * ((CC + 3) & ~3);
    const float* d = dl + buf * NT;
    float best = neg_inf();
    int arg = 0;
    if (act) {
      for (int i = 0; i < C; ++i) {
        const float x = d[i] + tile[i * C + tid];
        if (x > best) {  // strict: the smallest index attaining the max (reading R5)
          best = x;
          arg = i;
        }
      }
      bpc[t * C + tid] = (uint8_t)arg;
    }
    dl[(buf ^ 1) * NT + tid] = act ? best : neg_inf();
    buf ^= 1;
    __syncthreads();
  }
  cp_async_wait<0>();
}

// One CTA per chunk: thread j walks back from label j at the chunk's last node.
__global__ void __launch_bounds__(256) vch_maps_kernel(VChunkArgs a) {
  constexpr int kRows = 128;
  __shared__ uint8_t rows[kRows * 256];
  const int C = (int)a.C;
  const int64_t E = a.N - 1, s = blockIdx.x;
  const Chunk ch = chunk_of(a, s);
  const int tid = threadIdx.x;
  const uint8_t* bpc = a.bp + (ch.b * E + ch.t0) * C;
  int z = tid;
  for (int64_t hi = ch.n; hi > 0; hi -= kRows) {
    const int64_t lo = hi - kRows > 0 ? hi - kRows : 0;
    const int n = (int)(hi - lo);
    __syncthreads();
    for (int q = tid; q < n * C; q += blockDim.x) rows[q] = bpc[lo * C + q];
    __syncthreads();
    if (tid < C)
      for (int r = n - 1; r >= 0; --r) z = rows[r * C + z];
  }
  if (tid < C) a.maps[s * C + tid] = z;
}

// One thread per sequence: every chunk's end label, -1 fill of unused / flagged nodes.
__global__ void vch_endlabel_kernel(VChunkArgs a) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  const int64_t N = a.N, P = a.P, C = a.C;
  const int64_t len = seq_len(a.lengths, b, N);
  int e = a.zglob[b];
  int32_t* pb = a.path + b * N;
  if (len < 1 || e < 0) {  // BADLEN / EMPTY / NONFINITE: no path
    for (int64_t q = 0; q < N; ++q) pb[q] = -1;
    for (int64_t k = 0; k < P; ++k) a.zend[b * P + k] = -1;
    return;
  }
  for (int64_t q = len; q < N; ++q) pb[q] = -1;
  pb[len - 1] = e;  // the last node (also the only one when len = 1)
  for (int64_t k = P - 1; k >= 0; --k) {
    a.zend[b * P + k] = e;
    e = a.maps[(b * P + k) * C + e];
  }
}

// One warp per chunk (lane 0 walks): path nodes [t0, t0 + n] from the chunk's end label.
__global__ void vch_backtrack_kernel(VChunkArgs a) {
  const int64_t s = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= a.B * a.P || (threadIdx.x & 31) != 0) return;
  const Chunk ch = chunk_of(a, s);
  int z = a.zend[s];
  if (ch.n == 0 || z < 0) return;
  const int64_t C = a.C, E = a.N - 1;
  const uint8_t* bpc = a.bp + (ch.b * E + ch.t0) * C;
  int32_t* pb = a.path + ch.b * a.N + ch.t0;
  pb[ch.n] = z;
  for (int64_t t = ch.n - 1; t >= 0; --t) {
    z = bpc[t * C + z];
    pb[t] = z;
  }
}

namespace {
size_t vch_smem(int C, int extra_floats) {
  return (2 * (((size_t)C * C + 3) & ~(size_t)3) + (size_t)extra_floats) * sizeof(float);
}
template <typename K>
cudaError_t optin(K kern, std::atomic<uint64_t>& mask, size_t smem) {
  // the attribute is set once per kernel and device, so to the bound of every size a launch
  // may ask for (vchunk_ok: <= 200 KB), not to this call's size
  if (smem <= 48 * 1024) return cudaSuccess;
  return smem_optin_once(kern, mask, 200 * 1024);
}
std::atomic<uint64_t> g_attr_sum{0}, g_attr_fwd{0}, g_attr_mm[3];
std::atomic<int> g_vch_mm{1};
bool vch_mm_enabled() { return g_vch_mm.load() != 0; }
}  // namespace

void set_vchunk_mm(int enable) { g_vch_mm.store(enable ? 1 : 0); }

size_t vchunk_ws_floats(const VChunkArgs& a) {
  return (size_t)(a.B * a.P) * (size_t)(a.C * a.C + a.C);
}

bool vchunk_ok(int64_t C) { return C >= 1 && C <= 256 && vch_smem((int)C, 2 * kVcR * 256) <= 200 * 1024; }

bool vchunk_mm(int64_t C) { return (C == 128 || C == 64 || C == 32) && vch_mm_enabled(); }

cudaError_t launch_vchunk(const VChunkArgs& a, bool want_path, cudaStream_t st, int* launches) {
  const int C = (int)a.C;
  const int NT = ((C + 31) / 32) * 32;
  const unsigned nseg = (unsigned)(a.B * a.P);
  cudaError_t e;
  const bool mm = vchunk_mm(C) && (reinterpret_cast<uintptr_t>(a.pot) & 15) == 0;
  if (mm) {  // register-blocked max-plus products (FADD2 + FMNMX3)
    const size_t s_mm = ((size_t)C * (C + 4) + (size_t)2 * C * C) * sizeof(float);
    switch (C) {
      case 128:
        if ((e = optin(vch_summary_mm_kernel<128>, g_attr_mm[0], s_mm)) != cudaSuccess) return e;
        vch_summary_mm_kernel<128><<<nseg, 256, s_mm, st>>>(a);
        break;
      case 64:
        if ((e = optin(vch_summary_mm_kernel<64>, g_attr_mm[1], s_mm)) != cudaSuccess) return e;
        vch_summary_mm_kernel<64><<<nseg, 64, s_mm, st>>>(a);
        break;
      default:
        if ((e = optin(vch_summary_mm_kernel<32>, g_attr_mm[2], s_mm)) != cudaSuccess) return e;
        vch_summary_mm_kernel<32><<<nseg, 16, s_mm, st>>>(a);
        break;
    }
  } else {
    const size_t s_sum = vch_smem(C, 2 * kVcR * NT);
    if ((e = optin(vch_summary_kernel, g_attr_sum, s_sum)) != cudaSuccess) return e;
    vch_summary_kernel<<<dim3(nseg, (unsigned)((C + kVcR - 1) / kVcR)), NT, s_sum, st>>>(a);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  vch_combine_kernel<<<(unsigned)a.B, 256, 0, st>>>(a);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  int n = 2;
  if (want_path) {
    const size_t s_fwd = vch_smem(C, 2 * NT);
    if ((e = optin(vch_forward_kernel, g_attr_fwd, s_fwd)) != cudaSuccess) return e;
    vch_forward_kernel<<<nseg, NT, s_fwd, st>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    vch_maps_kernel<<<nseg, 256, 0, st>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    vch_endlabel_kernel<<<(unsigned)((a.B + 127) / 128), 128, 0, st>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    vch_backtrack_kernel<<<(nseg + 3) / 4, 128, 0, st>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    n += 4;
  }
  if (launches) *launches = n;
  return cudaSuccess;
}

}  // namespace tsb
