// fb_small.cu — one CTA per sequence, the whole sequence resident in shared memory:
// forward sweep (warp 0) and backward sweep (warp 1) run concurrently, then all warps
// compute the marginals.  Used when C <= 32 and the sequence fits in SMEM
// (BASELINE configs 1 and 2: the paper's Table 1 setting B=32, N=25, C=20).
//
// Per edge t (§5.2 P:252-256 forward, P:181-183 marginals,
// §6(c) P:330-331 stabilised product):
//   T_t  = max_ij l_t[i][j]                    (re-centring, natural units, exact)
//   x'   = (l_t - T_t) log2 e,  EX = 2^x' <= 1  (prepass, all warps; + row/col sums)
//   fwd (sum-normalised, Σ_i p_t[i] = 1, ah = log2 p):
//       s_j = Σ_i p_t[i] EX[i][j],  S_t = Σ_j s_j = Σ_i p_t[i] rowsum_i   (no reduction)
//       p_{t+1}[j] = s_j / S_t,  ah_{t+1}[j] = log2 s_j - log2 S_t,
//       O_{t+1} = O_t + T_t + ln2 log2 S_t   (fp64)
//   bwd: the same with EX transposed and column sums.
//   gate: s_j < 2^-60 -> exact per-cell-max recomputation from the log values (§6(c)).
//   mu_t[i][j] = 2^(ah_t[i] + x'_ij + bh_{t+1}[j] - log2 S_t - L_{t+1}),
//   L_n = log2 Σ_j 2^(ah_n[j] + bh_n[j])    (log2 Z in node n's frames).
// Tiles are stored with a compile-time row stride CT (C rounded up to a multiple of 4;
// padding x' = -inf, EX = 0) so every shared-memory address in the sweeps is an
// immediate offset: the per-step chain is latency-bound on one warp.
#include <atomic>

#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

#ifdef TS_PHASE_TIMING
__device__ long long g_phase[1024][8];
__device__ long long g_steps[2][64];
#define PHASE(k)                                                                   \
  do {                                                                             \
    if (threadIdx.x == 0 && blockIdx.x < 1024) g_phase[blockIdx.x][k] = clock64(); \
  } while (0)
#define PHASEW(k)                                                                         \
  do {                                                                                    \
    if ((threadIdx.x & 31) == 0 && blockIdx.x < 1024) g_phase[blockIdx.x][k] = clock64(); \
  } while (0)
#else
#define PHASE(k) \
  do {           \
  } while (0)
#define PHASEW(k) \
  do {            \
  } while (0)
#endif

constexpr int kSmallThreads = 512;
constexpr int kSmallWarps = kSmallThreads / 32;

inline __host__ __device__ int small_ct(int64_t C) { return (int)(((C + 3) / 4) * 4); }

struct SmallLayout {
  int64_t x, ex, ext, rs, cs, T, lS, lSb, alpha, beta, Ln, pb, total;  // float offsets
};

__host__ __device__ inline SmallLayout small_layout(int64_t N, int CT) {
  SmallLayout l;
  const int64_t E = N - 1, TT = (int64_t)CT * CT;  // CT % 4 == 0: tiles 16-byte aligned
  l.x = 0;
  l.ex = l.x + E * TT;
  l.ext = l.ex + E * TT;
  l.rs = l.ext + E * TT;  // [E][CT] row sums of EX
  l.cs = l.rs + E * CT;   // [E][CT] column sums of EX
  l.T = l.cs + E * CT;    // [E] tile max
  l.lS = l.T + E;         // [E] forward log2 S_t
  l.lSb = l.lS + E;       // [E] backward log2 S'_t
  l.alpha = (l.lSb + E + 3) & ~(int64_t)3;  // [N][32]
  l.beta = l.alpha + N * 32;               // [N][32]
  l.Ln = l.beta + N * 32;                  // [N]
  l.pb = (l.Ln + N + 3) & ~(int64_t)3;     // [2 sweeps][2 buffers][32]
  l.total = l.pb + 128 + 4;                // + flag word
  return l;
}

size_t small_smem_bytes(int64_t N, int64_t C) {
  return (size_t)small_layout(N, small_ct(C)).total * sizeof(float);
}

bool small_fits(int64_t N, int64_t C) {
  return C <= 32 && N >= 1 && small_smem_bytes(N, C) <= (size_t)200 * 1024;
}

namespace {

// Exact per-cell-max value log2 Σ_r 2^(v_r + X[r*xs]) over r < C (the §6(c) formula).
__device__ __forceinline__ float exact_lse(const float* __restrict__ v, const float* __restrict__ X,
                                           int xs, int C) {
  float q = neg_inf();
  for (int r = 0; r < C; ++r) q = fmaxf(q, v[r] + X[r * xs]);
  if (q == neg_inf()) return neg_inf();
  float ss = 0.f;
  for (int r = 0; r < C; ++r) ss += ex2(v[r] + X[r * xs] - q);
  return q + lg2(ss);
}

// One sweep.  FWD: lane j owns column j of EX (M = EX, W = row sums);
// !FWD: lane i owns row i (M = EX^T, W = column sums).  vec receives log2 vectors.
template <bool FWD, int CT>
__device__ __forceinline__ void sweep(const float* __restrict__ X, const float* __restrict__ M,
                                      const float* __restrict__ W, float* vec, float* lSv,
                                      const float* __restrict__ Tm, int Eb, int C, int lane,
                                      double* Oout, float* pbuf) {
  constexpr int TT = CT * CT;
  const bool act = lane < C;
  const int jj = lane < CT ? lane : 0;  // lanes >= CT read a padded column (value 0)
  float p = act ? 1.f / (float)C : 0.f;  // normalised start: uniform (log-one vector)
  vec[(FWD ? 0 : Eb) * 32 + lane] = act ? -lg2((float)C) : neg_inf();
  // step k handles edge t = FWD ? k : Eb-1-k; tiles advance by +-TT floats per step
  const int dT = FWD ? TT : -TT, dW = FWD ? CT : -CT, dV = FWD ? 32 : -32;
  const float* Mt = M + (FWD ? 0 : (Eb - 1) * TT) + jj;
  const float* Wt = W + (FWD ? 0 : (Eb - 1) * CT);
  float* vout = vec + (FWD ? 32 : (Eb - 1) * 32) + lane;
  float* lso = lSv + (FWD ? 0 : Eb - 1);
  for (int k = 0; k < Eb; ++k) {
    float mv[CT];
#pragma unroll
    for (int i = 0; i < CT; ++i) mv[i] = Mt[i * CT];
    float* pb = pbuf + (k & 1) * 32;
    pb[lane] = p;
    __syncwarp();
    float sa[4] = {0.f, 0.f, 0.f, 0.f}, Sa[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < CT; i += 4) {
      const float4 q = *reinterpret_cast<const float4*>(pb + i);  // broadcast
      const float4 w = *reinterpret_cast<const float4*>(Wt + i);
      sa[0] = fmaf(q.x, mv[i + 0], sa[0]);
      sa[1] = fmaf(q.y, mv[i + 1], sa[1]);
      sa[2] = fmaf(q.z, mv[i + 2], sa[2]);
      sa[3] = fmaf(q.w, mv[i + 3], sa[3]);
      Sa[0] = fmaf(q.x, w.x, Sa[0]);
      Sa[1] = fmaf(q.y, w.y, Sa[1]);
      Sa[2] = fmaf(q.z, w.z, Sa[2]);
      Sa[3] = fmaf(q.w, w.w, Sa[3]);
    }
    const float s = (sa[0] + sa[1]) + (sa[2] + sa[3]);
    const float S = (Sa[0] + Sa[1]) + (Sa[2] + Sa[3]);
    float lS = lg2(S);
    float np = __fdividef(s, S);
    float nh = lg2(s) - lS;
    const bool gated = act && !(s >= kGate);
    if (__any_sync(0xffffffffu, gated) || !(S >= kGate)) {
      // exact path for the gated lanes; exact normaliser when S itself is tiny
      const int t = FWD ? k : Eb - 1 - k;
      const float* vin = vec + (FWD ? t : t + 1) * 32;
      const float* xt = X + t * TT;
      const float tl = act ? (gated ? (FWD ? exact_lse(vin, xt + lane, CT, C)
                                           : exact_lse(vin, xt + lane * CT, 1, C))
                                    : lg2(s))
                           : neg_inf();
      if (!(S >= kGate)) lS = warp_lse2(tl);
      nh = (lS == neg_inf()) ? neg_inf() : tl - lS;
      np = act ? ex2(nh) : 0.f;
    }
    *vout = act ? nh : neg_inf();
    if (lane == 0) *lso = lS;
    p = act ? np : 0.f;
    Mt += dT;
    Wt += dW;
    vout += dV;
    lso += FWD ? 1 : -1;
#ifdef TS_PHASE_TIMING
    if (blockIdx.x == 0 && lane == 0 && k < 64) g_steps[FWD ? 0 : 1][k] = clock64();
#endif
  }
  __syncwarp();
  // frame offset O_E = log C + Σ_t (T_t + ln2 log2 S_t), summed in fp64 off the chain
  double part = 0.0;
  for (int t = lane; t < Eb; t += 32) part += (double)Tm[t] + kLn2 * (double)lSv[t];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  *Oout = (double)lg2((float)C) * kLn2 + part;
}

}  // namespace

template <int CT>
__global__ void __launch_bounds__(kSmallThreads) fb_small_kernel(SmallArgs a) {
  extern __shared__ __align__(16) float sm[];
  constexpr int TT = CT * CT;
  const int C = (int)a.C;
  const int64_t N = a.N, E = N - 1;
  const int CC = C * C;
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const SmallLayout Lay = small_layout(N, CT);
  float* X = sm + Lay.x;
  float* EX = sm + Lay.ex;
  float* EXT = sm + Lay.ext;
  float* RS = sm + Lay.rs;
  float* CS = sm + Lay.cs;
  float* Tm = sm + Lay.T;
  float* lS = sm + Lay.lS;
  float* lSb = sm + Lay.lSb;
  float* alpha = sm + Lay.alpha;
  float* beta = sm + Lay.beta;
  float* Ln = sm + Lay.Ln;
  float* pb = sm + Lay.pb;
  unsigned* sflag = reinterpret_cast<unsigned*>(sm + Lay.total - 4);

  const int64_t len = seq_len(a.lengths, b, N);
  float* mg = a.marg ? a.marg + b * E * CC : nullptr;
  if (len < 0) {  // BADLEN: logZ NaN, marginals 0
    if (mg)
      for (int64_t k = tid; k < E * CC; k += kSmallThreads) mg[k] = 0.f;
    if (tid == 0) {
      a.logz[b] = qnan();
      if (a.flags) a.flags[b] = TS_F_BADLEN;
    }
    return;
  }
  const int64_t Eb = len - 1;
  if (tid == 0) *sflag = 0u;
  PHASE(0);

  // ---- each warp stages its own tiles (rows into CT-strided SMEM rows) ----------------
  const float* src = a.pot + b * E * CC;
  const bool v4 = ((C & 3) == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
  for (int64_t t = warp; t < Eb; t += kSmallWarps) {
    float* xt = X + t * TT;
    const float* st = src + t * CC;
    if (v4) {
      const int q = C >> 2;
      for (int k = lane; k < C * q; k += 32) {
        const int i = k / q, c4 = k - i * q;
        cp_async16(xt + i * CT + 4 * c4, st + i * C + 4 * c4);
      }
    } else {
      for (int k = lane; k < CC; k += 32) {
        const int i = k / C, j = k - i * C;
        cp_async4(xt + i * CT + j, st + k);
      }
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  PHASE(1);
  // ---- prepass (same warp, same tiles): tile max, re-centred base-2 values, exps
  // (+ transposed copy), row / column sums ------------------------------------------------
  for (int64_t t = warp; t < Eb; t += kSmallWarps) {
    float* xt = X + t * TT;
    float* ex = EX + t * TT;
    float* ext = EXT + t * TT;
    constexpr int NE = (TT + 31) / 32;
    float v[NE];
    float mx = neg_inf();
    bool bad = false;
#pragma unroll
    for (int m = 0; m < NE; ++m) {
      const int k = lane + 32 * m;
      const int i = k / CT, j = k - (k / CT) * CT;
      const bool in = (k < TT) && (i < C) && (j < C);
      v[m] = in ? xt[k] : neg_inf();
      mx = fmaxf(mx, v[m]);
      bad |= (v[m] != v[m]) | (v[m] == pos_inf());
    }
    mx = warp_max(mx);
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(sflag, (unsigned)TS_F_NONFINITE);
    const float Tz = (mx == neg_inf()) ? 0.f : mx;  // all-masked tile: x' = -inf
    if (lane == 0) Tm[t] = Tz;
#pragma unroll
    for (int m = 0; m < NE; ++m) {
      const int k = lane + 32 * m;
      if (k < TT) {
        const int i = k / CT, j = k - (k / CT) * CT;
        const float x = (v[m] - Tz) * kLog2e;
        const float e = ex2(x);
        xt[k] = x;
        ex[k] = e;
        ext[j * CT + i] = e;
      }
    }
    __syncwarp();
    if (lane < CT) {
      float r = 0.f, c = 0.f;
#pragma unroll
      for (int q = 0; q < CT; ++q) {
        r += ext[q * CT + lane];  // row sum of EX (row = lane)
        c += ex[q * CT + lane];   // column sum of EX (column = lane)
      }
      RS[t * CT + lane] = r;
      CS[t * CT + lane] = c;
    }
  }
  __syncthreads();
  PHASE(2);
  if (*sflag & TS_F_NONFINITE) {
    if (mg)
      for (int64_t k = tid; k < E * CC; k += kSmallThreads) mg[k] = 0.f;
    if (tid == 0) {
      a.logz[b] = qnan();
      if (a.flags) a.flags[b] = TS_F_NONFINITE;
    }
    return;
  }

  if (warp == 0) {
    double O;
    sweep<true, CT>(X, EX, RS, alpha, lS, Tm, (int)Eb, C, lane, &O, pb);
    PHASEW(3);
    // logZ = O_E + ln2 log2 Σ_j 2^ah_E[j]  (the sum is 1 up to rounding)
    const float L = warp_lse2(alpha[Eb * 32 + lane]);
    if (lane == 0) {
      const bool empty = (L == neg_inf()) || (O == -INFINITY);
      a.logz[b] = empty ? neg_inf() : (float)(O + kLn2 * (double)L);
      if (empty) atomicOr(sflag, (unsigned)TS_F_EMPTY);
    }
  } else if (warp == 1 && mg) {
    double O;
    sweep<false, CT>(X, EXT, CS, beta, lSb, Tm, (int)Eb, C, lane, &O, pb + 64);
    PHASEW(4);
  }
  __syncthreads();
  PHASE(5);
  const unsigned fl = *sflag;
  if (tid == 0 && a.flags) a.flags[b] = fl;
  if (!mg) return;
  if (fl & TS_F_EMPTY) {
    for (int64_t k = tid; k < E * CC; k += kSmallThreads) mg[k] = 0.f;
    return;
  }
  // ---- node normalisers L_n, n = 1..Eb ---------------------------------------------------
  for (int64_t n = 1 + warp; n <= Eb; n += kSmallWarps) {
    const float Lv = warp_lse2(alpha[n * 32 + lane] + beta[n * 32 + lane]);
    if (lane == 0) Ln[n] = Lv;
  }
  __syncthreads();
  PHASE(6);
  // ---- marginals: one warp per edge, coalesced stores; zeros on padded edges --------------
  const int di = 32 / C, dj = 32 - di * C;
  for (int64_t t = warp; t < Eb; t += kSmallWarps) {
    const float cst = lS[t] + Ln[t + 1];
    const float* xt = X + t * TT;
    const float* at = alpha + t * 32;
    const float* bt = beta + (t + 1) * 32;
    float* out = mg + t * CC;
    int i = lane / C, j = lane - (lane / C) * C;
    for (int k = lane; k < CC; k += 32) {
      out[k] = ex2(at[i] + xt[i * CT + j] + bt[j] - cst);
      i += di;
      j += dj;
      if (j >= C) {
        j -= C;
        ++i;
      }
    }
  }
  for (int64_t k = Eb * CC + tid; k < E * CC; k += kSmallThreads) mg[k] = 0.f;
#ifdef TS_PHASE_TIMING
  __syncthreads();
  PHASE(7);
#endif
}

namespace {
template <int CT>
cudaError_t launch_small_ct(const SmallArgs& a, size_t smem, cudaStream_t st) {
  static std::atomic<uint64_t> attr_mask{0};  // one-time attribute setup per device
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_mask.load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(fb_small_kernel<CT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr_mask.fetch_or(bit);
  }
  fb_small_kernel<CT><<<(unsigned)a.B, kSmallThreads, smem, st>>>(a);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_small(const SmallArgs& a, cudaStream_t st) {
  const size_t smem = small_smem_bytes(a.N, a.C);
  switch (small_ct(a.C)) {
    case 4: return launch_small_ct<4>(a, smem, st);
    case 8: return launch_small_ct<8>(a, smem, st);
    case 12: return launch_small_ct<12>(a, smem, st);
    case 16: return launch_small_ct<16>(a, smem, st);
    case 20: return launch_small_ct<20>(a, smem, st);
    case 24: return launch_small_ct<24>(a, smem, st);
    case 28: return launch_small_ct<28>(a, smem, st);
    case 32: return launch_small_ct<32>(a, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tsb
