// fb_small.cu — one CTA per sequence, the whole sequence resident in shared memory:
// forward sweep (warp 0) and backward sweep (warp 1) run concurrently, then all warps
// compute the marginals.  Used when C <= 32 and 3*(N-1)*C*C floats fit in SMEM
// (BASELINE configs 1 and 2: the paper's Table 1 setting B=32, N=25, C=20).
//
// Per edge t (§5.2 P:252-256 forward, P:181-183 marginals,
// §6(c) P:330-331 stabilised product):
//   T_t  = max_ij l_t[i][j]                        (re-centring, natural units, exact)
//   x'   = (l_t - T_t) * log2 e,  EX = 2^x'        (prepass, all warps)
//   fwd:  a_i = 2^(ah_t[i] - m_t);  ah_{t+1}[j] = log2 sum_i a_i EX[i][j]
//   bwd:  b_j = 2^(bh_{t+1}[j] - m'_{t+1});  bh_t[i] = log2 sum_j EX[i][j] b_j
//   offsets O_{t+1} = O_t + ln2*m_t + T_t (fp64);  m_{t+1} = log2 C + max(ah_t) - m_t
//   (a lagged upper bound: a_i <= 1 always, the max-reduction is off the critical path)
//   gate: a sum below 2^-60 is recomputed exactly with the per-cell max of §6(c).
//   mu_t[i][j] = 2^(ah_t[i] + bh_{t+1}[j] + x'_ij - m_t - L_{t+1}),
//   L_n = log2 sum_j 2^(ah_n[j] + bh_n[j])   (= log2 Z in node n's frames)
#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

constexpr int kSmallThreads = 256;
constexpr int kSmallWarps = kSmallThreads / 32;

struct SmallLayout {
  int64_t x, ex, ext, T, alpha, beta, mF, Ln, total;  // float offsets
};

__host__ __device__ inline SmallLayout small_layout(int64_t N, int64_t C) {
  SmallLayout l;
  const int64_t E = N - 1, CC = C * C;
  l.x = 0;
  l.ex = l.x + E * CC;
  l.ext = l.ex + E * CC;
  l.T = l.ext + E * CC;
  l.alpha = l.T + E;
  l.beta = l.alpha + N * 32;
  l.mF = l.beta + N * 32;
  l.Ln = l.mF + N;
  l.total = l.Ln + N + 4;  // + flag word
  return l;
}

size_t small_smem_bytes(int64_t N, int64_t C) {
  return (size_t)small_layout(N, C).total * sizeof(float);
}

bool small_fits(int64_t N, int64_t C) {
  return C <= 32 && N >= 1 && small_smem_bytes(N, C) <= (size_t)200 * 1024;
}

__global__ void __launch_bounds__(kSmallThreads) fb_small_kernel(SmallArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int C = (int)a.C;
  const int64_t N = a.N, E = N - 1;
  const int CC = C * C;
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const SmallLayout Lay = small_layout(N, C);
  float* X = sm + Lay.x;
  float* EX = sm + Lay.ex;
  float* EXT = sm + Lay.ext;
  float* Tm = sm + Lay.T;
  float* alpha = sm + Lay.alpha;
  float* beta = sm + Lay.beta;
  float* mF = sm + Lay.mF;
  float* Ln = sm + Lay.Ln;
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
  const int64_t nused = Eb * CC;
  if (tid == 0) *sflag = 0u;

  // ---- stage l (the used edges) into SMEM with cp.async -------------------------------
  const float* src = a.pot + b * E * CC;
  if (nused > 0) {
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
      const int64_t n4 = nused >> 2;
      for (int64_t k = tid; k < n4; k += kSmallThreads) cp_async16(X + 4 * k, src + 4 * k);
      for (int64_t k = 4 * n4 + tid; k < nused; k += kSmallThreads) cp_async4(X + k, src + k);
    } else {
      for (int64_t k = tid; k < nused; k += kSmallThreads) cp_async4(X + k, src + k);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();

  // ---- prepass: per-tile max, re-centred base-2 values, exps (+ transposed copy) -------
  for (int64_t t = warp; t < Eb; t += kSmallWarps) {
    float* xt = X + t * CC;
    float mx = neg_inf();
    unsigned bad = 0u;
    for (int k = lane; k < CC; k += 32) {
      float v = xt[k];
      mx = fmaxf(mx, v);
      bad |= (v != v) | (v == pos_inf());
    }
    mx = warp_max(mx);
    bad = warp_or(bad);
    if (bad && lane == 0) atomicOr(sflag, (unsigned)TS_F_NONFINITE);
    const float Tz = (mx == neg_inf()) ? 0.f : mx;  // all-masked tile: x' = -inf
    if (lane == 0) Tm[t] = Tz;
    float* ext = EXT + t * CC;
    float* ex = EX + t * CC;
    for (int k = lane; k < CC; k += 32) {
      float x = (xt[k] - Tz) * kLog2e;
      float e = ex2(x);
      xt[k] = x;
      ex[k] = e;
      int i = k / C, j = k - i * C;
      ext[j * C + i] = e;
    }
  }
  __syncthreads();
  const unsigned pre = *sflag;
  if (pre & TS_F_NONFINITE) {
    if (mg)
      for (int64_t k = tid; k < E * CC; k += kSmallThreads) mg[k] = 0.f;
    if (tid == 0) {
      a.logz[b] = qnan();
      if (a.flags) a.flags[b] = TS_F_NONFINITE;
    }
    return;
  }

  const float log2C = lg2((float)C);
  const bool act = lane < C;
  const int jj = act ? lane : 0;

  if (warp == 0) {
    // ---- forward sweep: lane j owns column j ---------------------------------------------
    float ah = act ? 0.f : neg_inf();
    alpha[lane] = ah;
    float m = 0.f, mu = 0.f;
    double O = 0.0;
    __syncwarp();
    for (int64_t t = 0; t < Eb; ++t) {
      const float av = act ? ex2(ah - m) : 0.f;
      const float* ex = EX + t * CC;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      int i = 0;
      for (; i + 4 <= C; i += 4) {
        s0 = fmaf(__shfl_sync(0xffffffffu, av, i + 0), ex[(i + 0) * C + jj], s0);
        s1 = fmaf(__shfl_sync(0xffffffffu, av, i + 1), ex[(i + 1) * C + jj], s1);
        s2 = fmaf(__shfl_sync(0xffffffffu, av, i + 2), ex[(i + 2) * C + jj], s2);
        s3 = fmaf(__shfl_sync(0xffffffffu, av, i + 3), ex[(i + 3) * C + jj], s3);
      }
      for (; i < C; ++i) s0 = fmaf(__shfl_sync(0xffffffffu, av, i), ex[i * C + jj], s0);
      const float s = (s0 + s1) + (s2 + s3);
      float nh = lg2(s);
      if (act && !(s >= kGate)) {  // exact per-cell-max path (§6(c))
        const float* xt = X + t * CC;
        const float* at = alpha + t * 32;
        float q = neg_inf();
        for (int r = 0; r < C; ++r) q = fmaxf(q, at[r] + xt[r * C + lane]);
        if (q == neg_inf()) {
          nh = neg_inf();
        } else {
          float ss = 0.f;
          for (int r = 0; r < C; ++r) ss += ex2(at[r] + xt[r * C + lane] - q);
          nh = q + lg2(ss) - m;
        }
      }
      if (!act) nh = neg_inf();
      alpha[(t + 1) * 32 + lane] = nh;
      if (lane == 0) mF[t] = m;
      O += kLn2 * (double)m + (double)Tm[t];
      const float mu_next = warp_max(nh);
      const float m_next = (mu == neg_inf()) ? 0.f : (log2C + mu - m);
      mu = mu_next;
      m = m_next;
      ah = nh;
      __syncwarp();
    }
    const float L = warp_lse2(ah);
    if (lane == 0) {
      const double lz = (L == neg_inf()) ? -INFINITY : O + kLn2 * (double)L;
      a.logz[b] = (float)lz;
      if (L == neg_inf()) atomicOr(sflag, (unsigned)TS_F_EMPTY);
    }
  } else if (warp == 1 && mg) {
    // ---- backward sweep: lane i owns row i (reads the transposed exps) -------------------
    float bh = act ? 0.f : neg_inf();
    beta[Eb * 32 + lane] = bh;
    float m = 0.f, mu = 0.f;
    __syncwarp();
    for (int64_t t = Eb - 1; t >= 0; --t) {
      const float bv = act ? ex2(bh - m) : 0.f;
      const float* ext = EXT + t * CC;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      int j = 0;
      for (; j + 4 <= C; j += 4) {
        s0 = fmaf(__shfl_sync(0xffffffffu, bv, j + 0), ext[(j + 0) * C + jj], s0);
        s1 = fmaf(__shfl_sync(0xffffffffu, bv, j + 1), ext[(j + 1) * C + jj], s1);
        s2 = fmaf(__shfl_sync(0xffffffffu, bv, j + 2), ext[(j + 2) * C + jj], s2);
        s3 = fmaf(__shfl_sync(0xffffffffu, bv, j + 3), ext[(j + 3) * C + jj], s3);
      }
      for (; j < C; ++j) s0 = fmaf(__shfl_sync(0xffffffffu, bv, j), ext[j * C + jj], s0);
      const float s = (s0 + s1) + (s2 + s3);
      float nb = lg2(s);
      if (act && !(s >= kGate)) {
        const float* xt = X + t * CC + lane * C;
        const float* bt = beta + (t + 1) * 32;
        float q = neg_inf();
        for (int c = 0; c < C; ++c) q = fmaxf(q, xt[c] + bt[c]);
        if (q == neg_inf()) {
          nb = neg_inf();
        } else {
          float ss = 0.f;
          for (int c = 0; c < C; ++c) ss += ex2(xt[c] + bt[c] - q);
          nb = q + lg2(ss) - m;
        }
      }
      if (!act) nb = neg_inf();
      beta[t * 32 + lane] = nb;
      const float mu_next = warp_max(nb);
      const float m_next = (mu == neg_inf()) ? 0.f : (log2C + mu - m);
      mu = mu_next;
      m = m_next;
      bh = nb;
      __syncwarp();
    }
  }
  __syncthreads();
  const unsigned fl = *sflag;
  if (tid == 0 && a.flags) a.flags[b] = fl;
  if (!mg) return;
  if (fl & TS_F_EMPTY) {
    for (int64_t k = tid; k < E * CC; k += kSmallThreads) mg[k] = 0.f;
    return;
  }
  // ---- node normalisers L_n, n = 1..Eb ---------------------------------------------------
  for (int64_t n = 1 + warp; n <= Eb; n += kSmallWarps) {
    float v = act ? alpha[n * 32 + lane] + beta[n * 32 + lane] : neg_inf();
    float Lv = warp_lse2(v);
    if (lane == 0) Ln[n] = Lv;
  }
  __syncthreads();
  // ---- marginals (coalesced stores), zeros on padded edges --------------------------------
  for (int64_t k = tid; k < nused; k += kSmallThreads) {
    const int64_t t = k / CC;
    const int r = (int)(k - t * CC);
    const int i = r / C, j = r - i * C;
    const float u = alpha[t * 32 + i] + beta[(t + 1) * 32 + j] + X[k] - mF[t] - Ln[t + 1];
    mg[k] = ex2(u);
  }
  for (int64_t k = nused + tid; k < E * CC; k += kSmallThreads) mg[k] = 0.f;
}

cudaError_t launch_small(const SmallArgs& a, cudaStream_t st) {
  const size_t smem = small_smem_bytes(a.N, a.C);
  static bool attr_done = false;  // one-time attribute setup (max dynamic SMEM)
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(fb_small_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  fb_small_kernel<<<(unsigned)a.B, kSmallThreads, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace tsb
