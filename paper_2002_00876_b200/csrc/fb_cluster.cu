// fb_cluster.cu — short chains with C <= 32 (BASELINE configs 1-2; the paper's Table 1
// setting B=32, N=25, C=20): the chunked parallel scan of PAPER.md §6(a) mapped onto
// a thread-block CLUSTER of G CTAs per sequence (G SMs), exchanging chunk summaries
// through distributed shared memory (DSMEM).
//
// CTA `rank` of sequence b owns the contiguous edge chunk [t0, t1) (balanced split):
//   1. stage its tiles (cp.async), prepass: tile max T_t (re-centring), x' = (l - T) log2 e,
//      EX = 2^x' (+ transposed copy), row / column sums of EX.
//   2. chunk summary F = l_{t0} (x) ... (x) l_{t1-1} (C x C, log semiring): rows are
//      sum-normalised forward vectors (a small SIMT GEMM per edge) with fp64 row offsets;
//      exact log-space per-cell-max fallback (§6(c)) when flush-to-zero could
//      drop a term (a finite x' < -40 or a normalised value in (0, 2^-80)).
//   3. cluster barrier; read every peer's F through DSMEM.
//   4. boundary vectors: alpha_in = 0 (x) F_0 ... F_{rank-1} (warp 0),
//      beta_out = F_{rank+1} ... F_{G-1} (x) 0 (warp 1)   (exact log-space vector products).
//   5. local forward (warp 0) / backward (warp 1) sum-normalised sweeps from them
//      (s_j = Σ_i p_i EX[i][j], S = Σ_i p_i rowsum_i: no cross-lane reduction on the chain;
//      gate s < 2^-60 -> exact per-cell-max recomputation).
//   6. node normalisers L_n and marginals mu_t[i][j] = 2^(ah_t[i] + x'_ij + bh_{t+1}[j]
//      - log2 S_t - L_{t+1}); the last rank writes logZ and the flags.
// G = 1 degenerates to one CTA per sequence running the whole chain (no summary).
#include <cooperative_groups.h>

#include <atomic>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace tsb {

#ifdef TS_PHASE_TIMING
__device__ long long g_cl_phase[4096][10];
__device__ long long g_cl_steps[4][64];
#define CPHASE(k)                                                       \
  do {                                                                  \
    if (threadIdx.x == 0 && blockIdx.x < 4096) g_cl_phase[blockIdx.x][k] = clock64(); \
  } while (0)
#else
#define CPHASE(k) \
  do {            \
  } while (0)
#endif

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr float kTinyX = -40.f;
constexpr float kTinyP = 8.271806125530277e-25f;  // 2^-80

inline __host__ __device__ int ct_of(int64_t C) { return (int)(((C + 3) / 4) * 4); }

struct Layout {
  int64_t x, ex, ext, rs, cs, T, lS, lSb, alpha, beta, Ln, pb, P0, P1, Fh, Foff, Gh, Goff, vin,
      vout, flags, total;  // float offsets
};

__host__ __device__ inline Layout layout(int64_t EL, int CT, int G) {
  Layout l;
  const int64_t TT = (int64_t)CT * CT;
  auto a4 = [](int64_t v) { return (v + 3) & ~(int64_t)3; };
  l.x = 0;
  l.ex = l.x + EL * TT;
  l.ext = l.ex + EL * TT;
  l.rs = l.ext + EL * TT;
  l.cs = l.rs + EL * CT;
  l.T = l.cs + EL * CT;
  l.lS = a4(l.T + EL);
  l.lSb = a4(l.lS + EL);
  l.alpha = a4(l.lSb + EL);
  l.beta = l.alpha + (EL + 1) * 32;
  l.Ln = l.beta + (EL + 1) * 32;
  l.pb = a4(l.Ln + EL + 1);
  l.P0 = l.pb + 128;
  l.P1 = l.P0 + TT;
  l.Fh = l.P1 + TT;
  l.Foff = a4(l.Fh + TT);             // CT doubles
  l.Gh = l.Foff + 2 * CT;             // [G][TT]
  l.Goff = a4(l.Gh + (int64_t)G * TT);  // [G][CT] doubles
  l.vin = l.Goff + 2 * (int64_t)G * CT;  // [2][32] floats + [2] doubles
  l.vout = l.vin + 64;
  l.flags = l.vout + 8;
  l.total = l.flags + 8;
  return l;
}

__device__ __forceinline__ float exact_lse(const float* __restrict__ v, const float* __restrict__ X,
                                           int xs, int C) {
  float q = neg_inf();
  for (int r = 0; r < C; ++r) q = fmaxf(q, v[r] + X[r * xs]);
  if (q == neg_inf()) return neg_inf();
  float ss = 0.f;
  for (int r = 0; r < C; ++r) ss += ex2(v[r] + X[r * xs] - q);
  return q + lg2(ss);
}

__device__ __forceinline__ double warp_max_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, v, o);
    v = x > v ? x : v;
  }
  return v;
}

// Local sweep over `EL` tiles from a start log2 vector h0 (lane values) with natural offset
// O0.  FWD: lane j owns column j (M = EX, W = row sums); !FWD: lane i owns row i (M = EX^T,
// W = column sums).  Writes vec[node*32 + lane] (log2, sum-normalised frames) and lSv[t];
// returns the fp64 natural offset of the final node.
template <bool FWD, int CT>
__device__ double sweep(const float* __restrict__ X, const float* __restrict__ M,
                        const float* __restrict__ W, float* vec, float* lSv,
                        const float* __restrict__ Tm, int EL, int C, int lane, float h0, double O0,
                        float* pbuf) {
  constexpr int TT = CT * CT;
  const bool act = lane < C;
  const int jj = lane < CT ? lane : 0;
  // normalise the start vector: p = 2^(h0 - lse2(h0)), O += ln2 lse2(h0)
  const float L0 = warp_lse2(act ? h0 : neg_inf());
  double O = (L0 == neg_inf()) ? -INFINITY : O0 + kLn2 * (double)L0;
  float h = (act && L0 != neg_inf()) ? h0 - L0 : neg_inf();
  float p = act ? ex2(h) : 0.f;
  vec[(FWD ? 0 : EL) * 32 + lane] = h;
  const int dT = FWD ? TT : -TT, dW = FWD ? CT : -CT, dV = FWD ? 32 : -32;
  const float* Mt = M + (FWD ? 0 : (EL - 1) * TT) + jj;
  const float* Wt = W + (FWD ? 0 : (EL - 1) * CT);
  float* vout = vec + (FWD ? 32 : (EL - 1) * 32) + lane;
  float* lso = lSv + (FWD ? 0 : EL - 1);
  for (int k = 0; k < EL; ++k) {
    float mv[CT];
#pragma unroll
    for (int i = 0; i < CT; ++i) mv[i] = Mt[i * CT];
    float* pb = pbuf + (k & 1) * 32;
    pb[lane] = p;
    __syncwarp();
    float sa[4] = {0.f, 0.f, 0.f, 0.f}, Sa[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < CT; i += 4) {
      const float4 q = *reinterpret_cast<const float4*>(pb + i);
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
      const int t = FWD ? k : EL - 1 - k;
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
  }
  __syncwarp();
  double part = 0.0;
  for (int t = lane; t < EL; t += 32) part += (double)Tm[t] + kLn2 * (double)lSv[t];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  return O + part;
}

// Warp-level exact vector (x) matrix:  u_j = log Σ_r exp(v_r + F_r,j)  with v (lane r: log2
// value, natural offset vo) and F (log2 Fh[r][j] + natural row offsets Fo[r]).
__device__ void wvec_mat(float& v, double& vo, const float* Fh, const double* Fo, int C, int CT,
                         int lane, float* scr) {
  const bool act = lane < C;
  const double c = (act && v != neg_inf()) ? kLn2 * (double)v + Fo[lane] : -INFINITY;
  const double ref = warp_max_d(c);
  scr[lane] = (c == -INFINITY || ref == -INFINITY) ? neg_inf() : (float)((c - ref) * (double)kLog2e);
  __syncwarp();
  float u = neg_inf();
  if (act) u = exact_lse(scr, Fh + lane, CT, C);
  const float m = warp_max(u);
  __syncwarp();
  v = (act && m != neg_inf()) ? u - m : neg_inf();
  vo = (ref == -INFINITY || m == neg_inf()) ? 0.0 : vo + ref + kLn2 * (double)m;
}

// Warp-level exact matrix (x) vector:  u_r = log Σ_j exp(F_r,j + v_j).
__device__ void wmat_vec(float& v, double& vo, const float* Fh, const double* Fo, int C, int CT,
                         int lane, float* scr) {
  const bool act = lane < C;
  scr[lane] = act ? v : neg_inf();
  __syncwarp();
  float u = neg_inf();
  if (act) u = exact_lse(scr, Fh + lane * CT, 1, C);
  const double tot = (act && u != neg_inf()) ? Fo[lane] + vo + kLn2 * (double)u : -INFINITY;
  const double ref = warp_max_d(tot);
  __syncwarp();
  v = (tot == -INFINITY || ref == -INFINITY) ? neg_inf() : (float)((tot - ref) * (double)kLog2e);
  vo = (ref == -INFINITY) ? 0.0 : ref;
}

}  // namespace

template <int CT, int G>
__global__ void __launch_bounds__(kThreads, 1) fb_cluster_kernel(SmallArgs a) {
  extern __shared__ __align__(16) float sm[];
  constexpr int TT = CT * CT;
  const int C = (int)a.C;
  const int64_t N = a.N, E = N - 1;
  const int CC = C * C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int rank = (G > 1) ? (int)cg::this_cluster().block_rank() : 0;
  const int64_t b = blockIdx.x / G;
  const int64_t EL = (E + G - 1) / G;  // max chunk length (layout)
  const Layout Lay = layout(EL, CT, G);
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
  float* P0 = sm + Lay.P0;
  float* P1 = sm + Lay.P1;
  float* Fh = sm + Lay.Fh;
  double* Foff = reinterpret_cast<double*>(sm + Lay.Foff);
  float* Gh = sm + Lay.Gh;
  double* Goff = reinterpret_cast<double*>(sm + Lay.Goff);
  float* vin = sm + Lay.vin;
  unsigned* sflag = reinterpret_cast<unsigned*>(sm + Lay.flags);  // [0] nonfinite, [1] tiny

  const int64_t len = seq_len(a.lengths, b, N);
  float* mg = a.marg ? a.marg + b * E * CC : nullptr;
  if (len < 0) {  // BADLEN (uniform across the cluster): zeros, NaN logZ
    if (mg) {
      const int64_t q0 = E * CC * rank / G, q1 = E * CC * (rank + 1) / G;
      for (int64_t q = q0 + tid; q < q1; q += kThreads) mg[q] = 0.f;
    }
    if (rank == 0 && tid == 0) {
      a.logz[b] = qnan();
      if (a.flags) a.flags[b] = TS_F_BADLEN;
    }
    return;
  }
  const int64_t Eb = len - 1;
  // balanced split of this sequence's Eb edges over the G CTAs
  const int64_t base = Eb / G, extra = Eb - base * G;
  const int64_t t0 = rank * base + (rank < extra ? rank : extra);
  const int EL_me = (int)(base + (rank < extra ? 1 : 0));
  if (tid < 8) sflag[tid] = 0u;
  CPHASE(0);

  // ---- 1. stage this CTA's tiles and preprocess them ---------------------------------------
  const float* src = a.pot + (b * E + t0) * CC;
  const bool v4 = ((C & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.pot) & 15) == 0);
  if (v4) {  // all threads, flat over (tile, row, float4)
    const int q4 = C >> 2, per = C * q4;
    for (int q = tid; q < EL_me * per; q += kThreads) {
      const int t = q / per, r = q - (q / per) * per;
      const int i = r / q4, c4 = r - (r / q4) * q4;
      cp_async16(X + t * TT + i * CT + 4 * c4, src + (int64_t)t * CC + i * C + 4 * c4);
    }
  } else {
    for (int q = tid; q < EL_me * CC; q += kThreads) {
      const int t = q / CC, r = q - (q / CC) * CC;
      const int i = r / C, j = r - (r / C) * C;
      cp_async4(X + t * TT + i * CT + j, src + q);
    }
  }
  cp_async_commit();
  if (G > 1) cg::this_cluster().sync();  // flags zeroed in every CTA before any peer writes
  cp_async_wait<0>();
  __syncthreads();  // tiles and sflag init visible
  CPHASE(1);
  // prepass, block-wide over all (tile, element) pairs of this chunk:
  //   (a) tile max T_t (one warp per tile, strided) + NaN / +inf probe
  for (int t = warp; t < EL_me; t += kWarps) {
    const float* xt = X + t * TT;
    float mx = neg_inf();
    bool bad = false;
    for (int k = lane; k < TT; k += 32) {
      const int i = k / CT, j = k - (k / CT) * CT;
      if (i < C && j < C) {
        const float v = xt[k];
        mx = fmaxf(mx, v);
        bad |= (v != v) | (v == pos_inf());
      }
    }
    mx = warp_max(mx);
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&sflag[0], 1u);
    if (lane == 0) Tm[t] = (mx == neg_inf()) ? 0.f : mx;  // all-masked tile: x' = -inf
  }
  __syncthreads();
  //   (b) re-centred base-2 values, exps and the transposed exps, flat over the chunk
  {
    bool tiny = false;
    for (int q = tid; q < EL_me * TT; q += kThreads) {
      const int t = q / TT, k = q - (q / TT) * TT;
      const int i = k / CT, j = k - (k / CT) * CT;
      const bool in = (i < C) && (j < C);
      const float x = in ? (X[q] - Tm[t]) * kLog2e : neg_inf();
      tiny |= (x < kTinyX) & (x != neg_inf());
      const float e = ex2(x);
      X[q] = x;
      EX[q] = e;
      EXT[t * TT + j * CT + i] = e;
    }
    if (__any_sync(0xffffffffu, tiny) && lane == 0) atomicOr(&sflag[1], 1u);
  }
  __syncthreads();
  //   (c) row / column sums of EX (one thread per (tile, index))
  for (int q = tid; q < EL_me * CT; q += kThreads) {
    const int t = q / CT, l = q - (q / CT) * CT;
    const float* ex = EX + t * TT;
    const float* ext = EXT + t * TT;
    float r = 0.f, c = 0.f;
#pragma unroll
    for (int u = 0; u < CT; ++u) {
      r += ext[u * CT + l];
      c += ex[u * CT + l];
    }
    RS[q] = r;
    CS[q] = c;
  }
  __syncthreads();
  CPHASE(2);

  // ---- 2. chunk summary F (only when there are peers to combine with) --------------------
  if (G > 1) {
    if (EL_me == 0) {
      for (int q = tid; q < TT; q += kThreads) Fh[q] = ((q / CT) == (q % CT)) ? 0.f : neg_inf();
      for (int r = tid; r < CT; r += kThreads) Foff[r] = 0.0;
    } else {
      bool exact = sflag[1] != 0u;
      if (!exact) {
        // fast: rows are sum-normalised forward vectors, P <- P EX_t / rowsum (SIMT GEMM)
        for (int q = tid; q < TT; q += kThreads) {
          P0[q] = ((q / CT) == (q % CT) && (q / CT) < C) ? 1.f : 0.f;
          P1[q] = 0.f;
        }
        for (int r = tid; r < CT; r += kThreads) Foff[r] = 0.0;
        __syncthreads();
        float* Pc = P0;
        float* Pn = P1;
        constexpr int RPW = (CT + kWarps - 1) / kWarps;  // rows per warp (unrolled: ILP)
        constexpr int SW = (CT + RPW - 1) / RPW;          // warps with rows
        for (int t = 0; t < EL_me; ++t) {
          if (warp < SW) {
            const float* ex = EX + t * TT;
            const float* rs = RS + t * CT;
            const int jj = lane < CT ? lane : 0;
            float e[CT];
#pragma unroll
            for (int i = 0; i < CT; ++i) e[i] = ex[i * CT + jj];
            float acc[RPW], S[RPW];
#pragma unroll
            for (int x = 0; x < RPW; ++x) {
              acc[x] = 0.f;
              S[x] = 0.f;
            }
#pragma unroll
            for (int i = 0; i < CT; i += 4) {
              const float4 w = *reinterpret_cast<const float4*>(rs + i);
#pragma unroll
              for (int x = 0; x < RPW; ++x) {
                const int r = warp * RPW + x;
                const float4 pv = *reinterpret_cast<const float4*>(Pc + r * CT + i);  // broadcast
                acc[x] = fmaf(pv.x, e[i], acc[x]);
                S[x] = fmaf(pv.x, w.x, S[x]);
                acc[x] = fmaf(pv.y, e[i + 1], acc[x]);
                S[x] = fmaf(pv.y, w.y, S[x]);
                acc[x] = fmaf(pv.z, e[i + 2], acc[x]);
                S[x] = fmaf(pv.z, w.z, S[x]);
                acc[x] = fmaf(pv.w, e[i + 3], acc[x]);
                S[x] = fmaf(pv.w, w.w, S[x]);
              }
            }
            const double Tt = (double)Tm[t];
#pragma unroll
            for (int x = 0; x < RPW; ++x) {
              const int r = warp * RPW + x;
              if (r < C) {
                const float pn = (S[x] > 0.f) ? __fdividef(acc[x], S[x]) : 0.f;
                if (pn > 0.f && pn < kTinyP) atomicOr(&sflag[1], 1u);
                if (lane < CT) Pn[r * CT + lane] = (lane < C) ? pn : 0.f;
                if (lane == 0) {
                  const double o = Foff[r];
                  Foff[r] = (S[x] > 0.f && o != -INFINITY) ? o + Tt + kLn2 * (double)lg2(S[x])
                                                           : -INFINITY;
                }
              }
            }
          }
#ifdef TS_PHASE_TIMING
          if (blockIdx.x == 0 && tid == 0 && t < 64) g_cl_steps[0][t] = clock64();
#endif
          __syncthreads();
#ifdef TS_PHASE_TIMING
          if (blockIdx.x == 0 && tid == 0 && t < 64) g_cl_steps[1][t] = clock64();
#endif
          float* tmp = Pc;
          Pc = Pn;
          Pn = tmp;
        }
        exact = sflag[1] != 0u;
        if (!exact) {
          for (int q = tid; q < TT; q += kThreads) {
            const int r = q / CT;
            const float pv = Pc[q];
            Fh[q] = (pv > 0.f && Foff[r] != -INFINITY) ? lg2(pv) : neg_inf();
          }
          __syncthreads();
          for (int r = tid; r < CT; r += kThreads)
            if (Foff[r] == -INFINITY) Foff[r] = 0.0;
        }
      }
      if (exact) {
        // exact log-space product chain with the per-cell max of §6(c)
        for (int q = tid; q < TT; q += kThreads) P0[q] = ((q / CT) == (q % CT)) ? 0.f : neg_inf();
        for (int r = tid; r < CT; r += kThreads) Foff[r] = 0.0;
        __syncthreads();
        float* Pc = P0;
        float* Pn = P1;
        for (int t = 0; t < EL_me; ++t) {
          const float* xt = X + t * TT;
          for (int q = tid; q < TT; q += kThreads) {
            const int r = q / CT, j = q - (q / CT) * CT;
            Pn[q] = (r < C && j < C) ? exact_lse(Pc + r * CT, xt + j, CT, C) : neg_inf();
          }
          __syncthreads();
          for (int r = tid; r < CT; r += kThreads) {
            float m = neg_inf();
            for (int j = 0; j < C; ++j) m = fmaxf(m, Pn[r * CT + j]);
            const bool dead = (m == neg_inf()) || Foff[r] == -INFINITY || r >= C;
            for (int j = 0; j < CT; ++j) Pn[r * CT + j] = dead ? neg_inf() : Pn[r * CT + j] - m;
            Foff[r] = dead ? -INFINITY : Foff[r] + (double)Tm[t] + kLn2 * (double)m;
          }
          __syncthreads();
          float* tmp = Pc;
          Pc = Pn;
          Pn = tmp;
        }
        for (int q = tid; q < TT; q += kThreads) Fh[q] = Pc[q];
        __syncthreads();
        for (int r = tid; r < CT; r += kThreads)
          if (Foff[r] == -INFINITY) Foff[r] = 0.0;
      }
    }
    // ---- 3. exchange: push this CTA's summary and flags into every peer (DSMEM stores),
    // then ONE cluster barrier (release/acquire) makes them visible everywhere -----------
    cg::cluster_group cl = cg::this_cluster();
    __syncthreads();
    CPHASE(3);
    for (int g = 0; g < G; ++g) {
      float* rG = cl.map_shared_rank(Gh, g) + rank * TT;
      double* rO = cl.map_shared_rank(Goff, g) + rank * CT;
      for (int q = tid; q < TT; q += kThreads) rG[q] = Fh[q];
      for (int r = tid; r < CT; r += kThreads) rO[r] = Foff[r];
      if (tid == 0 && sflag[0]) atomicOr(cl.map_shared_rank(&sflag[2], g), 1u);
    }
    cl.sync();
    CPHASE(4);
    CPHASE(5);
  } else {
    if (tid == 0) sflag[2] = sflag[0];
  }
  __syncthreads();
  const bool nonfinite = (sflag[2] | sflag[0]) != 0u;
  if (nonfinite) {
    if (mg) {
      const int64_t q0 = (rank == 0) ? 0 : t0 * CC;
      const int64_t q1 = (rank == G - 1) ? E * CC : (t0 + EL_me) * CC;
      for (int64_t q = q0 + tid; q < q1; q += kThreads) mg[q] = 0.f;
    }
    if (rank == G - 1 && tid == 0) {
      a.logz[b] = qnan();
      if (a.flags) a.flags[b] = TS_F_NONFINITE;
    }
    return;
  }

  // ---- 4. boundary vectors, 5. local sweeps ---------------------------------------------------
  if (warp == 0) {
    float v = lane < C ? 0.f : neg_inf();
    double vo = 0.0;
    for (int g = 0; g < rank; ++g) wvec_mat(v, vo, Gh + g * TT, Goff + g * CT, C, CT, lane, vin);
    const double O = sweep<true, CT>(X, EX, RS, alpha, lS, Tm, EL_me, C, lane, v, vo, pb);
    if (rank == G - 1) {  // the end of the chain: logZ = O_E + ln2 log2 Σ_j 2^ah_E[j]
      const float L = warp_lse2(alpha[EL_me * 32 + lane]);
      if (lane == 0) {
        const bool empty = (L == neg_inf()) || (O == -INFINITY) || (O != O);
        a.logz[b] = empty ? neg_inf() : (float)(O + kLn2 * (double)L);
        if (a.flags) a.flags[b] = empty ? TS_F_EMPTY : 0u;
      }
    }
  } else if (warp == 1 && mg) {
    float v = lane < C ? 0.f : neg_inf();
    double vo = 0.0;
    for (int g = G - 1; g > rank; --g)
      wmat_vec(v, vo, Gh + g * TT, Goff + g * CT, C, CT, lane, vin + 32);
    sweep<false, CT>(X, EXT, CS, beta, lSb, Tm, EL_me, C, lane, v, vo, pb + 64);
  }
  __syncthreads();
  CPHASE(6);
  if (!mg) return;
  // ---- 6. node normalisers and marginals ----------------------------------------------------
  for (int n = warp; n <= EL_me; n += kWarps) {
    const float Lv = warp_lse2(alpha[n * 32 + lane] + beta[n * 32 + lane]);
    if (lane == 0) Ln[n] = Lv;
  }
  __syncthreads();
  const bool dead = !(Ln[0] > neg_inf());  // Z = 0 (EMPTY): every node normaliser is -inf
  float* out0 = mg + t0 * CC;
  if (dead) {
    for (int64_t q = tid; q < (int64_t)EL_me * CC; q += kThreads) out0[q] = 0.f;
  } else {
    for (int q = tid; q < EL_me * TT; q += kThreads) {
      const int t = q / TT, k = q - (q / TT) * TT;
      const int i = k / CT, j = k - (k / CT) * CT;
      if (i < C && j < C)
        out0[(int64_t)t * CC + i * C + j] =
            ex2(alpha[t * 32 + i] + X[q] + beta[(t + 1) * 32 + j] - lS[t] - Ln[t + 1]);
    }
  }
  if (rank == G - 1)
    for (int64_t q = Eb * CC + tid; q < E * CC; q += kThreads) mg[q] = 0.f;
#ifdef TS_PHASE_TIMING
  __syncthreads();
  CPHASE(7);
#endif
}

// ====================================================================================
// host side
// ====================================================================================
namespace {
template <int CT, int G>
cudaError_t launch_ct(const SmallArgs& a, size_t smem, cudaStream_t st) {
  static std::atomic<uint64_t> mask{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(mask.load() & bit)) {
    cudaError_t e = cudaFuncSetAttribute(fb_cluster_kernel<CT, G>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return e;
    mask.fetch_or(bit);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(a.B * G));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fb_cluster_kernel<CT, G>, a);
}

template <int G>
cudaError_t launch_g(const SmallArgs& a, size_t smem, cudaStream_t st) {
  switch (ct_of(a.C)) {
    case 4: return launch_ct<4, G>(a, smem, st);
    case 8: return launch_ct<8, G>(a, smem, st);
    case 12: return launch_ct<12, G>(a, smem, st);
    case 16: return launch_ct<16, G>(a, smem, st);
    case 20: return launch_ct<20, G>(a, smem, st);
    case 24: return launch_ct<24, G>(a, smem, st);
    case 28: return launch_ct<28, G>(a, smem, st);
    case 32: return launch_ct<32, G>(a, smem, st);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace

int cluster_g(int64_t B, int64_t N, int sms) {
  const int64_t E = N - 1;
  int G = 1;
  while (G < 4 && B * (2 * G) <= sms && E >= 4 * (2 * G)) G *= 2;  // >= 4 edges per CTA
  return G;
}

size_t cluster_smem_bytes(int64_t N, int64_t C, int G) {
  const int64_t E = N - 1;
  const int64_t EL = (E + G - 1) / G;
  return (size_t)layout(EL, ct_of(C), G).total * sizeof(float);
}

bool cluster_fits(int64_t N, int64_t C, int G) {
  return C <= 32 && N >= 1 && cluster_smem_bytes(N, C, G) <= (size_t)200 * 1024;
}

cudaError_t launch_cluster(const SmallArgs& a, int G, cudaStream_t st) {
  const size_t smem = cluster_smem_bytes(a.N, a.C, G);
  switch (G) {
    case 1: return launch_g<1>(a, smem, st);
    case 2: return launch_g<2>(a, smem, st);
    case 4: return launch_g<4>(a, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tsb
