// semimarkov.cu — semi-Markov CRF log-partition and marginals (Table 1
// 'Semi-Markov', "similar parallel approach ... semi-Markov", P:311;
// reading R17: pot [B][N-1][K][C][C], l[b,n,k-1,c1,c2] scores a segment covering the k
// steps n -> n+k with label c2 after label c1 at node n; K = 1 is the linear chain).
//
// Segmental forward-backward, one CTA per sequence: the first GS threads (GS = 128 or 256
// >= C) run the forward recursion, the next GS the backward one concurrently; within a
// group S = 8/4/2/1 lanes share a label (C * S <= GS), each taking every S-th candidate
// (k, c') as an online (max, sum) over chunks of 4 loads, merged by shuffles:
//   alpha_p[c] = LSE_{k <= min(K,p), c'} alpha_{p-k}[c'] + l[p-k, k-1, c', c]
//   beta_p[c]  = LSE_{k <= min(K,E-p), c'} l[p, k-1, c, c'] + beta_{p+k}[c']
// with the per-cell max of §6(c) and node vectors stored normalised (max 0) with
// fp64 natural offsets (the last K+1 vectors also in an SMEM ring).  Then all threads write
//   mu[n,k-1,c1,c2] = exp(alpha_n[c1] + l[n,k-1,c1,c2] + beta_{n+k}[c2] - A)
// (0 for parts beyond the sequence).  Flags as the linear chain.  With K = 1 this is also
// the exact fallback of ts_logpartition / ts_marginals for long chains with 128 < C <= 256.
#include <atomic>

#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

namespace {
template <int GS>
__device__ __forceinline__ float group_max(float v, float* red, int gw, int bar_id) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) red[gw] = v;
  named_bar(bar_id, GS);
  float r = red[0];
  for (int k = 1; k < GS / 32; ++k) r = fmaxf(r, red[k]);
  named_bar(bar_id, GS);
  return r;
}
}  // namespace

// lanes per label: the largest power of two <= 8 with C * S <= GS
__device__ __forceinline__ int semi_split(int C, int GS) {
  int S = 8;
  while (S > 1 && C * S > GS) S >>= 1;
  return S;
}

// GS = threads per recursion group: 128 (C <= 128) or 256 (C <= 256)
template <int GS>
__global__ void __launch_bounds__(2 * GS, 1) semimarkov_kernel(SemiArgs a) {
  constexpr int kSmG = GS;
  extern __shared__ __align__(16) float ssm[];
  const int C = (int)a.C, K = (int)a.K;
  const int64_t N = a.N, E = N - 1, KCC = (int64_t)K * C * C;
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, grp = tid / kSmG, c = tid % kSmG, gw = c >> 5;
  const int R = K + 1;                                   // ring rows
  float* ring = ssm + grp * R * kSmG;                    // [2][R][128] normalised vectors
  double* ooff = reinterpret_cast<double*>(ssm + 2 * R * kSmG) + grp * R;  // [2][R] offsets
  float* red0 = reinterpret_cast<float*>(reinterpret_cast<double*>(ssm + 2 * R * kSmG) + 2 * R);
  float* red = red0 + grp * 8;                           // [2][8] per-group reductions
  unsigned* sflag = reinterpret_cast<unsigned*>(red0 + 16);  // one word for the CTA
  float* stage = reinterpret_cast<float*>(sflag + 4);         // [2][GS] label values
  float* stg = stage + 2 * kSmG + grp * 2 * K * C * C;        // [2 grp][2][K][C][C] (a.staged)
  const float* pb = a.pot + b * E * KCC;
  float* mg = a.marg ? a.marg + b * E * KCC : nullptr;
  const int64_t len = seq_len(a.lengths, b, N);
  if (len < 0) {
    if (mg)
      for (int64_t q = tid; q < E * KCC; q += blockDim.x) mg[q] = 0.f;
    if (tid == 0) {
      a.logz[b] = qnan();
      if (a.flags) a.flags[b] = TS_F_BADLEN;
    }
    return;
  }
  const int64_t Eb = len - 1;
  if (tid == 0) *sflag = 0u;
  __syncthreads();
  const bool act = c < C;
  float* vh = (grp == 0 ? a.ah : a.bh) + b * N * C;      // [N][C] normalised vectors
  double* vo = (grp == 0 ? a.ao : a.bo) + b * N;         // [N] natural offsets
  bool bad = false;
  // node 0 (forward) / node Eb (backward): log-one vector, offset 0
  {
    const int64_t n0 = grp == 0 ? 0 : Eb;
    ring[(n0 % R) * kSmG + c] = act ? 0.f : neg_inf();
    if (act) vh[n0 * C + c] = 0.f;
    if (c == 0) {
      ooff[n0 % R] = 0.0;
      vo[n0] = 0.0;
    }
  }
  // staged: the tiles a step reads are copied to SMEM with cp.async one step ahead
  // (forward node p: l[p-k][k-1]; backward node p: l[p][k-1], k <= K within the sequence)
  const int64_t CC2 = (int64_t)C * C;
  auto issue = [&](int64_t ss) {
    const int64_t pp = grp == 0 ? ss : Eb - ss;
    const int km = (int)(grp == 0 ? (pp < K ? pp : K) : (Eb - pp < K ? Eb - pp : K));
    float* dst = stg + (ss & 1) * K * CC2;
    for (int k = 1; k <= km; ++k) {
      const float* src = grp == 0 ? pb + (pp - k) * KCC + (int64_t)(k - 1) * CC2
                                  : pb + pp * KCC + (int64_t)(k - 1) * CC2;
      for (int64_t r = c; r < CC2; r += kSmG) cp_async4(dst + (k - 1) * CC2 + r, src + r);
    }
    cp_async_commit();
  };
  if (a.staged && Eb >= 1) {
    issue(1);
    cp_async_wait<0>();
  }
  named_bar(1 + grp, kSmG);
  // S lanes per label: lane sl of label cl takes the candidates (k, c') with c' = sl (mod S),
  // an online (max, sum) over chunks of 4 loads, merged by shuffles
  const int S = semi_split(C, kSmG);
  const int cl = c / S, sl = c - cl * S;
  const bool actl = cl < C;
  for (int64_t s = 1; s <= Eb; ++s) {
    const int64_t p = grp == 0 ? s : Eb - s;             // node computed at this step
    const int64_t pr = grp == 0 ? p - 1 : p + 1;         // reference node (offset frame)
    const int kmax = (int)(grp == 0 ? (p < K ? p : K) : (Eb - p < K ? Eb - p : K));
    const double oref = ooff[pr % R];
    float m = neg_inf(), sum = 0.f;
    if (a.staged && s + 1 <= Eb) issue(s + 1);
    if (actl) {
      // per segment length k: the offset delta and the source rows are hoisted; lane sl
      // takes c' = sl, sl + S, ... in chunks of 4 (online (max, sum), log2 units)
      for (int k = 1; k <= kmax; ++k) {
        const int64_t q = grp == 0 ? p - k : p + k;      // the other end of the segment
        const int qs = (int)(q % R);
        const float d = (float)(ooff[qs] - oref);
        const float* vq = ring + qs * kSmG;
        const float* lt = a.staged ? stg + (s & 1) * K * CC2 + (k - 1) * CC2
                          : (grp == 0 ? pb + (p - k) * KCC + (int64_t)(k - 1) * CC2
                                      : pb + p * KCC + (int64_t)(k - 1) * CC2);
        // forward reads column cl (stride C), backward row cl (stride 1)
        const float* lp = grp == 0 ? lt + cl : lt + (int64_t)cl * C;
        const int ls = grp == 0 ? C : 1;
        for (int c0 = sl; c0 < C; c0 += 4 * S) {
          float x[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c2 = c0 + u * S;
            float xv = neg_inf();
            if (c2 < C) {
              const float lv = lp[c2 * ls];
              bad |= (lv != lv) | (lv == pos_inf());
              xv = (d + vq[c2] + lv) * kLog2e;
            }
            x[u] = xv;
          }
          const float bm = fmaxf(fmaxf(x[0], x[1]), fmaxf(x[2], x[3]));
          if (bm != neg_inf()) {
            const float mn = fmaxf(m, bm);
            float acc = (m == neg_inf()) ? 0.f : sum * ex2(m - mn);
#pragma unroll
            for (int u = 0; u < 4; ++u) acc += ex2(x[u] - mn);
            m = mn;
            sum = acc;
          }
        }
      }
    }
    for (int o = 1; o < S; o <<= 1) {  // merge the S partial (max, sum) pairs (log2 units)
      const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
      const float s2 = __shfl_xor_sync(0xffffffffu, sum, o);
      const float M2 = fmaxf(m, m2);
      if (M2 != neg_inf()) {
        sum = ((m == neg_inf()) ? 0.f : sum * ex2(m - M2)) + ((m2 == neg_inf()) ? 0.f : s2 * ex2(m2 - M2));
        m = M2;
      }
    }
    // the label's value, moved to thread c = label (the layout of the ring and vh)
    const float lval = (m == neg_inf()) ? neg_inf() : (m + lg2(sum)) * (float)kLn2;
    if (actl && sl == 0) stage[grp * kSmG + cl] = lval;
    named_bar(1 + grp, kSmG);
    const bool act2 = c < C;
    const float val = act2 ? stage[grp * kSmG + c] : neg_inf();
    const float M = group_max<GS>(val, red, gw, 1 + grp);
    const bool dead = (M == neg_inf());
    const float nv = (act && !dead) ? val - M : neg_inf();
    ring[(p % R) * kSmG + c] = nv;
    if (act) vh[p * C + c] = nv;
    if (c == 0) {
      const double o = dead ? oref : oref + (double)M;
      ooff[p % R] = o;
      vo[p] = dead ? -INFINITY : o;
    }
    if (a.staged) cp_async_wait<0>();
    named_bar(1 + grp, kSmG);
  }
  if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0) atomicOr(sflag, (unsigned)TS_F_NONFINITE);
  __syncthreads();
  // logZ = O_E + LSE_c alpha_hat_E[c]  (forward group, warp 0)
  if (tid < 32) {
    float x = neg_inf();
    for (int q = tid; q < C; q += 32) x = fmaxf(x, a.ah[(b * N + Eb) * C + q]);
    x = warp_max(x);
    float s = 0.f;
    if (x != neg_inf())
      for (int q = tid; q < C; q += 32) s += ex2((a.ah[(b * N + Eb) * C + q] - x) * kLog2e);
    s = warp_sum(s);
    if (tid == 0) {
      const double oE = a.ao[b * N + Eb];
      const unsigned f = *sflag;
      float lz;
      unsigned fl = 0;
      if (f & TS_F_NONFINITE) {
        lz = qnan();
        fl = TS_F_NONFINITE;
      } else if (x == neg_inf() || !(oE > -INFINITY)) {
        lz = neg_inf();
        fl = TS_F_EMPTY;
      } else {
        lz = (float)(oE + (double)x + kLn2 * (double)lg2(s));
        a.zbuf[b] = oE + (double)x + kLn2 * (double)lg2(s);
      }
      a.logz[b] = lz;
      if (a.flags) a.flags[b] = fl;
      *sflag = fl;
    }
  }
  __syncthreads();
  if (!mg) return;
  const unsigned fl = *sflag;
  const double A = fl ? 0.0 : a.zbuf[b];
  const float* ah = a.ah + b * N * C;
  const float* bh = a.bh + b * N * C;
  const double* ao = a.ao + b * N;
  const double* bo = a.bo + b * N;
  // one (n, k) tile at a time: the offsets are per tile, element indices need no 64-bit
  // division; warps take tiles round-robin, lanes stride the C x C elements
  const int64_t CCt = (int64_t)C * C;
  const int nw = blockDim.x >> 5, wid = tid >> 5, ln = tid & 31;
  for (int64_t nk = wid; nk < E * K; nk += nw) {
    const int64_t n = nk / K;
    const int k = (int)(nk - n * K) + 1;
    float* mq = mg + nk * CCt;
    const bool live = !fl && n + k <= Eb;
    const double offd = live ? ao[n] + bo[n + k] - A : 0.0;
    const bool ok = live && offd > -INFINITY;
    const float off = (float)offd;
    const float* lq = pb + nk * CCt;
    const float* ahn = ah + n * C;
    const float* bhn = bh + (n + k) * C;
    for (int r = ln; r < (int)CCt; r += 32) {
      float v = 0.f;
      if (ok) {
        const int c1 = r / C, c2 = r - c1 * C;
        const float x = off + ahn[c1] + lq[r] + bhn[c2];
        v = (x == neg_inf()) ? 0.f : ex2(x * kLog2e);
      }
      mq[r] = v;
    }
  }
}

constexpr size_t kSemiStageBytes = 96 * 1024;  // staged tiles only when 4 K C^2 floats fit

cudaError_t launch_semimarkov(const SemiArgs& a0, cudaStream_t st) {
  SemiArgs a = a0;
  const int R = (int)a.K + 1;
  const int GS = a.C <= 128 ? 128 : 256;
  const size_t stage_bytes = (size_t)4 * a.K * a.C * a.C * sizeof(float);
  a.staged = stage_bytes <= kSemiStageBytes ? 1 : 0;
  const size_t smem = (size_t)2 * R * GS * sizeof(float) + (size_t)2 * R * sizeof(double) +
                      16 * sizeof(float) + 16 + (size_t)2 * GS * sizeof(float) +
                      (a.staged ? stage_bytes : 0);
  static std::atomic<uint64_t> attr128{0}, attr256{0};
  const int mx = (int)((size_t)2 * 17 * 256 * sizeof(float) + 2 * 17 * sizeof(double) + 64 +
                       2 * 256 * sizeof(float) + kSemiStageBytes);
  cudaError_t ea = GS == 128 ? smem_optin_once(semimarkov_kernel<128>, attr128, mx)
                             : smem_optin_once(semimarkov_kernel<256>, attr256, mx);
  if (ea != cudaSuccess) return ea;
  if (GS == 128)
    semimarkov_kernel<128><<<(unsigned)a.B, 256, smem, st>>>(a);
  else
    semimarkov_kernel<256><<<(unsigned)a.B, 512, smem, st>>>(a);
  return cudaGetLastError();
}

// ---- semi-Markov Viterbi (max semiring over R17 segmentations; reading R18) -------------
//   delta_p[c] = max_{k <= min(K,p), c'} delta_{p-k}[c'] + l[p-k, k-1, c', c]
// thread c owns label c; candidates are scanned in (k asc, c' asc) order with a strict >, so
// the backpointer is the first maximiser (the oracle's rule); the last K+1 delta vectors
// live in an SMEM ring.  fp32 adds: exact (= the fp64 oracle) on dyadic inputs whose
// partial sums fit 24 bits.  The end label is the smallest arg-max; one thread backtracks.
__global__ void __launch_bounds__(256) semimarkov_viterbi_kernel(SemiVitArgs a) {
  extern __shared__ __align__(16) float vsm[];
  const int C = (int)a.C, K = (int)a.K, R = K + 1, NT = blockDim.x;
  const int64_t N = a.N, E = N - 1, KCC = (int64_t)K * C * C;
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  float* ring = vsm;                                    // [R][NT]
  float* rv = ring + R * NT;                            // [8] block arg-max values
  int* ri = reinterpret_cast<int*>(rv + 8);             // [8] block arg-max labels
  unsigned* sflag = reinterpret_cast<unsigned*>(ri + 8);
  float* stg = reinterpret_cast<float*>(sflag + 4);     // [2][K][C][C] staged tiles (a.staged)
  const float* pb = a.pot + b * E * KCC;
  int32_t* sg = a.seg + b * N;
  uint16_t* bp = a.bp + b * N * C;
  const int64_t len = seq_len(a.lengths, b, N);
  for (int64_t p = tid; p < N; p += NT) sg[p] = -1;
  if (len < 0) {
    if (tid == 0) {
      a.score[b] = qnan();
      if (a.flags) a.flags[b] = TS_F_BADLEN;
    }
    return;
  }
  const int64_t Eb = len - 1;
  const bool act = tid < C;                             // final arg-max: thread = label
  const int S = semi_split(C, 256);                     // step loop: S lanes per label
  const int cl = tid / S, sl = tid - cl * S;
  const bool actl = cl < C;
  if (tid == 0) *sflag = 0u;
  ring[tid] = act ? 0.f : neg_inf();                    // delta_0 = 0 (node 0 in slot 0)
  // staged: the tiles node p reads (l[p-k][k-1], k <= min(K,p)) are copied to SMEM with
  // cp.async one step ahead, so each step waits for one memory round trip, not one per batch
  const int64_t CC2 = (int64_t)C * C;
  auto issue = [&](int64_t pp) {
    float* dst = stg + (pp & 1) * K * CC2;
    const int km = (int)(pp < K ? pp : K);
    for (int k = 1; k <= km; ++k) {
      const float* src = pb + (pp - k) * KCC + (int64_t)(k - 1) * CC2;
      for (int64_t r = tid; r < CC2; r += NT) cp_async4(dst + (k - 1) * CC2 + r, src + r);
    }
    cp_async_commit();
  };
  if (a.staged && Eb >= 1) {
    issue(1);
    cp_async_wait<0>();
  }
  __syncthreads();
  bool bad = false;
  for (int64_t p = 1; p <= Eb; ++p) {
    float best = neg_inf();
    int arg = 0;
    if (a.staged && p + 1 <= Eb) issue(p + 1);
    if (actl) {
      const int kmax = (int)(p < K ? p : K);
      for (int k = 1; k <= kmax; ++k) {
        const float* dq = ring + (int)((p - k) % R) * NT;
        const float* col = a.staged ? stg + (p & 1) * K * CC2 + (k - 1) * CC2 + cl
                                    : pb + (p - k) * KCC + (int64_t)(k - 1) * CC2 + cl;
        for (int i0 = sl; i0 < C; i0 += 4 * S) {
          float lv[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) lv[u] = (i0 + u * S < C) ? col[(int64_t)(i0 + u * S) * C] : neg_inf();
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * S;
            bad |= (lv[u] != lv[u]) | (lv[u] == pos_inf());
            const float v = dq[i < C ? i : 0] + lv[u];
            if (v > best) {
              best = v;
              arg = (k - 1) * C + i;
            }
          }
        }
      }
    }
    // merge the S lanes of a label: max value, ties -> the smallest (k, c') (= serial order)
    for (int o = 1; o < S; o <<= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
      if (ov > best || (ov == best && oa < arg)) {
        best = ov;
        arg = oa;
      }
    }
    if (actl && sl == 0) {
      bp[p * C + cl] = (uint16_t)arg;
      ring[(p % R) * NT + cl] = best;
    }
    if (a.staged) cp_async_wait<0>();
    __syncthreads();
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(sflag, 1u);
  // end label: the smallest c attaining max delta_Eb
  float v = act ? ring[(Eb % R) * NT + tid] : neg_inf();
  int idx = (act && v != neg_inf()) ? tid : 0x7fffffff;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
  if (lane == 0) {
    rv[w] = v;
    ri[w] = idx;
  }
  __syncthreads();
  if (tid == 0) {
    float bv = rv[0];
    int bi = ri[0];
    for (int q = 1; q < NT / 32; ++q)
      if (rv[q] > bv || (rv[q] == bv && ri[q] < bi)) {
        bv = rv[q];
        bi = ri[q];
      }
    unsigned fl = 0;
    if (*sflag) {
      fl = TS_F_NONFINITE;
      a.score[b] = qnan();
    } else if (bv == neg_inf()) {
      fl = TS_F_EMPTY;
      a.score[b] = neg_inf();
    } else {
      a.score[b] = bv;
      int c = bi;
      int64_t p = Eb;
      while (p > 0) {
        sg[p] = c;
        const int v16 = bp[p * C + c];
        const int k = v16 / C + 1;
        c = v16 - (k - 1) * C;
        p -= k;
      }
      sg[0] = c;
    }
    if (a.flags) a.flags[b] = fl;
  }
}

constexpr size_t kSemiStageMax = 96 * 1024;  // staged tiles only when 2 K C^2 floats fit

int semimarkov_viterbi_threads(int64_t C) {
  int S = 8;
  while (S > 1 && C * S > 256) S >>= 1;
  return (int)(((C * S + 31) / 32) * 32);
}

size_t semimarkov_viterbi_smem(int64_t C, int64_t K, bool staged) {
  const int NT = semimarkov_viterbi_threads(C);
  return (size_t)(K + 1) * NT * sizeof(float) + 8 * sizeof(float) + 8 * sizeof(int) + 16 +
         (staged ? (size_t)2 * K * C * C * sizeof(float) : 0);
}

cudaError_t launch_semimarkov_viterbi(const SemiVitArgs& a0, cudaStream_t st) {
  SemiVitArgs a = a0;
  a.staged = (size_t)2 * a.K * a.C * a.C * sizeof(float) <= kSemiStageMax ? 1 : 0;
  const int NT = semimarkov_viterbi_threads(a.C);
  const size_t smem = semimarkov_viterbi_smem(a.C, a.K, a.staged != 0);
  static std::atomic<uint64_t> attr{0};  // one bit per device (the attribute is per device)
  const cudaError_t ea = smem_optin_once(semimarkov_viterbi_kernel, attr,
                                         (int)(semimarkov_viterbi_smem(256, 16, false) + kSemiStageMax));
  if (ea != cudaSuccess) return ea;
  semimarkov_viterbi_kernel<<<(unsigned)a.B, NT, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace tsb
