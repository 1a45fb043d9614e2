// fb_stream.cu — streaming forward / backward sweeps of the log semiring for chains
// whose tiles do not all fit in SMEM (C <= 128).  One CTA per (sequence, time chunk);
// C x C edge tiles stream HBM -> SMEM through a multi-stage cp.async ring.
//
// Forward (thread j owns column j; §5.2, §6(c)):
//   M_j = max_i l[i][j],  T = max_j M_j  (tile re-centring, natural units)
//   s_j = sum_i a_i 2^((l_ij - M_j) log2 e),  a_i = 2^(ah_t[i] - m_t) <= 1
//   ah_{t+1}[j] = (M_j - T) log2 e + log2 s_j      (frame O_{t+1} = O_t + ln2 m_t + T, fp64)
//   m_{t+1} = log2 C + max_i ah_t[i] - m_t         (lagged bound; reduction off the chain)
//   gate: s_j < 2^-60 -> exact per-cell max recomputation (the §6(c) formula).
// Backward (thread i owns row i; explicit backward scan, not autodiff — P:187 replaced):
//   bh_t[i] = (R_i - T) log2 e + log2 sum_j 2^((l_ij - R_i) log2 e) b_j,  b_j = 2^(bh_{t+1}[j] - m'_{t+1})
//   mu_t[i][j] = 2^(ah_t[i] + bh_{t+1}[j] + (l_ij - T) log2 e - m_t - L_{t+1})
//   L_n = log2 sum_k 2^(ah_n[k] + bh_n[k])  (log2 Z in node n's frames)
#include <atomic>

#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

namespace {

__host__ __device__ inline int fwd_tile_floats(int C) { return ((C * C) + 3) & ~3; }
__host__ __device__ inline int bwd_stride(int C, bool vec4) { return tile_stride(C, vec4); }
__host__ __device__ inline int bwd_tile_floats(int C, bool vec4) {
  return ((C * bwd_stride(C, vec4)) + 3) & ~3;
}

// block-wide max over one float per thread; `red` has >= nwarps floats; all threads get it.
__device__ __forceinline__ float block_max(float v, float* red, int nwarps) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = v;
  __syncthreads();
  float r = red[0];
  for (int k = 1; k < nwarps; ++k) r = fmaxf(r, red[k]);
  __syncthreads();
  return r;
}

// block-wide log2-sum-exp2 of one value per thread (-inf for inactive threads).
__device__ __forceinline__ float block_lse2(float v, float* redm, float* reds, int nwarps) {
  float wm = warp_max(v);
  float e = (wm == neg_inf()) ? 0.f : ex2(v - wm);
  float ws = warp_sum(e);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    redm[w] = wm;
    reds[w] = ws;
  }
  __syncthreads();
  float M = redm[0];
  for (int k = 1; k < nwarps; ++k) M = fmaxf(M, redm[k]);
  float S = 0.f;
  if (M != neg_inf())
    for (int k = 0; k < nwarps; ++k) S += (redm[k] == neg_inf()) ? 0.f : reds[k] * ex2(redm[k] - M);
  __syncthreads();
  return (M == neg_inf()) ? neg_inf() : M + lg2(S);
}

}  // namespace

// Thread layout (both kernels): NT = 256 threads = G groups x CW lanes, CW = C rounded up to
// a multiple of 32.  Forward: lane j of group g owns column j, rows [g*R, g*R + R); backward:
// lane i of group g owns row i, columns [g*R, g*R + R).  Each step: phase A (all groups,
// partial max + partial exp-shifted sum) -> barrier -> phase B (group 0 merges the G partials
// online-softmax style and finalises the vector) -> barrier.  Many short independent chains
// per SM instead of one long one (latency hiding).
constexpr int kNT = 256;
__host__ __device__ inline int cw_of(int C) { return ((C + 31) / 32) * 32; }

// ====================================================================================
// Forward sweep
// ====================================================================================
template <int CT, bool VEC4>
__global__ void __launch_bounds__(kNT) fwd_sweep_kernel(SweepArgs a, int S) {
  extern __shared__ __align__(16) float sm[];
  const int C = CT > 0 ? CT : (int)a.C, CC = C * C;
  const int64_t N = a.N, E = N - 1, P = a.P, L = a.L;
  const int64_t b = blockIdx.x / P, k = blockIdx.x - (blockIdx.x / P) * P;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  constexpr int NW = kNT / 32;
  const int CW = cw_of(C), G = kNT / CW, NW0 = CW / 32;
  const int g = tid / CW, j = tid - g * CW;
  const int R = (C + G - 1) / G, r0 = g * R, r1 = min(C, r0 + R);
  const int TF = fwd_tile_floats(C);
  float* ring = sm;
  float* a_s = ring + (size_t)S * TF;  // [2][CW]
  float* ah_s = a_s + 2 * CW;          // [2][CW]
  float* pm = ah_s + 2 * CW;           // [G][CW] partial column max
  float* ps = pm + kNT;                // [G][CW] partial sums
  float* red_T = ps + kNT;             // [NW]
  float* red_mu = red_T + NW;          // [2][NW]
  float* red_x = red_mu + 2 * NW;      // [2*NW]

  const int64_t len = seq_len(a.lengths, b, N);
  if (len < 0) {
    if (k == 0 && a.final_in_fwd && tid == 0) {
      a.logz[b] = qnan();
      if (a.flags) a.flags[b] = TS_F_BADLEN;
    }
    return;
  }
  const int64_t Eb = len - 1;
  const int64_t t0 = k * L;
  if (t0 >= Eb && k > 0) return;  // chunk beyond this sequence's end
  const int64_t t1 = (t0 + L < Eb) ? t0 + L : Eb;
  const int64_t nsteps = t1 - t0;
  const bool last = (t1 == Eb);
  const bool act = (j < C);          // this lane's column exists
  const bool own = act && (g == 0);  // finalises column j
  const int64_t bk = b * P + k;
  const float* potb = a.pot + b * E * (int64_t)CC;

  // start vector (chunk 0: log-one; otherwise alpha_in from the scan tree)
  float ah = own ? (a.alpha_in ? a.alpha_in[bk * C + j] : 0.f) : neg_inf();
  double O = a.alpha_in_off ? a.alpha_in_off[bk] : 0.0;
  float mu = block_max(ah, red_x, NW);
  float m = (mu == neg_inf()) ? 0.f : mu;
  if (a.alpha_hat && own) a.alpha_hat[(b * N + t0) * C + j] = ah;

  for (int u = 0; u < S - 1; ++u) {
    if (u < nsteps)
      stage_tile(ring + (size_t)(u % S) * TF, potb + (t0 + u) * (int64_t)CC, C, C, VEC4, tid, kNT);
    cp_async_commit();
  }
  if (g == 0) {
    a_s[j] = own ? ex2(ah - m) : 0.f;
    ah_s[j] = ah;
  }
  cp_async_wait_dyn(S - 2);
  __syncthreads();

  const float log2C = lg2((float)C);
  unsigned bad = 0u;
  int buf = 0;
  for (int64_t u = 0; u < nsteps; ++u) {
    const int64_t t = t0 + u;
    {
      const int64_t uu = u + S - 1;
      if (uu < nsteps)
        stage_tile(ring + (size_t)(uu % S) * TF, potb + (t0 + uu) * (int64_t)CC, C, C, VEC4, tid,
                   kNT);
      cp_async_commit();
    }
    const float* tile = ring + (size_t)(u % S) * TF;
    const float* av = a_s + buf * CW;
    // ---- phase A: partial column max and exp-shifted partial dot product -------------------
    float M = neg_inf(), s = 0.f;
    if (act && r0 < r1) {
      float m0 = neg_inf(), m1 = neg_inf();
      int i = r0;
      for (; i + 2 <= r1; i += 2) {
        m0 = fmaxf(m0, tile[i * C + j]);
        m1 = fmaxf(m1, tile[(i + 1) * C + j]);
      }
      if (i < r1) m0 = fmaxf(m0, tile[i * C + j]);
      M = fmaxf(m0, m1);
      if (M != neg_inf()) {
        float s0 = 0.f, s1 = 0.f;
        i = r0;
        for (; i + 2 <= r1; i += 2) {
          s0 = fmaf(av[i], ex2((tile[i * C + j] - M) * kLog2e), s0);
          s1 = fmaf(av[i + 1], ex2((tile[(i + 1) * C + j] - M) * kLog2e), s1);
        }
        if (i < r1) s0 = fmaf(av[i], ex2((tile[i * C + j] - M) * kLog2e), s0);
        s = s0 + s1;
      }
    }
    pm[g * CW + j] = M;
    ps[g * CW + j] = s;
    {
      const float wm = warp_max(M);
      if (lane == 0) red_T[w] = wm;
    }
    __syncthreads();
    float T = red_T[0];
#pragma unroll
    for (int q = 1; q < NW; ++q) T = fmaxf(T, red_T[q]);
    const float Tz = (T == neg_inf()) ? 0.f : T;
    const float m_next = (mu == neg_inf()) ? 0.f : (log2C + mu - m);
    // ---- phase B: every group merges the G partials of its column (redundantly, no idle
    // warps); group 0 finalises ah_{t+1}[j] ---------------------------------------------------
    {
      float nh = neg_inf();
      if (act) {
        float Mj = neg_inf();
        for (int q = 0; q < G; ++q) Mj = fmaxf(Mj, pm[q * CW + j]);
        if (Mj != neg_inf()) {
          float sj = 0.f;
          for (int q = 0; q < G; ++q) {
            const float mq = pm[q * CW + j];
            if (mq != neg_inf()) sj = fmaf(ps[q * CW + j], ex2((mq - Mj) * kLog2e), sj);
          }
          nh = (Mj - Tz) * kLog2e + lg2(sj);
          if (g == 0 && !(sj >= kGate)) {  // exact per-cell-max path (also reached by NaN)
            const float* ahv = ah_s + buf * CW;
            float q = neg_inf();
            for (int i = 0; i < C; ++i) q = fmaxf(q, ahv[i] + (tile[i * C + j] - Tz) * kLog2e);
            if (q == neg_inf()) {
              nh = neg_inf();
            } else {
              float ss = 0.f;
              for (int i = 0; i < C; ++i) ss += ex2(ahv[i] + (tile[i * C + j] - Tz) * kLog2e - q);
              nh = q + lg2(ss) - m;
            }
            if (sj != sj) nh = qnan();
          }
        }
        if (g == 0) {
          if (nh != nh || Mj == pos_inf()) bad = 1u;
          if (a.alpha_hat && t + 1 < t1) a.alpha_hat[(b * N + t + 1) * C + j] = nh;
        }
      }
      if (g == 0) {
        ah_s[(buf ^ 1) * CW + j] = nh;
        a_s[(buf ^ 1) * CW + j] = act ? ex2(nh - m_next) : 0.f;
        const float wm = warp_max(nh);
        if (lane == 0) red_mu[(buf ^ 1) * NW + w] = wm;
        ah = nh;
      }
    }
    if (tid == 0) {
      if (a.mlag) a.mlag[b * N + t] = m;
      if (a.tmax) a.tmax[b * E + t] = Tz;
    }
    O += kLn2 * (double)m + (double)Tz;
    cp_async_wait_dyn(S - 2);
    __syncthreads();
    float mx = red_mu[(buf ^ 1) * NW];
    for (int q = 1; q < NW0; ++q) mx = fmaxf(mx, red_mu[(buf ^ 1) * NW + q]);
    mu = mx;
    m = m_next;
    buf ^= 1;
  }
  cp_async_wait<0>();
  if (a.alpha_end && own) a.alpha_end[bk * C + j] = ah;
  if (a.alpha_end_off && tid == 0) a.alpha_end_off[bk] = O;
  // NONFINITE: any NaN/+inf propagates to a NaN column (0 * NaN = NaN in the dot product)
  const unsigned anybad = __syncthreads_or(bad);
  if (anybad && tid == 0 && a.wflags) atomicOr(&a.wflags[b], (unsigned)WF_NONFINITE);
  if (a.final_in_fwd && last) {
    const float Lz = block_lse2(own ? ah : neg_inf(), red_x, red_x + NW, NW);
    if (tid == 0) {
      uint32_t fl = 0;
      float lz;
      if (anybad) {
        fl = TS_F_NONFINITE;
        lz = qnan();
      } else if (Lz == neg_inf()) {
        fl = TS_F_EMPTY;
        lz = neg_inf();
      } else {
        lz = (float)(O + kLn2 * (double)Lz);
      }
      a.logz[b] = lz;
      if (a.flags) a.flags[b] = fl;
    }
  }
}

// ====================================================================================
// Backward sweep + marginals
// ====================================================================================
template <int CT, bool VEC4>
__global__ void __launch_bounds__(kNT) bwd_sweep_kernel(SweepArgs a, int S) {
  extern __shared__ __align__(16) float sm[];
  const int C = CT > 0 ? CT : (int)a.C, CC = C * C;
  const int64_t N = a.N, E = N - 1, P = a.P, L = a.L;
  const int64_t b = blockIdx.x / P, k = blockIdx.x - (blockIdx.x / P) * P;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  constexpr int NW = kNT / 32;
  const int CW = cw_of(C), G = kNT / CW, NW0 = CW / 32;
  const int g = tid / CW, i = tid - g * CW;
  int R = (C + G - 1) / G;
  if (VEC4) R = (R + 3) & ~3;
  const int c0 = min(C, g * R), c1 = min(C, c0 + R);
  const int SB = bwd_stride(C, VEC4);
  const int TF = bwd_tile_floats(C, VEC4);
  float* ring = sm;
  float* b_s = ring + (size_t)S * TF;  // [2][CW] b values
  float* bh_s = b_s + 2 * CW;          // [2][CW] bh values
  float* pr = bh_s + 2 * CW;           // [G][CW] partial row max
  float* ps = pr + kNT;                // [G][CW] partial sums
  float* red_mu = ps + kNT;            // [2][NW]
  float* red_lm = red_mu + 2 * NW;     // [2][NW]
  float* red_ls = red_lm + 2 * NW;     // [2][NW]
  float* red_x = red_ls + 2 * NW;      // [2*NW]

  const int64_t len = seq_len(a.lengths, b, N);
  float* mgb = a.marg + b * E * (int64_t)CC;
  if (len < 0) {  // BADLEN: chunk 0 zeroes everything
    if (k == 0) {
      for (int64_t q = tid; q < E * CC; q += kNT) mgb[q] = 0.f;
      if (tid == 0) {
        a.logz[b] = qnan();
        if (a.flags) a.flags[b] = TS_F_BADLEN;
      }
    }
    return;
  }
  const int64_t Eb = len - 1;
  const int64_t t0 = k * L;
  if (t0 >= Eb && k > 0) return;
  const int64_t t1 = (t0 + L < Eb) ? t0 + L : Eb;
  const int64_t nsteps = t1 - t0;
  const bool last = (t1 == Eb);
  const bool act = (i < C);
  const bool own = act && (g == 0);
  const int64_t bk = b * P + k;
  const float* potb = a.pot + b * E * (int64_t)CC;
  const uint32_t wf = a.wflags ? a.wflags[b] : 0u;

  // end-of-chunk vectors: beta_out (tree) or log-one; alpha in the chunk's own frame
  float bh = own ? (a.beta_out ? a.beta_out[bk * C + i] : 0.f) : neg_inf();
  const float ahe = own ? a.alpha_end[bk * C + i] : neg_inf();
  float Lnext = block_lse2(own ? ahe + bh : neg_inf(), red_x, red_x + NW, NW);
  float mu = block_max(bh, red_x, NW);
  float m = (mu == neg_inf()) ? 0.f : mu;

  const bool dead = (wf & WF_NONFINITE) || !(Lnext > neg_inf());  // also NaN (remote segment)
  if (last && !a.no_final) {  // zero the padded tail, publish logZ and flags
    for (int64_t q = Eb * CC + tid; q < E * CC; q += kNT) mgb[q] = 0.f;
    if (tid == 0) {
      uint32_t fl = 0;
      float lz;
      if (wf & WF_NONFINITE) {
        fl = TS_F_NONFINITE;
        lz = qnan();
      } else if (Lnext == neg_inf()) {
        fl = TS_F_EMPTY;
        lz = neg_inf();
      } else {
        const double Oa = a.alpha_end_off[bk];
        const double Ob = a.beta_out_off ? a.beta_out_off[bk] : 0.0;
        lz = (float)(Oa + Ob + kLn2 * (double)Lnext);
      }
      if (a.logz) a.logz[b] = lz;
      if (a.flags) a.flags[b] = fl;
    }
  }
  if (last && a.no_final)
    for (int64_t q = Eb * CC + tid; q < E * CC; q += kNT) mgb[q] = 0.f;
  if (dead) {
    for (int64_t q = t0 * CC + tid; q < t1 * CC; q += kNT) mgb[q] = 0.f;
    return;
  }

  for (int u = 0; u < S - 1; ++u) {
    if (u < nsteps)
      stage_tile(ring + (size_t)(u % S) * TF, potb + (t1 - 1 - u) * (int64_t)CC, C, SB, VEC4, tid,
                 kNT);
    cp_async_commit();
  }
  if (g == 0) {
    b_s[i] = own ? ex2(bh - m) : 0.f;
    bh_s[i] = bh;
  }
  cp_async_wait_dyn(S - 2);
  __syncthreads();

  const float log2C = lg2((float)C);
  int buf = 0;
  float aht = (act && nsteps > 0) ? a.alpha_hat[(b * N + t1 - 1) * C + i] : neg_inf();
  for (int64_t u = 0; u < nsteps; ++u) {
    const int64_t t = t1 - 1 - u;
    {
      const int64_t uu = u + S - 1;
      if (uu < nsteps)
        stage_tile(ring + (size_t)(uu % S) * TF, potb + (t1 - 1 - uu) * (int64_t)CC, C, SB, VEC4,
                   tid, kNT);
      cp_async_commit();
    }
    const float* tile = ring + (size_t)(u % S) * TF;
    const float* bv = b_s + buf * CW;
    const float* bhv = bh_s + buf * CW;
    const float Tt = a.tmax[b * E + t];
    const float mt = a.mlag[b * N + t];
    const float aht_cur = aht;
    if (act && u + 1 < nsteps) aht = a.alpha_hat[(b * N + t - 1) * C + i];  // prefetch
    // ---- phase A: partial row max, partial sum, and this group's marginals ------------------
    float Rg = neg_inf(), s = 0.f;
    if (act && c0 < c1) {
      const float* row = tile + i * SB;
      float* mrow = mgb + ((int64_t)t * C + i) * C;
      const float cst = aht_cur - mt - Lnext;
      if (VEC4) {
        for (int c = c0; c < c1; c += 4) {
          const float4 v = *reinterpret_cast<const float4*>(row + c);
          Rg = fmaxf(Rg, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
        }
        for (int c = c0; c < c1; c += 4) {
          const float4 v = *reinterpret_cast<const float4*>(row + c);
          const float4 bb = *reinterpret_cast<const float4*>(bv + c);
          const float4 hh = *reinterpret_cast<const float4*>(bhv + c);
          if (Rg != neg_inf()) {
            s = fmaf(ex2((v.x - Rg) * kLog2e), bb.x, s);
            s = fmaf(ex2((v.y - Rg) * kLog2e), bb.y, s);
            s = fmaf(ex2((v.z - Rg) * kLog2e), bb.z, s);
            s = fmaf(ex2((v.w - Rg) * kLog2e), bb.w, s);
          }
          float4 mu4;
          mu4.x = ex2(cst + hh.x + (v.x - Tt) * kLog2e);
          mu4.y = ex2(cst + hh.y + (v.y - Tt) * kLog2e);
          mu4.z = ex2(cst + hh.z + (v.z - Tt) * kLog2e);
          mu4.w = ex2(cst + hh.w + (v.w - Tt) * kLog2e);
          *reinterpret_cast<float4*>(mrow + c) = mu4;
        }
      } else {
        for (int c = c0; c < c1; ++c) Rg = fmaxf(Rg, row[c]);
        for (int c = c0; c < c1; ++c) {
          const float v = row[c];
          if (Rg != neg_inf()) s = fmaf(ex2((v - Rg) * kLog2e), bv[c], s);
          mrow[c] = ex2(cst + bhv[c] + (v - Tt) * kLog2e);
        }
      }
    }
    pr[g * CW + i] = Rg;
    ps[g * CW + i] = s;
    __syncthreads();
    const float m_next = (mu == neg_inf()) ? 0.f : (log2C + mu - m);
    // ---- phase B (group 0): merge, finalise bh_t[i], reductions for the next step -----------
    if (g == 0) {
      float nb = neg_inf();
      if (act) {
        float Ri = neg_inf();
        for (int q = 0; q < G; ++q) Ri = fmaxf(Ri, pr[q * CW + i]);
        if (Ri != neg_inf()) {
          float si = 0.f;
          for (int q = 0; q < G; ++q) {
            const float rq = pr[q * CW + i];
            if (rq != neg_inf()) si = fmaf(ps[q * CW + i], ex2((rq - Ri) * kLog2e), si);
          }
          nb = (Ri - Tt) * kLog2e + lg2(si);
          if (!(si >= kGate)) {  // exact per-cell-max path
            const float* row = tile + i * SB;
            float q = neg_inf();
            for (int c = 0; c < C; ++c) q = fmaxf(q, (row[c] - Tt) * kLog2e + bhv[c]);
            if (q == neg_inf()) {
              nb = neg_inf();
            } else {
              float ss = 0.f;
              for (int c = 0; c < C; ++c) ss += ex2((row[c] - Tt) * kLog2e + bhv[c] - q);
              nb = q + lg2(ss) - m;
            }
          }
        }
      }
      b_s[(buf ^ 1) * CW + i] = act ? ex2(nb - m_next) : 0.f;
      bh_s[(buf ^ 1) * CW + i] = nb;
      const float wm = warp_max(nb);
      const float v = act ? aht_cur + nb : neg_inf();
      const float lm = warp_max(v);
      const float le = (lm == neg_inf()) ? 0.f : ex2(v - lm);
      const float ls = warp_sum(le);
      if (lane == 0) {
        red_mu[(buf ^ 1) * NW + w] = wm;
        red_lm[(buf ^ 1) * NW + w] = lm;
        red_ls[(buf ^ 1) * NW + w] = ls;
      }
    }
    cp_async_wait_dyn(S - 2);
    __syncthreads();
    {
      const float* rm = red_mu + (buf ^ 1) * NW;
      const float* lmv = red_lm + (buf ^ 1) * NW;
      const float* lsv = red_ls + (buf ^ 1) * NW;
      float mx = rm[0], LM = lmv[0];
      for (int q = 1; q < NW0; ++q) {
        mx = fmaxf(mx, rm[q]);
        LM = fmaxf(LM, lmv[q]);
      }
      float LS = 0.f;
      if (LM != neg_inf())
        for (int q = 0; q < NW0; ++q) LS += (lmv[q] == neg_inf()) ? 0.f : lsv[q] * ex2(lmv[q] - LM);
      Lnext = (LM == neg_inf()) ? neg_inf() : LM + lg2(LS);
      mu = mx;
    }
    m = m_next;
    buf ^= 1;
  }
  cp_async_wait<0>();
}

// ====================================================================================
// host launchers
// ====================================================================================
namespace {
int fwd_stages(int C) {
  const size_t tile = (size_t)fwd_tile_floats(C) * 4;
  const size_t budget = (C > 64) ? 192 * 1024 : 96 * 1024;
  int S = (int)(budget / tile);
  return S < 2 ? 2 : (S > 8 ? 8 : S);
}
int bwd_stages(int C, bool vec4) {
  const size_t tile = (size_t)bwd_tile_floats(C, vec4) * 4;
  const size_t budget = (C > 64) ? 200 * 1024 : 96 * 1024;
  int S = (int)(budget / tile);
  return S < 2 ? 2 : (S > 8 ? 8 : S);
}
std::atomic<uint64_t> g_attr_fwd[64], g_attr_bwd[64];  // per-device masks, one per kernel id

template <typename K>
cudaError_t set_smem_once(K kern, std::atomic<uint64_t>* masks, int bit) {
  return smem_optin_once(kern, masks[bit], 220 * 1024);
}
}  // namespace

size_t fwd_smem_bytes(int64_t C, int stages) {
  const int CW = cw_of((int)C), NW = kNT / 32;
  return ((size_t)stages * fwd_tile_floats((int)C) + 4 * CW + 2 * kNT + 5 * NW) * sizeof(float);
}
size_t bwd_smem_bytes(int64_t C, int stages) {
  const bool vec4 = (C % 4) == 0;
  const int CW = cw_of((int)C), NW = kNT / 32;
  return ((size_t)stages * bwd_tile_floats((int)C, vec4) + 4 * CW + 2 * kNT + 8 * NW) * sizeof(float);
}

cudaError_t launch_fwd(const SweepArgs& a, cudaStream_t st) {
  if (stream2_ok(a)) return launch_fwd2(a, st);
  const int C = (int)a.C;
  const bool vec4 = (C % 4) == 0 && (reinterpret_cast<uintptr_t>(a.pot) & 15) == 0;
  const int S = fwd_stages(C);
  const size_t smem = fwd_smem_bytes(C, S);
  const dim3 grid((unsigned)(a.B * a.P)), block(kNT);
  cudaError_t e;
#define TS_FWD(CTV, V4, BIT)                                                                \
  do {                                                                                   \
    if ((e = set_smem_once(fwd_sweep_kernel<CTV, V4>, g_attr_fwd, BIT)) != cudaSuccess) \
      return e;                                                                          \
    fwd_sweep_kernel<CTV, V4><<<grid, block, smem, st>>>(a, S);                          \
  } while (0)
  if (vec4 && C == 64) TS_FWD(64, true, 0);
  else if (vec4 && C == 128) TS_FWD(128, true, 1);
  else if (vec4 && C == 32) TS_FWD(32, true, 2);
  else if (vec4) TS_FWD(0, true, 3);
  else TS_FWD(0, false, 4);
#undef TS_FWD
  return cudaGetLastError();
}

cudaError_t launch_bwd(const SweepArgs& a, cudaStream_t st) {
  if (stream2_ok(a)) return launch_bwd2(a, st);
  const int C = (int)a.C;
  const bool vec4 = (C % 4) == 0 && (reinterpret_cast<uintptr_t>(a.pot) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(a.marg) & 15) == 0;
  const int S = bwd_stages(C, vec4);
  const size_t smem = bwd_smem_bytes(C, S);
  const dim3 grid((unsigned)(a.B * a.P)), block(kNT);
  cudaError_t e;
#define TS_BWD(CTV, V4, BIT)                                                                \
  do {                                                                                   \
    if ((e = set_smem_once(bwd_sweep_kernel<CTV, V4>, g_attr_bwd, BIT)) != cudaSuccess) \
      return e;                                                                          \
    bwd_sweep_kernel<CTV, V4><<<grid, block, smem, st>>>(a, S);                          \
  } while (0)
  if (vec4 && C == 64) TS_BWD(64, true, 0);
  else if (vec4 && C == 128) TS_BWD(128, true, 1);
  else if (vec4 && C == 32) TS_BWD(32, true, 2);
  else if (vec4) TS_BWD(0, true, 3);
  else TS_BWD(0, false, 4);
#undef TS_BWD
  return cudaGetLastError();
}

}  // namespace tsb
