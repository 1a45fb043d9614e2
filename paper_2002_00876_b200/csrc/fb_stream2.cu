// fb_stream2.cu — register-blocked streaming sweeps for C in {32, 64, 128} (BASELINE cfg3
// and the cfg5 leaf sweeps).  Same mathematics and workspace contract as fb_stream.cu
// (DESIGN.md §4); the difference is the thread-to-tile mapping:
//
//   forward : thread (g, q) holds the 4 columns 4q..4q+3 for the R rows i = g + G*r of every
//             tile in registers (one LDS.128 per row: consecutive q -> consecutive 16 B,
//             conflict-free), computes the partial column max and the partial exp-shifted
//             dot product Σ_i a_i 2^((l_ij - M) log2 e) for its rows;
//   backward: thread (q, g) holds the 4 rows 4q..4q+3 for the R columns c = 4g + 4G*k (one
//             LDS.128 per row chunk, conflict-free with the padded C+4 stride), computes the
//             partial row max / sum and writes its marginals as coalesced float4 stores.
// Then one thread per column (row) merges the G partials online-softmax style and
// finalises the vector; the rest is identical to fb_stream.cu.  NT = 256, G = 256/(C/4).
#include <atomic>

#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

namespace {
constexpr int kNT2 = 256;

__device__ __forceinline__ float block_max2(float v, float* red) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = v;
  __syncthreads();
  float r = red[0];
#pragma unroll
  for (int k = 1; k < kNT2 / 32; ++k) r = fmaxf(r, red[k]);
  __syncthreads();
  return r;
}

__device__ __forceinline__ float block_lse2_2(float v, float* redm, float* reds) {
  const float wm = warp_max(v);
  const float e = (wm == neg_inf()) ? 0.f : ex2(v - wm);
  const float ws = warp_sum(e);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    redm[w] = wm;
    reds[w] = ws;
  }
  __syncthreads();
  float M = redm[0];
#pragma unroll
  for (int k = 1; k < kNT2 / 32; ++k) M = fmaxf(M, redm[k]);
  float S = 0.f;
  if (M != neg_inf())
#pragma unroll
    for (int k = 0; k < kNT2 / 32; ++k) S += (redm[k] == neg_inf()) ? 0.f : reds[k] * ex2(redm[k] - M);
  __syncthreads();
  return (M == neg_inf()) ? neg_inf() : M + lg2(S);
}

// cp.async staging of one dense C x C tile into SMEM rows of `stride` floats (C % 4 == 0).
template <int C>
__device__ __forceinline__ void stage2(float* dst, const float* __restrict__ src, int stride,
                                       int tid) {
  constexpr int Q = C / 4, n = C * Q;
#pragma unroll
  for (int k = tid; k < n; k += kNT2) {
    const int r = k / Q, c4 = k - (k / Q) * Q;
    cp_async16(dst + r * stride + 4 * c4, src + r * C + 4 * c4);
  }
}
}  // namespace

// ====================================================================================
// Forward
// ====================================================================================
template <int C>
__global__ void __launch_bounds__(kNT2) fwd2_kernel(SweepArgs a, int S) {
  constexpr int Q = C / 4, G = kNT2 / Q, R = C / G, CC = C * C, NW = kNT2 / 32;
  static_assert(C % 4 == 0 && kNT2 % Q == 0 && C % G == 0, "bad C");
  extern __shared__ __align__(16) float sm[];
  const int64_t N = a.N, E = N - 1, P = a.P, L = a.L;
  const int64_t b = blockIdx.x / P, k = blockIdx.x - (blockIdx.x / P) * P;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = tid / Q, q = tid - (tid / Q) * Q;
  float* ring = sm;                    // [S][CC]
  float* a_s = ring + (size_t)S * CC;  // [2][C]
  float* ah_s = a_s + 2 * C;           // [2][C]
  float* pm = ah_s + 2 * C;            // [G][C]
  float* ps = pm + G * C;              // [G][C]
  float* red_T = ps + G * C;           // [NW]
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
  if (t0 >= Eb && k > 0) return;
  const int64_t t1 = (t0 + L < Eb) ? t0 + L : Eb;
  const int64_t nsteps = t1 - t0;
  const bool last = (t1 == Eb);
  const bool own = tid < C;  // thread tid finalises column tid
  const int64_t bk = b * P + k;
  const float* potb = a.pot + b * E * (int64_t)CC;

  float ah = own ? (a.alpha_in ? a.alpha_in[bk * C + tid] : 0.f) : neg_inf();
  double O = a.alpha_in_off ? a.alpha_in_off[bk] : 0.0;
  float mu = block_max2(ah, red_x);
  float m = (mu == neg_inf()) ? 0.f : mu;
  if (a.alpha_hat && own) a.alpha_hat[(b * N + t0) * C + tid] = ah;

  for (int u = 0; u < S - 1; ++u) {
    if (u < nsteps) stage2<C>(ring + (size_t)(u % S) * CC, potb + (t0 + u) * (int64_t)CC, C, tid);
    cp_async_commit();
  }
  if (own) {
    a_s[tid] = ex2(ah - m);
    ah_s[tid] = ah;
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
        stage2<C>(ring + (size_t)(uu % S) * CC, potb + (t0 + uu) * (int64_t)CC, C, tid);
      cp_async_commit();
    }
    const float* tile = ring + (size_t)(u % S) * CC;
    const float* av = a_s + buf * C;
    // ---- phase A: 4 columns x R rows in registers ------------------------------------------
    float4 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = *reinterpret_cast<const float4*>(tile + (g + G * r) * C + 4 * q);
    float4 M4 = v[0];
#pragma unroll
    for (int r = 1; r < R; ++r) {
      M4.x = fmaxf(M4.x, v[r].x);
      M4.y = fmaxf(M4.y, v[r].y);
      M4.z = fmaxf(M4.z, v[r].z);
      M4.w = fmaxf(M4.w, v[r].w);
    }
    const float4 Mc = make_float4(M4.x == neg_inf() ? 0.f : M4.x, M4.y == neg_inf() ? 0.f : M4.y,
                                  M4.z == neg_inf() ? 0.f : M4.z, M4.w == neg_inf() ? 0.f : M4.w);
    float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const float ai = av[g + G * r];
      s4.x = fmaf(ai, ex2((v[r].x - Mc.x) * kLog2e), s4.x);
      s4.y = fmaf(ai, ex2((v[r].y - Mc.y) * kLog2e), s4.y);
      s4.z = fmaf(ai, ex2((v[r].z - Mc.z) * kLog2e), s4.z);
      s4.w = fmaf(ai, ex2((v[r].w - Mc.w) * kLog2e), s4.w);
    }
    *reinterpret_cast<float4*>(pm + g * C + 4 * q) = M4;
    *reinterpret_cast<float4*>(ps + g * C + 4 * q) = s4;
    {
      const float wm = warp_max(fmaxf(fmaxf(M4.x, M4.y), fmaxf(M4.z, M4.w)));
      if (lane == 0) red_T[w] = wm;
    }
    __syncthreads();
    float T = red_T[0];
#pragma unroll
    for (int x = 1; x < NW; ++x) T = fmaxf(T, red_T[x]);
    const float Tz = (T == neg_inf()) ? 0.f : T;
    const float m_next = (mu == neg_inf()) ? 0.f : (log2C + mu - m);
    // ---- phase B: thread j merges the G partials of column j ---------------------------------
    if (own) {
      const int j = tid;
      float Mj = neg_inf();
#pragma unroll
      for (int x = 0; x < G; ++x) Mj = fmaxf(Mj, pm[x * C + j]);
      float nh = neg_inf();
      if (Mj != neg_inf()) {
        float sj = 0.f;
#pragma unroll
        for (int x = 0; x < G; ++x) {
          const float mq = pm[x * C + j];
          if (mq != neg_inf()) sj = fmaf(ps[x * C + j], ex2((mq - Mj) * kLog2e), sj);
        }
        nh = (Mj - Tz) * kLog2e + lg2(sj);
        if (!(sj >= kGate)) {  // exact per-cell-max path (§6(c)); also reached by NaN
          const float* ahv = ah_s + buf * C;
          float qx = neg_inf();
          for (int i = 0; i < C; ++i) qx = fmaxf(qx, ahv[i] + (tile[i * C + j] - Tz) * kLog2e);
          if (qx == neg_inf()) {
            nh = neg_inf();
          } else {
            float ss = 0.f;
            for (int i = 0; i < C; ++i) ss += ex2(ahv[i] + (tile[i * C + j] - Tz) * kLog2e - qx);
            nh = qx + lg2(ss) - m;
          }
          if (sj != sj) nh = qnan();
        }
      }
      if (nh != nh || Mj == pos_inf()) bad = 1u;
      if (a.alpha_hat && t + 1 < t1) a.alpha_hat[(b * N + t + 1) * C + j] = nh;
      ah_s[(buf ^ 1) * C + j] = nh;
      a_s[(buf ^ 1) * C + j] = ex2(nh - m_next);
      ah = nh;
    }
    if (w < (C + 31) / 32) {
      const float wm = warp_max(own ? ah : neg_inf());
      if (lane == 0) red_mu[(buf ^ 1) * NW + w] = wm;
    }
    if (tid == 0) {
      if (a.mlag) a.mlag[b * N + t] = m;
      if (a.tmax) a.tmax[b * E + t] = Tz;
    }
    O += kLn2 * (double)m + (double)Tz;
    cp_async_wait_dyn(S - 2);
    __syncthreads();
    float mx = red_mu[(buf ^ 1) * NW];
#pragma unroll
    for (int x = 1; x < (C + 31) / 32; ++x) mx = fmaxf(mx, red_mu[(buf ^ 1) * NW + x]);
    mu = mx;
    m = m_next;
    buf ^= 1;
  }
  cp_async_wait<0>();
  if (a.alpha_end && own) a.alpha_end[bk * C + tid] = ah;
  if (a.alpha_end_off && tid == 0) a.alpha_end_off[bk] = O;
  const unsigned anybad = __syncthreads_or(bad);
  if (anybad && tid == 0 && a.wflags) atomicOr(&a.wflags[b], (unsigned)WF_NONFINITE);
  if (a.final_in_fwd && last) {
    const float Lz = block_lse2_2(own ? ah : neg_inf(), red_x, red_x + NW);
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
// Backward + marginals
// ====================================================================================
template <int C>
__global__ void __launch_bounds__(kNT2) bwd2_kernel(SweepArgs a, int S) {
  constexpr int Q = C / 4, G = kNT2 / Q, R = C / G, RQ = R / 4 > 0 ? R / 4 : 1;
  constexpr int SB = C + 4, TF = C * SB, CC = C * C, NW = kNT2 / 32;
  static_assert(R % 4 == 0 || R < 4, "bad C");
  extern __shared__ __align__(16) float sm[];
  const int64_t N = a.N, E = N - 1, P = a.P, L = a.L;
  const int64_t b = blockIdx.x / P, k = blockIdx.x - (blockIdx.x / P) * P;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // thread (q, g): rows 4q..4q+3, columns c = 4g + 4G*x, x < RQ (when R >= 4);
  // for R < 4 (C = 32: G = 32, R = 1) thread (q, g) holds column g of rows 4q..4q+3
  const int g = tid % G, q = tid / G;
  float* ring = sm;                    // [S][C][SB]
  float* b_s = ring + (size_t)S * TF;  // [2][C]
  float* bh_s = b_s + 2 * C;           // [2][C]
  float* pr = bh_s + 2 * C;            // [G][C] partial row max
  float* ps = pr + G * C;              // [G][C] partial sums
  float* red_mu = ps + G * C;          // [2][NW]
  float* red_lm = red_mu + 2 * NW;     // [2][NW]
  float* red_ls = red_lm + 2 * NW;     // [2][NW]
  float* red_x = red_ls + 2 * NW;      // [2*NW]

  const int64_t len = seq_len(a.lengths, b, N);
  float* mgb = a.marg + b * E * (int64_t)CC;
  if (len < 0) {
    if (k == 0) {
      for (int64_t x = tid; x < E * CC; x += kNT2) mgb[x] = 0.f;
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
  const bool own = tid < C;  // thread tid finalises row tid
  const int64_t bk = b * P + k;
  const float* potb = a.pot + b * E * (int64_t)CC;
  const uint32_t wf = a.wflags ? a.wflags[b] : 0u;

  float bh = own ? (a.beta_out ? a.beta_out[bk * C + tid] : 0.f) : neg_inf();
  const float ahe = own ? a.alpha_end[bk * C + tid] : neg_inf();
  float Lnext = block_lse2_2(own ? ahe + bh : neg_inf(), red_x, red_x + NW);
  float mu = block_max2(bh, red_x);
  float m = (mu == neg_inf()) ? 0.f : mu;

  const bool dead = (wf & WF_NONFINITE) || !(Lnext > neg_inf());
  if (last && !a.no_final) {
    for (int64_t x = Eb * CC + tid; x < E * CC; x += kNT2) mgb[x] = 0.f;
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
    for (int64_t x = Eb * CC + tid; x < E * CC; x += kNT2) mgb[x] = 0.f;
  if (dead) {
    for (int64_t x = t0 * CC + tid; x < t1 * CC; x += kNT2) mgb[x] = 0.f;
    return;
  }

  for (int u = 0; u < S - 1; ++u) {
    if (u < nsteps) stage2<C>(ring + (size_t)(u % S) * TF, potb + (t1 - 1 - u) * (int64_t)CC, SB, tid);
    cp_async_commit();
  }
  if (own) {
    b_s[tid] = ex2(bh - m);
    bh_s[tid] = bh;
  }
  cp_async_wait_dyn(S - 2);
  __syncthreads();

  const float log2C = lg2((float)C);
  int buf = 0;
  float4 aht4 = make_float4(neg_inf(), neg_inf(), neg_inf(), neg_inf());
  float aho = neg_inf();  // alpha_hat_t[tid] for the row owner
  if (nsteps > 0) {
    aht4 = *reinterpret_cast<const float4*>(a.alpha_hat + (b * N + t1 - 1) * C + 4 * q);
    if (own) aho = a.alpha_hat[(b * N + t1 - 1) * C + tid];
  }
  for (int64_t u = 0; u < nsteps; ++u) {
    const int64_t t = t1 - 1 - u;
    {
      const int64_t uu = u + S - 1;
      if (uu < nsteps)
        stage2<C>(ring + (size_t)(uu % S) * TF, potb + (t1 - 1 - uu) * (int64_t)CC, SB, tid);
      cp_async_commit();
    }
    const float* tile = ring + (size_t)(u % S) * TF;
    const float* bv = b_s + buf * C;
    const float* bhv = bh_s + buf * C;
    const float Tt = a.tmax[b * E + t];
    const float mt = a.mlag[b * N + t];
    const float4 ahc = aht4;
    const float aho_cur = aho;
    if (u + 1 < nsteps) {
      aht4 = *reinterpret_cast<const float4*>(a.alpha_hat + (b * N + t - 1) * C + 4 * q);
      if (own) aho = a.alpha_hat[(b * N + t - 1) * C + tid];
    }
    // ---- phase A: 4 rows x R columns ---------------------------------------------------------
    const float ahr[4] = {ahc.x, ahc.y, ahc.z, ahc.w};
    float Rm[4], sr[4];
    float* mrow0 = mgb + ((int64_t)t * C + 4 * q) * C;
    if constexpr (R >= 4) {
      float4 v[4][RQ];
#pragma unroll
      for (int rr = 0; rr < 4; ++rr)
#pragma unroll
        for (int x = 0; x < RQ; ++x)
          v[rr][x] = *reinterpret_cast<const float4*>(tile + (4 * q + rr) * SB + 4 * g + 4 * G * x);
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        float mx = neg_inf();
#pragma unroll
        for (int x = 0; x < RQ; ++x)
          mx = fmaxf(mx, fmaxf(fmaxf(v[rr][x].x, v[rr][x].y), fmaxf(v[rr][x].z, v[rr][x].w)));
        Rm[rr] = mx;
        sr[rr] = 0.f;
      }
#pragma unroll
      for (int x = 0; x < RQ; ++x) {
        const int c = 4 * g + 4 * G * x;
        const float4 bb = *reinterpret_cast<const float4*>(bv + c);
        const float4 hh = *reinterpret_cast<const float4*>(bhv + c);
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          const float Rz = (Rm[rr] == neg_inf()) ? 0.f : Rm[rr];
          const float4 vv = v[rr][x];
          sr[rr] = fmaf(ex2((vv.x - Rz) * kLog2e), bb.x, sr[rr]);
          sr[rr] = fmaf(ex2((vv.y - Rz) * kLog2e), bb.y, sr[rr]);
          sr[rr] = fmaf(ex2((vv.z - Rz) * kLog2e), bb.z, sr[rr]);
          sr[rr] = fmaf(ex2((vv.w - Rz) * kLog2e), bb.w, sr[rr]);
          const float cst = ahr[rr] - mt - Lnext;
          float4 mu4;
          mu4.x = ex2(cst + hh.x + (vv.x - Tt) * kLog2e);
          mu4.y = ex2(cst + hh.y + (vv.y - Tt) * kLog2e);
          mu4.z = ex2(cst + hh.z + (vv.z - Tt) * kLog2e);
          mu4.w = ex2(cst + hh.w + (vv.w - Tt) * kLog2e);
          *reinterpret_cast<float4*>(mrow0 + rr * C + c) = mu4;
        }
      }
    } else {  // R < 4 (C = 32): one column per thread
      const int c = g;
      const float bb = bv[c], hh = bhv[c];
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const float vv = tile[(4 * q + rr) * SB + c];
        Rm[rr] = vv;
        const float Rz = (vv == neg_inf()) ? 0.f : vv;
        sr[rr] = ex2((vv - Rz) * kLog2e) * bb;
        mrow0[rr * C + c] = ex2(ahr[rr] - mt - Lnext + hh + (vv - Tt) * kLog2e);
      }
    }
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
      pr[g * C + 4 * q + rr] = Rm[rr];
      ps[g * C + 4 * q + rr] = sr[rr];
    }
    __syncthreads();
    const float m_next = (mu == neg_inf()) ? 0.f : (log2C + mu - m);
    // ---- phase B: thread i merges the G partials of row i --------------------------------------
    float nb = neg_inf();
    if (own) {
      const int i = tid;
      float Ri = neg_inf();
#pragma unroll 8
      for (int x = 0; x < G; ++x) Ri = fmaxf(Ri, pr[x * C + i]);
      if (Ri != neg_inf()) {
        float si = 0.f;
#pragma unroll 8
        for (int x = 0; x < G; ++x) {
          const float rq = pr[x * C + i];
          if (rq != neg_inf()) si = fmaf(ps[x * C + i], ex2((rq - Ri) * kLog2e), si);
        }
        nb = (Ri - Tt) * kLog2e + lg2(si);
        if (!(si >= kGate)) {  // exact per-cell-max path
          const float* row = tile + i * SB;
          float qx = neg_inf();
          for (int c = 0; c < C; ++c) qx = fmaxf(qx, (row[c] - Tt) * kLog2e + bhv[c]);
          if (qx == neg_inf()) {
            nb = neg_inf();
          } else {
            float ss = 0.f;
            for (int c = 0; c < C; ++c) ss += ex2((row[c] - Tt) * kLog2e + bhv[c] - qx);
            nb = qx + lg2(ss) - m;
          }
        }
      }
      b_s[(buf ^ 1) * C + i] = ex2(nb - m_next);
      bh_s[(buf ^ 1) * C + i] = nb;
    }
    if (w < (C + 31) / 32) {
      const float wm = warp_max(nb);
      const float v = own ? aho_cur + nb : neg_inf();
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
      constexpr int NW0 = (C + 31) / 32;
      const float* rm = red_mu + (buf ^ 1) * NW;
      const float* lmv = red_lm + (buf ^ 1) * NW;
      const float* lsv = red_ls + (buf ^ 1) * NW;
      float mx = rm[0], LM = lmv[0];
#pragma unroll
      for (int x = 1; x < NW0; ++x) {
        mx = fmaxf(mx, rm[x]);
        LM = fmaxf(LM, lmv[x]);
      }
      float LS = 0.f;
      if (LM != neg_inf())
#pragma unroll
        for (int x = 0; x < NW0; ++x) LS += (lmv[x] == neg_inf()) ? 0.f : lsv[x] * ex2(lmv[x] - LM);
      Lnext = (LM == neg_inf()) ? neg_inf() : LM + lg2(LS);
      mu = mx;
    }
    m = m_next;
    buf ^= 1;
  }
  cp_async_wait<0>();
}

// ====================================================================================
// host side
// ====================================================================================
namespace {
std::atomic<uint64_t> g_attr2[64];  // one per-device mask per kernel (`bit` = kernel id)
template <typename K>
cudaError_t set_smem2(K kern, int bit) {
  return smem_optin_once(kern, g_attr2[bit], 220 * 1024);
}
template <int C>
size_t fwd2_smem(int S) {
  constexpr int Q = C / 4, G = kNT2 / Q;
  return ((size_t)S * C * C + 4 * C + 2 * G * C + 5 * (kNT2 / 32)) * sizeof(float);
}
template <int C>
size_t bwd2_smem(int S) {
  constexpr int Q = C / 4, G = kNT2 / Q;
  return ((size_t)S * C * (C + 4) + 4 * C + 2 * G * C + 8 * (kNT2 / 32)) * sizeof(float);
}
template <int C>
int stages2(size_t tile_bytes) {
  const size_t budget = (C > 64) ? 196 * 1024 : 96 * 1024;
  int S = (int)(budget / tile_bytes);
  return S < 2 ? 2 : (S > 8 ? 8 : S);
}
template <int C>
cudaError_t fwd2(const SweepArgs& a, cudaStream_t st) {
  const int S = stages2<C>((size_t)C * C * 4);
  cudaError_t e = set_smem2(fwd2_kernel<C>, C == 32 ? 0 : (C == 64 ? 1 : 2));
  if (e != cudaSuccess) return e;
  fwd2_kernel<C><<<(unsigned)(a.B * a.P), kNT2, fwd2_smem<C>(S), st>>>(a, S);
  return cudaGetLastError();
}
template <int C>
cudaError_t bwd2(const SweepArgs& a, cudaStream_t st) {
  const int S = stages2<C>((size_t)C * (C + 4) * 4);
  cudaError_t e = set_smem2(bwd2_kernel<C>, C == 32 ? 3 : (C == 64 ? 4 : 5));
  if (e != cudaSuccess) return e;
  bwd2_kernel<C><<<(unsigned)(a.B * a.P), kNT2, bwd2_smem<C>(S), st>>>(a, S);
  return cudaGetLastError();
}
}  // namespace

bool stream2_ok(const SweepArgs& a) {
  const bool al = (reinterpret_cast<uintptr_t>(a.pot) & 15) == 0 &&
                  (!a.marg || (reinterpret_cast<uintptr_t>(a.marg) & 15) == 0);
  return al && (a.C == 32 || a.C == 64 || a.C == 128);
}

cudaError_t launch_fwd2(const SweepArgs& a, cudaStream_t st) {
  switch (a.C) {
    case 32: return fwd2<32>(a, st);
    case 64: return fwd2<64>(a, st);
    case 128: return fwd2<128>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_bwd2(const SweepArgs& a, cudaStream_t st) {
  switch (a.C) {
    case 32: return bwd2<32>(a, st);
    case 64: return bwd2<64>(a, st);
    case 128: return bwd2<128>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tsb
