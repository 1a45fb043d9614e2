// fb_meet.cu — meet-in-the-middle forward/backward sweep with fused marginals, C = 64
// (BASELINE cfg3: B=256, N=512, C=64).  One CTA of 512 threads per sequence, two
// independent 256-thread "engines" (own named barrier, own TMA ring):
//
//   phase 1   engine F: alpha_hat over edges [0, h)        (forward recursion, eq. for A(l))
//             engine B: beta_hat  over edges [E_b-1 .. h]  (backward recursion)
//   middle    log Z = O_F + O_B + ln2 * log2 sum_j 2^(ah_h[j] + bh_h[j])        (h = E_b/2)
//   phase 2   engine F continues over [h, E_b): alpha_{t+1} and mu_t from beta_hat[t+1]
//             engine B continues over [h-1 .. 0]: beta_t and mu_t from alpha_hat[t]
//
// so every edge tile is read from HBM twice (once per engine, as with separate forward and
// backward kernels) but the two serial chains run concurrently: the SM has twice the
// independent work to overlap, and each sweep is E_b steps instead of 2 E_b.  The marginal
// of edge t is mu_t(i,j) = alpha_t(i) psi_t(i,j) beta_{t+1}(j) / Z (paper §3, gradient of
// A(l)), evaluated in whichever engine reaches edge t second (DESIGN.md §4 "meet").
//
// Numerics: node vectors are log2 values relative to a lagged bound m
// (linear-space weights a = 2^(ah - m)); tile weights e = 2^((l - T_s) log2 e) with a
// per-step natural shift T_s.  In phase 1 T_s is the previous tile's max, verified against
// the current tile max after the partial sums (|T - T_s| log2 e <= 40, else the step is redone
// with T_s = T); phase 2 reuses the shift the other engine recorded for that edge.  Merged
// partial sums below 2^-60 take the exact per-cell-max path (§6(c)).  Marginals use the
// product form mu = a_i e_ij c_j (F) / e_ij b_j r_i (B), exact exp form when a factor leaves
// [0, 2^80].  Tiles arrive by 1-D TMA bulk copies (cp.async.bulk + mbarrier), 3 stages.
#include <atomic>

#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

namespace {
constexpr int kC = 64, kCC = kC * kC, kNTE = 256, kNT = 512, kS = 3;
constexpr int kQ = kC / 4, kG = kNTE / kQ, kR = kC / kG, kNW = kNTE / 32, kPS = kC + 4;
constexpr uint32_t kTileBytes = kCC * 4;
constexpr float kShiftTol = 40.f;               // log2 units
constexpr float kBig = 1.2089258196146292e24f;  // 2^80
static_assert(kR == 4 && kG == 16, "layout assumes C = 64");

struct __align__(16) MeetSmem {
  float ring[2][kS][kCC];  // [engine][stage] tiles
  float a_s[2][kC];        // F: 2^(ah - m), double-buffered
  float ah_s[2][kC];       // F: ah
  float b_s[2][kC];        // B: 2^(bh - m)
  float bh_s[2][kC];       // B: bh
  float ps[2][kG][kPS];    // [engine] partial sums per thread group
  float redT[2][kNW];
  float redmu[2][kNW];
  float redlm[2][kNW];
  float redls[2][kNW];
  double O[2];
  double xred[2][kNW];
  uint32_t bad[2];
  float Lh;
  int dead;
  uint64_t full[2][kS];
};

struct EState {
  float Ts, m, mu, Lnext;
  int buf;
  uint32_t bad;
  double O;
  int64_t u;       // tiles consumed by this engine
  int64_t issued;  // tiles issued (producer thread only)
  double xacc;     // fused f1 epilogue: this thread's Σ mu·x over its elements (fixed order)
};

__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void sts4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float max4(float4 v) { return fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)); }
__device__ __forceinline__ bool finite_f(float x) { return fabsf(x) < pos_inf(); }

__device__ __forceinline__ void issue(MeetSmem& s, int eng, EState& st, int64_t Eb,
                                      const float* potb) {
  const int64_t u = st.issued++;
  const int slot = (int)(u % kS);
  const int64_t t = eng == 0 ? u : Eb - 1 - u;
  bulk_load(s.ring[eng][slot], potb + t * kCC, kTileBytes, &s.full[eng][slot]);
}

// Σ mu·x over one float4 of marginals (terms with mu = 0 skipped: masked parts may hold -inf
// in l or anything in r, reading R13/R13b)
__device__ __forceinline__ float xdot4(float4 mu, float4 x) {
  float s = 0.f;
  if (mu.x != 0.f) s = fmaf(mu.x, x.x, s);
  if (mu.y != 0.f) s = fmaf(mu.y, x.y, s);
  if (mu.z != 0.f) s = fmaf(mu.z, x.z, s);
  if (mu.w != 0.f) s = fmaf(mu.w, x.w, s);
  return s;
}

// merge the 256-thread engine's two-warp owner reductions (log2-sum-exp of kC values)
__device__ __forceinline__ float lse_parts(const float* lm, const float* ls) {
  const float LM = fmaxf(lm[0], lm[1]);
  if (LM == neg_inf()) return neg_inf();
  float LS = 0.f;
  if (lm[0] != neg_inf()) LS += ls[0] * ex2(lm[0] - LM);
  if (lm[1] != neg_inf()) LS += ls[1] * ex2(lm[1] - LM);
  return LM + lg2(LS);
}

// ----------------------------------------------------------------------------------------
// engine F: thread (g, q) holds rows g + 16 r (r < 4) x columns 4q..4q+3 of each tile
// ----------------------------------------------------------------------------------------
template <bool P2, int XM>
__device__ __forceinline__ void f_run(MeetSmem& s, const MeetArgs& a, EState& st, int64_t b,
                                      int64_t t_lo, int64_t t_hi, int64_t Eb, const float* potb,
                                      int e, float log2C) {
  const int g = e / kQ, q = e - (e / kQ) * kQ, lane = e & 31, w = e >> 5;
  const bool own = e < kC;
  const int64_t N = a.N, E = N - 1;
  float4 bh4n = make_float4(0.f, 0.f, 0.f, 0.f);
  float bhjn = neg_inf(), Tn = 0.f;
  if (P2 && t_lo < t_hi) {
    const float* bp = a.beta_hat + (b * N + t_lo + 1) * kC;
    bh4n = lds4(bp + 4 * q);
    if (own) bhjn = bp[e];
    Tn = a.tshift[b * E + t_lo];
  }
  for (int64_t t = t_lo; t < t_hi; ++t) {
    const int64_t u = st.u;
    const int slot = (int)(u % kS);
    float4 bh4 = bh4n;
    float bhj = bhjn;
    if (P2) {
      st.Ts = Tn;
      if (t + 1 < t_hi) {
        const float* bp = a.beta_hat + (b * N + t + 2) * kC;
        bh4n = lds4(bp + 4 * q);
        if (own) bhjn = bp[e];
        Tn = a.tshift[b * E + t + 1];
      }
    }
    mbar_wait(&s.full[0][slot], (uint32_t)((u / kS) & 1));
    const float* tile = s.ring[0][slot];
    const float* av = s.a_s[st.buf];
    float ai[kR];
    float4 v[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      ai[r] = av[g + kG * r];
      v[r] = lds4(tile + (g + kG * r) * kC + 4 * q);
    }
    if (!P2) {
      float lm = max4(v[0]);
#pragma unroll
      for (int r = 1; r < kR; ++r) lm = fmaxf(lm, max4(v[r]));
      lm = warp_max(lm);
      if (lane == 0) s.redT[0][w] = lm;
    }
    float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      v[r].x = ex2((v[r].x - st.Ts) * kLog2e);
      v[r].y = ex2((v[r].y - st.Ts) * kLog2e);
      v[r].z = ex2((v[r].z - st.Ts) * kLog2e);
      v[r].w = ex2((v[r].w - st.Ts) * kLog2e);
      s4.x = fmaf(ai[r], v[r].x, s4.x);
      s4.y = fmaf(ai[r], v[r].y, s4.y);
      s4.z = fmaf(ai[r], v[r].z, s4.z);
      s4.w = fmaf(ai[r], v[r].w, s4.w);
    }
    sts4(&s.ps[0][g][4 * q], s4);
    named_bar(1, kNTE);
    if (e == 0 && u >= 1 && st.issued < Eb) issue(s, 0, st, Eb, potb);
    float Tz = st.Ts;
    if (!P2) {
      float T = s.redT[0][0];
#pragma unroll
      for (int x = 1; x < kNW; ++x) T = fmaxf(T, s.redT[0][x]);
      if (T == pos_inf()) st.bad = 1u;
      Tz = finite_f(T) ? T : (finite_f(st.Ts) ? st.Ts : 0.f);
      if (!(fabsf(Tz - st.Ts) * kLog2e <= kShiftTol)) {  // rare: redo with the exact shift
        st.Ts = Tz;
        s4 = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          v[r] = lds4(tile + (g + kG * r) * kC + 4 * q);
          v[r].x = ex2((v[r].x - Tz) * kLog2e);
          v[r].y = ex2((v[r].y - Tz) * kLog2e);
          v[r].z = ex2((v[r].z - Tz) * kLog2e);
          v[r].w = ex2((v[r].w - Tz) * kLog2e);
          s4.x = fmaf(ai[r], v[r].x, s4.x);
          s4.y = fmaf(ai[r], v[r].y, s4.y);
          s4.z = fmaf(ai[r], v[r].z, s4.z);
          s4.w = fmaf(ai[r], v[r].w, s4.w);
        }
        sts4(&s.ps[0][g][4 * q], s4);
        named_bar(1, kNTE);
      }
    }
    const float m = st.m;
    const float m_next = (st.mu == neg_inf()) ? 0.f : (log2C + st.mu - m);
    float nh = neg_inf();
    if (own) {
      const int j = e;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
      for (int x = 0; x < kG; x += 4) {
        s0 += s.ps[0][x][j];
        s1 += s.ps[0][x + 1][j];
        s2 += s.ps[0][x + 2][j];
        s3 += s.ps[0][x + 3][j];
      }
      const float sj = (s0 + s1) + (s2 + s3);
      nh = lg2(sj);
      if (!(sj >= kGate) || sj == pos_inf()) {  // exact per-cell-max path (§6(c)); NaN too
        const float* ahv = s.ah_s[st.buf];
        float qx = neg_inf();
        for (int i = 0; i < kC; ++i) qx = fmaxf(qx, ahv[i] + (tile[i * kC + j] - st.Ts) * kLog2e);
        if (qx == neg_inf() || qx == pos_inf()) {
          nh = qx;
        } else {
          float ss = 0.f;
          for (int i = 0; i < kC; ++i) ss += ex2(ahv[i] + (tile[i * kC + j] - st.Ts) * kLog2e - qx);
          nh = qx + lg2(ss) - m;
        }
        if (sj != sj) nh = qnan();
      }
      if (nh != nh || nh == pos_inf()) st.bad = 1u;
      if (!P2) a.alpha_hat[(b * N + t + 1) * kC + j] = nh;
      s.ah_s[st.buf ^ 1][j] = nh;
      s.a_s[st.buf ^ 1][j] = ex2(nh - m_next);
    }
    if (w < kC / 32) {
      const float wm = warp_max(nh);
      if (lane == 0) s.redmu[0][w] = wm;
      if (P2) {
        const float lv = nh + bhj;
        const float lm = warp_max(lv);
        const float ls = warp_sum(lm == neg_inf() ? 0.f : ex2(lv - lm));
        if (lane == 0) {
          s.redlm[0][w] = lm;
          s.redls[0][w] = ls;
        }
      }
    }
    if (e == 0) {
      if (!P2) {
        a.mlag[b * N + t] = m;
        a.tshift[b * E + t] = st.Ts;
      }
      st.O += kLn2 * (double)m + (double)st.Ts;
    }
    named_bar(1, kNTE);
    st.mu = fmaxf(s.redmu[0][0], s.redmu[0][1]);
    if (P2) {  // mu_t(i,j) = a_i e_ij 2^(bh_{t+1}[j] - L_{t+1})
      const float L = lse_parts(s.redlm[0], s.redls[0]);
      const float c0 = ex2(bh4.x - L), c1 = ex2(bh4.y - L), c2 = ex2(bh4.z - L), c3 = ex2(bh4.w - L);
      float* mt = a.marg + ((b * E + t) * kC) * kC + 4 * q;
      const float* xt = XM == 2 ? a.xr + ((b * E + t) * kC) * kC + 4 * q : nullptr;
      float xe = 0.f;  // this edge's Σ mu·x over the thread's elements
      if (c0 <= kBig && c1 <= kBig && c2 <= kBig && c3 <= kBig) {
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          const float4 o = make_float4(ai[r] * c0 * v[r].x, ai[r] * c1 * v[r].y,
                                       ai[r] * c2 * v[r].z, ai[r] * c3 * v[r].w);
          __stcs(reinterpret_cast<float4*>(mt + (g + kG * r) * kC), o);
          if (XM)
            xe += xdot4(o, XM == 1 ? lds4(tile + (g + kG * r) * kC + 4 * q)
                                        : __ldcs(reinterpret_cast<const float4*>(xt + (g + kG * r) * kC)));
        }
      } else {
        const float* ahv = s.ah_s[st.buf];
        const float bhk[4] = {bh4.x, bh4.y, bh4.z, bh4.w};
#pragma unroll
        for (int r = 0; r < kR; ++r) {
          const int i = g + kG * r;
          float o[4];
#pragma unroll
          for (int k = 0; k < 4; ++k)
            o[k] = ex2(ahv[i] + (tile[i * kC + 4 * q + k] - st.Ts) * kLog2e + bhk[k] - m - L);
          const float4 o4 = make_float4(o[0], o[1], o[2], o[3]);
          __stcs(reinterpret_cast<float4*>(mt + i * kC), o4);
          if (XM)
            xe += xdot4(o4, XM == 1 ? lds4(tile + i * kC + 4 * q)
                                         : __ldcs(reinterpret_cast<const float4*>(xt + i * kC)));
        }
      }
      if (XM) st.xacc += (double)xe;
    }
    st.m = m_next;
    st.buf ^= 1;
    st.Ts = Tz;
    st.u = u + 1;
  }
}

// ----------------------------------------------------------------------------------------
// engine B: thread (q, g) holds rows 4q..4q+3 x columns 4g..4g+3 of each tile
// ----------------------------------------------------------------------------------------
template <bool P2, int XM>
__device__ __forceinline__ void b_run(MeetSmem& s, const MeetArgs& a, EState& st, int64_t b,
                                      int64_t t_lo, int64_t t_hi, int64_t Eb, const float* potb,
                                      int e, float log2C) {
  const int g = e % kG, q = e / kG, lane = e & 31, w = e >> 5;
  const bool own = e < kC;
  const int64_t N = a.N, E = N - 1;
  float4 ah4n = make_float4(0.f, 0.f, 0.f, 0.f);
  float ahon = neg_inf(), mFn = 0.f, TFn = 0.f;
  if (P2 && t_lo < t_hi) {
    const int64_t t = t_hi - 1;
    const float* ap = a.alpha_hat + (b * N + t) * kC;
    ah4n = lds4(ap + 4 * q);
    if (own) ahon = ap[e];
    mFn = a.mlag[b * N + t];
    TFn = a.tshift[b * E + t];
  }
  for (int64_t t = t_hi - 1; t >= t_lo; --t) {
    const int64_t u = st.u;
    const int slot = (int)(u % kS);
    const float4 ah4 = ah4n;
    const float aho = ahon, mF = mFn;
    if (P2) {
      st.Ts = TFn;
      if (t - 1 >= t_lo) {
        const float* ap = a.alpha_hat + (b * N + t - 1) * kC;
        ah4n = lds4(ap + 4 * q);
        if (own) ahon = ap[e];
        mFn = a.mlag[b * N + t - 1];
        TFn = a.tshift[b * E + t - 1];
      }
    }
    mbar_wait(&s.full[1][slot], (uint32_t)((u / kS) & 1));
    const float* tile = s.ring[1][slot];
    const float4 bb = lds4(s.b_s[st.buf] + 4 * g);
    float4 v[4];
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) v[rr] = lds4(tile + (4 * q + rr) * kC + 4 * g);
    if (!P2) {
      float lm = fmaxf(fmaxf(max4(v[0]), max4(v[1])), fmaxf(max4(v[2]), max4(v[3])));
      lm = warp_max(lm);
      if (lane == 0) s.redT[1][w] = lm;
    }
    float sr[4];
    if (P2) {  // mu_t(i,j) = e_ij b_j 2^(ah_t[i] - m_t^F - L_{t+1} + m)
      const float ahr[4] = {ah4.x, ah4.y, ah4.z, ah4.w};
      float* mt = a.marg + ((b * E + t) * kC + 4 * q) * kC + 4 * g;
      const float* xt = XM == 2 ? a.xr + ((b * E + t) * kC + 4 * q) * kC + 4 * g : nullptr;
      float xe = 0.f;
      const float L = st.Lnext;
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const float rf = ex2(ahr[rr] - mF - L + st.m);
        const float e0 = ex2((v[rr].x - st.Ts) * kLog2e), e1 = ex2((v[rr].y - st.Ts) * kLog2e);
        const float e2 = ex2((v[rr].z - st.Ts) * kLog2e), e3 = ex2((v[rr].w - st.Ts) * kLog2e);
        const float p0 = e0 * bb.x, p1 = e1 * bb.y, p2 = e2 * bb.z, p3 = e3 * bb.w;
        sr[rr] = (p0 + p1) + (p2 + p3);
        float4 o;
        if (rf <= kBig) {
          o = make_float4(p0 * rf, p1 * rf, p2 * rf, p3 * rf);
        } else {
          const float4 bh = lds4(s.bh_s[st.buf] + 4 * g);
          const float cst = ahr[rr] - mF - L;
          o.x = ex2(cst + (v[rr].x - st.Ts) * kLog2e + bh.x);
          o.y = ex2(cst + (v[rr].y - st.Ts) * kLog2e + bh.y);
          o.z = ex2(cst + (v[rr].z - st.Ts) * kLog2e + bh.z);
          o.w = ex2(cst + (v[rr].w - st.Ts) * kLog2e + bh.w);
        }
        __stcs(reinterpret_cast<float4*>(mt + rr * kC), o);
        if (XM)
          xe += xdot4(o, XM == 1 ? v[rr] : __ldcs(reinterpret_cast<const float4*>(xt + rr * kC)));
      }
      if (XM) st.xacc += (double)xe;
    } else {
#pragma unroll
      for (int rr = 0; rr < 4; ++rr) {
        const float p0 = ex2((v[rr].x - st.Ts) * kLog2e) * bb.x;
        const float p1 = ex2((v[rr].y - st.Ts) * kLog2e) * bb.y;
        const float p2 = ex2((v[rr].z - st.Ts) * kLog2e) * bb.z;
        const float p3 = ex2((v[rr].w - st.Ts) * kLog2e) * bb.w;
        sr[rr] = (p0 + p1) + (p2 + p3);
      }
    }
    sts4(&s.ps[1][g][4 * q], make_float4(sr[0], sr[1], sr[2], sr[3]));
    named_bar(2, kNTE);
    if (e == 0 && u >= 1 && st.issued < Eb) issue(s, 1, st, Eb, potb);
    float Tz = st.Ts;
    if (!P2) {
      float T = s.redT[1][0];
#pragma unroll
      for (int x = 1; x < kNW; ++x) T = fmaxf(T, s.redT[1][x]);
      if (T == pos_inf()) st.bad = 1u;
      Tz = finite_f(T) ? T : (finite_f(st.Ts) ? st.Ts : 0.f);
      if (!(fabsf(Tz - st.Ts) * kLog2e <= kShiftTol)) {
        st.Ts = Tz;
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
          const float4 x = lds4(tile + (4 * q + rr) * kC + 4 * g);
          sr[rr] = (ex2((x.x - Tz) * kLog2e) * bb.x + ex2((x.y - Tz) * kLog2e) * bb.y) +
                   (ex2((x.z - Tz) * kLog2e) * bb.z + ex2((x.w - Tz) * kLog2e) * bb.w);
        }
        sts4(&s.ps[1][g][4 * q], make_float4(sr[0], sr[1], sr[2], sr[3]));
        named_bar(2, kNTE);
      }
    }
    const float m = st.m;
    const float m_next = (st.mu == neg_inf()) ? 0.f : (log2C + st.mu - m);
    float nb = neg_inf();
    if (own) {
      const int i = e;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
      for (int x = 0; x < kG; x += 4) {
        s0 += s.ps[1][x][i];
        s1 += s.ps[1][x + 1][i];
        s2 += s.ps[1][x + 2][i];
        s3 += s.ps[1][x + 3][i];
      }
      const float si = (s0 + s1) + (s2 + s3);
      nb = lg2(si);
      if (!(si >= kGate) || si == pos_inf()) {  // exact per-cell-max path
        const float* row = tile + i * kC;
        const float* bhv = s.bh_s[st.buf];
        float qx = neg_inf();
        for (int c = 0; c < kC; ++c) qx = fmaxf(qx, (row[c] - st.Ts) * kLog2e + bhv[c]);
        if (qx == neg_inf() || qx == pos_inf()) {
          nb = qx;
        } else {
          float ss = 0.f;
          for (int c = 0; c < kC; ++c) ss += ex2((row[c] - st.Ts) * kLog2e + bhv[c] - qx);
          nb = qx + lg2(ss) - m;
        }
        if (si != si) nb = qnan();
      }
      if (nb != nb || nb == pos_inf()) st.bad = 1u;
      if (!P2) a.beta_hat[(b * N + t) * kC + i] = nb;
      s.bh_s[st.buf ^ 1][i] = nb;
      s.b_s[st.buf ^ 1][i] = ex2(nb - m_next);
    }
    if (w < kC / 32) {
      const float wm = warp_max(nb);
      if (lane == 0) s.redmu[1][w] = wm;
      if (P2) {
        const float lv = aho + nb;
        const float lm = warp_max(lv);
        const float ls = warp_sum(lm == neg_inf() ? 0.f : ex2(lv - lm));
        if (lane == 0) {
          s.redlm[1][w] = lm;
          s.redls[1][w] = ls;
        }
      }
    }
    if (e == 0) {
      if (!P2) a.tshift[b * E + t] = st.Ts;
      st.O += kLn2 * (double)m + (double)st.Ts;
    }
    named_bar(2, kNTE);
    st.mu = fmaxf(s.redmu[1][0], s.redmu[1][1]);
    if (P2) st.Lnext = lse_parts(s.redlm[1], s.redls[1]);
    st.m = m_next;
    st.buf ^= 1;
    st.Ts = Tz;
    st.u = u + 1;
  }
}

__device__ __forceinline__ void zero_range(float* p, int64_t n4, int tid) {
  float4* p4 = reinterpret_cast<float4*>(p);
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int64_t x = tid; x < n4; x += kNT) __stcs(p4 + x, z);
}

template <int XM>
__global__ void __launch_bounds__(kNT, 2) meet64_kernel(MeetArgs a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  MeetSmem& s = *reinterpret_cast<MeetSmem*>(smraw);
  const int tid = threadIdx.x, eng = tid >> 8, e = tid & (kNTE - 1);
  const int64_t b = blockIdx.x, N = a.N, E = N - 1;
  float* mgb = a.marg + b * E * (int64_t)kCC;
  const int64_t len = seq_len(a.lengths, b, N);
  if (len < 0) {
    zero_range(mgb, E * kCC / 4, tid);
    if (tid == 0) {
      a.logz[b] = qnan();
      if (a.flags) a.flags[b] = TS_F_BADLEN;
      if (XM) a.xsum[2 * b] = a.xsum[2 * b + 1] = 0.0;
    }
    return;
  }
  const int64_t Eb = len - 1, h = Eb / 2;
  const float* potb = a.pot + b * E * (int64_t)kCC;
  const float log2C = 6.f;  // log2(64)
  if (tid == 0) {
    for (int x = 0; x < kS; ++x) {
      mbar_init(&s.full[0][x], 1);
      mbar_init(&s.full[1][x], 1);
    }
    s.bad[0] = s.bad[1] = 0u;
    fence_mbar_init();
  }
  if (e < kC) {
    if (eng == 0) {
      s.a_s[0][e] = 1.f;
      s.ah_s[0][e] = 0.f;
      a.alpha_hat[(b * N) * kC + e] = 0.f;
    } else {
      s.b_s[0][e] = 1.f;
      s.bh_s[0][e] = 0.f;
      a.beta_hat[(b * N + Eb) * kC + e] = 0.f;
    }
  }
  __syncthreads();
  EState st{qnan(), 0.f, 0.f, neg_inf(), 0, 0u, 0.0, 0, 0, 0.0};
  if (e == 0)
    while (st.issued < kS && st.issued < Eb) issue(s, eng, st, Eb, potb);
  zero_range(mgb + Eb * kCC, (E - Eb) * kCC / 4, tid);

  // ---- phase 1 -----------------------------------------------------------------------
  if (eng == 0)
    f_run<false, XM>(s, a, st, b, 0, h, Eb, potb, e, log2C);
  else
    b_run<false, XM>(s, a, st, b, h, Eb, Eb, potb, e, log2C);
  if (e == 0) s.O[eng] = st.O;
  if (st.bad) atomicOr(&s.bad[eng], 1u);
  __syncthreads();
  // ---- middle: log Z from the meeting node h --------------------------------------------
  if (tid < 32) {
    const int fb = (int)(h & 1), bbuf = (int)((Eb - h) & 1);
    const float v0 = s.ah_s[fb][tid] + s.bh_s[bbuf][tid];
    const float v1 = s.ah_s[fb][tid + 32] + s.bh_s[bbuf][tid + 32];
    const float mx = warp_max(fmaxf(v0, v1));
    const float sm = warp_sum(mx == neg_inf() ? 0.f : ex2(v0 - mx) + ex2(v1 - mx));
    const float Lh = (mx == neg_inf()) ? neg_inf() : mx + lg2(sm);
    const bool bad = (s.bad[0] | s.bad[1]) != 0u || Lh != Lh;
    if (tid == 0) {
      uint32_t fl = 0;
      float lz;
      if (bad) {
        fl = TS_F_NONFINITE;
        lz = qnan();
      } else if (Lh == neg_inf()) {
        fl = TS_F_EMPTY;
        lz = neg_inf();
      } else {
        lz = (float)(s.O[0] + s.O[1] + kLn2 * (double)Lh);
      }
      a.logz[b] = lz;
      if (a.flags) a.flags[b] = fl;
      s.Lh = Lh;
      s.dead = (bad || Lh == neg_inf()) ? 1 : 0;
    }
  }
  __syncthreads();
  if (s.dead) {
    zero_range(mgb, Eb * kCC / 4, tid);
    if (XM && tid < 2) a.xsum[2 * b + tid] = 0.0;
    if (e == 0)  // drain this engine's outstanding bulk copies before the CTA exits
      for (int64_t u = st.u; u < st.issued; ++u)
        mbar_wait(&s.full[eng][u % kS], (uint32_t)((u / kS) & 1));
    return;
  }
  // ---- phase 2 -----------------------------------------------------------------------
  if (eng == 0) {
    f_run<true, XM>(s, a, st, b, h, Eb, Eb, potb, e, log2C);
  } else {
    st.Lnext = s.Lh;
    b_run<true, XM>(s, a, st, b, 0, h, Eb, potb, e, log2C);
  }
  if (XM) {  // fused f1 epilogue: fixed-order engine reduction of the threads' Σ mu·x
    double v = st.xacc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((e & 31) == 0) s.xred[eng][e >> 5] = v;
    named_bar(1 + eng, kNTE);
    if (e == 0) {
      double tot = 0.0;
      for (int x = 0; x < kNW; ++x) tot += s.xred[eng][x];
      a.xsum[2 * b + eng] = tot;
    }
  }
}

std::atomic<uint64_t> g_meet_attr[3];
template <int XM>
cudaError_t launch_meet_x(const MeetArgs& a, cudaStream_t st) {
  cudaError_t e = smem_optin_once(meet64_kernel<XM>, g_meet_attr[XM], (int)sizeof(MeetSmem));
  if (e != cudaSuccess) return e;
  meet64_kernel<XM><<<(unsigned)a.B, kNT, sizeof(MeetSmem), st>>>(a);
  return cudaGetLastError();
}
}  // namespace

bool meet_ok(int64_t C, const float* pot, const float* marg) {
  return C == kC && (reinterpret_cast<uintptr_t>(pot) & 15) == 0 &&
         (reinterpret_cast<uintptr_t>(marg) & 15) == 0;
}

cudaError_t launch_meet(const MeetArgs& a, int64_t C, cudaStream_t st) {
  if (C != kC) return cudaErrorInvalidValue;
  if (a.xmode == 1) return launch_meet_x<1>(a, st);
  if (a.xmode == 2) return launch_meet_x<2>(a, st);
  return launch_meet_x<0>(a, st);
}

}  // namespace tsb
