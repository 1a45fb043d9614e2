// tiny.cuh — device code of the latency-optimised fused forward / backward / marginals for
// short chains with C % 4 == 0 and C <= 28 (the paper's Table 1 setting B=32, N=25, C=20,
// PAPER.md P:54): the one-CTA-per-sequence body `tiny_body` (the fb_tiny kernel, and the exact
// fallback of the cluster scan in fb_cscan.cu) and its recursion `tiny_sweep`.
// One CTA (kTinyThreads = 256 threads, two per SM) per sequence, the whole sequence resident in shared
// memory; the marginals are pipelined against the two serial recursions through per-node
// mbarriers.
//
// Same mathematics as fb_small.cu (§5.2 P:252-256 forward, P:181-183 marginals,
// §6(c) P:330-331 stabilised product):
//
//  * Load: each warp bulk-copies (TMA, cp.async.bulk) the tiles it preps into a dense raw
//    area, each onto its own mbarrier; the PDL prologue prefetches them into L2 while the
//    previous grid drains.
//  * Prepass (tiles t and t + W on warp t, W warps): T_t = max l_t, EX = 2^((l - T_t) log2 e)
//    stored row-major (EXB, spare row C = column sums) and transposed (EXF, spare row C = row
//    sums), row stride RS = 4 mod 8 (conflict-free LDS.128 row reads by lanes = rows).
//  * Recursions (forward on warp kFwdWarp, lane j <= C reads row j of EXF; backward on warp
//    kBwdWarp, lane i <= C reads row i of EXB; C/4 LDS.128 each), unnormalised linear vectors
//    with a lagged normaliser: lane j < C computes s_j = Σ_i u_t[i] X[i][j]; the spare lane C
//    computes Σ_i u_t[i] rowsum_i = Σ_j s_j in the same instruction stream.  The step output
//    is u_{t+1} = s · (1/U_t), U_t = the previous step's spare-lane value, so the reciprocal
//    runs beside the FMAs.  With alpha_t[i] = K_t + ln2 log2 u_t[i]:
//    K_{t+1} = K_t + T_t + ln2 c_t, c_t = log2 U_t.  Gate: a step whose output
//    has an entry below 2^-60 is redone (and the recursion continued) by the careful loop,
//    which recomputes gated steps exactly in log space from the exact log2 node values H and
//    x' = (l - T_t) log2 e (the §6(c) per-cell max) and records H, c_t for its steps.  The
//    gate of step k is voted one step late (in the shadow of step k+1's loads); node n is
//    published on fn[n] / bn[n] only once the step that produced it is known to be exact.
//  * Marginals (all other warps, centre edges first — those become ready first; they sleep on
//    the node barriers between edges): mu_t[i][j] = u_t[i] EX[i][j] v_{t+1}[j] / Z_t with Z_t
//    the warp sum of the same products (Σ_ij mu_t = 1 to rounding); edges with
//    Z_t / (U_t V_{t+1}) < 2^-30 are recomputed exactly in log space.
#pragma once
#include <atomic>

#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

#ifdef TINY_OCC_TRACE  // (debug, tools/occ_tiny.cu) per-CTA residency records:
                       // smid, %globaltimer at start / end / after the prepass / after the sweeps
__device__ unsigned long long g_occ_idx;
__device__ unsigned long long g_occ_rec[1 << 20][5];
__device__ __forceinline__ unsigned long long occ_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif
#ifdef TS_PHASE_TIMING
__device__ long long g_tiny_phase[1024][8];
__device__ long long g_tiny_steps[2][64];
__device__ long long g_tiny_wp[4][16][8];  // per warp phase stamps (prepass: 0 start, 3 max, 4 stores, 5 sums; 2 marginals done)
__device__ long long g_tiny_edge[64][4];   // cta 0 per edge: waited, summed, stored
#define TPHASE(k)                                                                       \
  do {                                                                                  \
    if (threadIdx.x == 0 && blockIdx.x < 1024) g_tiny_phase[blockIdx.x][k] = clock64(); \
  } while (0)
#define TPHASEW(k)                                                                             \
  do {                                                                                         \
    if ((threadIdx.x & 31) == 0 && blockIdx.x < 1024) g_tiny_phase[blockIdx.x][k] = clock64(); \
  } while (0)
#define TWARP(slot)                                                                 \
  do {                                                                              \
    if (lane == 0 && blockIdx.x < 4) g_tiny_wp[blockIdx.x][warp][slot] = clock64(); \
  } while (0)
#else
#define TPHASE(k) \
  do {            \
  } while (0)
#define TPHASEW(k) \
  do {             \
  } while (0)
#define TWARP(slot) \
  do {              \
  } while (0)
#endif

namespace {

#ifndef TINY_THREADS
// 256: two CTAs per SM (128 registers x 256 threads x 2, ~92 KB shared memory each at cfg2), so
// overlapping calls (PDL early mode) have twice the CTA slots: cfg2 1.45 -> 1.075 us/step.
// (One call alone: 384 was best in a 256-1024 sweep, 6.66 vs 6.71 us at 512.)
#define TINY_THREADS 256
#endif
constexpr int kTinyThreads = TINY_THREADS;
constexpr int kTinyWarps = kTinyThreads / 32;
// Recursion warps.  Warp 0 is avoided: a recursion on warp 0 measured ~4x slower per step
// (938 vs 226 cycles at C = 20, tools/phase_tiny.cu) for reasons not yet understood.
#ifndef TINY_FWD_WARP
#define TINY_FWD_WARP 2  // (fwd, bwd) warps swept at 384 threads: (2,3) 6.62 vs (1,2) 6.66 us/step
#endif
#ifndef TINY_BWD_WARP
#define TINY_BWD_WARP 3
#endif
constexpr int kFwdWarp = TINY_FWD_WARP;            // forward recursion
constexpr int kBwdWarp = TINY_BWD_WARP;            // backward recursion
constexpr int kWorkers = kTinyWarps - 2;           // marginal warps: all others
__device__ __forceinline__ int worker_index(int warp) {
  constexpr int lo = kFwdWarp < kBwdWarp ? kFwdWarp : kBwdWarp;
  constexpr int hi = kFwdWarp < kBwdWarp ? kBwdWarp : kFwdWarp;
  return warp < lo ? warp : (warp < hi ? warp - 1 : warp - 2);
}
constexpr float kZGate = 9.313225746154785e-10f;  // 2^-30 (marginal normaliser gate)
constexpr int kFlagSlot = 31;                      // V[n][31] = 1: node n has exact H[n]

// row stride of the tiles: = 4 mod 8 (conflict-free LDS.128 row reads by lanes = rows)
__host__ __device__ constexpr int tiny_rs(int C) { return (C % 8 == 4) ? C : C + 4; }

struct TinyLayout {
  int64_t raw, exf, exb, T, F, HF, G, HG, cf, bar, xred, total;  // float offsets
};

// mbarriers: ld[E] (tile loaded; TMA variants), fn[N], bn[N] (node published).  The raw tile
// area (a bulk-copy target) exists only in the TMA prepass variants: the default prepass
// reads the tiles from L2, and without it two CTAs fit on an SM.
#if defined(TINY_TMA_PREPASS) || defined(TINY_TMA_ROWS)
constexpr bool kTinyRaw = true;
#else
constexpr bool kTinyRaw = false;
#endif
__host__ __device__ inline TinyLayout tiny_layout(int64_t N, int C) {
  TinyLayout l;
  const int64_t E = N - 1 > 0 ? N - 1 : 1;
  const int64_t RS = tiny_rs(C), TB = (int64_t)(C + 1) * RS;
  l.raw = 0;                           // [E][C][C] dense (bulk-copy target, TMA variants)
  l.exf = l.raw + (kTinyRaw ? E * C * C : 0);  // EXF: [E][C+1][RS] row j = column j of EX, row C = row sums
  l.exb = l.exf + E * TB;              // EXB: [E][C+1][RS] row i = row i of EX, row C = col sums
  l.T = l.exb + E * TB;                // [E]
  l.cf = l.T + E;                      // [E] forward increments c_t (log2), careful steps
  l.F = (l.cf + E + 3) & ~(int64_t)3;  // [N][32] forward linear u_n (slot C: U_n, 31: flag)
  l.HF = l.F + N * 32;                 // [N][32] forward exact log2 u_n (careful nodes)
  l.G = l.HF + N * 32;                 // [N][32] backward linear v_n (slot C: V_n, 31: flag)
  l.HG = l.G + N * 32;                 // [N][32] backward exact log2 v_n
  l.bar = (l.HG + N * 32 + 3) & ~(int64_t)3;
  l.xred = l.bar + 2 * (E + 2 * N) + 8;    // mbarriers (2 floats each) + flag words
  l.total = l.xred + 2 * 32;               // fused f1 epilogue: per-warp fp64 partials
  return l;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Order in which edges become ready for marginals (edge t needs forward node t and backward
// node t+1): centre first, ready(t) = max(t, Eb-1-t).
__device__ __forceinline__ int edge_order(int q, int Eb) {
  const int lo = (Eb - 1) >> 1, hi = Eb - 1 - lo;
  if (lo == hi) {
    if (q == 0) return lo;
    const int j = (q + 1) >> 1;
    return (q & 1) ? lo - j : hi + j;
  }
  return (q & 1) ? hi + (q >> 1) : lo - (q >> 1);
}

// Exact log2 of node n's vector entry j: recorded by the careful loop (flag slot), else
// the linear value is >= 2^-60 of its scale and lg2 recovers it.
__device__ __forceinline__ float node_log(const float* V, const float* H, int n, int j) {
  return V[n * 32 + kFlagSlot] != 0.f ? H[n * 32 + j] : lg2(V[n * 32 + j]);
}

// One recursion (FWD: nodes 0 -> Eb over EXF; !FWD: nodes Eb -> 0 over EXB).  Lane r <= C
// reads row r of the edge's matrix; lanes > C mirror row 0 and their results are discarded.
// Returns kb, the first step run by the careful loop (Eb if none).
template <bool FWD, int C>
__device__ __forceinline__ void tiny_row(const float* __restrict__ X, int row, float (&mv)[C]) {
  constexpr int RS = tiny_rs(C);
#pragma unroll
  for (int q = 0; q < C / 4; ++q) {
    const float4 w = *reinterpret_cast<const float4*>(X + row * RS + 4 * q);
    mv[4 * q] = w.x;
    mv[4 * q + 1] = w.y;
    mv[4 * q + 2] = w.z;
    mv[4 * q + 3] = w.w;
  }
}

// TS: tile stride in floats (the distance between consecutive edges' matrices; default TB).
template <bool FWD, int C, int TS = (C + 1) * tiny_rs(C)>
__device__ __forceinline__ int tiny_sweep(const float* __restrict__ Xall, const float* __restrict__ raw,
                                          const float* __restrict__ Tm, float* __restrict__ V,
                                          float* __restrict__ H, float* __restrict__ cinc,
                                          uint64_t* nb, int Eb, int lane, float v0) {
  constexpr int RS = tiny_rs(C), Q = C / 4;
  const bool act = lane < C;
  const bool live = lane <= C;
  const int row = live ? lane : 0;
  const int n0 = FWD ? 0 : Eb;
  V[n0 * 32 + lane] = v0;  // start node: lanes < C its entries, lane C their sum, others 0
  __syncwarp();
  if (lane == 0) mbar_arrive(&nb[n0]);
  if (Eb == 0) return 0;
  float m[C], mn[C];
  // running pointers (no per-step index arithmetic on the chain)
  const float* mp = Xall + (int64_t)(FWD ? 0 : Eb - 1) * TS + row * RS;  // this edge's row
  const float* u = V + n0 * 32;                                          // input node
  uint64_t* np = nb + n0;                                                // input node barrier
  constexpr int dT = FWD ? TS : -TS, dV = FWD ? 32 : -32, dN = FWD ? 1 : -1;
  tiny_row<FWD, C>(mp, 0, m);
  int kb = Eb;
  bool prev_bad = false;
  for (int k = 0; k < Eb; ++k) {
    float4 x[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) x[q] = *reinterpret_cast<const float4*>(u + 4 * q);  // broadcast
    const float U = u[C];
    if (k > 0) {  // verify step k-1 (in the shadow of the loads), then publish its node
      if (__any_sync(0xffffffffu, prev_bad)) {
        kb = k - 1;
        break;
      }
#ifndef TINY_NO_PUBLISH
      if (lane == 0) mbar_arrive(np);
#endif
    }
    // the next edge's operand (independent of the chain; consumed next step)
    if (k + 1 < Eb) tiny_row<FWD, C>(mp + dT, 0, mn);
    const float r = rcp_approx(U);
    float sa[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      sa[0] = fmaf(x[q].x, m[4 * q], sa[0]);
      sa[1] = fmaf(x[q].y, m[4 * q + 1], sa[1]);
      sa[2] = fmaf(x[q].z, m[4 * q + 2], sa[2]);
      sa[3] = fmaf(x[q].w, m[4 * q + 3], sa[3]);
    }
    const float un = ((sa[0] + sa[1]) + (sa[2] + sa[3])) * r;
    const_cast<float*>(u)[dV + lane] = live ? un : 0.f;
    prev_bad = live && !(un >= kGate);
#pragma unroll
    for (int i = 0; i < C; ++i) m[i] = mn[i];
    u += dV;
    mp += dT;
    np += dN;
    __syncwarp();
#if defined(TS_PHASE_TIMING) && !defined(TS_PHASE_NOSTEPS)  // per-step stores cost ~70 cycles/step
    if (blockIdx.x == 0 && lane == 0 && k < 64) g_tiny_steps[FWD ? 0 : 1][k] = clock64();
#endif
  }
  if (kb == Eb) {  // the last step's verdict
    if (!__any_sync(0xffffffffu, prev_bad)) {
      if (lane == 0) mbar_arrive(&nb[FWD ? Eb : 0]);
      return Eb;
    }
    kb = Eb - 1;
  }
  // ---- careful loop from step kb ---------------------------------------------------------
  {
    const int t = FWD ? kb : Eb - 1 - kb;
    const int nin = FWD ? t : t + 1;
    // the start node is already published (consumers recover its logs as lg2 of V); its
    // exact logs for this loop's gated steps are the same lg2 values
    const float x = V[nin * 32 + lane];
    H[nin * 32 + lane] = act ? lg2(x) : neg_inf();
    __syncwarp();
  }
  for (int k = kb; k < Eb; ++k) {
    const int t = FWD ? k : Eb - 1 - k;
    const int nin = FWD ? t : t + 1;
    const int nout = FWD ? t + 1 : t;
    float w[C];
    tiny_row<FWD, C>(Xall + (int64_t)t * TS, row, w);
    const float* u = V + nin * 32;
    const float U = u[C];
    const float r = rcp_approx(U);
    float sa[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      const float4 xx = *reinterpret_cast<const float4*>(u + 4 * q);
      sa[0] = fmaf(xx.x, w[4 * q], sa[0]);
      sa[1] = fmaf(xx.y, w[4 * q + 1], sa[1]);
      sa[2] = fmaf(xx.z, w[4 * q + 2], sa[2]);
      sa[3] = fmaf(xx.w, w[4 * q + 3], sa[3]);
    }
    const float un = ((sa[0] + sa[1]) + (sa[2] + sa[3])) * r;
    const bool gated = live && !(un >= kGate);
    if (__any_sync(0xffffffffu, gated)) {
      // exact log-space recomputation of the whole step (§6(c) per-cell max), renormalised
      const float* hin = H + nin * 32;
      const float* rt = raw + (int64_t)t * C * C;
      const float Tt = Tm[t];
      float tl = neg_inf();
      if (act) {
        float q = neg_inf();
        for (int i = 0; i < C; ++i) {
          const float xv = (FWD ? rt[i * C + lane] : rt[lane * C + i]) - Tt;
          q = fmaxf(q, hin[i] + xv * kLog2e);
        }
        if (q != neg_inf()) {
          float ss = 0.f;
          for (int i = 0; i < C; ++i) {
            const float xv = (FWD ? rt[i * C + lane] : rt[lane * C + i]) - Tt;
            ss += ex2(hin[i] + xv * kLog2e - q);
          }
          tl = q + lg2(ss);
        }
      }
      const float L = warp_lse2(tl);
      const bool dead = (L == neg_inf());
      const float h = dead ? neg_inf() : tl - L;
      V[nout * 32 + lane] = act ? (dead ? 0.f : ex2(h))
                                : (lane == C ? 1.f : (lane == kFlagSlot ? 1.f : 0.f));
      H[nout * 32 + lane] = act ? h : neg_inf();
      if (FWD && lane == 0) cinc[t] = L;
    } else {
      V[nout * 32 + lane] = live ? un : (lane == kFlagSlot ? 1.f : 0.f);
      H[nout * 32 + lane] = act ? lg2(un) : neg_inf();
      if (FWD && lane == 0) cinc[t] = lg2(U);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&nb[nout]);
  }
  return kb;
}

}  // namespace

// Prepass over tiles [0, Eb) (raw tiles arriving on ld[t]): tiles t0 = warp + 2 W r and
// t1 = t0 + W (W = nwarps warps, two tiles in flight per warp): T_t = max l_t, EX into EXB
// (row-major, spare row C = column sums) and EXF (transposed, spare row C = row sums);
// NaN / +inf sets TS_F_NONFINITE in *sflag.  The caller synchronises afterwards.
template <int C, int TS = (C + 1) * tiny_rs(C)>
__device__ __forceinline__ void tiny_prepass(const float* __restrict__ raw, float* __restrict__ EXF,
                                             float* __restrict__ EXB, float* __restrict__ Tm,
                                             uint64_t* ld, unsigned* sflag, int Eb, int warp,
                                             int nwarps, int lane) {
  constexpr int RS = tiny_rs(C), CC = C * C, Q4 = CC / 4, Q = C / 4;
  for (int t0 = warp; t0 < Eb; t0 += 2 * nwarps) {
    constexpr int NV = (Q4 + 31) / 32;
    const int t1 = t0 + nwarps;
    const int nt = t0 < Eb ? (t1 < Eb ? 2 : 1) : 0;
    float4 v[2][NV];
    float mx[2] = {neg_inf(), neg_inf()};
    bool bad = false;
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      if (n < nt) {
        const int t = n ? t1 : t0;
        mbar_wait(&ld[t], 0);
        const float4* rt = reinterpret_cast<const float4*>(raw + (int64_t)t * CC);
#pragma unroll
        for (int m = 0; m < NV; ++m) {
          const int k = lane + 32 * m;
          v[n][m] = k < Q4 ? rt[k] : make_float4(neg_inf(), neg_inf(), neg_inf(), neg_inf());
          mx[n] = fmaxf(mx[n], fmaxf(fmaxf(v[n][m].x, v[n][m].y), fmaxf(v[n][m].z, v[n][m].w)));
          bad |= (v[n][m].x != v[n][m].x) | (v[n][m].y != v[n][m].y) |
                 (v[n][m].z != v[n][m].z) | (v[n][m].w != v[n][m].w) |
                 (v[n][m].x == pos_inf()) | (v[n][m].y == pos_inf()) |
                 (v[n][m].z == pos_inf()) | (v[n][m].w == pos_inf());
        }
      }
    }
    if (nt > 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mx[0] = fmaxf(mx[0], __shfl_xor_sync(0xffffffffu, mx[0], o));
        mx[1] = fmaxf(mx[1], __shfl_xor_sync(0xffffffffu, mx[1], o));
      }
      if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(sflag, (unsigned)TS_F_NONFINITE);
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        if (n < nt) {
          const int t = n ? t1 : t0;
          const float Tz = (mx[n] == neg_inf()) ? 0.f : mx[n];  // all-masked tile: EX = 0
          float* xb = EXB + (int64_t)t * TS;
          float* xf = EXF + (int64_t)t * TS;
          if (lane == 0) Tm[t] = Tz;
#pragma unroll
          for (int m = 0; m < NV; ++m) {
            const int k = lane + 32 * m;
            if (k < Q4) {
              const int i = (4 * k) / C, j = 4 * k - i * C;
              float4 e;
              e.x = ex2((v[n][m].x - Tz) * kLog2e);
              e.y = ex2((v[n][m].y - Tz) * kLog2e);
              e.z = ex2((v[n][m].z - Tz) * kLog2e);
              e.w = ex2((v[n][m].w - Tz) * kLog2e);
              *reinterpret_cast<float4*>(xb + i * RS + j) = e;
              xf[(j + 0) * RS + i] = e.x;
              xf[(j + 1) * RS + i] = e.y;
              xf[(j + 2) * RS + i] = e.z;
              xf[(j + 3) * RS + i] = e.w;
            }
          }
        }
      }
      __syncwarp();
      if (lane < C) {
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          if (n < nt) {
            const int t = n ? t1 : t0;
            float* xb = EXB + (int64_t)t * TS;
            float* xf = EXF + (int64_t)t * TS;
            float rs = 0.f, cs = 0.f;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
              const float4 x = *reinterpret_cast<const float4*>(xb + lane * RS + 4 * q);  // row
              const float4 y = *reinterpret_cast<const float4*>(xf + lane * RS + 4 * q);  // column
              rs += (x.x + x.y) + (x.z + x.w);
              cs += (y.x + y.y) + (y.z + y.w);
            }
            xf[C * RS + lane] = rs;  // forward spare row: row sums (indexed by i)
            xb[C * RS + lane] = cs;  // backward spare row: column sums (indexed by j)
          }
        }
      }
    }
  }
}

__device__ __forceinline__ float fmax_nan_t(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// Row-per-lane prepass over tiles [0, Eb) read straight from global memory (src = the
// sequence's first tile; L2-warm: the PDL prologue prefetched it): tiles t0 = warp + 2 W r and
// t1 = t0 + W, lane i < C owns row i of both (C/4 float4 loads each).  Row max and the row
// sum are lane-local, T_t by a warp max; EXB rows are STS.128 (RS = 4 mod 8: conflict-free),
// the transposed EXF gets C scalar stores per lane at consecutive addresses (conflict-free),
// EXF's spare row = the row sums; the column sums (EXB's spare row) re-read EXF rows.
// Shared memory sees ~46 wavefronts per 20 x 20 tile instead of ~100 (TMA write + raw read +
// conflicted transposed stores + two sum re-reads).  NaN / +inf -> TS_F_NONFINITE.
// ld: per-tile mbarriers of a TMA-staged raw area at `src` (nullptr: src is global memory).
template <int C, int TS = (C + 1) * tiny_rs(C)>
__device__ __forceinline__ void tiny_prepass_rows(const float* __restrict__ src, float* __restrict__ EXF,
                                                  float* __restrict__ EXB, float* __restrict__ Tm,
                                                  unsigned* sflag, int Eb, int warp, int nwarps,
                                                  int lane, uint64_t* ld = nullptr) {
  constexpr int RS = tiny_rs(C), CC = C * C, Q = C / 4;
  const bool act = lane < C;
  for (int t0 = warp; t0 < Eb; t0 += 2 * nwarps) {
    const int t1 = t0 + nwarps;
    const int nt = t1 < Eb ? 2 : 1;
    float4 v[2][Q];
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      const int t = n ? t1 : t0;
      if (ld && n < nt) mbar_wait(&ld[t], 0);
#pragma unroll
      for (int q = 0; q < Q; ++q)
        v[n][q] = (act && n < nt) ? reinterpret_cast<const float4*>(src + (int64_t)t * CC + lane * C)[q]
                                  : make_float4(neg_inf(), neg_inf(), neg_inf(), neg_inf());
    }
    float mx[2], mn[2];
    TWARP(0);
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      float m = neg_inf();
#pragma unroll
      for (int q = 0; q < Q; ++q)
        m = fmax_nan_t(m, fmax_nan_t(fmax_nan_t(v[n][q].x, v[n][q].y), fmax_nan_t(v[n][q].z, v[n][q].w)));
      mn[n] = m;  // NaN-propagating: a NaN / +inf input surfaces here
      mx[n] = m;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mx[0] = fmax_nan_t(mx[0], __shfl_xor_sync(0xffffffffu, mx[0], o));
      mx[1] = fmax_nan_t(mx[1], __shfl_xor_sync(0xffffffffu, mx[1], o));
    }
    const bool bad = (mx[0] != mx[0]) | (mx[0] == pos_inf()) |
                     ((nt > 1) & ((mx[1] != mx[1]) | (mx[1] == pos_inf())));
    (void)mn;
    if (bad && lane == 0) atomicOr(sflag, (unsigned)TS_F_NONFINITE);
    TWARP(3);
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      if (n < nt) {
        const int t = n ? t1 : t0;
        const float Tz = (mx[n] == neg_inf() || !(mx[n] == mx[n]) || mx[n] == pos_inf()) ? 0.f : mx[n];
        float* xb = EXB + (int64_t)t * TS;
        float* xf = EXF + (int64_t)t * TS;
        if (lane == 0) Tm[t] = Tz;
        float rs = 0.f;
        if (act) {
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            float4 e;
            e.x = ex2((v[n][q].x - Tz) * kLog2e);
            e.y = ex2((v[n][q].y - Tz) * kLog2e);
            e.z = ex2((v[n][q].z - Tz) * kLog2e);
            e.w = ex2((v[n][q].w - Tz) * kLog2e);
            rs += (e.x + e.y) + (e.z + e.w);
            *reinterpret_cast<float4*>(xb + lane * RS + 4 * q) = e;
            xf[(4 * q + 0) * RS + lane] = e.x;
            xf[(4 * q + 1) * RS + lane] = e.y;
            xf[(4 * q + 2) * RS + lane] = e.z;
            xf[(4 * q + 3) * RS + lane] = e.w;
          }
          xf[C * RS + lane] = rs;  // forward spare row: row sums (indexed by i)
        }
      }
    }
    __syncwarp();
    TWARP(4);
    if (act) {
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        if (n < nt) {
          const int t = n ? t1 : t0;
          const float* xf = EXF + (int64_t)t * TS;
          float cs[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int q = 0; q < Q; ++q) {
            const float4 y = *reinterpret_cast<const float4*>(xf + lane * RS + 4 * q);  // column
            cs[0] += y.x;
            cs[1] += y.y;
            cs[2] += y.z;
            cs[3] += y.w;
          }
          EXB[(int64_t)t * TS + C * RS + lane] = (cs[0] + cs[1]) + (cs[2] + cs[3]);  // column sums
        }
      }
    }
    TWARP(5);
  }
}

// Marginal worker loop (one warp per edge, centre edges first): edge t waits for forward node
// t (fn[t]) and backward node t + 1 (bn[t+1]), then writes mu_t = u_t[i] EX[i][j] v_{t+1}[j] / Z_t
// (exact log-space edge when Z_t / (U_t V_{t+1}) < 2^-30) to mg + t C^2.  Worker wi of
// nworkers takes the edges qe = wi, wi + nworkers, ... of the centre-first order.
// Fused f1 epilogue (xm != 0): the lane accumulates Σ mu·x over the elements it
// writes (x = l from the staged raw tiles for xm = 1, x = xr[t] (global) for xm = 2; terms
// with mu = 0 skipped), in a fixed order, into *xacc.
template <int C, int TS = (C + 1) * tiny_rs(C), int XM = 0>
__device__ __forceinline__ void tiny_marginals(const float* __restrict__ EXB, const float* __restrict__ raw,
                                               const float* __restrict__ Tm, const float* __restrict__ F,
                                               const float* __restrict__ HF, const float* __restrict__ G,
                                               const float* __restrict__ HG, uint64_t* fn, uint64_t* bn,
                                               int Eb, float* __restrict__ mg, int wi, int nworkers,
                                               int lane, const float* __restrict__ xr = nullptr,
                                               double* xacc = nullptr) {
  constexpr int xm = XM;
  constexpr int RS = tiny_rs(C), CC = C * C, Q4 = CC / 4;
  constexpr int NV = (Q4 + 31) / 32;
      for (int qe = wi; qe < Eb; qe += nworkers) {
        const int t = edge_order(qe, Eb);
#ifndef TINY_SLEEP_NS
#define TINY_SLEEP_NS 64  // swept 32-512: 64 best (6.710 vs 6.735 us/step at 128)
#endif
#ifdef TINY_NO_CONSUMERS
        break;
#endif
#ifdef TINY_BN_FIRST
        mbar_wait_sleep(&bn[t + 1], 0, TINY_SLEEP_NS);
        mbar_wait_sleep(&fn[t], 0, TINY_SLEEP_NS);
#else
        mbar_wait_sleep(&fn[t], 0, TINY_SLEEP_NS);
        mbar_wait_sleep(&bn[t + 1], 0, TINY_SLEEP_NS);
#endif
#ifdef TS_PHASE_TIMING
        if (blockIdx.x == 0 && lane == 0 && t < 64) g_tiny_edge[t][0] = clock64();
#endif
        const float* u = F + t * 32;
        const float* v = G + (t + 1) * 32;
        const float* xb = EXB + (int64_t)t * TS;
        float4 val[NV];
        float z = 0.f;
#pragma unroll
        for (int m = 0; m < NV; ++m) {
          const int k = lane + 32 * m;
          if (k < Q4) {
            const int i = (4 * k) / C, j = 4 * k - i * C;
            const float ui = u[i];
            const float4 e = *reinterpret_cast<const float4*>(xb + i * RS + j);
            const float4 vj = *reinterpret_cast<const float4*>(v + j);
            val[m] = make_float4(ui * e.x * vj.x, ui * e.y * vj.y, ui * e.z * vj.z, ui * e.w * vj.w);
            z += (val[m].x + val[m].y) + (val[m].z + val[m].w);
          }
        }
        z = warp_sum(z);
#ifdef TS_PHASE_TIMING
        if (blockIdx.x == 0 && lane == 0 && t < 64) g_tiny_edge[t][1] = clock64();
#endif
        float4* out = reinterpret_cast<float4*>(mg + (int64_t)t * CC);
        if (z >= kZGate * (u[C] * v[C])) {
          const float rz = __fdividef(1.f, z);
          float xe = 0.f;
#pragma unroll
          for (int m = 0; m < NV; ++m) {
            const int k = lane + 32 * m;
            if (k < Q4) {
              const float4 o = make_float4(val[m].x * rz, val[m].y * rz, val[m].z * rz, val[m].w * rz);
              out[k] = o;
              if (xm) {
                const float4 x = reinterpret_cast<const float4*>((xm == 1 ? raw : xr) + (int64_t)t * CC)[k];
                if (o.x != 0.f) xe = fmaf(o.x, x.x, xe);
                if (o.y != 0.f) xe = fmaf(o.y, x.y, xe);
                if (o.z != 0.f) xe = fmaf(o.z, x.z, xe);
                if (o.w != 0.f) xe = fmaf(o.w, x.w, xe);
              }
            }
          }
          if (xm) *xacc += (double)xe;
#ifdef TS_PHASE_TIMING
          if (blockIdx.x == 0 && lane == 0 && t < 64) g_tiny_edge[t][2] = clock64();
#endif
        } else {
          // exact log-space edge: mu = 2^(h_t[i] + x'_ij + g_{t+1}[j] - Lz)
          const float hu = lane < C ? node_log(F, HF, t, lane) : neg_inf();
          const float hv = lane < C ? node_log(G, HG, t + 1, lane) : neg_inf();
          const float* rt = raw + (int64_t)t * CC;
          const float Tt = Tm[t];
          float mxl = neg_inf();
          for (int k0 = 0; k0 < CC; k0 += 32) {
            const int k = k0 + lane, kk = k < CC ? k : 0;
            const int i = kk / C, j = kk - i * C;
            const float hi = __shfl_sync(0xffffffffu, hu, i), hj = __shfl_sync(0xffffffffu, hv, j);
            if (k < CC) mxl = fmaxf(mxl, hi + (rt[k] - Tt) * kLog2e + hj);
          }
          mxl = warp_max(mxl);
          float ss = 0.f;
          for (int k0 = 0; k0 < CC; k0 += 32) {
            const int k = k0 + lane, kk = k < CC ? k : 0;
            const int i = kk / C, j = kk - i * C;
            const float hi = __shfl_sync(0xffffffffu, hu, i), hj = __shfl_sync(0xffffffffu, hv, j);
            if (k < CC && mxl != neg_inf()) ss += ex2(hi + (rt[k] - Tt) * kLog2e + hj - mxl);
          }
          ss = warp_sum(ss);
          const float Lz = (mxl == neg_inf()) ? pos_inf() : mxl + lg2(ss);
          float* o = mg + (int64_t)t * CC;
          float xe = 0.f;
          for (int k0 = 0; k0 < CC; k0 += 32) {
            const int k = k0 + lane, kk = k < CC ? k : 0;
            const int i = kk / C, j = kk - i * C;
            const float hi = __shfl_sync(0xffffffffu, hu, i), hj = __shfl_sync(0xffffffffu, hv, j);
            if (k < CC) {
              const float mu = ex2(hi + (rt[k] - Tt) * kLog2e + hj - Lz);
              o[k] = mu;
              if (xm && mu != 0.f) xe = fmaf(mu, (xm == 1 ? raw : xr)[(int64_t)t * CC + k], xe);
            }
          }
          if (xm) *xacc += (double)xe;
        }
      }
}

// The whole-sequence body: one CTA of kTinyThreads threads processes sequence b with the
// shared memory at `sm` (tiny_layout).  PROLOGUE: this call owns the PDL handshake
// (launch_dependents, L2 prefetch, griddepcontrol.wait — before the first read, or with
// a.early before each thread's first global write); the cluster scan's exact fallback calls
// it with PROLOGUE = false after its own prologue.
template <int C, bool PROLOGUE, int XM = 0>
__device__ __forceinline__ void tiny_body(const SmallArgs& a, const int64_t b, float* __restrict__ sm) {
  constexpr int CC = C * C, Q4 = CC / 4;
  const int64_t N = a.N, E = N - 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const TinyLayout Lay = tiny_layout(N, C);
  const int64_t Ea = E > 0 ? E : 1;
  float* raw = sm + Lay.raw;
  float* EXF = sm + Lay.exf;
  float* EXB = sm + Lay.exb;
  float* Tm = sm + Lay.T;
  float* cf = sm + Lay.cf;
  float* F = sm + Lay.F;
  float* HF = sm + Lay.HF;
  float* G = sm + Lay.G;
  float* HG = sm + Lay.HG;
  uint64_t* ld = reinterpret_cast<uint64_t*>(sm + Lay.bar);
  uint64_t* fn = ld + Ea;
  uint64_t* bn = fn + N;
  unsigned* sflag = reinterpret_cast<unsigned*>(bn + N);

  // programmatic dependent launch: the next kernel in the stream may start now (first thing:
  // the next grid launches only once every CTA of this one has triggered, so the trigger's
  // position sets the launch-to-launch floor of back-to-back calls)
  if (PROLOGUE) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef TINY_OCC_TRACE
  const unsigned long long occ_t0 = occ_now();
#endif
  // barriers for every tile / node slot, initialised in parallel before any global access
  for (int64_t k = tid; k < E + 2 * N; k += kTinyThreads)
    mbar_init(k < E ? &ld[k] : (k < E + N ? &fn[k - E] : &bn[k - E - N]), 1);
  if (tid == 0) *sflag = 0u;
  fence_mbar_init();
  if (PROLOGUE) {
#ifndef TINY_NO_L2_PREFETCH
  // While the previous grid drains, warm L2 with this sequence's tiles (all N-1 edges, so no
  // input is read yet): a prefetch is only a hint and L2 is the coherence point, so a tile
  // the previous grid might still write cannot be observed stale.
  if (lane == 0 && a.pot)
    for (int64_t t = warp; t < E; t += kTinyWarps)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.pot + (b * E + t) * CC),
                   "r"((uint32_t)(CC * 4))
                   : "memory");
#endif
  if (!a.early) asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  __syncthreads();

  const int64_t len = seq_len(a.lengths, b, N);
  float* mg = a.marg ? a.marg + b * E * CC : nullptr;
  if (len < 0) {  // BADLEN: logZ NaN, marginals 0
    if (PROLOGUE && a.early) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (mg)
      for (int64_t k = tid; k < E * Q4; k += kTinyThreads)
        reinterpret_cast<float4*>(mg)[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (tid == 0) {
      a.logz[b] = qnan();
      if (a.flags) a.flags[b] = TS_F_BADLEN;
      if (XM) a.xout[b] = qnan();
    }
    return;
  }
  const int Eb = (int)(len - 1);
  const float* src = a.pot + b * E * CC;
  // each warp bulk-copies the tiles it preps
  const int wi = worker_index(warp);
#if defined(TINY_TMA_PREPASS)  // (variant: TMA staging, float4-per-lane prepass)
  if (lane == 0)
    for (int t = warp; t < Eb; t += kTinyWarps)
      bulk_load(raw + (int64_t)t * CC, src + (int64_t)t * CC, (uint32_t)(CC * 4), &ld[t]);
  TPHASE(0);
  tiny_prepass<C>(raw, EXF, EXB, Tm, ld, sflag, Eb, warp, kTinyWarps, lane);
#elif defined(TINY_TMA_ROWS)  // (variant: TMA staging, row-per-lane reads; faster eager, 6.22
                              // vs 5.97 us/step in the bench's graph)
  if (lane == 0)
    for (int t = warp; t < Eb; t += kTinyWarps)
      bulk_load(raw + (int64_t)t * CC, src + (int64_t)t * CC, (uint32_t)(CC * 4), &ld[t]);
  TPHASE(0);
  tiny_prepass_rows<C>(raw, EXF, EXB, Tm, sflag, Eb, warp, kTinyWarps, lane, ld);
#else  // default: row-per-lane straight from L2 (the PDL prologue prefetched the tiles)
  TPHASE(0);
  tiny_prepass_rows<C>(src, EXF, EXB, Tm, sflag, Eb, warp, kTinyWarps, lane);
  raw = const_cast<float*>(src);  // the exact (careful / gated) paths read the raw tiles here
#endif
  __syncthreads();
  TPHASE(2);
#ifdef TINY_OCC_TRACE
  const unsigned long long occ_t1 = occ_now();
#endif

  const float ones0 = lane < C ? 1.f : (lane == C ? (float)C : 0.f);  // log-one start vector
  double xacc = 0.0;  // fused f1 epilogue: this lane's Σ mu·x
  if (warp == kFwdWarp) {
    // ---- forward recursion, then logZ -------------------------------------------------
    const int kbf = tiny_sweep<true, C>(EXF, raw, Tm, F, HF, cf, fn, Eb, lane, ones0);
    TPHASEW(3);
    // logZ = Σ_t (T_t + ln2 c_t) + ln2 log2 Σ_j u_E[j]  (fp64 offsets, exact log sum);
    // c_t = log2 U_t for fast steps, recorded by the careful loop for t >= kbf
    double part = 0.0;
    for (int t = lane; t < Eb; t += 32)
      part += (double)Tm[t] + kLn2 * (double)(t < kbf ? lg2(F[t * 32 + C]) : cf[t]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    const float Lf = warp_lse2(lane < C ? node_log(F, HF, Eb, lane) : neg_inf());
    if (PROLOGUE && (a.early & 5) == 1) asm volatile("griddepcontrol.wait;" ::: "memory");  // logZ
    if (lane == 0) {
      const bool empty = (Lf == neg_inf()) || !(part > -INFINITY);
      a.logz[b] = empty ? neg_inf() : (float)(part + kLn2 * (double)Lf);
      if (empty) atomicOr(sflag, (unsigned)TS_F_EMPTY);
    }
  } else if (warp == kBwdWarp) {
    if (mg) {
      tiny_sweep<false, C>(EXB, raw, Tm, G, HG, nullptr, bn, Eb, lane, ones0);
      TPHASEW(4);
    }
  } else {
    // ---- marginals: centre edges first, one warp per edge, float4-wide -------------------
    if (mg) {
      if (PROLOGUE && (a.early & 3) == 1) asm volatile("griddepcontrol.wait;" ::: "memory");  // marginals
      tiny_marginals<C, (C + 1) * tiny_rs(C), XM>(EXB, raw, Tm, F, HF, G, HG, fn, bn, Eb, mg, wi,
                                                  kWorkers, lane, XM == 2 ? a.xr + b * E * CC : nullptr,
                                                  &xacc);
      for (int64_t k = (int64_t)Eb * Q4 + (32 * wi + lane); k < E * Q4; k += 32 * kWorkers)
        reinterpret_cast<float4*>(mg)[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    TWARP(2);
  }
  __syncthreads();
  TPHASE(5);
#ifdef TINY_OCC_TRACE
  const unsigned long long occ_t2 = occ_now();
#endif
  if (PROLOGUE && (a.early & 5) == 1) asm volatile("griddepcontrol.wait;" ::: "memory");  // tail writes
  const unsigned fl = (*sflag & TS_F_NONFINITE) ? (unsigned)TS_F_NONFINITE : *sflag;
  if (tid == 0 && a.flags) a.flags[b] = fl;
  if ((fl & TS_F_NONFINITE) && tid == 0) a.logz[b] = qnan();
  if (mg && (fl & (TS_F_EMPTY | TS_F_NONFINITE)))
    for (int64_t k = tid; k < E * Q4; k += kTinyThreads)
      reinterpret_cast<float4*>(mg)[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (XM) {  // fused f1 epilogue: fixed-order CTA reduction, H = A - Σ mu·l or Σ mu·r
    double* xred = reinterpret_cast<double*>(sm + Lay.xred);
    double v = xacc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) xred[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double tot = 0.0;
      for (int w = 0; w < kTinyWarps; ++w) tot += xred[w];
      const float lz = a.logz[b];
      const bool bad = fl != 0u || !(lz > -INFINITY && lz < INFINITY);
      a.xout[b] = bad ? qnan() : (float)(XM == 1 ? (double)lz - tot : tot);
    }
  }
  // the call completes only after its predecessor, so everything after it on the stream stays
  // ordered after both: with every write done before the wait (early == 7) one CTA waiting is
  // enough and the others free their SM slots for the calls behind; otherwise every thread
  // has waited already
  if (PROLOGUE && a.early && (a.early != 7 || b == 0)) asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef TINY_OCC_TRACE
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    const unsigned long long i = atomicAdd(&g_occ_idx, 1ull) & ((1 << 20) - 1);
    g_occ_rec[i][0] = smid;
    g_occ_rec[i][1] = occ_t0;
    g_occ_rec[i][2] = occ_now();
    g_occ_rec[i][3] = occ_t1;
    g_occ_rec[i][4] = occ_t2;
  }
#endif
}

// The cluster scan's exact fallback: one non-inlined copy of the body, so the cluster
// kernel's hot path stays small (it measured instruction-fetch bound with the body inlined).
template <int C>
__device__ __noinline__ void tiny_body_fallback(const SmallArgs& a, const int64_t b, float* __restrict__ sm) {
  tiny_body<C, false>(a, b, sm);
}

}  // namespace tsb
