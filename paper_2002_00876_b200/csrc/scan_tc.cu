// scan_tc.cu — leaf chunk summaries of the time-chunked scan (§6(a)) on
// the sm_100a tensor cores, for 64 < C <= 128 (even C).  A leaf summary is the log-semiring
// product S_k = l_{s_k} (x) ... (x) l_{e_k - 1} of the chunk's C x C edge tiles (Fig. 4
// leaves).  In the exp-shifted form of §6(c) each log product becomes a real
// matrix product of non-negative matrices:
//
//   S_{u+1}[m][j] = LSE_i(S_u[m][i] + l_u[i][j])
//                 = off_m + R_u + ln sum_i (Ahat_u[m][i] w_i) X_u[i][j]
//   r_i = max_j l_u[i][j] (row shift), R_u = max_i r_i, w_i = e^(r_i - R_u) <= 1,
//   X_u[i][j] = e^(l_u[i][j] - r_i) <= 1,  S_u[m][i] = off_m + ln Ahat_u[m][i]
//
// D = (Ahat o w) . X runs on tcgen05 kind::tf32 as 3xTF32 (hi.hi + hi.lo + lo.hi, fp32
// accumulate in TMEM; measured max relative error 2.9e-6 per 128^3 product vs 3.7e-4 for a
// single TF32 pass, tools/tc_probe.cu).  Default shift (predicted): one scalar per tile, r_i =
// R_u = T_u for every row, so w = 1 and X_u = e^(l_u - T_u) with T_u = the previous tile's
// max (tile 0: its own) — the producers need ONE pass per tile and the epilogue never waits for
// them; a tile whose max is off the prediction by more than 2^40 either way, or with a finite
// entry 2^40 below it, flags the chunk for the exact kernel (TC_ROW_SHIFT builds the per-row
// shifts of the formula above in a second pass: 3.51 vs 3.17 us per step).  Each row of D is
// then renormalised by its sum s_m
// (Ahat_{u+1} = D / c_m, off_m += R_u + ln c_m, fp64) with the LAGGED row scale c_m = the
// previous step's row sum s_m (any positive scale is exact), so the epilogue converts D_u to
// A_{u+1} in one pass, block by block, releasing each 32-column block of A to the MMA issuer
// at once: with D double-buffered in TMEM, MMA(u+1) overlaps the rest of epilogue(u).  The
// gate of DESIGN.md §4 is kept:
// chunks where a re-centred entry, a row weight or a normalised value is tiny enough that
// flush-to-zero could drop a significant term are flagged (cflag) and recomputed by the
// exact per-cell-max kernel (summary_exact_kernel, scan.cu).
//
// CTA = one (sequence, chunk), 288 threads, warp-specialised:
//   warps 0-3  epilogue: TMEM lane m = row m of D / A; normalise, scale by the next
//              tile's row weights, split hi/lo, tcgen05.st into the A columns;
//   warps 4-7  producers: warp p owns rows [32p, 32p+32) of every tile (K-block p): TMA
//              bulk load HBM -> staging, row max (31-shuffle transpose reduction), exps,
//              hi/lo split, K-major UMMA layout in the 4-stage B ring;
//   warp 8     TMEM allocation + the single MMA-issuing thread.
// TMEM: D[0] cols [0,128), D[1] [128,256), A_hi [256,384), A_lo [384,512) (512 allocated;
// 1 CTA per SM).
#include <atomic>
#include <cstdio>

#include "common.cuh"
#include "kernels.cuh"
#include "tc.cuh"

namespace tsb {

#ifdef TS_TC_TIMING
__device__ long long g_tc_t[64][8];
__device__ long long g_tc_p[64][6];  // producer warp 0: staged, pass 1 done, B stage free, pass 2 done
#define TCP(u, k)                                                                          \
  do {                                                                                     \
    if (blockIdx.x == 0 && pw == 0 && lane == 0 && (u) < 64) g_tc_p[(u)][(k)] = clock64(); \
  } while (0)
#define TCT(u, k)                                                      \
  do {                                                                 \
    if (blockIdx.x == 0 && (u) < 64) g_tc_t[(u)][(k)] = clock64();     \
  } while (0)
#else
#define TCT(u, k) \
  do {            \
  } while (0)
#define TCP(u, k) \
  do {            \
  } while (0)
#endif

namespace {
constexpr int kPW = 8;                      // producer warps (16 rows of every tile each)
constexpr int kPR = 128 / kPW;              // rows per producer warp
constexpr int kMmaWarp = 4 + kPW;           // the MMA-issuing warp (also allocates TMEM)
constexpr int kTcThreads = 32 * (kMmaWarp + 1);
constexpr int kBlk = 16384;                 // one B stage (32 rows x 128 cols fp32), bytes
constexpr int kOffBhi = 0;                  // [4][16 KB] tf32-hi  (K-major UMMA layout)
constexpr int kOffBlo = 4 * kBlk;           // [4][16 KB] tf32-lo
constexpr int kOffStg = 8 * kBlk;           // [kPW][16 KB / kPW x 4] raw staging (kPR rows each)
constexpr int kOffW = 12 * kBlk;            // float wbuf[2][132]: w[128], R (natural)
constexpr int kOffRs = kOffW + 2 * 132 * 4; // float rsc[4][32] row maxes of the current tile
constexpr int kOffRp = kOffRs + 4 * 32 * 4; // float Rp[4][kPW] per-warp maxes (and mins)
constexpr int kOffBar = kOffRp + 4 * kPW * 4;  // mbarriers
// bars: full[4] empty[4] stg[kPW] wready[2] dfull aready[4] (one per 32-column block of A)
constexpr int kBarFull = 0, kBarEmpty = 4, kBarStg = 8, kBarW = 8 + kPW, kBarD = kBarW + 2,
              kBarA = kBarD + 1;
constexpr int kOffMisc = kOffBar + (kBarA + 4) * 8;  // u32 tmem base, flags[2]
constexpr int kTcSmem = kOffMisc + 16;
#ifndef TC_AHEAD
#define TC_AHEAD 2
#endif
constexpr int kTcAhead = TC_AHEAD;
#ifndef TC_P2_UNROLL
#define TC_P2_UNROLL 2
#endif
constexpr int kP2Unroll = TC_P2_UNROLL;  // producer pass-2 unroll over 4-row groups  // L2 prefetch distance (tiles) of the producers' staging
constexpr float kTinyXtc = -40.f;  // log2 re-centred tile entry
constexpr float kTinyWtc = -30.f;  // log2 row weight
constexpr float kTinyPtc = 9.313225746154785e-10f;  // 2^-30 normalised value

__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// UMMA descriptors: B stage, K-major, no swizzle: core matrix 8 n-rows x 16 B (4 k's),
// k-groups at LBO = 128 B, n-groups (8 columns) at SBO = 1024 B (32 k's per stage).
__device__ __forceinline__ uint32_t bstage_off(int n, int kg) {
  return (uint32_t)((n >> 3) * 1024 + kg * 128 + (n & 7) * 16);
}
// mbarrier wait; with -DTS_TC_WATCHDOG a stuck wait reports (tag, u, block) and traps
__device__ __forceinline__ void tc_wait(uint64_t* bar, uint32_t parity, int tag, int u) {
#ifdef TS_TC_WATCHDOG
  const uint32_t b = smem_u32(bar);
  uint32_t done = 0;
  const long long t_start = clock64();
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
    if (!done && clock64() - t_start > 4000000000ll) {
      printf("TC watchdog: block %d thread %d tag %d u %d parity %u\n", blockIdx.x, threadIdx.x,
             tag, u, parity);
      __trap();
    }
  } while (!done);
#else
  (void)tag;
  (void)u;
  mbar_wait(bar, parity);
#endif
}
}  // namespace

// CF = compile-time C (128: every producer block is 32 full rows, all index arithmetic folds
// into immediates) or 0 for a runtime C in (64, 128).
template <int NP, int CF>
__global__ void __launch_bounds__(kTcThreads, 1) summary_tc_kernel(ScanArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int C = CF ? CF : (int)a.C, CC = C * C;
  const int64_t N = a.N, E = N - 1, P = a.P, Ppad = a.Ppad, L = a.L;
  const int64_t b = blockIdx.x / Ppad, k = blockIdx.x - (blockIdx.x / Ppad) * Ppad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t node = b * a.nodes + k;
  const int64_t len = seq_len(a.lengths, b, N);
  const int64_t Eb = len < 0 ? 0 : len - 1;
  const int64_t t0 = k * L;
  const int64_t t1 = (t0 + L < Eb) ? t0 + L : Eb;
  if ((k >= P) || (t0 >= Eb) || len < 0) {
    if (tid == 0) {
      a.ident[node] = 1;
      a.cflag[b * Ppad + k] = 0;
    }
    return;
  }
  const int n = (int)(t1 - t0);
  const float* potb = a.pot + b * E * (int64_t)CC;

  float* wbuf = reinterpret_cast<float*>(smem + kOffW);
  float* rsc = reinterpret_cast<float*>(smem + kOffRs);
  float* Rp = reinterpret_cast<float*>(smem + kOffRp);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBar);
  uint32_t* misc = reinterpret_cast<uint32_t*>(smem + kOffMisc);

  if (warp == kMmaWarp) tc::tmem_alloc<512>(&misc[0]);
  if (tid == 0) {
    for (int q = 0; q < 4; ++q) {
      mbar_init(&bars[kBarFull + q], 32 * (kPW / 4));
      mbar_init(&bars[kBarEmpty + q], 1);
    }
    for (int q = 0; q < kPW; ++q) mbar_init(&bars[kBarStg + q], 1);
    mbar_init(&bars[kBarW + 0], 32 * kPW);
    mbar_init(&bars[kBarW + 1], 32 * kPW);
    mbar_init(&bars[kBarD], 1);
    for (int c = 0; c < 4; ++c) mbar_init(&bars[kBarA + c], 128);
    misc[1] = 0u;  // bit 0: non-finite input, bit 1: precision gate (cflag)
    fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tm = misc[0];
  // TMEM: D double-buffered (step u writes D[u & 1]) so MMA(u+1) overlaps the epilogue of
  // step u; A (hi, lo) single-buffered, rewritten block by block once MMA(u) is complete
  const uint32_t tD0 = tm, tAh = tm + 256, tAl = tm + 384;

  if (warp >= 4 && warp < 4 + kPW) {
    // =============================== producers ===============================
    // warp pw owns rows [kPR pw, kPR pw + kPR) of every tile: half (or a quarter) of the
    // K-block p = pw / (kPW / 4) of the B operand
    const int pw = warp - 4, i0 = kPR * pw, p = pw / (kPW / 4), kg0 = (i0 - 32 * p) / 4;
    const int rows = CF == 128 ? kPR : ((C - i0) < 0 ? 0 : ((C - i0) > kPR ? kPR : (C - i0)));
    constexpr int kStg = kPR * 128 * 4;  // staging bytes per warp
    const float* stg = reinterpret_cast<const float*>(smem + kOffStg + pw * kStg);
    uint8_t* bhi = smem + kOffBhi + p * kBlk;
    uint8_t* blo = smem + kOffBlo + p * kBlk;
    const uint32_t blk_bytes = (uint32_t)(rows * C * 4);
    bool bad = false, tiny = false;
    if (lane == 0 && rows > 0) {
      bulk_load(smem + kOffStg + pw * kStg, potb + t0 * CC + (int64_t)i0 * C, blk_bytes,
                &bars[kBarStg + pw]);
#ifndef TC_NO_L2_AHEAD
      for (int v = 1; v < kTcAhead && v < n; ++v)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                         potb + (t0 + v) * CC + (int64_t)i0 * C),
                     "r"(blk_bytes)
                     : "memory");
#endif
    }
#ifndef TC_ROW_SHIFT
    // Single pass per tile with a PREDICTED shift: X_u = 2^((l - T_u) log2 e) with one scalar
    // T_u per tile = the previous tile's max (tile 0: its own max, one extra pass), so there are
    // no row weights (w = 1) and the epilogue never waits for this tile's pass; the tile's max
    // and finite min are gathered in the same pass and a prediction off by more than 2^40
    // either way (or a finite entry 2^40 below the shift) flags the chunk for the exact kernel.
    float Tp = 0.f;
    for (int u = 0; u < n; ++u) {
      if (rows > 0) tc_wait(&bars[kBarStg + pw], (uint32_t)(u & 1), 1, u);
      TCP(u, 0);
      if (u == 0) {  // tile 0: exact max
        float m = neg_inf();
#pragma unroll
        for (int rr = 0; rr < kPR; ++rr)
#pragma unroll
          for (int jb = 0; jb < 4; ++jb) {
            const int j = 32 * jb + lane;
            m = fmax_nan(m, (rr < rows && j < C) ? stg[rr * C + j] : neg_inf());
          }
        m = warp_max(m);
        if (lane == 0) Rp[kPW + pw] = m;
        named_bar(1, 32 * kPW);
        float R = Rp[kPW];
#pragma unroll
        for (int q = 1; q < kPW; ++q) R = fmaxf(R, Rp[kPW + q]);
        Tp = (R == neg_inf() || !(R == R) || R == pos_inf()) ? 0.f : R;
      }
      const float Tcur = Tp, tl = Tp * kLog2e;
      // B stage p free (the MMA of tile u-1 is done with it)?  Then publish this tile's shift.
      if (u > 0) tc_wait(&bars[kBarEmpty + p], (uint32_t)((u - 1) & 1), 2, u);
      TCP(u, 2);
      if (pw == 0 && lane == 0) wbuf[(u & 1) * 132 + 128] = Tp;
      mbar_arrive(&bars[kBarW + (u & 1)]);
      float mx = neg_inf(), mnf = pos_inf();
      float lvn[16];
#pragma unroll
      for (int x = 0; x < 16; ++x) {
        const int rr = x & 3, j = 32 * (x >> 2) + lane;
        lvn[x] = (rr < rows && j < C) ? stg[rr * C + j] : neg_inf();
      }
#pragma unroll kP2Unroll
      for (int kg = 0; kg < kPR / 4; ++kg) {
        float lv[16];
#pragma unroll
        for (int x = 0; x < 16; ++x) lv[x] = lvn[x];
        if (kg + 1 < kPR / 4) {
#pragma unroll
          for (int x = 0; x < 16; ++x) {
            const int rr = 4 * (kg + 1) + (x & 3), j = 32 * (x >> 2) + lane;
            lvn[x] = (rr < rows && j < C) ? stg[rr * C + j] : neg_inf();
          }
        }
#pragma unroll
        for (int x = 0; x < 16; ++x) {
          mx = fmax_nan(mx, lv[x]);
          mnf = fminf(mnf, lv[x] == neg_inf() ? pos_inf() : lv[x]);
        }
#pragma unroll
        for (int jb = 0; jb < 4; ++jb) {
          const int j = 32 * jb + lane;
          float e[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) e[q] = ex2(fmaf(lv[4 * jb + q], kLog2e, -tl));
          float4 h, l;
          tc::split_tf32(e[0], h.x, l.x);
          tc::split_tf32(e[1], h.y, l.y);
          tc::split_tf32(e[2], h.z, l.z);
          tc::split_tf32(e[3], h.w, l.w);
          const uint32_t off = bstage_off(j, kg0 + kg);
          *reinterpret_cast<float4*>(bhi + off) = h;
          if (NP == 3) *reinterpret_cast<float4*>(blo + off) = l;
        }
      }
      TCP(u, 4);
      tc::fence_async_smem();
      __syncwarp();
      TCP(u, 5);
      if (lane == 0 && rows > 0 && u + 1 < n)
        bulk_load(smem + kOffStg + pw * kStg, potb + (t0 + u + 1) * CC + (int64_t)i0 * C,
                  blk_bytes, &bars[kBarStg + pw]);
#ifndef TC_NO_L2_AHEAD
      if (lane == 0 && rows > 0 && u + kTcAhead < n)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                         potb + (t0 + u + kTcAhead) * CC + (int64_t)i0 * C),
                     "r"(blk_bytes)
                     : "memory");
#endif
      tc::fence_async_smem();
      if (pw == 0 && lane == 0) TCT(u, 7);
      TCP(u, 3);
      mbar_arrive(&bars[kBarFull + p]);
      // this tile's max (the next tile's shift) and gates
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mx = fmax_nan(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mnf = fminf(mnf, __shfl_xor_sync(0xffffffffu, mnf, o));
      }
      bad |= (mx != mx) | (mx == pos_inf());
      if (lane == 0) {
        Rp[(u & 1) * kPW + pw] = mx;
        Rp[2 * kPW + (u & 1) * kPW + pw] = mnf;
      }
      named_bar(1, 32 * kPW);
      float M = Rp[(u & 1) * kPW], Mn = Rp[2 * kPW + (u & 1) * kPW];
#pragma unroll
      for (int q = 1; q < kPW; ++q) {
        M = fmaxf(M, Rp[(u & 1) * kPW + q]);
        Mn = fminf(Mn, Rp[2 * kPW + (u & 1) * kPW + q]);
      }
      if (M != neg_inf() && M == M && M != pos_inf()) {
        const float dM = (M - Tp) * kLog2e;
        tiny |= (dM > 40.f) | (dM < -40.f);  // the prediction was off by more than 2^40
        Tp = M;
      }
      tiny |= (Mn != pos_inf()) & ((Mn - Tcur) * kLog2e < kTinyXtc);
    }
#else
    for (int u = 0; u < n; ++u) {
      // ---- tile u, rows i0.., columns j = 32 jb + lane; pass 1: row max and finite min ----
      if (rows > 0) tc_wait(&bars[kBarStg + pw], (uint32_t)(u & 1), 1, u);
      TCP(u, 0);
      float rm[kPR], rn[kPR];
#pragma unroll
      for (int rr = 0; rr < kPR; ++rr) {
        float m = neg_inf(), mn = pos_inf();
#pragma unroll
        for (int jb = 0; jb < 4; ++jb) {
          const int j = 32 * jb + lane;
          const float x = (rr < rows && j < C) ? stg[rr * C + j] : neg_inf();
          m = fmax_nan(m, x);  // NaN-propagating: NaN / +inf inputs surface in the row max
          mn = fminf(mn, x == neg_inf() ? pos_inf() : x);
        }
        bad |= (m != m) | (m == pos_inf());
        rm[rr] = m;
        rn[rr] = mn;
      }
      // transpose reductions: lane L ends with the max (min) of row i0 + (L mod kPR)
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
        if (o >= kPR) {  // more lanes than rows: plain combine
#pragma unroll
          for (int q = 0; q < kPR; ++q) {
            rm[q] = fmaxf(rm[q], __shfl_xor_sync(0xffffffffu, rm[q], o));
            rn[q] = fminf(rn[q], __shfl_xor_sync(0xffffffffu, rn[q], o));
          }
        } else {
#pragma unroll
          for (int q = 0; q < o; ++q) {
            const float send = up ? rm[q] : rm[q + o];
            const float keep = up ? rm[q + o] : rm[q];
            rm[q] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, o));
            const float sendn = up ? rn[q] : rn[q + o];
            const float keepn = up ? rn[q + o] : rn[q];
            rn[q] = fminf(keepn, __shfl_xor_sync(0xffffffffu, sendn, o));
          }
        }
      }
      const float rmy = rm[0];
      // gate: a finite re-centred entry (l - r_i) log2 e below -40
      tiny |= (rn[0] != pos_inf()) & ((rn[0] - rmy) * kLog2e < kTinyXtc);
      if (lane < kPR) rsc[i0 + lane] = rmy;
      const float wmax = warp_max(rmy);
      if (lane == 0) Rp[(u & 1) * kPW + pw] = wmax;
      named_bar(1, 32 * kPW);
      float R = Rp[(u & 1) * kPW + 0];
#pragma unroll
      for (int q = 1; q < kPW; ++q) R = fmaxf(R, Rp[(u & 1) * kPW + q]);
      const float Rz = (R == neg_inf()) ? 0.f : R;
      const float xw = (rmy - Rz) * kLog2e;
      const float wv = (rmy == neg_inf()) ? 0.f : ex2(xw);
      tiny |= (rmy != neg_inf()) & (xw < kTinyWtc);
      TCP(u, 1);
      // B stage p free (the MMA of tile u-1 is done with it)?
      if (u > 0) tc_wait(&bars[kBarEmpty + p], (uint32_t)((u - 1) & 1), 2, u);
      TCP(u, 2);
      if (lane < kPR) wbuf[(u & 1) * 132 + i0 + lane] = wv;
      if (pw == 0 && lane == 0) wbuf[(u & 1) * 132 + 128] = Rz;
      mbar_arrive(&bars[kBarW + (u & 1)]);
      // ---- pass 2 (on the chain: MMA(u) K-block p waits for it): X = 2^(l log2 e - r_i log2 e)
      // as one FFMA + ex2 (an all -inf row gets shift +inf: every X = 2^-inf = 0), hi/lo
      // split, K-major stores (4 k's per 16 B)
      float lvn[16];  // the next 4-row group's 16 values, loaded ahead (the stores into the
                      // B stage would otherwise pin every later load behind them: aliasing)
#pragma unroll
      for (int x = 0; x < 16; ++x) {
        const int rr = x & 3, j = 32 * (x >> 2) + lane;
        lvn[x] = (rr < rows && j < C) ? stg[rr * C + j] : neg_inf();
      }
#pragma unroll kP2Unroll
      for (int kg = 0; kg < kPR / 4; ++kg) {
        float lv[16];
#pragma unroll
        for (int x = 0; x < 16; ++x) lv[x] = lvn[x];
        if (kg + 1 < kPR / 4) {
#pragma unroll
          for (int x = 0; x < 16; ++x) {
            const int rr = 4 * (kg + 1) + (x & 3), j = 32 * (x >> 2) + lane;
            lvn[x] = (rr < rows && j < C) ? stg[rr * C + j] : neg_inf();
          }
        }
        float rl[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float r = rsc[i0 + 4 * kg + q];
          rl[q] = (r == neg_inf()) ? pos_inf() : r * kLog2e;
        }
#pragma unroll
        for (int jb = 0; jb < 4; ++jb) {
          const int j = 32 * jb + lane;
          float e[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
#ifdef TC_EXP_NOMUFU
            e[q] = fmaf(lv[4 * jb + q], kLog2e, -rl[q]);
#else
            e[q] = ex2(fmaf(lv[4 * jb + q], kLog2e, -rl[q]));
#endif
          }
          float4 h, l;
          tc::split_tf32(e[0], h.x, l.x);
          tc::split_tf32(e[1], h.y, l.y);
          tc::split_tf32(e[2], h.z, l.z);
          tc::split_tf32(e[3], h.w, l.w);
          const uint32_t off = bstage_off(j, kg0 + kg);
          *reinterpret_cast<float4*>(bhi + off) = h;
          if (NP == 3) *reinterpret_cast<float4*>(blo + off) = l;
        }
      }
      TCP(u, 4);
      // staging consumed: prefetch the next tile's block (generic reads before async write)
      tc::fence_async_smem();
      __syncwarp();
      TCP(u, 5);
      if (lane == 0 && rows > 0 && u + 1 < n)
        bulk_load(smem + kOffStg + pw * kStg, potb + (t0 + u + 1) * CC + (int64_t)i0 * C,
                  blk_bytes, &bars[kBarStg + pw]);
#ifndef TC_NO_L2_AHEAD
      // the staging block is single-buffered (smem is full), so its refill latency is on the
      // per-step chain: warm L2 with the block kTcAhead tiles ahead
      if (lane == 0 && rows > 0 && u + kTcAhead < n)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                         potb + (t0 + u + kTcAhead) * CC + (int64_t)i0 * C),
                     "r"(blk_bytes)
                     : "memory");
#endif
      tc::fence_async_smem();
      if (pw == 0 && lane == 0) TCT(u, 7);
      TCP(u, 3);
      mbar_arrive(&bars[kBarFull + p]);
    }
#endif  // !TC_ROW_SHIFT
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&misc[1], 1u);
    if (__any_sync(0xffffffffu, tiny) && lane == 0) atomicOr(&misc[1], 2u);
  } else if (warp == kMmaWarp) {
    // =============================== MMA issuer ===============================
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_tf32(128, 128, 0, 0);
      for (int u = 0; u < n; ++u) {
        TCT(u, 0);
        const uint32_t tD = tD0 + 128u * (uint32_t)(u & 1);
        for (int p = 0; p < 4; ++p) {
          // K-block p needs A_u columns [32p, 32p+32) (epilogue of step u-1, block p) and
          // the B stage p of tile u (producer warp p)
          tc_wait(&bars[kBarA + p], (uint32_t)(u & 1), 3, u);
          tc_wait(&bars[kBarFull + p], (uint32_t)(u & 1), 10 + p, u);
          tc::fence_after();
          if (p == 0) TCT(u, 1);
          const uint8_t* bh = smem + kOffBhi + p * kBlk;
          const uint8_t* bl = smem + kOffBlo + p * kBlk;
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const uint32_t kc = (uint32_t)(32 * p + 8 * s);
            const uint64_t dh = tc::smem_desc(bh + s * 256, 128, 1024);
            tc::mma_tf32_ts(tD, tAh + kc, dh, idesc, (p | s) != 0);
            if (NP == 3) {
              const uint64_t dl = tc::smem_desc(bl + s * 256, 128, 1024);
              tc::mma_tf32_ts(tD, tAh + kc, dl, idesc, 1u);
              tc::mma_tf32_ts(tD, tAl + kc, dh, idesc, 1u);
            }
          }
          tc::commit(&bars[kBarEmpty + p]);
        }
        tc::commit(&bars[kBarD]);
        TCT(u, 2);
      }
    }
    __syncwarp();
  } else {
    // =============================== epilogue ===============================
    const int m = tid;  // row m <-> TMEM lane m
    const uint32_t lb = (uint32_t)(32 * warp) << 16;
    double off = 0.0;
    bool dead = (m >= C);
    bool tinyp = false;
    // A_0 = I (the identity start; with the TC_ROW_SHIFT variant diag(w^(0)), tile 0's row
    // weights)
#ifdef TC_ROW_SHIFT
    tc_wait(&bars[kBarW + 0], 0u, 4, 0);
#endif
    {
      float wh, wl;
#ifndef TC_ROW_SHIFT
      tc::split_tf32(dead ? 0.f : 1.f, wh, wl);
#else
      tc::split_tf32(dead ? 0.f : wbuf[m], wh, wl);
#endif
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t vh[32], vl[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const bool d = (32 * c + q == m);
          vh[q] = __float_as_uint(d ? wh : 0.f);
          vl[q] = __float_as_uint(d ? wl : 0.f);
        }
        tc::st32(tAh + lb + 32 * c, vh);
        if (NP == 3) tc::st32(tAl + lb + 32 * c, vl);
      }
      tc::wait_st();
      tc::fence_before();
#pragma unroll
      for (int c = 0; c < 4; ++c) mbar_arrive(&bars[kBarA + c]);
    }
    // Lagged normaliser: A_{u+1} = D_u * (1 / s_{u-1}) * w^(u+1) with s_{u-1} the previous row
    // sum (s_{-1} = 1), so each 32-column block of A_{u+1} is written (and released to the
    // MMA issuer) as soon as it is converted — MMA(u+1) K-block c starts while blocks c+1..
    // are still in flight.  Any positive row scale is exact (off_m absorbs its log); the row
    // sum s_u is accumulated in the same pass and the precision gate is evaluated against
    // it afterwards (min normalised entry < 2^-30 of s_u, the same test as before).
    float inv = dead ? 0.f : 1.f;
    float Rprev_ls = 0.f;  // log2 of the scale applied at this step
    float* S = a.mat + node * (int64_t)CC;
    for (int u = 0; u < n; ++u) {
      const uint32_t tD = tD0 + 128u * (uint32_t)(u & 1);
      tc_wait(&bars[kBarD], (uint32_t)(u & 1), 5, u);
      tc::fence_after();
      if (tid == 0) TCT(u, 3);
#ifndef TC_ROW_SHIFT
      tc_wait(&bars[kBarW + (u & 1)], (uint32_t)((u >> 1) & 1), 6, u);  // this tile's shift
#endif
      const float Ru = wbuf[(u & 1) * 132 + 128];
      if (u + 1 < n) {
        const int nb = (u + 1) & 1;
        if (tid == 0) TCT(u, 4);
#ifdef TC_ROW_SHIFT
        tc_wait(&bars[kBarW + nb], (uint32_t)(((u + 1) >> 1) & 1), 6, u);
#endif
        if (tid == 0) TCT(u, 5);
        const float* w = wbuf + nb * 132;
        (void)w;
        float s4[4] = {0.f, 0.f, 0.f, 0.f};
        float pmin = pos_inf();
#if !defined(TC_EPI_NOPIPE) && !defined(TC_ROW_SHIFT)
        // blocks double-buffered in registers: block c+1's TMEM load is in flight while block
        // c is converted (hi in place of D, lo beside it)
        uint32_t va[32], vb[32], vl[32];
        tc::ld32_async(tD + lb, va);
        tc::wait_ld32(va);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t(&v)[32] = (c & 1) ? vb : va;
          uint32_t(&vn)[32] = (c & 1) ? va : vb;
          if (c + 1 < 4) tc::ld32_async(tD + lb + 32 * (c + 1), vn);
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const float x = __uint_as_float(v[q]);
            s4[q & 3] += x;
            const float p = x * inv;
            if (p > 0.f) pmin = fminf(pmin, p);
            float h, l;
            tc::split_tf32(p, h, l);
            v[q] = __float_as_uint(h);
            vl[q] = __float_as_uint(l);
          }
          tc::st32(tAh + lb + 32 * c, v);
          if (NP == 3) tc::st32(tAl + lb + 32 * c, vl);
          tc::wait_st();
          tc::fence_before();
          mbar_arrive(&bars[kBarA + c]);
          if (c + 1 < 4) tc::wait_ld32(vn);
        }
#else
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32], vh[32], vl[32];
          tc::ld32(tD + lb + 32 * c, v);
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const float x = __uint_as_float(v[q]);
            s4[q & 3] += x;
            const float p = x * inv;
            if (p > 0.f) pmin = fminf(pmin, p);
            float h, l;
#ifndef TC_ROW_SHIFT
            tc::split_tf32(p, h, l);
#else
            tc::split_tf32(p * w[32 * c + q], h, l);
#endif
            vh[q] = __float_as_uint(h);
            vl[q] = __float_as_uint(l);
          }
          tc::st32(tAh + lb + 32 * c, vh);
          if (NP == 3) tc::st32(tAl + lb + 32 * c, vl);
          tc::wait_st();
          tc::fence_before();
          mbar_arrive(&bars[kBarA + c]);
        }
#endif
        const float s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
        if (!dead) off += (double)Ru + kLn2 * (double)Rprev_ls;
        dead |= !(s > 0.f);
        // gate: the smallest normalised entry relative to this step's row sum
        tinyp |= !dead && (pmin < pos_inf()) && (pmin * (1.f / (s * inv)) < kTinyPtc);
        inv = dead ? 0.f : 1.f / s;
        Rprev_ls = dead ? 0.f : lg2(s);
        if (tid == 0) TCT(u, 6);
      } else {
        // final: leaf LogMat row m = log2 of the row normalised by its own sum (+ fp64 natural
        // offset).  tcgen05.ld is .sync.aligned: every lane of the warp loads, rows >= C only
        // skip the stores.
        float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32];
          tc::ld32(tD + lb + 32 * c, v);
#pragma unroll
          for (int q = 0; q < 32; ++q) s4[q & 3] += __uint_as_float(v[q]);
        }
        const float s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
        dead |= !(s > 0.f);
        const float ls = dead ? 0.f : lg2(s);
        // true S_n = off + R_{n-1} + ln D_{n-1}: normalised by its own row sum, entries are
        // log2(D / s) and the offset takes R_{n-1} + ln s (the lagged scales are already in off)
        if (!dead) off += (double)Ru + kLn2 * (double)ls;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32];
          tc::ld32(tD + lb + 32 * c, v);
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const int j = 32 * c + q;
            const float x = __uint_as_float(v[q]);
            if (m < C && j < C) S[m * C + j] = (dead || !(x > 0.f)) ? neg_inf() : lg2(x) - ls;
          }
        }
        if (m < C) a.off[node * (int64_t)C + m] = dead ? 0.0 : off;
      }
    }
    if (__any_sync(0xffffffffu, tinyp) && lane == 0) atomicOr(&misc[1], 2u);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == kMmaWarp) tc::tmem_dealloc<512>(tm);
  if (tid == 0) {
    const uint32_t f = misc[1];
    a.ident[node] = 0;
    a.cflag[b * Ppad + k] = (f & 2u) ? 1u : 0u;
    if ((f & 1u) && a.wflags) atomicOr(&a.wflags[b], (unsigned)WF_NONFINITE);
  }
}

namespace {
std::atomic<int> g_tc_summary{3};  // 0 = SIMT summaries, 1 = 1xTF32, 3 = 3xTF32 (default)
template <int NP, int CF>
cudaError_t launch_np(const ScanArgs& a, cudaStream_t st) {
  static std::atomic<uint64_t> attr{0};  // per instantiation, one bit per device
  cudaError_t e = smem_optin_once(summary_tc_kernel<NP, CF>, attr, kTcSmem);
  if (e != cudaSuccess) return e;
  summary_tc_kernel<NP, CF><<<(unsigned)(a.B * a.Ppad), kTcThreads, kTcSmem, st>>>(a);
  return cudaGetLastError();
}
}  // namespace

#ifndef TC_MIN_C
#define TC_MIN_C 64
#endif
constexpr int kTcMinC = TC_MIN_C;  // tensor-core summaries for kTcMinC < C <= 128

bool summary_tc_ok(const ScanArgs& a) {
  return g_tc_summary.load() != 0 && a.C > kTcMinC && a.C <= 128 && (a.C % 2) == 0 &&
         (reinterpret_cast<uintptr_t>(a.pot) & 15) == 0;
}

cudaError_t launch_summary_tc(const ScanArgs& a, cudaStream_t st) {
  if (a.C == 128)
    return g_tc_summary.load() == 1 ? launch_np<1, 128>(a, st) : launch_np<3, 128>(a, st);
  return g_tc_summary.load() == 1 ? launch_np<1, 0>(a, st) : launch_np<3, 0>(a, st);
}

void set_tc_summary(int mode) { g_tc_summary.store(mode == 1 || mode == 3 ? mode : 0); }
int get_tc_summary() { return g_tc_summary.load(); }

}  // namespace tsb
