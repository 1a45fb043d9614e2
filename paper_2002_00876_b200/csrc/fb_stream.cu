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
inline int nthreads_for(int64_t C) { return (int)(((C + 31) / 32) * 32); }

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

// ====================================================================================
// Forward sweep
// ====================================================================================
template <bool VEC4>
__global__ void __launch_bounds__(128) fwd_sweep_kernel(SweepArgs a, int S) {
  extern __shared__ __align__(16) float sm[];
  const int C = (int)a.C, CC = C * C;
  const int64_t N = a.N, E = N - 1, P = a.P, L = a.L;
  const int64_t b = blockIdx.x / P, k = blockIdx.x - (blockIdx.x / P) * P;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int NT = blockDim.x, NW = NT >> 5;
  const int TF = fwd_tile_floats(C);
  float* ring = sm;
  float* a_s = ring + (size_t)S * TF;  // [2][NT]
  float* ah_s = a_s + 2 * NT;          // [2][NT]
  float* red_mu = ah_s + 2 * NT;       // [2][NW]
  float* red_T = red_mu + 2 * NW;      // [NW]
  float* red_x = red_T + NW;           // [2*NW] scratch

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
  const bool act = tid < C;
  const int64_t bk = b * P + k;
  const float* potb = a.pot + b * E * (int64_t)CC;

  // start vector (chunk 0: log-one; otherwise alpha_in from the scan tree)
  float ah = act ? (a.alpha_in ? a.alpha_in[bk * C + tid] : 0.f) : neg_inf();
  double O = a.alpha_in_off ? a.alpha_in_off[bk] : 0.0;
  float mu = block_max(ah, red_x, NW);
  float m = (mu == neg_inf()) ? 0.f : mu;
  if (a.alpha_hat && act) a.alpha_hat[(b * N + t0) * C + tid] = ah;

  // prologue: stage the first S-1 tiles
  for (int u = 0; u < S - 1; ++u) {
    if (u < nsteps)
      stage_tile(ring + (size_t)(u % S) * TF, potb + (t0 + u) * (int64_t)CC, C, C, VEC4, tid, NT);
    cp_async_commit();
  }
  a_s[tid] = act ? ex2(ah - m) : 0.f;
  ah_s[tid] = ah;
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
                   NT);
      cp_async_commit();
    }
    const float* tile = ring + (size_t)(u % S) * TF;
    const float* av = a_s + buf * NT;
    // ---- phase A: column max and exp-shifted dot product --------------------------
    float M = neg_inf(), s = 0.f;
    if (act) {
      for (int i = 0; i < C; ++i) M = fmaxf(M, tile[i * C + tid]);
      if (M != neg_inf()) {
        float s0 = 0.f, s1 = 0.f;
        int i = 0;
        for (; i + 2 <= C; i += 2) {
          s0 = fmaf(av[i], ex2((tile[i * C + tid] - M) * kLog2e), s0);
          s1 = fmaf(av[i + 1], ex2((tile[(i + 1) * C + tid] - M) * kLog2e), s1);
        }
        if (i < C) s0 = fmaf(av[i], ex2((tile[i * C + tid] - M) * kLog2e), s0);
        s = s0 + s1;
      }
    }
    {
      float wm = warp_max(M);
      if (lane == 0) red_T[w] = wm;
    }
    __syncthreads();
    float T = red_T[0];
    for (int q = 1; q < NW; ++q) T = fmaxf(T, red_T[q]);
    const float Tz = (T == neg_inf()) ? 0.f : T;
    // ---- phase B: finalise ah_{t+1}[j] -------------------------------------------------
    float nh = neg_inf();
    if (act && M != neg_inf()) {
      nh = (M - Tz) * kLog2e + lg2(s);
      if (!(s >= kGate)) {  // exact per-cell-max path (also reached by NaN)
        const float* ahv = ah_s + buf * NT;
        float q = neg_inf();
        for (int i = 0; i < C; ++i) q = fmaxf(q, ahv[i] + (tile[i * C + tid] - Tz) * kLog2e);
        if (q == neg_inf()) {
          nh = neg_inf();
        } else {
          float ss = 0.f;
          for (int i = 0; i < C; ++i) ss += ex2(ahv[i] + (tile[i * C + tid] - Tz) * kLog2e - q);
          nh = q + lg2(ss) - m;
        }
        if (s != s) nh = qnan();
      }
    }
    if (nh != nh || M == pos_inf()) bad = 1u;
    if (a.alpha_hat && act && t + 1 < t1) a.alpha_hat[(b * N + t + 1) * C + tid] = nh;
    if (tid == 0) {
      if (a.mlag) a.mlag[b * N + t] = m;
      if (a.tmax) a.tmax[b * E + t] = Tz;
    }
    O += kLn2 * (double)m + (double)Tz;
    const float m_next = (mu == neg_inf()) ? 0.f : (log2C + mu - m);
    ah_s[(buf ^ 1) * NT + tid] = nh;
    a_s[(buf ^ 1) * NT + tid] = act ? ex2(nh - m_next) : 0.f;
    {
      float wm = warp_max(nh);
      if (lane == 0) red_mu[(buf ^ 1) * NW + w] = wm;
    }
    cp_async_wait_dyn(S - 2);
    __syncthreads();
    float mx = red_mu[(buf ^ 1) * NW];
    for (int q = 1; q < NW; ++q) mx = fmaxf(mx, red_mu[(buf ^ 1) * NW + q]);
    mu = mx;
    m = m_next;
    ah = nh;
    buf ^= 1;
  }
  cp_async_wait<0>();
  if (a.alpha_end && act) a.alpha_end[bk * C + tid] = ah;
  if (a.alpha_end_off && tid == 0) a.alpha_end_off[bk] = O;
  // NONFINITE: any NaN/+inf propagates to a NaN column (0 * NaN = NaN in the dot product)
  const unsigned anybad = __syncthreads_or(bad);
  if (anybad && tid == 0 && a.wflags) atomicOr(&a.wflags[b], (unsigned)WF_NONFINITE);
  if (a.final_in_fwd && last) {
    const float Lz = block_lse2(act ? ah : neg_inf(), red_x, red_x + NW, NW);
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
template <bool VEC4>
__global__ void __launch_bounds__(128) bwd_sweep_kernel(SweepArgs a, int S) {
  extern __shared__ __align__(16) float sm[];
  const int C = (int)a.C, CC = C * C;
  const int64_t N = a.N, E = N - 1, P = a.P, L = a.L;
  const int64_t b = blockIdx.x / P, k = blockIdx.x - (blockIdx.x / P) * P;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int NT = blockDim.x, NW = NT >> 5;
  const int SB = bwd_stride(C, VEC4);
  const int TF = bwd_tile_floats(C, VEC4);
  float* ring = sm;
  float* b_s = ring + (size_t)S * TF;  // [2][NT] b values
  float* bh_s = b_s + 2 * NT;          // [2][NT] bh values
  float* red_mu = bh_s + 2 * NT;       // [2][NW]
  float* red_lm = red_mu + 2 * NW;     // [2][NW]
  float* red_ls = red_lm + 2 * NW;     // [2][NW]
  float* red_x = red_ls + 2 * NW;      // [2*NW]

  const int64_t len = seq_len(a.lengths, b, N);
  float* mgb = a.marg + b * E * (int64_t)CC;
  if (len < 0) {  // BADLEN: chunk 0 zeroes everything
    if (k == 0) {
      for (int64_t q = tid; q < E * CC; q += NT) mgb[q] = 0.f;
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
  const bool act = tid < C;
  const int64_t bk = b * P + k;
  const float* potb = a.pot + b * E * (int64_t)CC;
  const uint32_t wf = a.wflags ? a.wflags[b] : 0u;

  // end-of-chunk vectors: beta_out (tree) or log-one; alpha in the chunk's own frame
  float bh = act ? (a.beta_out ? a.beta_out[bk * C + tid] : 0.f) : neg_inf();
  const float ahe = act ? a.alpha_end[bk * C + tid] : neg_inf();
  float Lnext = block_lse2(act ? ahe + bh : neg_inf(), red_x, red_x + NW, NW);
  float mu = block_max(bh, red_x, NW);
  float m = (mu == neg_inf()) ? 0.f : mu;

  const bool dead = (wf & WF_NONFINITE) || !(Lnext > neg_inf());  // also NaN (remote segment)
  if (last && !a.no_final) {  // zero the padded tail, publish logZ and flags
    for (int64_t q = Eb * CC + tid; q < E * CC; q += NT) mgb[q] = 0.f;
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
    for (int64_t q = Eb * CC + tid; q < E * CC; q += NT) mgb[q] = 0.f;
  if (dead) {
    for (int64_t q = t0 * CC + tid; q < t1 * CC; q += NT) mgb[q] = 0.f;
    return;
  }

  for (int u = 0; u < S - 1; ++u) {
    if (u < nsteps)
      stage_tile(ring + (size_t)(u % S) * TF, potb + (t1 - 1 - u) * (int64_t)CC, C, SB, VEC4,
                 tid, NT);
    cp_async_commit();
  }
  b_s[tid] = act ? ex2(bh - m) : 0.f;
  bh_s[tid] = bh;
  cp_async_wait_dyn(S - 2);
  __syncthreads();

  const float log2C = lg2((float)C);
  int buf = 0;
  for (int64_t u = 0; u < nsteps; ++u) {
    const int64_t t = t1 - 1 - u;
    {
      const int64_t uu = u + S - 1;
      if (uu < nsteps)
        stage_tile(ring + (size_t)(uu % S) * TF, potb + (t1 - 1 - uu) * (int64_t)CC, C, SB, VEC4,
                   tid, NT);
      cp_async_commit();
    }
    const float* tile = ring + (size_t)(u % S) * TF;
    const float* bv = b_s + buf * NT;
    const float* bhv = bh_s + buf * NT;
    const float Tt = a.tmax[b * E + t];
    const float mt = a.mlag[b * N + t];
    float aht = act ? a.alpha_hat[(b * N + t) * C + tid] : neg_inf();
    float nb = neg_inf();
    if (act) {
      const float* row = tile + tid * SB;
      float* mrow = mgb + ((int64_t)t * C + tid) * C;
      const float cst = aht - mt - Lnext;
      float R = neg_inf();
      float s = 0.f;
      if (VEC4) {
        for (int j = 0; j < C; j += 4) {
          float4 v = *reinterpret_cast<const float4*>(row + j);
          R = fmaxf(R, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
        }
        for (int j = 0; j < C; j += 4) {
          const float4 v = *reinterpret_cast<const float4*>(row + j);
          const float4 bb = *reinterpret_cast<const float4*>(bv + j);
          const float4 hh = *reinterpret_cast<const float4*>(bhv + j);
          if (R != neg_inf()) {
            s = fmaf(ex2((v.x - R) * kLog2e), bb.x, s);
            s = fmaf(ex2((v.y - R) * kLog2e), bb.y, s);
            s = fmaf(ex2((v.z - R) * kLog2e), bb.z, s);
            s = fmaf(ex2((v.w - R) * kLog2e), bb.w, s);
          }
          float4 mu4;
          mu4.x = ex2(cst + hh.x + (v.x - Tt) * kLog2e);
          mu4.y = ex2(cst + hh.y + (v.y - Tt) * kLog2e);
          mu4.z = ex2(cst + hh.z + (v.z - Tt) * kLog2e);
          mu4.w = ex2(cst + hh.w + (v.w - Tt) * kLog2e);
          *reinterpret_cast<float4*>(mrow + j) = mu4;
        }
      } else {
        for (int j = 0; j < C; ++j) R = fmaxf(R, row[j]);
        for (int j = 0; j < C; ++j) {
          const float v = row[j];
          if (R != neg_inf()) s = fmaf(ex2((v - R) * kLog2e), bv[j], s);
          mrow[j] = ex2(cst + bhv[j] + (v - Tt) * kLog2e);
        }
      }
      if (R != neg_inf()) {
        nb = (R - Tt) * kLog2e + lg2(s);
        if (!(s >= kGate)) {  // exact per-cell-max path
          float q = neg_inf();
          for (int j = 0; j < C; ++j) q = fmaxf(q, (row[j] - Tt) * kLog2e + bhv[j]);
          if (q == neg_inf()) {
            nb = neg_inf();
          } else {
            float ss = 0.f;
            for (int j = 0; j < C; ++j) ss += ex2((row[j] - Tt) * kLog2e + bhv[j] - q);
            nb = q + lg2(ss) - m;
          }
        }
      }
    }
    const float m_next = (mu == neg_inf()) ? 0.f : (log2C + mu - m);
    b_s[(buf ^ 1) * NT + tid] = act ? ex2(nb - m_next) : 0.f;
    bh_s[(buf ^ 1) * NT + tid] = nb;
    {
      float wm = warp_max(nb);
      const float v = act ? aht + nb : neg_inf();
      float lm = warp_max(v);
      float le = (lm == neg_inf()) ? 0.f : ex2(v - lm);
      float ls = warp_sum(le);
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
      for (int q = 1; q < NW; ++q) {
        mx = fmaxf(mx, rm[q]);
        LM = fmaxf(LM, lmv[q]);
      }
      float LS = 0.f;
      if (LM != neg_inf())
        for (int q = 0; q < NW; ++q) LS += (lmv[q] == neg_inf()) ? 0.f : lsv[q] * ex2(lmv[q] - LM);
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
std::atomic<uint64_t> g_attr_fwd{0}, g_attr_bwd{0};

template <typename K>
cudaError_t set_smem_once(K kern, std::atomic<uint64_t>& mask, int bit) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t m = 1ull << ((dev & 15) * 4 + bit);
  if (mask.load() & m) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  if (e == cudaSuccess) mask.fetch_or(m);
  return e;
}
}  // namespace

size_t fwd_smem_bytes(int64_t C, int stages) {
  const int NT = nthreads_for(C), NW = NT / 32;
  return ((size_t)stages * fwd_tile_floats((int)C) + 4 * NT + 5 * NW) * sizeof(float);
}
size_t bwd_smem_bytes(int64_t C, int stages) {
  const bool vec4 = (C % 4) == 0;
  const int NT = nthreads_for(C), NW = NT / 32;
  return ((size_t)stages * bwd_tile_floats((int)C, vec4) + 4 * NT + 8 * NW) * sizeof(float);
}

cudaError_t launch_fwd(const SweepArgs& a, cudaStream_t st) {
  const int C = (int)a.C;
  const bool vec4 = (C % 4) == 0 && (reinterpret_cast<uintptr_t>(a.pot) & 15) == 0;
  const int S = fwd_stages(C);
  const size_t smem = fwd_smem_bytes(C, S);
  const dim3 grid((unsigned)(a.B * a.P)), block(nthreads_for(C));
  cudaError_t e;
  if (vec4) {
    if ((e = set_smem_once(fwd_sweep_kernel<true>, g_attr_fwd, 0)) != cudaSuccess) return e;
    fwd_sweep_kernel<true><<<grid, block, smem, st>>>(a, S);
  } else {
    if ((e = set_smem_once(fwd_sweep_kernel<false>, g_attr_fwd, 1)) != cudaSuccess) return e;
    fwd_sweep_kernel<false><<<grid, block, smem, st>>>(a, S);
  }
  return cudaGetLastError();
}

cudaError_t launch_bwd(const SweepArgs& a, cudaStream_t st) {
  const int C = (int)a.C;
  const bool vec4 = (C % 4) == 0 && (reinterpret_cast<uintptr_t>(a.pot) & 15) == 0 &&
                    (reinterpret_cast<uintptr_t>(a.marg) & 15) == 0;
  const int S = bwd_stages(C, vec4);
  const size_t smem = bwd_smem_bytes(C, S);
  const dim3 grid((unsigned)(a.B * a.P)), block(nthreads_for(C));
  cudaError_t e;
  if (vec4) {
    if ((e = set_smem_once(bwd_sweep_kernel<true>, g_attr_bwd, 0)) != cudaSuccess) return e;
    bwd_sweep_kernel<true><<<grid, block, smem, st>>>(a, S);
  } else {
    if ((e = set_smem_once(bwd_sweep_kernel<false>, g_attr_bwd, 1)) != cudaSuccess) return e;
    bwd_sweep_kernel<false><<<grid, block, smem, st>>>(a, S);
  }
  return cudaGetLastError();
}

}  // namespace tsb
