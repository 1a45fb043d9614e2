// fb_wide.cu — logZ and marginals for wide label sets, 128 < C <= 256 (SURVEY §8(a) rows
// a5/a6/a9 for the shapes the SMEM-resident kernels cannot hold: a C x C tile is up to 256 KB).
//
// Pass 1, grid (B, 2): CTA (b, 0) runs the forward recursion, CTA (b, 1) the backward one,
// concurrently, each with 1024 threads and the exact per-cell max of §6(c):
//   alpha_{t+1}[j] = LSE_i alpha_t[i] + l_t[i][j]        beta_t[i] = LSE_j l_t[i][j] + beta_{t+1}[j]
// evaluated in log2 units as an online (max, sum) per output cell over batches of 8 terms
// (one ex2 per term plus one per batch), so no range gate is needed.  Node vectors are
// stored normalised (max 0) with fp64 offsets.  Forward: thread (j, q) reduces column j over
// rows i = q (mod 4) (loads coalesced along j), four partials combined through SMEM.
// Backward: warp w reduces rows i = w (mod 32), lanes along j, (max, sum) combined by
// shuffles.  The forward CTA also writes logZ = ln2 (O_E + log2 Σ_j 2^alpha_hat_E[j]) and the
// flags (NONFINITE from its scan of every used edge).
// Pass 2, one CTA per edge over the whole machine (marginals only):
//   mu_t[i][j] = 2^(alpha_hat_t[i] + l_t[i][j] log2 e + beta_hat_{t+1}[j] + O^a_t + O^b_{t+1} - A log2 e)
// (P:181-183), 0 beyond the sequence and for flagged sequences.
// Pass 1 streams the tiles through a bulk-copy SMEM ring when C % 4 == 0
// (fb_wide_ring_kernel, below) and with coalesced register loads otherwise.
// Traffic: 2 reads of l in pass 1 (one per direction) + 1 read and 1 write in pass 2.
// Measured at B64 N1024 C256: pass 1 8.5 ms (2 reads, 62 % of HBM with 128 of 148 SMs
// streaming; 9.6 ms in profiles/r1e_wide_launches.csv, before the producer warp), pass 2
// 5.2 ms (1 read + 1 write at ~6.6 TB/s).
#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

namespace {
constexpr int kWideThreads = 1024;
constexpr int kWideMaxC = 256;
constexpr int kBatch = 8;

// (m, s) <- (m, s) (+) batch of NB terms x[] (log2 domain), online: NB + 1 ex2
template <int NB = kBatch>
__device__ __forceinline__ void online_add(float& m, float& s, const float* x) {
  float bm = x[0];
#pragma unroll
  for (int k = 1; k < NB; ++k) bm = fmaxf(bm, x[k]);
  if (bm == neg_inf()) return;
  const float mn = fmaxf(m, bm);
  float acc = (m == neg_inf()) ? 0.f : s * ex2(m - mn);
#pragma unroll
  for (int k = 0; k < NB; ++k) acc += ex2(x[k] - mn);
  m = mn;
  s = acc;
}

__device__ __forceinline__ void lse_merge(float& m, float& s, float m2, float s2) {
  const float M = fmaxf(m, m2);
  if (M == neg_inf()) return;
  s = ((m == neg_inf()) ? 0.f : s * ex2(m - M)) + ((m2 == neg_inf()) ? 0.f : s2 * ex2(m2 - M));
  m = M;
}
}  // namespace

__global__ void __launch_bounds__(kWideThreads, 1) fb_wide_sweep_kernel(SemiArgs a) {
  __shared__ float vec[2][kWideMaxC];
  __shared__ float pm[4][kWideMaxC], ps[4][kWideMaxC];
  __shared__ float red[32];
  __shared__ unsigned sbad;
  const int C = (int)a.C;
  const int64_t N = a.N, E = N - 1, CC = (int64_t)C * C;
  const int64_t b = blockIdx.x;
  const bool fwd = blockIdx.y == 0;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t len = seq_len(a.lengths, b, N);
  if (len < 0) {
    if (fwd && tid == 0) {
      a.logz[b] = qnan();
      a.zbuf[b] = (double)qnan();
      if (a.flags) a.flags[b] = TS_F_BADLEN;
    }
    return;
  }
  const int64_t Eb = len - 1;
  float* vh = (fwd ? a.ah : a.bh) + b * N * C;
  double* vo = (fwd ? a.ao : a.bo) + b * N;
  const int64_t n0 = fwd ? 0 : Eb;
  if (tid < C) {
    vec[0][tid] = 0.f;
    vh[n0 * C + tid] = 0.f;
  }
  if (tid == 0) {
    sbad = 0u;
    vo[n0] = 0.0;
  }
  __syncthreads();
  bool bad = false;
  double off = 0.0;  // log2 units, identical in every thread
  bool dead = false;
  for (int64_t s = 1; s <= Eb; ++s) {
    const int64_t p = fwd ? s : Eb - s;      // node computed at this step
    const int64_t t = fwd ? p - 1 : p;       // its edge
    const float* tile = a.pot + (b * E + t) * CC;
    const float* v = vec[(s - 1) & 1];
    float* vn = vec[s & 1];
    float val = neg_inf();
    if (fwd) {
      const int j = tid & (kWideMaxC - 1), q = tid >> 8;
      float m = neg_inf(), sum = 0.f;
      if (j < C) {
        for (int i0 = q; i0 < C; i0 += 4 * kBatch) {
          float x[kBatch];
#pragma unroll
          for (int k = 0; k < kBatch; ++k) {
            const int i = i0 + 4 * k;
            const float lv = (i < C) ? tile[(int64_t)i * C + j] : neg_inf();
            bad |= (lv != lv) | (lv == pos_inf());
            x[k] = (i < C) ? fmaf(lv, kLog2e, v[i]) : neg_inf();
          }
          online_add<kBatch>(m, sum, x);
        }
      }
      pm[q][j] = m;
      ps[q][j] = sum;
      __syncthreads();
      if (tid < C) {
        float M = pm[0][tid], S = ps[0][tid];
#pragma unroll
        for (int k = 1; k < 4; ++k) lse_merge(M, S, pm[k][tid], ps[k][tid]);
        val = (M == neg_inf()) ? neg_inf() : M + lg2(S);
      }
    } else {
      constexpr int KJ = kWideMaxC / 32;  // columns per lane
      for (int i0 = w; i0 < C; i0 += 64) {  // rows i0 and i0 + 32: 16 loads in flight
        float x[2][KJ];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = i0 + 32 * h;
#pragma unroll
          for (int k = 0; k < KJ; ++k) {
            const int j = lane + 32 * k;
            const float lv = (i < C && j < C) ? tile[(int64_t)i * C + j] : neg_inf();
            x[h][k] = (i < C && j < C) ? fmaf(lv, kLog2e, v[j]) : neg_inf();
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float m = x[h][0];
#pragma unroll
          for (int k = 1; k < KJ; ++k) m = fmaxf(m, x[h][k]);
          m = warp_max(m);
          float sum = 0.f;
          if (m != neg_inf())
#pragma unroll
            for (int k = 0; k < KJ; ++k) sum += ex2(x[h][k] - m);
          sum = warp_sum(sum);
          const int i = i0 + 32 * h;
          if (lane == 0 && i < C) pm[0][i] = (m == neg_inf()) ? neg_inf() : m + lg2(sum);
        }
      }
      __syncthreads();
      if (tid < C) val = pm[0][tid];
    }
    // normalise by the vector max (8 warps hold the C <= 256 values)
    if (tid < kWideMaxC) {
      const float wm = warp_max(val);
      if (lane == 0) red[w] = wm;
    }
    __syncthreads();
    float Mx = red[0];
#pragma unroll
    for (int k = 1; k < kWideMaxC / 32; ++k) Mx = fmaxf(Mx, red[k]);
    dead = dead || (Mx == neg_inf());
    if (tid < C) {
      const float nv = dead ? neg_inf() : val - Mx;
      vn[tid] = nv;
      vh[p * C + tid] = nv;
    }
    if (!dead) off += (double)Mx;
    if (tid == 0) vo[p] = dead ? -INFINITY : off;
    __syncthreads();
  }
  if (!fwd) return;
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&sbad, 1u);
  __syncthreads();
  if (tid < 32) {
    const float* vE = vec[Eb & 1];
    float sum = 0.f;
    for (int j = tid; j < C; j += 32) sum += ex2(vE[j]);  // normalised: max 0, no overflow
    sum = warp_sum(sum);
    if (tid == 0) {
      unsigned fl = 0;
      double A;
      if (sbad) {
        fl = TS_F_NONFINITE;
        A = (double)qnan();
      } else if (dead) {
        fl = TS_F_EMPTY;
        A = -INFINITY;
      } else {
        A = kLn2 * (off + (double)lg2(sum));
      }
      a.zbuf[b] = A;
      a.logz[b] = (float)A;
      if (a.flags) a.flags[b] = fl;
    }
  }
}

// one CTA per edge (b, t); block 256
__global__ void __launch_bounds__(256) fb_wide_marg_kernel(SemiArgs a) {
  __shared__ float sa[kWideMaxC], sb[kWideMaxC];
  const int C = (int)a.C;
  const int64_t N = a.N, E = N - 1, CC = (int64_t)C * C;
  const int64_t e = blockIdx.x, b = e / E, t = e - b * E;
  const int tid = threadIdx.x;
  const int64_t len = seq_len(a.lengths, b, N);
  const double A = a.zbuf[b];
  float* mg = a.marg + e * CC;
  const float* l = a.pot + e * CC;
  bool zero = len < 0 || t >= len - 1 || !(A > -INFINITY && A < INFINITY);
  double dd = 0.0;
  if (!zero) {
    dd = a.ao[b * N + t] + a.bo[b * N + t + 1] - A / kLn2;
    zero = !(dd > -INFINITY);
  }
  if (zero) {
    if ((CC & 3) == 0) {
      float4* m4 = reinterpret_cast<float4*>(mg);
      for (int64_t k = tid; k < CC / 4; k += 256) m4[k] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      for (int64_t k = tid; k < CC; k += 256) mg[k] = 0.f;
    }
    return;
  }
  const float d = (float)dd;
  if (tid < C) {
    sa[tid] = a.ah[(b * N + t) * C + tid];
    sb[tid] = a.bh[(b * N + t + 1) * C + tid] + d;
  }
  __syncthreads();
  if ((CC & 3) == 0) {
    const float4* l4 = reinterpret_cast<const float4*>(l);
    float4* m4 = reinterpret_cast<float4*>(mg);
    // element index q = 4k: track (i, j) = divmod(q, C) incrementally (no integer division)
    const int step = 1024 % C, istep = 1024 / C;
    int i = (4 * tid) / C, j = 4 * tid - i * C;
    for (int64_t k = tid; k < CC / 4; k += 256) {
      const float4 v = l4[k];
      float r[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool wrap = j + u >= C;  // C > 128: at most one wrap in 4 elements
        const int ii = wrap ? i + 1 : i, jj = wrap ? j + u - C : j + u;
        r[u] = ex2(sa[ii] + fmaf(r[u], kLog2e, sb[jj]));
      }
      m4[k] = make_float4(r[0], r[1], r[2], r[3]);
      j += step;
      i += istep;
      if (j >= C) {
        j -= C;
        ++i;
      }
    }
  } else {
    for (int64_t k = tid; k < CC; k += 256) {
      const int i = (int)(k / C), j = (int)(k - (int64_t)i * C);
      mg[k] = ex2(sa[i] + fmaf(l[k], kLog2e, sb[j]));
    }
  }
}

// ---- TMA-ring variant (C % 4 == 0: every 32-row block of a tile is 16-byte aligned) -------
// A producer warp streams each tile as ceil(C/32) contiguous 32-row blocks (1-D bulk
// copies, up to 32 KB) into a kWideRing-slot SMEM ring, across steps, as fast as the 16
// consumer warps free slots, so up to ~190 KB of l is in flight per SM independently of
// registers.  Forward: thread (j, q) takes rows q, q+2, ... of each block (16 terms, online
// LSE); backward: warp w takes rows w and w+16 of each block (lanes along j).  Each consumer
// warp releases a slot with one arrival on its `empty` barrier (count 16).
constexpr int kWideRing = 6;

__device__ __forceinline__ void wide_issue(const SemiArgs& a, int64_t b, bool fwd, int64_t Eb,
                                           int nblk, int64_t h, float* ring, uint64_t* full,
                                           uint64_t* empty) {
  const int C = (int)a.C;
  const int64_t sh = h / nblk + 1;  // step of block h
  if (sh > Eb) return;
  const int kb = (int)(h - (sh - 1) * nblk);
  const int64_t p = fwd ? sh : Eb - sh;
  const int64_t t = fwd ? p - 1 : p;
  const int slot = (int)(h % kWideRing);
  if (h >= kWideRing) mbar_wait(&empty[slot], (uint32_t)(((h / kWideRing) - 1) & 1));
  const int r0 = kb * 32, rows = (C - r0 < 32) ? C - r0 : 32;
  const float* src = a.pot + ((b * (a.N - 1) + t) * C + r0) * (int64_t)C;
  bulk_load(ring + (size_t)slot * 32 * C, src, (uint32_t)(rows * C * 4), &full[slot]);
}

constexpr int kRingConsumers = 512;                  // 16 consumer warps
constexpr int kRingThreads = kRingConsumers + 32;    // + 1 producer warp
constexpr int kRingCW = kRingConsumers / 32;

__global__ void __launch_bounds__(kRingThreads, 1) fb_wide_ring_kernel(SemiArgs a) {
  extern __shared__ __align__(128) float wring[];
  __shared__ float vec[2][kWideMaxC];
  __shared__ float pm[2][kWideMaxC], ps[2][kWideMaxC];
  __shared__ float red[32];
  __shared__ unsigned sbad;
  __shared__ __align__(8) uint64_t full[kWideRing], empty[kWideRing];
  const int C = (int)a.C;
  const int64_t N = a.N;
  const int64_t b = blockIdx.x;
  const bool fwd = blockIdx.y == 0;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t len = seq_len(a.lengths, b, N);
  if (len < 0) {
    if (fwd && tid == 0) {
      a.logz[b] = qnan();
      a.zbuf[b] = (double)qnan();
      if (a.flags) a.flags[b] = TS_F_BADLEN;
    }
    return;
  }
  const int64_t Eb = len - 1;
  const int nblk = (C + 31) / 32;
  float* vh = (fwd ? a.ah : a.bh) + b * N * C;
  double* vo = (fwd ? a.ao : a.bo) + b * N;
  const int64_t n0 = fwd ? 0 : Eb;
  if (tid < C) {
    vec[0][tid] = 0.f;
    vh[n0 * C + tid] = 0.f;
  }
  if (tid == 0) {
    sbad = 0u;
    vo[n0] = 0.0;
    for (int k = 0; k < kWideRing; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], kRingCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (w == kRingCW) {  // producer warp: stream every block of every step through the ring
    if (lane == 0) {
      const int64_t total = Eb * nblk;
      for (int64_t h = 0; h < total; ++h) wide_issue(a, b, fwd, Eb, nblk, h, wring, full, empty);
    }
    return;
  }
  bool bad = false;
  double off = 0.0;
  bool dead = false;
  int64_t g = 0;  // blocks consumed so far
  for (int64_t s = 1; s <= Eb; ++s) {
    const int64_t p = fwd ? s : Eb - s;
    const float* v = vec[(s - 1) & 1];
    float* vn = vec[s & 1];
    float val = neg_inf();
    const int j = tid & (kWideMaxC - 1), q = tid >> 8;  // q in {0, 1}: rows = q (mod 2)
    float m = neg_inf(), sum = 0.f;
    for (int kb = 0; kb < nblk; ++kb, ++g) {
      const int slot = (int)(g % kWideRing);
      mbar_wait(&full[slot], (uint32_t)((g / kWideRing) & 1));
      const float* blk = wring + (size_t)slot * 32 * C;
      const int r0 = kb * 32;
      if (fwd) {
        if (j < C) {
          float x[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int r = q + 2 * k, i = r0 + r;
            const float lv = (i < C) ? blk[r * C + j] : neg_inf();
            bad |= (lv != lv) | (lv == pos_inf());
            x[k] = (i < C) ? fmaf(lv, kLog2e, v[i]) : neg_inf();
          }
          online_add<16>(m, sum, x);
        }
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // rows w and w + 16 of the block
          const int i = r0 + w + kRingCW * h;
          if (i < C) {
            float x[kWideMaxC / 32];
            float mm = neg_inf();
#pragma unroll
            for (int k = 0; k < kWideMaxC / 32; ++k) {
              const int jj = lane + 32 * k;
              x[k] = (jj < C) ? fmaf(blk[(w + kRingCW * h) * C + jj], kLog2e, v[jj]) : neg_inf();
              mm = fmaxf(mm, x[k]);
            }
            mm = warp_max(mm);
            float ss = 0.f;
            if (mm != neg_inf())
#pragma unroll
              for (int k = 0; k < kWideMaxC / 32; ++k) ss += ex2(x[k] - mm);
            ss = warp_sum(ss);
            if (lane == 0) pm[0][i] = (mm == neg_inf()) ? neg_inf() : mm + lg2(ss);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
    if (fwd) {
      pm[q][j] = m;
      ps[q][j] = sum;
    }
    named_bar(1, kRingConsumers);
    if (tid < C) {
      if (fwd) {
        float M = pm[0][tid], S = ps[0][tid];
        lse_merge(M, S, pm[1][tid], ps[1][tid]);
        val = (M == neg_inf()) ? neg_inf() : M + lg2(S);
      } else {
        val = pm[0][tid];
      }
    }
    if (tid < kWideMaxC) {
      const float wm = warp_max(val);
      if (lane == 0) red[w] = wm;
    }
    named_bar(1, kRingConsumers);
    float Mx = red[0];
#pragma unroll
    for (int k = 1; k < kWideMaxC / 32; ++k) Mx = fmaxf(Mx, red[k]);
    dead = dead || (Mx == neg_inf());
    if (tid < C) {
      const float nv = dead ? neg_inf() : val - Mx;
      vn[tid] = nv;
      vh[p * C + tid] = nv;
    }
    if (!dead) off += (double)Mx;
    if (tid == 0) vo[p] = dead ? -INFINITY : off;
    named_bar(1, kRingConsumers);
  }
  if (!fwd) return;
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&sbad, 1u);
  named_bar(1, kRingConsumers);
  if (tid < 32) {
    const float* vE = vec[Eb & 1];
    float sum = 0.f;
    for (int jj = tid; jj < C; jj += 32) sum += ex2(vE[jj]);
    sum = warp_sum(sum);
    if (tid == 0) {
      unsigned fl = 0;
      double A;
      if (sbad) {
        fl = TS_F_NONFINITE;
        A = (double)qnan();
      } else if (dead) {
        fl = TS_F_EMPTY;
        A = -INFINITY;
      } else {
        A = kLn2 * (off + (double)lg2(sum));
      }
      a.zbuf[b] = A;
      a.logz[b] = (float)A;
      if (a.flags) a.flags[b] = fl;
    }
  }
}

int g_wide_ring = 1;  // debug knob (tests): 0 forces the register-path sweep

cudaError_t launch_fb_wide(const SemiArgs& a, cudaStream_t st) {
  const dim3 grid((unsigned)a.B, a.marg ? 2u : 1u);
  if (a.C % 4 == 0 && g_wide_ring) {
    const size_t smem = (size_t)kWideRing * 32 * a.C * sizeof(float);
    static std::atomic<uint64_t> attr{0};
    cudaError_t ea = smem_optin_once(fb_wide_ring_kernel, attr,
                                     (int)((size_t)kWideRing * 32 * kWideMaxC * sizeof(float)));
    if (ea != cudaSuccess) return ea;
    fb_wide_ring_kernel<<<grid, kRingThreads, smem, st>>>(a);
  } else {
    fb_wide_sweep_kernel<<<grid, kWideThreads, 0, st>>>(a);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !a.marg || a.N < 2) return e;
  fb_wide_marg_kernel<<<(unsigned)(a.B * (a.N - 1)), 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace tsb
