// kbest.cu — K-best Viterbi (Table 2 'K-Max' semiring).
//
// delta_{t+1}[j] = the top-KM (score, i, r) of delta_t[i][r] + l_t[i][j] over all labels i and
// ranks r, ordered by (score desc, i asc, r asc); delta_0[j] = [(0)].  That order is the
// global order of DESIGN.md reading R16 (Score desc, then reverse-lexicographic asc)
// restricted to partial paths ending at (t+1, j), so the final merge over (score desc,
// j asc, r asc) yields the first K labelings of that order.  KM = the next power of two
// >= K (keeping more candidates than K never changes the top K).  fp32 sums of dyadic
// inputs are exact, so the result equals the fp64 oracle bit for bit.
//
// One CTA per sequence; column j is owned by a group of S consecutive lanes (S in {8,4,2,1},
// a template parameter), lane s of the group handling the labels i = s (mod S).  Each step:
//  * the next edge's C x C tile is staged into shared memory with cp.async while this step
//    runs (rows padded to LD = 32/S (mod 32) floats: the warp's S label rows of 32/S columns
//    land on distinct banks); C > 128 reads the tile from global memory instead;
//  * pass 1 (values only, min/max network): the KM largest heads h_i = delta_t[i][0] +
//    l[i][j] of the lane, merged over the group by a shuffle butterfly (bitonic max + sort):
//    T = the column's KM-th largest head.  A candidate with score < T has KM heads strictly
//    above it, so only candidates with score >= T can enter the column's list;
//  * pass 2: the lane's labels with h_i >= T (a register bit mask; usually ~KM/S of them)
//    insert their candidates with score >= T into a sorted register list (ties keep the
//    (i, r) order since labels and ranks are visited in ascending order);
//  * KM rounds of a shuffle arg-max over the S list heads under the (score desc, i asc,
//    r asc) key (packed (i, r, lane) in one int) write delta_{t+1}[j] and the backpointers
//    (i | r << 8, uint16 [B][E][C][KM]).
#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

namespace {
std::atomic<int> g_kbest_split{0};
__device__ __forceinline__ float fmax_nan(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
}  // namespace
void set_kbest_split(int S) { g_kbest_split.store((S == 1 || S == 2 || S == 4 || S == 8) ? S : 0); }

// padded tile row stride: >= C, a multiple of 4, and == 32/S (mod 32) for S >= 2
__host__ __device__ inline int kbest_ld(int C, int S) {
  const int r = S >= 2 ? 32 / S : 0;
  int ld = (C + 3) & ~3;
  if (S >= 2) ld += ((r - ld % 32) + 32) % 32;
  return ld;
}
constexpr int kKbStageMaxC = 128;  // two staged tiles fit in shared memory up to here
// dynamic shared memory opt-in (once per instantiation and device): above every kbest_smem
constexpr int kKbSmemOptin = 200 * 1024;

constexpr int kKbL2Ahead = 3;      // edges prefetched into L2 beyond the staged ring
// staged ring depth: 3 tiles when they fit in ~110 KB (two CTAs per SM), else 2
__host__ __device__ inline int kbest_stages(int C, int S) {
  return 3 * (size_t)C * kbest_ld(C, S) * sizeof(float) <= 110 * 1024 ? 3 : 2;
}

__host__ __device__ inline size_t kbest_dl_floats(int C, int KM) { return ((size_t)2 * C * KM + 3) & ~(size_t)3; }

template <int KM, int S>
__global__ void __launch_bounds__(512) kbest_kernel(KbestArgs a) {
  extern __shared__ __align__(16) float ksm[];
  const int C = (int)a.C;
  const bool staged = C <= kKbStageMaxC;
  const int LD = kbest_ld(C, S);
  const int64_t N = a.N, E = N - 1, CC = (int64_t)C * C;
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, NW = blockDim.x >> 5;
  const bool act = tid < C;                        // final merge: thread = column
  const int jcol = tid / S, sidx = tid - jcol * S;  // step loop: S lanes per column
  const bool actc = jcol < C;
  float* dl = ksm;                                  // [2][C][KM]
  float* tiles = dl + kbest_dl_floats(C, KM);       // [2][C][LD] when staged
  float* rs = tiles + (staged ? (size_t)kbest_stages(C, S) * C * LD : 0);  // [NW] block-reduction scores
  int* ri = reinterpret_cast<int*>(rs + 16);        // [NW] block-reduction labels
  int* sel = ri + 16;                               // [K][2] final (j, r)
  unsigned* bad = reinterpret_cast<unsigned*>(sel + 2 * a.K);
  const int K = (int)a.K;
  int32_t* pb = a.paths + b * (int64_t)K * N;
  float* sb = a.scores + b * K;
  const int64_t len = seq_len(a.lengths, b, N);
  if (len < 0) {
    for (int64_t q = tid; q < (int64_t)K * N; q += blockDim.x) pb[q] = -1;
    for (int q = tid; q < K; q += blockDim.x) sb[q] = qnan();
    if (tid == 0 && a.flags) a.flags[b] = TS_F_BADLEN;
    return;
  }
  const int64_t Eb = len - 1;
  const bool vec = (C % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.pot) & 15) == 0);
  const int NST = kbest_stages(C, S);  // staged tile ring depth (2 or 3)
  // cp.async mapping: thread tid copies the 16-byte pieces q = tid + NT k of a tile, i.e.
  // (row, quad) = (tid / C4 + k NT / C4, tid % C4) when NT is a multiple of C4 = C / 4
  const int C4 = C / 4, NT = (int)blockDim.x;
  const bool fastmap = vec && (NT % C4 == 0);
  const int row0 = fastmap ? tid / C4 : 0, qd0 = fastmap ? tid - (tid / C4) * C4 : 0;
  const int rstep = fastmap ? NT / C4 : 0;
  auto stage = [&](int64_t t) {  // cp.async the tile of edge t into tiles[t % NST]
    if (t < Eb) {
      const float* src = a.pot + (b * E + t) * CC;
      float* dst = tiles + (size_t)(t % NST) * C * LD;
      if (fastmap) {
        for (int row = row0; row < C; row += rstep)
          cp_async16(dst + row * LD + 4 * qd0, src + (int64_t)row * C + 4 * qd0);
      } else if (vec) {
        for (int q = tid; q < C * C4; q += NT) {
          const int row = q / C4, c4 = q - row * C4;
          cp_async16(dst + row * LD + 4 * c4, src + (int64_t)row * C + 4 * c4);
        }
      } else {
        for (int q = tid; q < C * C; q += NT) {
          const int row = q / C, c = q - row * C;
          cp_async4(dst + row * LD + c, src + q);
        }
      }
    }
    cp_async_commit();  // (an empty group past the end keeps the group count uniform)
  };
  auto prefetch_l2 = [&](int64_t t) {  // the tile of edge t into L2, ahead of its cp.async
    if (t >= Eb) return;
    const float* src = a.pot + (b * E + t) * CC;
    if (vec) {
      if (tid == 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"((unsigned)(CC * 4)));
    } else {
      for (int64_t q = (int64_t)tid * 32; q < CC; q += (int64_t)blockDim.x * 32)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(src + q));
    }
  };
  if (tid == 0) *bad = 0u;
  if (act) {
#pragma unroll
    for (int r = 0; r < KM; ++r) dl[tid * KM + r] = (r == 0) ? 0.f : neg_inf();
  }
  if (staged && Eb > 0) {
    for (int q = 0; q < NST - 1; ++q) stage(q);
    for (int q = 0; q < kKbL2Ahead; ++q) prefetch_l2(NST - 1 + q);
    cp_async_wait_dyn(NST - 2);  // tile 0 landed
  }
  __syncthreads();
  const int U = (C + S - 1) / S;  // labels i = sidx + S u of this lane, u < U
  constexpr int kHR = (512 / (S * S)) < 32 ? (512 / (S * S)) : 32;  // heads kept in registers
  float sc[KM];
  int ii[KM], rr[KM];
  int cur = 0;
  float lmax = neg_inf();  // NaN-propagating max of every potential read: NaN / +inf flag
  for (int64_t t = 0; t < Eb; ++t) {
    if (staged) {
      stage(t + NST - 1);
      prefetch_l2(t + NST - 1 + kKbL2Ahead);
    }
    const float* d = dl + (size_t)cur * C * KM;
    const float* lcol = staged ? tiles + (size_t)(t % NST) * C * LD + jcol : a.pot + (b * E + t) * CC + jcol;
    const int64_t lst = staged ? LD : C;
    // pass 1 (values only): the KM largest heads of this lane, then of the column
    float tv[KM], hv[kHR];
#pragma unroll
    for (int k = 0; k < KM; ++k) tv[k] = neg_inf();
#pragma unroll
    for (int u = 0; u < kHR; ++u) hv[u] = neg_inf();
    if (actc) {
#pragma unroll
      for (int u0 = 0; u0 < kHR; u0 += 8) {
        if (u0 < U) {
#pragma unroll
          for (int u = u0; u < u0 + 8; ++u) {
            const int i = sidx + S * u;
            if (u < U && i < C) {
              const float lv = lcol[i * lst];
              lmax = fmax_nan(lmax, lv);
              const float h = d[i * KM] + lv;
              hv[u] = h;
#pragma unroll
              for (int k = KM - 1; k > 0; --k) tv[k] = fmaxf(tv[k], fminf(tv[k - 1], h));
              tv[0] = fmaxf(tv[0], h);
            }
          }
        }
      }
      for (int u = kHR; u < U; ++u) {
        const int i = sidx + S * u;
        if (i >= C) break;
        const float lv = lcol[i * lst];
        lmax = fmax_nan(lmax, lv);
        const float h = d[i * KM] + lv;
#pragma unroll
        for (int k = KM - 1; k > 0; --k) tv[k] = fmaxf(tv[k], fminf(tv[k - 1], h));
        tv[0] = fmaxf(tv[0], h);
      }
    }
#pragma unroll
    for (int o = 1; o < S; o <<= 1) {  // merge two sorted KM-lists: bitonic max, then sort
      float pv[KM];
#pragma unroll
      for (int k = 0; k < KM; ++k) pv[k] = __shfl_xor_sync(0xffffffffu, tv[k], o);
#pragma unroll
      for (int k = 0; k < KM; ++k) tv[k] = fmaxf(tv[k], pv[KM - 1 - k]);
#pragma unroll
      for (int ln = KM / 2; ln > 0; ln >>= 1)
#pragma unroll
        for (int k = 0; k < KM; ++k)
          if ((k & ln) == 0) {
            const float hi = fmaxf(tv[k], tv[k + ln]), lo = fminf(tv[k], tv[k + ln]);
            tv[k] = hi;
            tv[k + ln] = lo;
          }
    }
    const float T = tv[KM - 1];
    // pass 2: the qualifying labels (h_i >= T, finite) of this lane in ascending i
#pragma unroll
    for (int r = 0; r < KM; ++r) {
      sc[r] = neg_inf();
      ii[r] = 0;
      rr[r] = 0;
    }
    if (actc) {
      for (int w0 = 0; w0 < U; w0 += 32) {
        uint32_t m = 0u;
        if (w0 == 0) {
#pragma unroll
          for (int u0 = 0; u0 < kHR; u0 += 8)
            if (u0 < U) {
#pragma unroll
              for (int u = u0; u < u0 + 8; ++u)
                if (hv[u] >= T && hv[u] > neg_inf()) m |= 1u << u;
            }
        } else {
          const int wn = (U - w0) < 32 ? (U - w0) : 32;
          for (int q = 0; q < wn; ++q) {
            const int i = sidx + S * (w0 + q);
            if (i >= C) break;
            const float h = d[i * KM] + lcol[i * lst];
            if (h >= T && h > neg_inf()) m |= 1u << q;
          }
        }
        while (m) {
          const int q = __ffs(m) - 1;
          m &= m - 1;
          const int i = sidx + S * (w0 + q);
          const float lv = lcol[i * lst];
          for (int r = 0; r < KM; ++r) {
            const float v = d[i * KM + r] + lv;
            if (!(v >= T) || !(v > sc[KM - 1])) break;  // lists are sorted: no later r enters
            int pos = 0;
#pragma unroll
            for (int q2 = 0; q2 < KM; ++q2) pos += (sc[q2] >= v) ? 1 : 0;
#pragma unroll
            for (int p2 = KM - 1; p2 > 0; --p2)
              if (p2 > pos) {
                sc[p2] = sc[p2 - 1];
                ii[p2] = ii[p2 - 1];
                rr[p2] = rr[p2 - 1];
              }
#pragma unroll
            for (int p2 = 0; p2 < KM; ++p2)
              if (p2 == pos) {
                sc[p2] = v;
                ii[p2] = i;
                rr[p2] = r;
              }
          }
        }
      }
    }
    // merge the S partial lists of the group: KM rounds of a (score desc, key asc) arg-max
    // over the group heads, key = i << 8 | r << 3 | lane-in-group (i < 256, r < 16, S <= 8)
    {
      float* dn = dl + (size_t)(cur ^ 1) * C * KM + (size_t)jcol * KM;
      uint16_t* bpo = a.bp + ((b * E + t) * C + jcol) * KM;
      int h = 0;
#pragma unroll
      for (int out = 0; out < KM; ++out) {
        float hv2 = neg_inf();
        int hk = 0;
#pragma unroll
        for (int q = 0; q < KM; ++q)
          if (q == h) {
            hv2 = sc[q];
            hk = (ii[q] << 8) | (rr[q] << 3) | sidx;
          }
        if (hv2 == neg_inf()) hk = sidx;  // -inf padding: (i, r) = (0, 0)
#pragma unroll
        for (int o = 1; o < S; o <<= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, hv2, o);
          const int ok = __shfl_xor_sync(0xffffffffu, hk, o);
          if (ov > hv2 || (ov == hv2 && ok < hk)) {
            hv2 = ov;
            hk = ok;
          }
        }
        if ((hk & 7) == sidx) ++h;
        if (sidx == 0 && actc) {
          dn[out] = hv2;
          bpo[out] = (uint16_t)((hk >> 8) | (((hk >> 3) & 31) << 8));
        }
      }
    }
    cur ^= 1;
    if (staged) cp_async_wait_dyn(NST - 2);  // tile t + 1 landed
    __syncthreads();
  }
  const bool nonfin = (lmax != lmax) || (lmax == pos_inf());
  if (__any_sync(0xffffffffu, nonfin) && lane == 0) atomicOr(bad, 1u);
  // final merge over (score desc, j asc, r asc): K rounds of a block arg-max over list heads
  const float* d = dl + (size_t)cur * C * KM;
  int h = 0;
  for (int q = 0; q < K; ++q) {
    float v = (act && h < KM) ? d[tid * KM + h] : neg_inf();
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
      rs[w] = v;
      ri[w] = idx;
    }
    __syncthreads();
    if (tid == 0) {
      float bv = rs[0];
      int bi = ri[0];
      for (int k = 1; k < NW; ++k)
        if (rs[k] > bv || (rs[k] == bv && ri[k] < bi)) {
          bv = rs[k];
          bi = ri[k];
        }
      sb[q] = bv;
      sel[2 * q] = (bv == neg_inf()) ? -1 : bi;
      sel[2 * q + 1] = -1;
      rs[0] = bv;
      ri[0] = bi;
    }
    __syncthreads();
    if (rs[0] != neg_inf() && tid == ri[0]) {  // the winner reports its rank and advances
      sel[2 * q + 1] = h;
      ++h;
    }
    __syncthreads();
  }
  const bool nf = *bad != 0u;
  if (tid == 0 && a.flags) {
    const bool empty = !nf && (K > 0) && sb[0] == neg_inf();
    a.flags[b] = nf ? (unsigned)TS_F_NONFINITE : (empty ? (unsigned)TS_F_EMPTY : 0u);
  }
  // backtrack: thread q < K walks its path back through the backpointers
  if (tid < K) {
    const int q = tid;
    int32_t* pq = pb + (int64_t)q * N;
    int z = sel[2 * q], slot = sel[2 * q + 1];
    if (nf) {
      sb[q] = qnan();
      z = -1;
    }
    for (int64_t n = len; n < N; ++n) pq[n] = -1;
    if (z < 0 || slot < 0) {
      for (int64_t n = 0; n < len; ++n) pq[n] = -1;
    } else {
      pq[Eb] = z;
      for (int64_t t = Eb - 1; t >= 0; --t) {
        const uint16_t v = a.bp[((b * E + t) * C + z) * KM + slot];
        z = v & 0xFF;
        slot = v >> 8;
        pq[t] = z;
      }
    }
  }
}


int kbest_km(int64_t K) {
  int km = 1;
  while (km < K) km <<= 1;
  return km;
}

namespace {
int kbest_split_for(int64_t B, int64_t C, int sms) {
  const int knob = g_kbest_split.load();
  int S = knob ? knob : (B >= sms ? 4 : 8);
  while (S > 1 && C * S > 512) S >>= 1;
  return S;
}
}  // namespace

size_t kbest_smem(int64_t C, int64_t K, int S) {
  const int km = kbest_km(K);
  const size_t tiles = C <= kKbStageMaxC ? (size_t)kbest_stages((int)C, S) * C * kbest_ld((int)C, S) : 0;
  return (kbest_dl_floats((int)C, km) + tiles + 16) * sizeof(float) + 16 * sizeof(int) +
         2 * (size_t)K * sizeof(int) + 16;
}

template <int KM>
cudaError_t launch_kbest_km(const KbestArgs& a, int S, size_t smem, cudaStream_t st) {
  static std::atomic<uint64_t> attr[4];
  const int NT = (int)(((a.C * S + 31) / 32) * 32);
  cudaError_t e = cudaSuccess;
  switch (S) {
    case 1:
      if ((e = smem_optin_once(kbest_kernel<KM, 1>, attr[0], kKbSmemOptin)) != cudaSuccess) return e;
      kbest_kernel<KM, 1><<<(unsigned)a.B, NT, smem, st>>>(a);
      break;
    case 2:
      if ((e = smem_optin_once(kbest_kernel<KM, 2>, attr[1], kKbSmemOptin)) != cudaSuccess) return e;
      kbest_kernel<KM, 2><<<(unsigned)a.B, NT, smem, st>>>(a);
      break;
    case 4:
      if ((e = smem_optin_once(kbest_kernel<KM, 4>, attr[2], kKbSmemOptin)) != cudaSuccess) return e;
      kbest_kernel<KM, 4><<<(unsigned)a.B, NT, smem, st>>>(a);
      break;
    default:
      if ((e = smem_optin_once(kbest_kernel<KM, 8>, attr[3], kKbSmemOptin)) != cudaSuccess) return e;
      kbest_kernel<KM, 8><<<(unsigned)a.B, NT, smem, st>>>(a);
      break;
  }
  return cudaGetLastError();
}

cudaError_t launch_kbest(const KbestArgs& a, cudaStream_t st) {
  const int km = kbest_km(a.K);
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int S = kbest_split_for(a.B, a.C, sms);
  const size_t smem = kbest_smem(a.C, a.K, S);
  switch (km) {
    case 1: return launch_kbest_km<1>(a, S, smem, st);
    case 2: return launch_kbest_km<2>(a, S, smem, st);
    case 4: return launch_kbest_km<4>(a, S, smem, st);
    case 8: return launch_kbest_km<8>(a, S, smem, st);
    case 16: return launch_kbest_km<16>(a, S, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tsb
