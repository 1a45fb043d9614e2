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
// One CTA per sequence; column j is owned by a group of S consecutive lanes (S = 8, 4, 2, 1
// as C allows <= 512 threads): lane s of the group inserts the candidates of labels
// i = s (mod S) into a sorted register list, then the S partial lists are merged with KM
// rounds of a shuffle arg-max over the group heads under the same (score desc, i asc,
// r asc) key (the partial lists cover disjoint label sets, so the merge is exact).  Lists
// live in SMEM between steps; backpointers (i | r << 8) as uint16 [B][E][C][KM].
#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

// lanes per column: the largest power of two <= 8 with C * S <= 512
__host__ __device__ inline int kbest_split(int C) {
  int S = 8;
  while (S > 1 && C * S > 512) S >>= 1;
  return S;
}

template <int KM>
__global__ void __launch_bounds__(512) kbest_kernel(KbestArgs a) {
  extern __shared__ __align__(16) float ksm[];
  const int C = (int)a.C;
  const int64_t N = a.N, E = N - 1, CC = (int64_t)C * C;
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, NW = blockDim.x >> 5;
  const bool act = tid < C;                        // final merge: thread = column
  const int S = kbest_split(C);
  const int jcol = tid / S, sidx = tid - jcol * S;  // step loop: S lanes per column
  const bool actc = jcol < C;
  float* dl = ksm;                                  // [2][C][KM]
  float* rs = dl + 2 * (size_t)C * KM;              // [NW] block-reduction scores
  int* ri = reinterpret_cast<int*>(rs + NW);        // [NW] block-reduction labels
  int* sel = ri + NW;                               // [K][2] final (j, r)
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
  if (tid == 0) *bad = 0u;
  if (act) {
#pragma unroll
    for (int r = 0; r < KM; ++r) dl[tid * KM + r] = (r == 0) ? 0.f : neg_inf();
  }
  __syncthreads();
  float sc[KM];
  int ii[KM], rr[KM];
  int cur = 0;
  bool nonfin = false;
  for (int64_t t = 0; t < Eb; ++t) {
#pragma unroll
    for (int r = 0; r < KM; ++r) {
      sc[r] = neg_inf();
      ii[r] = 0;
      rr[r] = 0;
    }
    const float* d = dl + (size_t)cur * C * KM;
    if (actc) {
      const float* col = a.pot + (b * E + t) * CC + jcol;
      constexpr int kPf = 16;  // column values loaded per batch (independent loads in flight)
      for (int i0 = sidx; i0 < C; i0 += S * kPf) {
        float lvs[kPf];
#pragma unroll
        for (int u = 0; u < kPf; ++u)
          lvs[u] = (i0 + S * u < C) ? col[(int64_t)(i0 + S * u) * C] : neg_inf();
#pragma unroll 1
        for (int u = 0; u < kPf && i0 + S * u < C; ++u) {
        const int i = i0 + S * u;
        const float lv = lvs[u];
        nonfin |= (lv != lv) | (lv == pos_inf());
        if (lv == neg_inf()) continue;
        for (int r = 0; r < KM; ++r) {
          const float v = d[i * KM + r] + lv;
          if (!(v > sc[KM - 1])) break;  // lists are sorted: no later r can enter
          int pos = 0;
#pragma unroll
          for (int q = 0; q < KM; ++q) pos += (sc[q] >= v) ? 1 : 0;
#pragma unroll
          for (int p = KM - 1; p > 0; --p)
            if (p > pos) {
              sc[p] = sc[p - 1];
              ii[p] = ii[p - 1];
              rr[p] = rr[p - 1];
            }
#pragma unroll
          for (int p = 0; p < KM; ++p)
            if (p == pos) {
              sc[p] = v;
              ii[p] = i;
              rr[p] = r;
            }
        }
        }
      }
    }
    // merge the S partial lists of the group: KM rounds of a (score desc, i asc, r asc)
    // arg-max over the group heads (every lane of the warp takes part in the shuffles)
    {
      float* dn = dl + (size_t)(cur ^ 1) * C * KM + (size_t)jcol * KM;
      uint16_t* bpo = a.bp + ((b * E + t) * C + jcol) * KM;
      int h = 0;
#pragma unroll
      for (int out = 0; out < KM; ++out) {
        float hv = neg_inf();
        int hi = 0, hr = 0;
#pragma unroll
        for (int q = 0; q < KM; ++q)
          if (q == h) {
            hv = sc[q];
            hi = ii[q];
            hr = rr[q];
          }
        int src = sidx;
        for (int o = 1; o < S; o <<= 1) {
          const float ov = __shfl_xor_sync(0xffffffffu, hv, o);
          const int oi = __shfl_xor_sync(0xffffffffu, hi, o);
          const int orr = __shfl_xor_sync(0xffffffffu, hr, o);
          const int os = __shfl_xor_sync(0xffffffffu, src, o);
          if (ov > hv || (ov == hv && (oi < hi || (oi == hi && (orr < hr || (orr == hr && os < src)))))) {
            hv = ov;
            hi = oi;
            hr = orr;
            src = os;
          }
        }
        if (src == sidx) ++h;
        if (sidx == 0 && actc) {
          dn[out] = hv;
          bpo[out] = (uint16_t)(hi | (hr << 8));
        }
      }
    }
    cur ^= 1;
    __syncthreads();
  }
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

size_t kbest_smem(int64_t C, int64_t K) {
  const int km = kbest_km(K);
  return (2 * (size_t)C * km + 16) * sizeof(float) + 16 * sizeof(int) + 2 * (size_t)K * sizeof(int) + 16;
}

cudaError_t launch_kbest(const KbestArgs& a, cudaStream_t st) {
  const int km = kbest_km(a.K);
  const int NT = (int)(((a.C * kbest_split((int)a.C) + 31) / 32) * 32);
  const size_t smem = kbest_smem(a.C, a.K);
  switch (km) {
    case 1: kbest_kernel<1><<<(unsigned)a.B, NT, smem, st>>>(a); break;
    case 2: kbest_kernel<2><<<(unsigned)a.B, NT, smem, st>>>(a); break;
    case 4: kbest_kernel<4><<<(unsigned)a.B, NT, smem, st>>>(a); break;
    case 8: kbest_kernel<8><<<(unsigned)a.B, NT, smem, st>>>(a); break;
    case 16: kbest_kernel<16><<<(unsigned)a.B, NT, smem, st>>>(a); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace tsb
