// dist_ops.cu — distribution properties on top of the hot path (
// PAPER.md §3: Sampling, Density, Entropy; Table 2; P:267 FFBS).
//
//  * entropy:  H_b = A_b - Σ_{t,i,j} mu[b,t,i,j] l[b,t,i,j]   (log p(z) = Score(z) - A,
//              P:176-177, and linearity of expectation over the parts).  A two-
//              stage deterministic reduction over the marginals the hot path just wrote:
//              grid (B, S) slices accumulate fp64 partials, one CTA per sequence sums them in
//              slice order.  Terms with mu = 0 are skipped (0 * -inf masks).
//  * expectation: E_p[Σ_p r_p z_p] = Σ_{t,i,j} mu[b,t,i,j] r[b,t,i,j] for a caller-given
//              additive feature r (Table 2 'Exp.' row; the expectation semiring's
//              moment over all structures equals this sum by linearity): the same
//              two-stage reduction with r in place of l, out = the sum.
//  * score:    Score_b(z) = Σ_{t < len-1} l[b,t,z_t,z_{t+1}], fp64; log_prob =
//              Score - A.
//  * sampling: forward-filtering backward-sampling.  The forward node vectors alpha_hat
//              (log2, one scalar frame per node) come from the streaming forward sweep; one
//              warp per (sample k, sequence b) walks back:
//                z_{n-1} ~ 2^(ah_{n-1}[j]),  z_t ~ 2^(ah_t[i] + (l_t[i][z_{t+1}] - c) log2 e)
//              (c = the column max, exact re-centring), drawing by inverse CDF with the
//              caller's uniform u[k][b][t]: the smallest i whose inclusive prefix sum exceeds
//              u * total (the oracle's rule, oracle.ffbs_sample).
#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

namespace {
constexpr int kRedThreads = 256;

__device__ __forceinline__ double block_sum_d(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];  // fixed order
  return s;
}
}  // namespace

// partial[b][s] = Σ mu * l (expectation: mu * r) over edges [s*Ls, min((s+1)*Ls, Eb)) of sequence b
__global__ void __launch_bounds__(kRedThreads) entropy_partial_kernel(DistArgs a) {
  __shared__ double red[kRedThreads / 32];
  const int64_t b = blockIdx.x, s = blockIdx.y;
  const int64_t N = a.N, E = N - 1, C = a.C, CC = C * C;
  const int64_t len = seq_len(a.lengths, b, N);
  const int64_t Eb = len < 1 ? 0 : len - 1;
  const int64_t t0 = s * a.Ls, t1 = (t0 + a.Ls < Eb) ? t0 + a.Ls : Eb;
  double acc = 0.0;
  if (t0 < t1) {
    const float* mu = a.marg + (b * E + t0) * CC;
    const float* l = (a.r ? a.r : a.pot) + (b * E + t0) * CC;
    const int64_t n = (t1 - t0) * CC;
    if ((CC & 3) == 0) {
      const float4* mu4 = reinterpret_cast<const float4*>(mu);
      const float4* l4 = reinterpret_cast<const float4*>(l);
      for (int64_t k = threadIdx.x; k < n / 4; k += kRedThreads) {
        const float4 m = mu4[k], v = l4[k];
        if (m.x != 0.f) acc += (double)m.x * (double)v.x;
        if (m.y != 0.f) acc += (double)m.y * (double)v.y;
        if (m.z != 0.f) acc += (double)m.z * (double)v.z;
        if (m.w != 0.f) acc += (double)m.w * (double)v.w;
      }
    } else {
      for (int64_t k = threadIdx.x; k < n; k += kRedThreads)
        if (mu[k] != 0.f) acc += (double)mu[k] * (double)l[k];
    }
  }
  const double tot = block_sum_d(acc, red);
  if (threadIdx.x == 0) a.partial[b * gridDim.y + s] = tot;
}

__global__ void entropy_final_kernel(DistArgs a, int S) {
  const int64_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  double sum = 0.0;
  for (int s = 0; s < S; ++s) sum += a.partial[b * S + s];  // slice order: deterministic
  const float lz = a.logz[b];
  const bool bad = (a.flags && a.flags[b] != 0) || !(lz > -INFINITY && lz < INFINITY);
  a.out[b] = bad ? qnan() : (float)(a.r ? sum : (double)lz - sum);
}

// Score(z) (and log_prob = Score - logz when logz is given), one CTA per sequence.
__global__ void __launch_bounds__(kRedThreads) score_kernel(DistArgs a) {
  __shared__ double red[kRedThreads / 32];
  __shared__ int bad;
  const int64_t b = blockIdx.x;
  const int64_t N = a.N, E = N - 1, C = a.C, CC = C * C;
  const int64_t len = seq_len(a.lengths, b, N);
  if (threadIdx.x == 0) bad = (len < 0);
  __syncthreads();
  double acc = 0.0;
  if (len > 0) {
    const int32_t* z = a.z + b * N;
    for (int64_t t = threadIdx.x; t < len; t += kRedThreads) {
      const int32_t zi = z[t];
      if (zi < 0 || zi >= C) bad = 1;
      else if (t + 1 < len) {
        const int32_t zj = z[t + 1];
        if (zj >= 0 && zj < C) acc += (double)a.pot[(b * E + t) * CC + (int64_t)zi * C + zj];
      }
    }
  }
  const double tot = block_sum_d(acc, red);
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = tot;
    if (a.logz) {
      const float lz = a.logz[b];
      v = (lz > -INFINITY && lz < INFINITY) ? tot - (double)lz : (double)qnan();
    }
    a.out[b] = bad ? qnan() : (float)v;
  }
}

// FFBS: one warp per (k, b).  ah: [B][N][C] forward node vectors (nodes < Eb), aend: [B][C]
// node Eb (the streaming forward's chunk-end vector, P = 1).
__global__ void __launch_bounds__(128) sample_kernel(DistArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (w >= a.K * a.B) return;
  const int64_t k = w / a.B, b = w - (w / a.B) * a.B;
  const int64_t N = a.N, E = N - 1, C = a.C, CC = C * C;
  int32_t* zo = a.zout + (k * a.B + b) * N;
  const float* u = a.uniforms + (k * a.B + b) * N;
  const int64_t len = seq_len(a.lengths, b, N);
  const bool flagged = len < 0 || (a.flags && a.flags[b] != 0);
  if (flagged) {
    for (int64_t t = lane; t < N; t += 32) zo[t] = -1;
    return;
  }
  for (int64_t t = len + lane; t < N; t += 32) zo[t] = -1;
  constexpr int R = 8;  // labels per lane (C <= 256): lane owns i in [R*lane, R*lane + R)
  const int i0 = R * lane;
  float lw[R];
  // z_{len-1} ~ 2^(ah_{len-1}[j])
  const float* v = a.aend_in_ah ? a.ah + (b * N + len - 1) * C : a.aend + b * C;
  if (len - 1 == 0) {  // single node: every label has weight 1 (alpha_0 = 0)
#pragma unroll
    for (int r = 0; r < R; ++r) lw[r] = (i0 + r < C) ? 0.f : neg_inf();
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r) lw[r] = (i0 + r < C) ? v[i0 + r] : neg_inf();
  }
  int32_t z = 0;
  for (int64_t t = len - 1; t >= 0; --t) {
    if (t < len - 1) {  // z_t | z_{t+1} = z:  ah_t[i] + (l_t[i][z] - c) log2 e
      const float* ahp = a.ah + (b * N + t) * C;
      const float* col = a.pot + (b * E + t) * CC + z;
      float lv[R];
      float c = neg_inf();
#pragma unroll
      for (int r = 0; r < R; ++r) {
        lv[r] = (i0 + r < C) ? col[(int64_t)(i0 + r) * C] : neg_inf();
        c = fmaxf(c, lv[r]);
      }
      c = warp_max(c);
      const float cz = (c == neg_inf()) ? 0.f : c;
#pragma unroll
      for (int r = 0; r < R; ++r)
        lw[r] = (i0 + r < C) ? ahp[i0 + r] + (lv[r] - cz) * kLog2e : neg_inf();
    }
    // inverse CDF: smallest i with inclusive prefix sum > u * total
    float m = neg_inf();
#pragma unroll
    for (int r = 0; r < R; ++r) m = fmaxf(m, lw[r]);
    m = warp_max(m);
    float pre[R];
    float run = 0.f;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      run += (m == neg_inf() || lw[r] == neg_inf()) ? 0.f : ex2(lw[r] - m);
      pre[r] = run;
    }
    float incl = run;  // warp inclusive scan of the lane totals
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const float y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const float total = __shfl_sync(0xffffffffu, incl, 31);
    const float excl = incl - run;
    const float target = u[t] * total;
    int hit = R;
#pragma unroll
    for (int r = R - 1; r >= 0; --r)
      if (i0 + r < C && excl + pre[r] > target) hit = r;
    const unsigned bal = __ballot_sync(0xffffffffu, hit < R);
    int zz;
    if (bal) {
      const int src = __ffs(bal) - 1;
      zz = R * src + __shfl_sync(0xffffffffu, hit, src);
    } else {  // u * total >= total through rounding: the last label with nonzero weight
      int last = -1;
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (i0 + r < C && lw[r] != neg_inf() && m != neg_inf()) last = i0 + r;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) last = max(last, __shfl_xor_sync(0xffffffffu, last, o));
      zz = last < 0 ? 0 : last;
    }
    z = zz;
    if (lane == 0) zo[t] = z;
  }
}

// ---- launchers ---------------------------------------------------------------------------
int entropy_slices(const DistArgs& a) {
  const int64_t E = a.N - 1 > 0 ? a.N - 1 : 1;
  int64_t S = (2 * 148 + a.B - 1) / a.B;
  if (S > E) S = E;
  if (S > 4096) S = 4096;
  return (int)(S < 1 ? 1 : S);
}

cudaError_t launch_entropy(DistArgs a, cudaStream_t st) {
  const int S = entropy_slices(a);
  const int64_t E = a.N - 1 > 0 ? a.N - 1 : 1;
  a.Ls = (E + S - 1) / S;
  entropy_partial_kernel<<<dim3((unsigned)a.B, (unsigned)S), kRedThreads, 0, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  entropy_final_kernel<<<(unsigned)((a.B + 127) / 128), 128, 0, st>>>(a, S);
  return cudaGetLastError();
}

cudaError_t launch_entropy_final(const DistArgs& a, int S, cudaStream_t st) {
  entropy_final_kernel<<<(unsigned)((a.B + 127) / 128), 128, 0, st>>>(a, S);
  return cudaGetLastError();
}

cudaError_t launch_score(const DistArgs& a, cudaStream_t st) {
  score_kernel<<<(unsigned)a.B, kRedThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_sample(const DistArgs& a, cudaStream_t st) {
  const int64_t warps = a.K * a.B;
  sample_kernel<<<(unsigned)((warps + 3) / 4), 128, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace tsb
