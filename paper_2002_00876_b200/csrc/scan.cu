// scan.cu — the time-chunked parallel scan of PAPER.md §6(a) (Fig. 4):
//   leaves  : chunk summaries S_k = l_{s_k} (x) ... (x) l_{e_k - 1}   (C x C, log semiring)
//   up-sweep: balanced tree of semiring matrix products, padded with I to a power of two
//   down    : prefix / suffix vectors alpha_in[k] = 0 (x) S_0 ... S_{k-1},
//             beta_out[k] = S_{k+1} ... S_{P-1} (x) 0   (vector x matrix at tree nodes)
// The leaf forward/backward sweeps (fb_stream.cu) then start from alpha_in / beta_out.
//
// Representations:
//   LogMat: S[r][j] = off[r] + ln2 * s[r][j]   (fp32 log2 values, fp64 natural row offsets)
//   LogVec: v[j]    = off    + ln2 * v[j]
// Products use the max-shifted log product of §6(c), except the leaf summaries,
// which run as a sum-normalised linear-space SIMT GEMM (each row is a forward sweep) and
// fall back to the exact log-space product for any chunk where flush-to-zero could drop a
// significant term (a finite re-centred tile entry below 2^-40 or a normalised value in
// (0, 2^-80)).
#include <atomic>

#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

namespace {
constexpr int kScanThreads = 256;
constexpr float kTinyX = -40.f;                     // re-centred tile entry (log2) bound
constexpr float kTinyP = 8.271806125530277e-25f;    // 2^-80

}  // namespace

// offset (in nodes) of level l inside one sequence's tree: Σ_{l'<l} Ppad >> l'
__host__ __device__ inline int64_t level_off(int l, int64_t Ppad) {
  int64_t o = 0;
  for (int q = 0; q < l; ++q) o += Ppad >> q;
  return o;
}

// ====================================================================================
// Leaf summaries: fast linear-space SIMT GEMM path.  RB = register block (CP = 16*RB >= C).
// ====================================================================================
template <int RB>
__global__ void __launch_bounds__(kScanThreads) summary_fast_kernel(ScanArgs a) {
  constexpr int CP = 16 * RB;
  constexpr int AS = CP + 1;  // AT row stride (floats)
  extern __shared__ __align__(16) float sm[];
  const int C = (int)a.C, CC = C * C;
  const int64_t N = a.N, E = N - 1, P = a.P, Ppad = a.Ppad, L = a.L;
  const int64_t b = blockIdx.x / Ppad, k = blockIdx.x - (blockIdx.x / Ppad) * Ppad;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int ty = tid >> 4, tx = tid & 15;
  float* AT = sm;                      // [CP][AS] normalised row vectors, transposed
  float* EXs = AT + CP * AS;           // [CP][CP] exps of the current tile (zero padding)
  float* raw = EXs + CP * CP;          // [C*C] staged tile (dense)
  double* Off = reinterpret_cast<double*>(raw + ((CC + 3) & ~3));  // [CP]
  float* red = reinterpret_cast<float*>(Off + CP);                 // [8]
  unsigned* sflag = reinterpret_cast<unsigned*>(red + 8);          // [2]

  const int64_t node = b * a.nodes + k;  // level-0 node
  const int64_t len = seq_len(a.lengths, b, N);
  const int64_t Eb = len < 0 ? 0 : len - 1;
  const int64_t t0 = k * L;
  const int64_t t1 = (t0 + L < Eb) ? t0 + L : Eb;
  const bool empty = (k >= P) || (t0 >= Eb) || len < 0;
  if (empty) {
    if (tid == 0) {
      a.ident[node] = 1;
      a.cflag[b * Ppad + k] = 0;
    }
    return;
  }
  const float* potb = a.pot + b * E * (int64_t)CC;
  const bool v4 = ((CC & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.pot) & 15) == 0);
  auto stage = [&](int64_t t) {
    const float* src = potb + t * CC;
    if (v4) {
      for (int q = tid; q < (CC >> 2); q += kScanThreads) cp_async16(raw + 4 * q, src + 4 * q);
    } else {
      for (int q = tid; q < CC; q += kScanThreads) cp_async4(raw + q, src + q);
    }
    cp_async_commit();
  };
  stage(t0);
  // identity start: row r is the one-hot vector e_r
  for (int q = tid; q < CP * AS; q += kScanThreads) {
    const int i = q / AS, r = q - (q / AS) * AS;
    AT[q] = (i == r && r < C) ? 1.f : 0.f;
  }
  for (int q = tid; q < CP * CP; q += kScanThreads) EXs[q] = 0.f;
  for (int q = tid; q < CP; q += kScanThreads) Off[q] = 0.0;
  if (tid == 0) sflag[0] = sflag[1] = 0u;

  float ah[RB][RB];
#pragma unroll
  for (int x = 0; x < RB; ++x)
#pragma unroll
    for (int y = 0; y < RB; ++y) ah[x][y] = neg_inf();

  for (int64_t t = t0; t < t1; ++t) {
    cp_async_wait<0>();
    __syncthreads();
    // ---- tile max (re-centring) and NaN / +inf probe --------------------------------
    float mx = neg_inf();
    bool bad = false;
    for (int q = tid; q < CC; q += kScanThreads) {
      const float v = raw[q];
      mx = fmaxf(mx, v);
      bad |= (v != v) | (v == pos_inf());
    }
    mx = warp_max(mx);
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&sflag[0], 1u);
    if (lane == 0) red[w] = mx;
    __syncthreads();
    float T = red[0];
#pragma unroll
    for (int q = 1; q < kScanThreads / 32; ++q) T = fmaxf(T, red[q]);
    const float Tz = (T == neg_inf()) ? 0.f : T;
    bool tiny = false;
    for (int q = tid; q < CC; q += kScanThreads) {
      const int i = q / C, j = q - (q / C) * C;
      const float x = (raw[q] - Tz) * kLog2e;
      tiny |= (x < kTinyX) & (x != neg_inf());
      EXs[i * CP + j] = ex2(x);
    }
    if (__any_sync(0xffffffffu, tiny) && lane == 0) atomicOr(&sflag[1], 1u);
    __syncthreads();  // EXs ready, raw free
    if (t + 1 < t1) stage(t + 1);
    // ---- s = A . EX  (A rows = normalised forward vectors) ------------------------------
    float acc[RB][RB];
#pragma unroll
    for (int x = 0; x < RB; ++x)
#pragma unroll
      for (int y = 0; y < RB; ++y) acc[x][y] = 0.f;
    for (int i = 0; i < C; ++i) {
      float av[RB], ev[RB];
#pragma unroll
      for (int x = 0; x < RB; ++x) av[x] = AT[i * AS + ty + 16 * x];
#pragma unroll
      for (int y = 0; y < RB; ++y) ev[y] = EXs[i * CP + tx + 16 * y];
#pragma unroll
      for (int x = 0; x < RB; ++x)
#pragma unroll
        for (int y = 0; y < RB; ++y) acc[x][y] = fmaf(av[x], ev[y], acc[x][y]);
    }
    // ---- row sums (over the 16 tx lanes of this half-warp), normalise ---------------------
    float lS[RB];
    bool tinyp = false;
#pragma unroll
    for (int x = 0; x < RB; ++x) {
      float s = 0.f;
#pragma unroll
      for (int y = 0; y < RB; ++y) s += acc[x][y];
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      const float inv = (s > 0.f) ? 1.f / s : 0.f;
      lS[x] = (s > 0.f) ? lg2(s) : neg_inf();
#pragma unroll
      for (int y = 0; y < RB; ++y) {
        const float pv = acc[x][y] * inv;
        tinyp |= (pv > 0.f) & (pv < kTinyP);
        ah[x][y] = (s > 0.f) ? lg2(acc[x][y]) - lS[x] : neg_inf();
        acc[x][y] = pv;
      }
    }
    if (__any_sync(0xffffffffu, tinyp) && lane == 0) atomicOr(&sflag[1], 1u);
    __syncthreads();  // all reads of AT / EXs done
#pragma unroll
    for (int x = 0; x < RB; ++x) {
      const int r = ty + 16 * x;
#pragma unroll
      for (int y = 0; y < RB; ++y) {
        const int j = tx + 16 * y;
        AT[j * AS + r] = (r < C && j < C) ? acc[x][y] : 0.f;
      }
      if (tx == 0 && r < C) {
        const double o = Off[r];
        Off[r] = (lS[x] == neg_inf() || o == -INFINITY) ? -INFINITY
                                                         : o + (double)Tz + kLn2 * (double)lS[x];
      }
    }
  }
  __syncthreads();
  // ---- write the leaf LogMat --------------------------------------------------------------
  float* S = a.mat + node * (int64_t)CC;
  double* O = a.off + node * (int64_t)C;
#pragma unroll
  for (int x = 0; x < RB; ++x) {
    const int r = ty + 16 * x;
    if (r >= C) continue;
    const bool dead = (Off[r] == -INFINITY);
#pragma unroll
    for (int y = 0; y < RB; ++y) {
      const int j = tx + 16 * y;
      if (j < C) S[r * C + j] = dead ? neg_inf() : ah[x][y];
    }
  }
  for (int r = tid; r < C; r += kScanThreads) O[r] = (Off[r] == -INFINITY) ? 0.0 : Off[r];
  if (tid == 0) {
    a.ident[node] = 0;
    a.cflag[b * Ppad + k] = sflag[1];
    if (sflag[0] && a.wflags) atomicOr(&a.wflags[b], (unsigned)WF_NONFINITE);
  }
}

// ====================================================================================
// Exact log-space leaf summary for flagged chunks (the §6(c) per-cell max), one CTA per
// flagged chunk; other CTAs exit immediately.
// ====================================================================================
__global__ void __launch_bounds__(kScanThreads) summary_exact_kernel(ScanArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int C = (int)a.C, CC = C * C;
  const int64_t N = a.N, E = N - 1, Ppad = a.Ppad, L = a.L;
  const int64_t b = blockIdx.x / Ppad, k = blockIdx.x - (blockIdx.x / Ppad) * Ppad;
  if (!a.cflag[b * Ppad + k]) return;
  const int tid = threadIdx.x;
  const int CC4 = (CC + 3) & ~3;
  float* A = sm;          // [C][C] current log rows (relative to row offsets)
  float* X = A + CC4;     // [C][C] re-centred tile (log2)
  float* R = X + CC4;     // [C][C] next rows
  double* Off = reinterpret_cast<double*>(R + CC4);  // [C]
  float* red = reinterpret_cast<float*>(Off + C);                 // [8]
  const int64_t node = b * a.nodes + k;
  const int64_t len = seq_len(a.lengths, b, N);
  const int64_t Eb = len < 0 ? 0 : len - 1;
  const int64_t t0 = k * L;
  const int64_t t1 = (t0 + L < Eb) ? t0 + L : Eb;
  const float* potb = a.pot + b * E * (int64_t)CC;
  for (int q = tid; q < CC; q += kScanThreads) A[q] = ((q / C) == (q % C)) ? 0.f : neg_inf();
  for (int q = tid; q < C; q += kScanThreads) Off[q] = 0.0;
  __syncthreads();
  for (int64_t t = t0; t < t1; ++t) {
    const float* src = potb + t * CC;
    float mx = neg_inf();
    for (int q = tid; q < CC; q += kScanThreads) mx = fmaxf(mx, src[q]);
    mx = warp_max(mx);
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    __syncthreads();
    float T = red[0];
    for (int q = 1; q < kScanThreads / 32; ++q) T = fmaxf(T, red[q]);
    const float Tz = (T == neg_inf()) ? 0.f : T;
    for (int q = tid; q < CC; q += kScanThreads) X[q] = (src[q] - Tz) * kLog2e;
    __syncthreads();
    for (int q = tid; q < CC; q += kScanThreads) {
      const int r = q / C, j = q - (q / C) * C;
      float m = neg_inf();
      for (int i = 0; i < C; ++i) m = fmaxf(m, A[r * C + i] + X[i * C + j]);
      float s = 0.f;
      if (m != neg_inf())
        for (int i = 0; i < C; ++i) s += ex2(A[r * C + i] + X[i * C + j] - m);
      R[q] = (m == neg_inf()) ? neg_inf() : m + lg2(s);
    }
    __syncthreads();
    // row renormalisation: subtract the row max, move it to the row offset
    for (int r = tid; r < C; r += kScanThreads) {
      float m = neg_inf();
      for (int j = 0; j < C; ++j) m = fmaxf(m, R[r * C + j]);
      const bool dead = (m == neg_inf()) || Off[r] == -INFINITY;
      for (int j = 0; j < C; ++j) A[r * C + j] = dead ? neg_inf() : R[r * C + j] - m;
      Off[r] = dead ? -INFINITY : Off[r] + (double)Tz + kLn2 * (double)m;
    }
    __syncthreads();
  }
  float* S = a.mat + node * (int64_t)CC;
  double* O = a.off + node * (int64_t)C;
  for (int q = tid; q < CC; q += kScanThreads) S[q] = A[q];
  for (int r = tid; r < C; r += kScanThreads) O[r] = (Off[r] == -INFINITY) ? 0.0 : Off[r];
}

// ====================================================================================
// Up-sweep: node(l,k) = node(l-1,2k) (x) node(l-1,2k+1)  (exact per-cell max, §6(c))
// ====================================================================================
__global__ void __launch_bounds__(kScanThreads) tree_up_kernel(ScanArgs a, int l) {
  extern __shared__ __align__(16) float sm[];
  const int C = (int)a.C, CC = C * C;
  const int64_t Ppad = a.Ppad;
  const int64_t nl = Ppad >> l;
  const int64_t b = blockIdx.x / nl, k = blockIdx.x - (blockIdx.x / nl) * nl;
  const int tid = threadIdx.x;
  const int64_t nd = b * a.nodes + level_off(l, Ppad) + k;
  const int64_t n1 = b * a.nodes + level_off(l - 1, Ppad) + 2 * k, n2 = n1 + 1;
  const bool i1 = a.ident[n1], i2 = a.ident[n2];
  float* Sd = a.mat + nd * CC;
  double* Od = a.off + nd * C;
  if (i1 && i2) {
    if (tid == 0) a.ident[nd] = 1;
    return;
  }
  if (i1 || i2) {  // product with the identity I (P:338 padding): copy
    const int64_t ns = i1 ? n2 : n1;
    for (int q = tid; q < CC; q += kScanThreads) Sd[q] = a.mat[ns * CC + q];
    for (int q = tid; q < C; q += kScanThreads) Od[q] = a.off[ns * C + q];
    if (tid == 0) a.ident[nd] = 0;
    return;
  }
  // Linear-space product (§6(c) exp-shifted form): with W[r][i] = (ln2 S1[r][i] + O2[i] -
  // ref_r) log2 e <= 0 (ref_r = row max) and S2[i][j] <= 0,
  //   R[r][j] = log2 Σ_i 2^W[r][i] 2^S2[i][j]
  // is a real 128 x 128 x C GEMM of values in [0, 1] (8 x 8 register tile per thread).  A cell
  // whose sum falls below 2^-60 may have lost significant terms to flush-to-zero and is
  // recomputed exactly with the per-cell max from the global operands (the gate of §4).
  constexpr int CP = 128;
  float* wT = sm;            // [CP][CP] wT[i][r] = 2^W[r][i]
  float* e2 = wT + CP * CP;  // [CP][CP] e2[i][j] = 2^S2[i][j]
  float* R = e2 + CP * CP;   // [C][C] log2 results; first the staged S1 rows (stride CP+1)
  double* ref = reinterpret_cast<double*>(R + CP * (CP + 1));  // [CP] row maxima
  double* O2s = ref + CP;                                      // [CP] staged O2
  const float* S1g = a.mat + n1 * CC;
  const double* O1 = a.off + n1 * C;
  const float* S2g = a.mat + n2 * CC;
  const double* O2 = a.off + n2 * C;
  // stage S1 (coalesced global reads; padded stride -> conflict-free column reads) and O2
  for (int q = tid; q < CC; q += kScanThreads) {
    const int r = q / C, i = q - (q / C) * C;
    R[r * (CP + 1) + i] = S1g[q];
  }
  for (int i = tid; i < C; i += kScanThreads) O2s[i] = O2[i];
  for (int q = tid; q < CP * CP; q += kScanThreads) {
    const int i = q >> 7, j = q & (CP - 1);
    e2[q] = (i < C && j < C) ? ex2(S2g[i * C + j]) : 0.f;
  }
  __syncthreads();
  {  // row maxima ref_r = max_i (ln2 S1[r][i] + O2[i]): one warp per row, lanes over i
    const int lane = tid & 31, w = tid >> 5;
    for (int r = w; r < C; r += kScanThreads / 32) {
      double m = -INFINITY;
      for (int i = lane; i < C; i += 32) {
        const float s1 = R[r * (CP + 1) + i];
        if (s1 != neg_inf()) {
          const double c = kLn2 * (double)s1 + O2s[i];
          m = c > m ? c : m;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double x = __shfl_xor_sync(0xffffffffu, m, o);
        m = x > m ? x : m;
      }
      if (lane == 0) ref[r] = m;
    }
  }
  __syncthreads();
  // wT[i][r] = 2^((ln2 S1[r][i] + O2[i] - ref_r) log2 e), flat over (i, r): coalesced stores
  for (int q = tid; q < CP * CP; q += kScanThreads) {
    const int i = q >> 7, r = q & (CP - 1);
    float v = 0.f;
    if (i < C && r < C) {
      const float s1 = R[r * (CP + 1) + i];
      const double m = ref[r];
      if (s1 != neg_inf() && m != -INFINITY)
        v = ex2((float)((kLn2 * (double)s1 + O2s[i] - m) * (double)kLog2e));
    }
    wT[q] = v;
  }
  __syncthreads();
  {
    const int ty = tid >> 4, tx = tid & 15, r0 = 8 * ty, j0 = 8 * tx;
    float acc[8][8];
#pragma unroll
    for (int x = 0; x < 8; ++x)
#pragma unroll
      for (int y = 0; y < 8; ++y) acc[x][y] = 0.f;
    if (r0 < C && j0 < C) {
      for (int i = 0; i < C; ++i) {
        const float4 a0 = *reinterpret_cast<const float4*>(wT + i * CP + r0);
        const float4 a1 = *reinterpret_cast<const float4*>(wT + i * CP + r0 + 4);
        const float4 b0 = *reinterpret_cast<const float4*>(e2 + i * CP + j0);
        const float4 b1 = *reinterpret_cast<const float4*>(e2 + i * CP + j0 + 4);
        const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int x = 0; x < 8; ++x)
#pragma unroll
          for (int y = 0; y < 8; ++y) acc[x][y] = fmaf(av[x], bv[y], acc[x][y]);
      }
    }
#pragma unroll
    for (int x = 0; x < 8; ++x) {
      const int r = r0 + x;
#pragma unroll
      for (int y = 0; y < 8; ++y) {
        const int j = j0 + y;
        if (r < C && j < C) {
          float v;
          if (acc[x][y] >= kGate) {
            v = lg2(acc[x][y]);
          } else {  // exact per-cell max (§6(c)) from the global operands
            const double rr = ref[r];
            float m = neg_inf();
            for (int i = 0; i < C; ++i) {
              const float s1 = S1g[r * C + i];
              const float w = (s1 == neg_inf() || rr == -INFINITY)
                                  ? neg_inf()
                                  : (float)((kLn2 * (double)s1 + O2[i] - rr) * (double)kLog2e);
              m = fmaxf(m, w + S2g[i * C + j]);
            }
            float sum = 0.f;
            if (m != neg_inf())
              for (int i = 0; i < C; ++i) {
                const float s1 = S1g[r * C + i];
                const float w = (s1 == neg_inf() || rr == -INFINITY)
                                    ? neg_inf()
                                    : (float)((kLn2 * (double)s1 + O2[i] - rr) * (double)kLog2e);
                sum += ex2(w + S2g[i * C + j] - m);
              }
            v = (m == neg_inf()) ? neg_inf() : m + lg2(sum);
          }
          R[r * C + j] = v;
        }
      }
    }
  }
  __syncthreads();
  // row normalisation: one warp per row, lanes over j (conflict-free SMEM, coalesced stores)
  {
    const int lane = tid & 31, w = tid >> 5;
    for (int r = w; r < C; r += kScanThreads / 32) {
      float m = neg_inf();
      for (int j = lane; j < C; j += 32) m = fmaxf(m, R[r * C + j]);
      m = warp_max(m);
      const bool dead = (m == neg_inf()) || ref[r] == -INFINITY;
      for (int j = lane; j < C; j += 32) Sd[r * C + j] = dead ? neg_inf() : R[r * C + j] - m;
      if (lane == 0) Od[r] = dead ? 0.0 : O1[r] + ref[r] + kLn2 * (double)m;
    }
  }
  if (tid == 0) a.ident[nd] = 0;
}

// ====================================================================================
// Down-sweep: from level l to its children.  alpha: left = parent, right = parent (x) left;
// beta: right = parent, left = right (x) parent.  Vectors are LogVec (C floats + offset).
// ====================================================================================
namespace {
// u_j = LSE_i(v_i + S[i][j]) with S a LogMat; returns normalised u (max 0) and offset.
__device__ void vec_mat(const float* v, double vo, const float* S, const double* So, int C,
                        float* out, double* out_off, float* scratch, int tid) {
  // scratch: [C] w values, [C] u values, [2*8] reductions
  float* w = scratch;
  float* u = scratch + ((C + 3) & ~3);
  double* dref = reinterpret_cast<double*>(u + ((C + 3) & ~3));
  if (tid == 0) {
    double m = -INFINITY;
    for (int i = 0; i < C; ++i)
      if (v[i] != neg_inf()) {
        const double c = kLn2 * (double)v[i] + So[i];
        m = c > m ? c : m;
      }
    dref[0] = m;
  }
  __syncthreads();
  const double ref = dref[0];
  for (int i = tid; i < C; i += kScanThreads)
    w[i] = (v[i] == neg_inf() || ref == -INFINITY)
               ? neg_inf()
               : (float)((kLn2 * (double)v[i] + So[i] - ref) * (double)kLog2e);
  __syncthreads();
  for (int j = tid; j < C; j += kScanThreads) {
    float m = neg_inf();
    for (int i = 0; i < C; ++i) m = fmaxf(m, w[i] + S[i * C + j]);
    float s = 0.f;
    if (m != neg_inf())
      for (int i = 0; i < C; ++i) s += ex2(w[i] + S[i * C + j] - m);
    u[j] = (m == neg_inf()) ? neg_inf() : m + lg2(s);
  }
  __syncthreads();
  if (tid == 0) {
    float m = neg_inf();
    for (int j = 0; j < C; ++j) m = fmaxf(m, u[j]);
    dref[1] = (m == neg_inf()) ? 0.0 : (double)m;
    *out_off = (ref == -INFINITY || m == neg_inf()) ? 0.0 : vo + ref + kLn2 * (double)m;
  }
  __syncthreads();
  const float m = (float)dref[1];
  for (int j = tid; j < C; j += kScanThreads) out[j] = u[j] - m;
  __syncthreads();
}

// u_r = LSE_j(S[r][j] + v_j): returns normalised u and offset.
__device__ void mat_vec(const float* S, const double* So, const float* v, double vo, int C,
                        float* out, double* out_off, float* scratch, int tid) {
  double* tot = reinterpret_cast<double*>(scratch);  // [C]
  double* dref = tot + C;
  {  // one warp per row, lanes over j (conflict-free SMEM row reads)
    const int lane = tid & 31, w = tid >> 5;
    for (int r = w; r < C; r += kScanThreads / 32) {
      float m = neg_inf();
      for (int j = lane; j < C; j += 32) m = fmaxf(m, S[r * C + j] + v[j]);
      m = warp_max(m);
      float s = 0.f;
      if (m != neg_inf())
        for (int j = lane; j < C; j += 32) s += ex2(S[r * C + j] + v[j] - m);
      s = warp_sum(s);
      if (lane == 0) tot[r] = (m == neg_inf()) ? -INFINITY : So[r] + vo + kLn2 * (double)(m + lg2(s));
    }
  }
  __syncthreads();
  if (tid == 0) {
    double m = -INFINITY;
    for (int r = 0; r < C; ++r) m = tot[r] > m ? tot[r] : m;
    dref[0] = m;
    *out_off = (m == -INFINITY) ? 0.0 : m;
  }
  __syncthreads();
  const double ref = dref[0];
  for (int r = tid; r < C; r += kScanThreads)
    out[r] = (tot[r] == -INFINITY || ref == -INFINITY)
                 ? neg_inf()
                 : (float)((tot[r] - ref) * (double)kLog2e);
  __syncthreads();
}
}  // namespace

__global__ void __launch_bounds__(kScanThreads) tree_down_kernel(ScanArgs a, int l) {
  extern __shared__ __align__(16) float sm[];
  const int C = (int)a.C, CC = C * C;
  const int64_t Ppad = a.Ppad;
  const int64_t nl = Ppad >> l;
  const int64_t b = blockIdx.x / nl, k = blockIdx.x - (blockIdx.x / nl) * nl;
  const int tid = threadIdx.x;
  const int64_t base = b * a.nodes;
  const int64_t np = base + level_off(l, Ppad) + k;
  const int64_t nlft = base + level_off(l - 1, Ppad) + 2 * k, nrgt = nlft + 1;
  float* S = sm;                       // [C][C] staged matrix
  float* scratch = S + ((CC + 3) & ~3);  // 16-byte aligned
  const float* av = a.valpha + np * C;
  const double ao = a.oalpha[np];
  const float* bv = a.vbeta + np * C;
  const double bo = a.obeta[np];
  // alpha: left child = parent
  for (int j = tid; j < C; j += kScanThreads) {
    a.valpha[nlft * C + j] = av[j];
    a.vbeta[nrgt * C + j] = bv[j];
  }
  if (tid == 0) {
    a.oalpha[nlft] = ao;
    a.obeta[nrgt] = bo;
  }
  // alpha: right child = parent (x) left
  if (a.ident[nlft]) {
    for (int j = tid; j < C; j += kScanThreads) a.valpha[nrgt * C + j] = av[j];
    if (tid == 0) a.oalpha[nrgt] = ao;
  } else {
    for (int q = tid; q < CC; q += kScanThreads) S[q] = a.mat[nlft * CC + q];
    __syncthreads();
    vec_mat(av, ao, S, a.off + nlft * C, C, a.valpha + nrgt * C, a.oalpha + nrgt, scratch, tid);
  }
  __syncthreads();
  // beta: left child = right (x) parent
  if (a.ident[nrgt]) {
    for (int j = tid; j < C; j += kScanThreads) a.vbeta[nlft * C + j] = bv[j];
    if (tid == 0) a.obeta[nlft] = bo;
  } else {
    for (int q = tid; q < CC; q += kScanThreads) S[q] = a.mat[nrgt * CC + q];
    __syncthreads();
    mat_vec(S, a.off + nrgt * C, bv, bo, C, a.vbeta + nlft * C, a.obeta + nlft, scratch, tid);
  }
}

// Root vectors: log-one (0) start / end vectors.
__global__ void tree_root_kernel(ScanArgs a) {
  const int C = (int)a.C;
  const int64_t b = blockIdx.x;
  const int64_t np = b * a.nodes + level_off(a.H, a.Ppad);
  for (int j = threadIdx.x; j < C; j += blockDim.x) {
    a.valpha[np * C + j] = 0.f;
    a.vbeta[np * C + j] = 0.f;
  }
  if (threadIdx.x == 0) {
    a.oalpha[np] = 0.0;
    a.obeta[np] = 0.0;
  }
}

// logZ from the root: A = LSE_{r,j} (off[r] + ln2 s[r][j])  (start and end vectors log-one).
__global__ void __launch_bounds__(kScanThreads) tree_logz_kernel(ScanArgs a) {
  __shared__ double red[kScanThreads / 32];
  const int C = (int)a.C;
  const int64_t b = blockIdx.x;
  const int64_t N = a.N;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t len = seq_len(a.lengths, b, N);
  const uint32_t wf = a.wflags ? a.wflags[b] : 0u;
  if (len < 0 || (wf & WF_NONFINITE)) {
    if (tid == 0) {
      a.logz[b] = qnan();
      if (a.flags) a.flags[b] = (len < 0) ? TS_F_BADLEN : TS_F_NONFINITE;
    }
    return;
  }
  const int64_t nr = b * a.nodes + level_off(a.H, a.Ppad);
  if (a.ident[nr]) {
    if (tid == 0) {
      a.logz[b] = (float)log((double)C);
      if (a.flags) a.flags[b] = 0u;
    }
    return;
  }
  const float* S = a.mat + nr * (int64_t)C * C;
  const double* O = a.off + nr * C;
  double m = -INFINITY;
  for (int q = tid; q < C * C; q += kScanThreads) {
    const float s = S[q];
    if (s != neg_inf()) {
      const double v = O[q / C] + kLn2 * (double)s;
      m = v > m ? v : m;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double x = __shfl_xor_sync(0xffffffffu, m, o);
    m = x > m ? x : m;
  }
  if (lane == 0) red[w] = m;
  __syncthreads();
  m = red[0];
  for (int q = 1; q < kScanThreads / 32; ++q) m = red[q] > m ? red[q] : m;
  __syncthreads();
  double sum = 0.0;
  if (m != -INFINITY)
    for (int q = tid; q < C * C; q += kScanThreads) {
      const float s = S[q];
      if (s != neg_inf()) sum += exp(O[q / C] + kLn2 * (double)s - m);
    }
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) red[w] = sum;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int q = 0; q < kScanThreads / 32; ++q) t += red[q];
    const double lz = (m == -INFINITY) ? -INFINITY : m + log(t);
    a.logz[b] = (float)lz;
    if (a.flags) a.flags[b] = (lz == -INFINITY) ? TS_F_EMPTY : 0u;
  }
}

// Copy the leaf vectors (level 0, k < P) into the [B][P] arrays the leaf sweeps read.
__global__ void tree_leaves_kernel(ScanArgs a) {
  const int C = (int)a.C;
  const int64_t b = blockIdx.x / a.P, k = blockIdx.x - (blockIdx.x / a.P) * a.P;
  const int64_t n0 = b * a.nodes + k;
  const int64_t d = b * a.P + k;
  for (int j = threadIdx.x; j < C; j += blockDim.x) {
    a.leaf_alpha[d * C + j] = a.valpha[n0 * C + j];
    a.leaf_beta[d * C + j] = a.vbeta[n0 * C + j];
  }
  if (threadIdx.x == 0) {
    a.leaf_alpha_off[d] = a.oalpha[n0];
    a.leaf_beta_off[d] = a.obeta[n0];
  }
}

// ====================================================================================
// Time sharding: export the local root as this segment's summary; combine
// all gathered segment summaries into the local root vectors and the global logZ.
// Summary layout: [B][C][C] fp32 log2 values, then [B][C] fp64 natural row offsets, each
// section padded to 16 bytes (seg_mat_floats / seg_total_floats, kernels.cuh).
// ====================================================================================
__global__ void __launch_bounds__(kScanThreads) segment_export_kernel(ScanArgs a, float* summ) {
  const int C = (int)a.C, CC = C * C;
  const int64_t b = blockIdx.x;
  const int64_t nr = b * a.nodes + level_off(a.H, a.Ppad);
  float* S = summ + b * CC;
  double* O = reinterpret_cast<double*>(summ + seg_mat_floats(a.B, C)) + b * C;
  const bool id = a.ident[nr];
  // a NaN / +inf anywhere in this segment poisons its summary so every rank sees it
  const bool bad = a.wflags && (a.wflags[b] & WF_NONFINITE);
  for (int q = threadIdx.x; q < CC; q += kScanThreads)
    S[q] = bad ? qnan() : id ? (((q / C) == (q % C)) ? 0.f : neg_inf()) : a.mat[nr * CC + q];
  for (int r = threadIdx.x; r < C; r += kScanThreads) O[r] = id ? 0.0 : a.off[nr * C + r];
}

__global__ void __launch_bounds__(kScanThreads) segment_combine_kernel(ScanArgs a,
                                                                       const float* all_summ,
                                                                       int rank, int world,
                                                                       int write_root) {
  extern __shared__ __align__(16) float sm[];
  const int C = (int)a.C, CC = C * C;
  const int64_t B = a.B, b = blockIdx.x;
  const int tid = threadIdx.x;
  const int CC4 = (CC + 3) & ~3, C4 = (C + 3) & ~3;
  float* S = sm;               // staged summary
  float* va = S + CC4;         // running vector
  float* vb = va + C4;         // output vector
  float* scratch = vb + C4;
  double* vo = reinterpret_cast<double*>(scratch + 4 * C4 + 32);  // [2]
  const size_t seg_floats = (size_t)seg_total_floats(B, C);  // one rank's slice
  const size_t mat_floats = (size_t)seg_mat_floats(B, C);
  auto segS = [&](int g) { return all_summ + (size_t)g * seg_floats + b * CC; };
  auto segO = [&](int g) {
    return reinterpret_cast<const double*>(all_summ + (size_t)g * seg_floats + mat_floats) + b * C;
  };
  const int64_t nr = b * a.nodes + level_off(a.H, a.Ppad);
  // a poisoned (NaN) summary anywhere -> NONFINITE on every rank, local sweeps zeroed
  int nan = 0;
  for (int g = 0; g < world; ++g)
    for (int q = tid; q < CC; q += kScanThreads) nan |= (segS(g)[q] != segS(g)[q]);
  if (__syncthreads_or(nan)) {
    if (tid == 0) {
      a.logz[b] = qnan();
      if (a.flags) a.flags[b] = TS_F_NONFINITE;
    }
    if (write_root) {
      for (int j = tid; j < C; j += kScanThreads) {
        a.valpha[nr * C + j] = qnan();
        a.vbeta[nr * C + j] = qnan();
      }
      if (tid == 0) {
        a.oalpha[nr] = 0.0;
        a.obeta[nr] = 0.0;
      }
    }
    return;
  }
  // ---- alpha_in(rank) = 0 (x) S_0 (x) ... (x) S_{rank-1}; then the full chain for logZ ----
  for (int j = tid; j < C; j += kScanThreads) va[j] = 0.f;
  if (tid == 0) vo[0] = 0.0;
  __syncthreads();
  for (int g = 0; g < world; ++g) {
    if (g == rank && write_root) {
      for (int j = tid; j < C; j += kScanThreads) a.valpha[nr * C + j] = va[j];
      if (tid == 0) a.oalpha[nr] = vo[0];
    }
    for (int q = tid; q < CC; q += kScanThreads) S[q] = segS(g)[q];
    __syncthreads();
    vec_mat(va, vo[0], S, segO(g), C, vb, &vo[1], scratch, tid);
    for (int j = tid; j < C; j += kScanThreads) va[j] = vb[j];
    if (tid == 0) vo[0] = vo[1];
    __syncthreads();
  }
  // logZ = LSE_j(alpha_E[j]) in the same order on every rank (bit-identical across ranks)
  if (tid == 0) {
    float m = neg_inf();
    bool nan = false;
    for (int j = 0; j < C; ++j) {
      m = fmaxf(m, va[j]);
      nan |= (va[j] != va[j]);
    }
    double lz;
    if (nan || vo[0] != vo[0]) {
      lz = NAN;
    } else if (m == neg_inf()) {
      lz = -INFINITY;
    } else {
      double ssum = 0.0;
      for (int j = 0; j < C; ++j) ssum += exp(kLn2 * (double)(va[j] - m));
      lz = vo[0] + kLn2 * (double)m + log(ssum);
    }
    a.logz[b] = (float)lz;
    if (a.flags) a.flags[b] = (lz != lz) ? TS_F_NONFINITE : (lz == -INFINITY ? TS_F_EMPTY : 0u);
  }
  if (!write_root) return;
  // ---- beta_out(rank) = S_{rank+1} (x) ... (x) S_{world-1} (x) 0 ------------------------------
  __syncthreads();
  for (int j = tid; j < C; j += kScanThreads) va[j] = 0.f;
  if (tid == 0) vo[0] = 0.0;
  __syncthreads();
  for (int g = world - 1; g > rank; --g) {
    for (int q = tid; q < CC; q += kScanThreads) S[q] = segS(g)[q];
    __syncthreads();
    mat_vec(S, segO(g), va, vo[0], C, vb, &vo[1], scratch, tid);
    for (int j = tid; j < C; j += kScanThreads) va[j] = vb[j];
    if (tid == 0) vo[0] = vo[1];
    __syncthreads();
  }
  for (int j = tid; j < C; j += kScanThreads) a.vbeta[nr * C + j] = va[j];
  if (tid == 0) a.obeta[nr] = vo[0];
}

// ====================================================================================
// host side
// ====================================================================================
namespace {
std::atomic<uint64_t> g_attr_scan[64];  // one per-device mask per kernel (`bit` = kernel id)
template <typename K>
cudaError_t set_smem(K kern, int bit) {
  return smem_optin_once(kern, g_attr_scan[bit], 225 * 1024);
}
template <int RB>
size_t fast_smem(int C) {
  constexpr int CP = 16 * RB;
  return (size_t)(CP * (CP + 1) + CP * CP + ((C * C + 3) & ~3)) * 4 + CP * 8 + 64;
}
template <int RB>
cudaError_t launch_fast(const ScanArgs& a, cudaStream_t st) {
  cudaError_t e = set_smem(summary_fast_kernel<RB>, RB);
  if (e != cudaSuccess) return e;
  summary_fast_kernel<RB><<<(unsigned)(a.B * a.Ppad), kScanThreads, fast_smem<RB>((int)a.C), st>>>(a);
  return cudaGetLastError();
}
}  // namespace

size_t scan_mat_smem(int64_t C) {  // tree_up: 2 [128][128] + 1 [128][129] fp32 buffers, 2x128 fp64
  (void)C;
  return (size_t)(2 * 128 * 128 + 128 * 129) * 4 + (size_t)2 * 128 * 8 + 64;
}

cudaError_t launch_scan_up(const ScanArgs& a, cudaStream_t st, int* launches) {
  const int C = (int)a.C;
  cudaError_t e;
  int n = 0;
  if (summary_tc_ok(a)) {
    e = launch_summary_tc(a, st);
  } else switch ((C + 15) / 16) {
    case 1: e = launch_fast<1>(a, st); break;
    case 2: e = launch_fast<2>(a, st); break;
    case 3: e = launch_fast<3>(a, st); break;
    case 4: e = launch_fast<4>(a, st); break;
    case 5: e = launch_fast<5>(a, st); break;
    case 6: e = launch_fast<6>(a, st); break;
    case 7: e = launch_fast<7>(a, st); break;
    case 8: e = launch_fast<8>(a, st); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  ++n;
  const size_t msm = scan_mat_smem(C);
  if ((e = set_smem(summary_exact_kernel, 9)) != cudaSuccess) return e;
  summary_exact_kernel<<<(unsigned)(a.B * a.Ppad), kScanThreads, msm, st>>>(a);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  ++n;
  if ((e = set_smem(tree_up_kernel, 10)) != cudaSuccess) return e;
  for (int l = 1; l <= a.H; ++l) {
    tree_up_kernel<<<(unsigned)(a.B * (a.Ppad >> l)), kScanThreads, msm, st>>>(a, l);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++n;
  }
  if (launches) *launches += n;
  return cudaSuccess;
}

cudaError_t launch_scan_down(const ScanArgs& a, cudaStream_t st, int* launches, bool set_root) {
  cudaError_t e;
  int n = 0;
  if (set_root) {
    tree_root_kernel<<<(unsigned)a.B, 128, 0, st>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++n;
  }
  const size_t dsm = (size_t)(((a.C * a.C + 3) & ~3) + 4 * a.C + 32) * 4 + (size_t)(a.C + 8) * 8;
  if ((e = set_smem(tree_down_kernel, 11)) != cudaSuccess) return e;
  for (int l = a.H; l >= 1; --l) {
    tree_down_kernel<<<(unsigned)(a.B * (a.Ppad >> l)), kScanThreads, dsm, st>>>(a, l);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    ++n;
  }
  tree_leaves_kernel<<<(unsigned)(a.B * a.P), 128, 0, st>>>(a);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  ++n;
  if (launches) *launches += n;
  return cudaSuccess;
}

cudaError_t launch_segment_export(const ScanArgs& a, float* summ, cudaStream_t st) {
  segment_export_kernel<<<(unsigned)a.B, kScanThreads, 0, st>>>(a, summ);
  return cudaGetLastError();
}

cudaError_t launch_segment_combine(const ScanArgs& a, const float* all_summ, int rank, int world,
                                   bool write_root, cudaStream_t st) {
  const int C = (int)a.C;
  const size_t smem = (size_t)(((C * C + 3) & ~3) + 6 * ((C + 3) & ~3) + 64) * 4 + 64;
  cudaError_t e = set_smem(segment_combine_kernel, 12);
  if (e != cudaSuccess) return e;
  segment_combine_kernel<<<(unsigned)a.B, kScanThreads, smem, st>>>(a, all_summ, rank, world,
                                                                    write_root ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_scan_logz(const ScanArgs& a, cudaStream_t st) {
  tree_logz_kernel<<<(unsigned)a.B, kScanThreads, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace tsb
