// semi_expand.cu — the semi-Markov CRF (Table 1 'Semi-Markov') on the scan of §6(a)
// ("Similar parallel approach can also be used for ... semi-Markov") through the
// expanded-state reduction: a labelled segmentation with segments of at most K steps is a
// path of a first-order chain over the S = C K states (r, c) = (label c, r more steps to the
// next segment boundary), state index r C + c (r = 0: a boundary node with label c).
//
// Edge n of the expanded chain (reading R17, l[n][k-1][c][c'] = a segment n -> n + k with
// label c' after label c):
//   (0, c)  -> (k-1, c') : l[n][k-1][c][c']   (a segment of k steps starts at boundary n)
//   (r, c)  -> (r-1, c)  : 0                  (r >= 1: inside a segment)
//   anything else         : -inf
// with the state (r, c) at node u admissible only when u + r <= E_b (segments end inside the
// sequence, so parts ending beyond it get mu = 0) and only boundary states at node 0 (rows
// r >= 1 of edge 0 are -inf).  Every admissible path then ends on a boundary state, the chain's
// final sum over all states is the semi-Markov partition function, and the marginal of the
// expanded entry ((0, c), (k-1, c')) at edge n is the part marginal mu[n][k-1][c][c']
// (P:181-183).  len = 1 has no edges: the chain returns ln(C K) over its start states, the
// semi-Markov value is ln C (fixed up by the gather).  Cost: S^2 = K^2 C^2 per edge instead of
// K C^2 (the banded structure is not exploited), in exchange for every plan of the chain —
// the chunked scan, its tensor-core summaries (S <= 128), the Fig. 4 tree, the time-sharded
// segments — and the max semiring's Viterbi (reading R18's order is the expanded chain's
// first-index order: boundary predecessors (k = 1) come before the continuation state, and
// within a segment length the labels ascend).
#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

// one thread per expanded entry, row-major over [B][E][S][S]
__global__ void semi_expand_kernel(SemiExpandArgs a) {
  const int64_t C = a.C, K = a.K, S = C * K, E = a.N - 1;
  const int64_t total = a.B * E * S * S;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = q % S, i = (q / S) % S, n = (q / (S * S)) % E, b = q / (S * S * E);
    const int64_t len = seq_len(a.lengths, b, a.N);
    const int64_t Eb = len < 1 ? 0 : len - 1;
    const int64_t ri = i / C, ci = i - ri * C, rj = j / C, cj = j - rj * C;
    float v = neg_inf();
    const bool adm = (n + 1 + rj <= Eb);  // the target state (rj, cj) at node n + 1
    if (ri == 0) {
      if (adm) v = a.pot[(((b * E + n) * K + rj) * C + ci) * C + cj];  // segment of rj + 1 steps
    } else if (n > 0 && rj == ri - 1 && cj == ci && adm) {
      v = 0.f;
    }
    a.xpot[q] = v;
  }
}

// mu[b][n][k-1][c][c'] = mu_x[b][n][(0, c)][(k-1, c')]; logz fix-up for len = 1
__global__ void semi_gather_kernel(SemiExpandArgs a) {
  const int64_t C = a.C, K = a.K, S = C * K, E = a.N - 1;
  const int64_t total = a.marg ? a.B * E * K * C * C : 0;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c2 = q % C, c1 = (q / C) % C, k = (q / (C * C)) % K, bn = q / (C * C * K);
    a.marg[q] = a.xmarg[(bn * S + c1) * S + k * C + c2];
  }
  if (blockIdx.x == 0)
    for (int64_t b = threadIdx.x; b < a.B; b += blockDim.x)
      if (seq_len(a.lengths, b, a.N) == 1 && a.logz && a.logz[b] == a.logz[b])
        a.logz[b] = (float)log((double)C);
}

// Semi-Markov Viterbi output from the expanded path: the label at boundary nodes (r = 0),
// -1 at interior nodes and wherever the expanded path is -1
__global__ void semi_seg_kernel(SemiExpandArgs a) {
  const int64_t C = a.C, total = a.B * a.N;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = a.xpath[q];
    a.seg[q] = (s >= 0 && s < C) ? s : -1;
  }
}

namespace {
unsigned grid_for(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return (unsigned)(g < 148 * 16 ? (g < 1 ? 1 : g) : 148 * 16);
}
}  // namespace

cudaError_t launch_semi_expand(const SemiExpandArgs& a, cudaStream_t st) {
  const int64_t S = a.C * a.K, E = a.N - 1;
  if (E < 1) return cudaSuccess;
  semi_expand_kernel<<<grid_for(a.B * E * S * S), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_semi_gather(const SemiExpandArgs& a, cudaStream_t st) {
  const int64_t E = a.N - 1;
  semi_gather_kernel<<<grid_for(a.marg && E > 0 ? a.B * E * a.K * a.C * a.C : 1), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_semi_seg(const SemiExpandArgs& a, cudaStream_t st) {
  semi_seg_kernel<<<grid_for(a.B * a.N), 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace tsb
