/*
 * ts_b200.h — C ABI of the B200-native linear-chain CRF hot path
 * (Torch-Struct, Rush 2020, arXiv 2002.00876: PAPER.md §5.1-§6).
 *
 * WHAT IS COMPUTED.  A batch of B linear-chain CRFs over N positions and C labels
 * whose parts are the edges (Table 1, "Edges (TC^2)"): the
 * log-potential of labelling position t with i and position t+1 with j is
 *     pot[b][t][i][j] = l(z_t = i, z_{t+1} = j),      t in [0, N-1).
 * With Score(z) = sum_t pot[b][t][z_t][z_{t+1}]:
 *   logZ_b      = A(l) = log sum_z exp Score(z)
 *   marg[b][t]  = dA/dl = p(z_t=i, z_{t+1}=j)
 *   score_b     = A*(l) = max_z Score(z);  path_b = argmax
 * computed with the semirings of Table 2: TS_LOG = (logsumexp, +),
 * TS_MAX = (max, +), as a chunked parallel scan of C x C semiring matrix products
 * (§6(a), Fig. 4) with the max-shifted log product of §6(c)
 * (P:330-331).  Marginals come from an explicit backward scan (not autodiff).
 *
 * Readings of the paper: no start/final/unary parts (R3: alpha_0 = 0,
 * final (+) over all labels); Viterbi ties -> among all optimal labelings the one that
 * is lexicographically smallest read from the last position backwards (R5);
 * lengths: edges t >= len_b - 1 are ignored, marg = 0 and path = -1 there (R10).
 *
 * CONVENTIONS (all entry points).
 *  - Every buffer is caller-owned DEVICE memory unless the name says host; the library
 *    never allocates in a hot call and keeps no pointer after the enqueued work.
 *  - Calls are asynchronous: work is enqueued on `stream` (a cudaStream_t; NULL = the
 *    legacy default stream) and the call returns without synchronising.
 *  - Synchronous errors come back as ts_status; nothing is enqueued on error:
 *      TS_E_INVALID     null required pointer, B/N/C out of range, pot/marg not 16-byte
 *                       aligned, other pointers not 4-byte aligned, bad semiring/op;
 *      TS_E_UNSUPPORTED the current device is not sm_100 (B200); there is no CPU path;
 *                       or the (semiring, C) combination is not implemented yet;
 *      TS_E_WORKSPACE   ws_bytes < ts_workspace_bytes(...) or ws misaligned (256 B);
 *      TS_E_CUDA        a launch or async-copy enqueue failed.
 *  - Data-dependent conditions go to the per-sequence device `flags` array:
 *      TS_F_EMPTY     every labelling has score -inf: logZ/score = -inf, marg = 0, path = -1;
 *      TS_F_NONFINITE NaN or +inf on a used edge:   logZ/score = NaN,  marg = 0, path = -1;
 *      TS_F_BADLEN    lengths[b] not in [1, N]:       logZ/score = NaN,  marg = 0, path = -1.
 *    len_b = 1 (no edges): logZ = ln C, path = [0, -1, ...], score = 0.
 *  - Deterministic: identical inputs give bit-identical outputs (fixed reduction orders,
 *    no floating-point atomics).  Re-entrant: the only global state is one-time kernel
 *    attribute setup and the debug plan knob below.
 *  - Layouts are row-major and 64-bit indexed (B*(N-1)*C*C may exceed 2^31).
 */
#ifndef TS_B200_H
#define TS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(_WIN32)
#define TS_API
#else
#define TS_API __attribute__((visibility("default")))
#endif

typedef enum { TS_LOG = 0, TS_MAX = 1 } ts_semiring;

typedef enum {
  TS_OK = 0,
  TS_E_INVALID = 1,
  TS_E_UNSUPPORTED = 2,
  TS_E_WORKSPACE = 3,
  TS_E_CUDA = 4
} ts_status;

enum { TS_F_EMPTY = 1u, TS_F_NONFINITE = 2u, TS_F_BADLEN = 4u }; /* per-sequence flags */

/* `op` argument of ts_workspace_bytes */
enum {
  TS_OP_LOGZ = 0,      /* ts_logpartition                                   */
  TS_OP_MARG = 1,      /* ts_marginals                                      */
  TS_OP_VITERBI = 2,   /* ts_viterbi                                        */
  TS_OP_MARG_HOST = 3, /* ts_marginals_host (adds device staging of I/O)    */
  TS_OP_SEGMENT = 4,   /* ts_segment_summary + ts_segment_finish            */
  TS_OP_ENTROPY = 5,   /* ts_entropy (TS_LOG)                               */
  TS_OP_SAMPLE = 6,    /* ts_sample (TS_LOG)                                */
  TS_OP_SEGMENT_VITERBI = 7, /* ts_segment_viterbi_maps + _finish (same ws)  */
  TS_OP_KBEST = 8,     /* ts_kbest: size via ts_kbest_workspace_bytes(c, K)  */
  TS_OP_EXPECTATION = 9 /* ts_expectation (TS_LOG; same size as TS_OP_ENTROPY) */
};

/* One batch of chains.  N >= 1 positions (N-1 edges), 1 <= B, 1 <= C <= 256.
 * pot:     [B][N-1][C][C] fp32, row-major, 16-byte aligned; pot[b][t][i][j] =
 *          l(z_t = i, z_{t+1} = j) (reading R1: first label index = earlier position).
 *          May be NULL only when N == 1.  -inf is a legal mask value.
 * lengths: [B] int32 device array with values in [1, N], or NULL => every len_b = N. */
typedef struct {
  int64_t B, N, C;
  const float *pot;
  const int32_t *lengths;
} ts_chain;

/* Bytes of device workspace the given call needs (0 is possible).  Returns 0 and the
 * call will fail with TS_E_INVALID if the chain is invalid. */
TS_API size_t ts_workspace_bytes(const ts_chain *c, int op, ts_semiring s);

/* A(l) per sequence (§5.1; TS_MAX: A*(l)).
 * logz [B] fp32 out; flags [B] u32 out or NULL. */
TS_API ts_status ts_logpartition(const ts_chain *c, ts_semiring s, float *logz, uint32_t *flags,
                                 void *ws, size_t ws_bytes, void *stream);

/* Marginals dA/dl for TS_LOG; for TS_MAX the one-hot indicator of the
 * canonical argmax structure, d(A^*)/d(l).  marg [B][N-1][C][C] fp32 out
 * (16-byte aligned; may be NULL only when N == 1, i.e. no edges); logz [B] out (required
 * for TS_LOG, may be NULL for TS_MAX); flags [B] out or NULL. */
TS_API ts_status ts_marginals(const ts_chain *c, ts_semiring s, float *marg, float *logz,
                              uint32_t *flags, void *ws, size_t ws_bytes, void *stream);

/* Viterbi argmax with backpointers (max semiring; tie rule R5).
 * path [B][N] int32 out (-1 beyond len_b); score [B] fp32 out; flags [B] out or NULL. */
TS_API ts_status ts_viterbi(const ts_chain *c, int32_t *path, float *score, uint32_t *flags,
                            void *ws, size_t ws_bytes, void *stream);

/* ---- semi-Markov CRF (Table 1 'Semi-Markov') -------------
 * Reading R17: c->pot is [B][N-1][K][C][C] fp32; l[b][n][k-1][c1][c2] scores a
 * segment covering the k steps n -> n+k (1 <= k <= K <= 16) with label c2 after label c1
 * at node n; a labelled segmentation of nodes 0 .. len-1 scores the sum of its segments.
 * K = 1 is exactly the linear chain.  logz [B] out (required); marg (same layout as pot, 0
 * for parts that end beyond the sequence) out or NULL; flags as ts_marginals.  C <= 256.
 * Plans: the segmental forward-backward on one CTA per sequence (per-cell max, fp64
 * offsets), or — when ts_set_plan_chunk asks for a chunk length, or automatically for long
 * chains (N-1 >= 256) with C K <= 128 — the scan of §6(a) on the expanded-state
 * chain of S = C K states (label, steps to the next boundary): the potentials are expanded
 * to [B][N-1][S][S] in the workspace, every linear-chain plan runs on them (chunked scan
 * with tensor-core summaries, Fig. 4 tree, serial sweeps), and the part marginals are
 * gathered back; ts_semimarkov_viterbi likewise runs the max plans (serial, time-chunked)
 * on the expanded chain, whose first-index order is reading R18's.
 * ws: ts_semimarkov_workspace_bytes(c, K) bytes, 256-byte aligned (the expanded plan needs
 * 2 B (N-1) S^2 floats plus the chain's own workspace). */
TS_API size_t ts_semimarkov_workspace_bytes(const ts_chain *c, int64_t K);
/* Semi-Markov Viterbi (the max semiring, over the segmentations of R17):
 * the best labelled segmentation, canonical by reading R18 (backpointers = the first
 * (k asc, c' asc) maximiser, end label = the smallest arg-max: the lexicographically
 * smallest (y_m, k_m, y_{m-1}, ..., y_0) read from the end).  c->pot [B][N-1][K][C][C] as
 * ts_semimarkov, 1 <= K <= 16, C <= 256.  seg [B][N] int32 out: the label at each segment
 * boundary node (0, p_1, ..., len-1), -1 at interior nodes, beyond len and for flagged
 * sequences; score [B] fp32 out (fp32 adds: equal to the fp64 oracle on dyadic inputs;
 * -inf EMPTY, NaN NONFINITE / BADLEN); flags [B] out or NULL.
 * ws: ts_semimarkov_viterbi_workspace_bytes(c, K) bytes (uint16 backpointers [B][N][C]),
 * 256-byte aligned. */
TS_API size_t ts_semimarkov_viterbi_workspace_bytes(const ts_chain *c, int64_t K);
TS_API ts_status ts_semimarkov_viterbi(const ts_chain *c, int64_t K, int32_t *seg, float *score,
                                       uint32_t *flags, void *ws, size_t ws_bytes, void *stream);
TS_API ts_status ts_semimarkov(const ts_chain *c, int64_t K, float *marg, float *logz,
                               uint32_t *flags, void *ws, size_t ws_bytes, void *stream);

/* ---- K-best Viterbi (Table 2 'K-Max') ---------------------------
 * The first K labelings (1 <= K <= 16) of the order: Score descending, then reverse-
 * lexicographic ascending (z_{len-1} compared first — reading R5 extended, R16),
 * by the k-best max-plus recursion with backpointers.  paths [B][K][N] int32 out (-1 beyond
 * len, for missing entries when fewer than K labelings have a finite score, and for flagged
 * sequences); scores [B][K] fp32 out (-inf missing, NaN flagged); flags [B] or NULL.
 * Bit-identical to the fp64 oracle on inputs whose path sums are exact in fp32.
 * ws: ts_kbest_workspace_bytes(c, K) bytes (backpointers), 256-byte aligned. */
TS_API size_t ts_kbest_workspace_bytes(const ts_chain *c, int64_t K);
TS_API ts_status ts_kbest(const ts_chain *c, int64_t K, int32_t *paths, float *scores,
                          uint32_t *flags, void *ws, size_t ws_bytes, void *stream);

/* ---- time-sharded Viterbi (the max-plus form of the §6(a) scan,
 * P:307-311, across devices; Table 2 'Max' P:200; tie rule R5) -------------------
 * Each rank holds edges [edge_begin, edge_begin + local->N - 1) of every length-n_global
 * chain (local->lengths must be NULL; C <= 128).  The caller performs two all-gathers on
 * its NCCL group:
 *   1. ts_segment_viterbi_summary: summary [B][C][C] fp32 (ts_segment_viterbi_summary_bytes)
 *      = the max-plus product of the local edges, S[b][m][j] = best local path score from
 *      label m at the first local node to label j at the last.
 *      all_gather(summary -> all_summaries [world][B][C][C]).
 *   2. ts_segment_viterbi_maps: combines all_summaries in a fixed order (identical on every
 *      rank): boundary vector 0 (x) S_0 ... S_{rank-1}, global A* (score [B], optional) and
 *      flags [B] (optional); runs the local forward with backpointers (kept in ws) and
 *      writes maps [B][C] int32: the first-local-node label reached by backtracking from
 *      each last-local-node label.   all_gather(maps -> all_maps [world][B][C]).
 *   3. ts_segment_viterbi_finish (same ws): this rank's end label = maps_{rank+1}[...
 *      maps_{world-1}[z_E]] (z_E = the smallest global argmax), then the local backtrack:
 *      path [B][local->N] int32 (global nodes edge_begin .. edge_begin + local->N - 1;
 *      -1 for EMPTY / NONFINITE sequences).
 * With inputs whose partial path sums are exact in fp32 (the dyadic generator), the result
 * equals the unsharded ts_viterbi bit for bit.  ws: ts_workspace_bytes(local,
 * TS_OP_SEGMENT_VITERBI, TS_MAX) bytes, 256-byte aligned, shared by steps 2 and 3. */
TS_API size_t ts_segment_viterbi_summary_bytes(const ts_chain *local);
TS_API ts_status ts_segment_viterbi_summary(const ts_chain *local, int64_t edge_begin,
                                            int64_t n_global, float *summary, void *stream);
TS_API ts_status ts_segment_viterbi_maps(const ts_chain *local, int64_t edge_begin,
                                         int64_t n_global, int rank, int world,
                                         const float *all_summaries, int32_t *maps, float *score,
                                         uint32_t *flags, void *ws, size_t ws_bytes, void *stream);
TS_API ts_status ts_segment_viterbi_finish(const ts_chain *local, int64_t edge_begin,
                                           int64_t n_global, int rank, int world,
                                           const int32_t *all_maps, int32_t *path, void *ws,
                                           size_t ws_bytes, void *stream);

/* ---- distribution properties (§3) ----------
 *
 * Entropy (Table 2 'Entropy') of p(z) = exp(Score(z) - A), written out through
 * log p(z) = Score(z) - A and linearity of expectation over the parts
 * (P:181-183):   H_b = A_b - Σ_{t,i,j} mu[b][t][i][j] l[b][t][i][j].
 * Runs the ts_marginals(TS_LOG) hot path into `marg` (required, as ts_marginals) and `logz`
 * (required) and reduces mu·l (terms with mu = 0 skipped) deterministically: fused into the
 * marginal kernel's epilogue where the plan's kernel supports it (the one-CTA short-chain
 * kernel: no extra launch; meet-in-the-middle C = 64: per-engine fp64 partials + a B-thread
 * final kernel), else a two-stage fp64 reduction pass over mu and l.  Fixed thread -> element
 * mapping and fixed reduction orders in every variant (bit-reproducible).  entropy [B] fp32
 * out; NaN for EMPTY / NONFINITE / BADLEN sequences.
 * ws: ts_workspace_bytes(c, TS_OP_ENTROPY, TS_LOG) bytes, 256-byte aligned. */
TS_API ts_status ts_entropy(const ts_chain *c, float *marg, float *logz, float *entropy,
                            uint32_t *flags, void *ws, size_t ws_bytes, void *stream);

/* Expectation of an additive feature (Table 2 'Exp.' row; the expectation semiring
 * of li2009first evaluated through the marginals):
 *     out[b] = E_{z ~ p}[Σ_{t<len-1} r[b][t][z_t][z_{t+1}]] = Σ_{t,i,j} mu[b][t][i][j] r[b][t][i][j]
 * r [B][N-1][C][C] fp32 device, 16-byte aligned (same layout as pot; required, TS_E_INVALID
 * when NULL).  Runs the ts_marginals(TS_LOG) hot path into `marg` and `logz` (both required
 * as for ts_entropy) and the same deterministic reduction of mu·r (fused or a separate pass,
 * as for ts_entropy; terms with mu = 0 skipped, so r may hold anything at masked parts).  out [B] fp32; NaN for
 * EMPTY / NONFINITE / BADLEN sequences.  r = l gives E_p[Score] = A - H.
 * ws: ts_workspace_bytes(c, TS_OP_EXPECTATION, TS_LOG) bytes, 256-byte aligned. */
TS_API ts_status ts_expectation(const ts_chain *c, const float *r, float *marg, float *logz,
                                float *out, uint32_t *flags, void *ws, size_t ws_bytes,
                                void *stream);

/* Density: out[b] = Score_b(z) - logz[b] with Score(z) = Σ_{t < len-1}
 * l[b][t][z_t][z_{t+1}] accumulated in fp64.  z [B][N] int32 labels
 * (positions >= len ignored); logz [B] device (from ts_logpartition) or NULL, in which case
 * out = Score(z).  out[b] = NaN when a used label is outside [0, C), len is bad, or logz[b]
 * is not finite.  No workspace; asynchronous on `stream`. */
TS_API ts_status ts_log_prob(const ts_chain *c, const int32_t *z, const float *logz,
                             float *out, void *stream);

/* Exact sampling by forward-filtering backward-sampling (Table 2 'Sample'):
 * K independent draws z ~ p(z) per sequence.  The random numbers are INPUTS: uniforms
 * [K][B][N] fp32 in [0, 1), u[k][b][t] drives the draw of z_t (inverse CDF: the smallest
 * label whose inclusive prefix sum of p(z_t | z_{t+1}) exceeds u * total; z_{len-1} from
 * p(z_{len-1})).  z [K][B][N] int32 out (-1 beyond len and for flagged sequences); logz [B]
 * out (required); flags [B] out or NULL.  TS_LOG only; C <= 128 filters with the streaming
 * forward sweep, 128 < C <= 256 with the forward recursion of the wide-label path.
 * ws: ts_workspace_bytes(c, TS_OP_SAMPLE, TS_LOG) bytes (forward node vectors [B][N][C]). */
TS_API ts_status ts_sample(const ts_chain *c, const float *uniforms, int64_t K, int32_t *z,
                           float *logz, uint32_t *flags, void *ws, size_t ws_bytes, void *stream);

/* End-to-end variant of ts_marginals with HOST buffers: host_chain->pot / ->lengths and
 * host_marg / host_logz / host_flags are host pointers (pinned for overlap); the call
 * enqueues the H2D copies, the scan and the D2H copies on `stream` using device staging
 * inside `ws` (size from TS_OP_MARG_HOST).  Synchronise the stream before reading.
 * The batch is cut into <= 4 chunks pipelined over library-owned streams (chunk k's copy
 * back overlaps chunk k+1's kernels and copy in).  A repeated call with the same I/O
 * binding (all pointers, sizes, semiring, workspace) replays a CUDA graph of the whole
 * pipeline captured on its second sighting (ts_set_host_graphs(0) disables this); every
 * copy and kernel still runs on every call.  Thread-safe (one lock per device).
 * Payloads below 4 MB (one chunk) are pipelined ACROSS calls instead: the inputs are copied
 * on a library stream into one of two device staging buffers (alternating per call), so
 * call k's copy-in overlaps call k-1's copy-back on `stream` (PCIe is full duplex); the
 * scan and the copy-back stay ordered on `stream` after the copy-in.  Contract of that
 * mode: the host inputs must be ready when the call is made and must not alias the host
 * outputs of an earlier call still in flight; the copy-in is ordered after the previous
 * call that used the same staging buffer (and, for each buffer's first use, after the work
 * already on `stream`), not after other work enqueued on `stream` in between — so `ws`
 * must not be shared with calls of OTHER entry points while pipelined calls may be in
 * flight.  A change of binding (B, N, C, ws, semiring) or an intervening stream-ordered
 * ts_marginals_host call re-orders the next copy-in after all work on `stream`.
 * ts_set_host_pipeline(0) restores plain stream order.  In that mode, outputs laid out back
 * to back in host memory (host_logz == host_marg + B (N-1) C^2, host_flags == (uint32_t *)
 * (host_logz + B)) come back in ONE device-to-host copy (each extra small copy costs a few
 * microseconds per call on PCIe). */
TS_API ts_status ts_marginals_host(const ts_chain *host_chain, ts_semiring s, float *host_marg,
                                   float *host_logz, uint32_t *host_flags, void *ws,
                                   size_t ws_bytes, void *stream);

/* Debug/testing: 1 (default) = graph replay of repeated ts_marginals_host bindings,
 * 0 = always enqueue eagerly. */
TS_API void ts_set_host_graphs(int on);

/* Debug/testing: the cross-call pipeline of ts_marginals_host for single-chunk payloads
 * (see there).  2 (default) = three stages: call k+1's copy-in, call k's kernels and call
 * k-1's copy-back run concurrently on library streams (input and output staging
 * double-buffered; `stream` waits for each call's copy-back); 1 = the two-stream copy pipeline
 * (copy-in on a library stream, kernels and copy-back on `stream`); 0 = every call fully
 * ordered on its stream. */
TS_API void ts_set_host_pipeline(int mode);

/* Debug/testing: leaf chunk summaries of the time-chunked scan for 64 < C <= 128 run on
 * the tensor cores (tcgen05 kind::tf32): 3 = 3xTF32 split (default), 1 = one TF32 pass,
 * 0 = SIMT fp32 kernel.  Chunks the precision gate flags are recomputed exactly in every
 * mode. */
TS_API void ts_set_tc_summary(int mode);
TS_API int  ts_get_tc_summary(void);

/* Page-locked host staging buffers for ts_marginals_host (cudaHostAlloc, portable).
 * Returns NULL on failure or bytes == 0; release with ts_host_free.  Buffers from this
 * allocator sustain full PCIe rate for the host->device copies (pinned registrations of
 * ordinary pages can be several times slower to DMA-read under an IOMMU). */
TS_API void *ts_host_alloc(size_t bytes);
TS_API void  ts_host_free(void *p);

/* ---- time-sharded chains (§6(a) scan across devices) --------------------
 * A chain of n_global positions is split into contiguous segments; a rank holds edges
 * [edge_begin, edge_begin + local->N - 1) in local->pot (local->N = local edge count + 1)
 * for every sequence of the batch (local->lengths must be NULL: full-length chains).
 * Step 1: ts_segment_summary writes this segment's C x C transfer matrix per sequence
 *         (the semiring product of its edges) into `summary` (16-byte aligned),
 *         laid out as ts_segment_summary_bytes(local) bytes: [B][C][C] fp32 log2-domain
 *         values relative to per-row fp64 natural-log offsets (this section padded to a
 *         multiple of 4 floats), followed by [B][C] fp64 offsets (padded to an even count),
 *         so the size is a multiple of 16 bytes and every gathered slice stays aligned.  The workspace (size: ts_workspace_bytes(local, TS_OP_SEGMENT, s)) holds
 *         the local scan tree and MUST be passed unchanged to ts_segment_finish.
 * Step 2: the caller all-gathers the summaries of all `world` segments, in rank order,
 *         into all_summaries ([world] x ts_segment_summary_bytes) — e.g. NCCL
 *         all_gather_into_tensor over NVLink.
 * Step 3: ts_segment_finish combines them (every rank computes the same prefix/suffix
 *         products in the same order, so logZ is bit-identical across ranks) and runs the
 *         local forward/backward sweeps: logz [B] (global A), marg (local edges) or NULL.
 * Only TS_LOG is implemented (TS_MAX returns TS_E_UNSUPPORTED); C <= 128; lengths NULL.
 * logz/flags are global (identical on every rank); marg covers the local edges. */
TS_API size_t ts_segment_summary_bytes(const ts_chain *local);
TS_API ts_status ts_segment_summary(const ts_chain *local, int64_t edge_begin, int64_t n_global,
                                    ts_semiring s, void *summary, void *ws, size_t ws_bytes,
                                    void *stream);
TS_API ts_status ts_segment_finish(const ts_chain *local, int64_t edge_begin, int64_t n_global,
                                   int rank, int world, ts_semiring s, const void *all_summaries,
                                   float *marg_or_null, float *logz, uint32_t *flags, void *ws,
                                   size_t ws_bytes, void *stream);

/* Plan knob (process-global): chunk length L of the time-chunked scan.
 * 0 = automatic; 1 = the paper's pure Fig. 4 tree (every edge a leaf); >= N-1 = serial
 * sweep (no tree).  Applies to the log semiring (logZ, marginals, f1) and to the max
 * semiring (ts_viterbi, ts_logpartition / ts_marginals with TS_MAX; C <= 158): max-plus
 * chunk summaries, a fixed-order combine of the boundary vectors, chunk-local forwards with
 * first-index backpointers, end-label maps and chunk backtracks (the automatic plan keeps
 * the serial sweep for Viterbi).  Results agree across plans within the parity tolerances
 * (Viterbi: bit-identical on inputs whose partial path sums are exact, e.g. the dyadic
 * generator). */
TS_API void ts_set_plan_chunk(int64_t L);
TS_API int64_t ts_get_plan_chunk(void);

/* Plan knob (process-global) for short log-semiring chains with C % 4 == 0, C <= 28 and
 * 2G <= N-1 <= 8G: the chunked parallel scan of PAPER.md §6(a) on a thread-block
 * cluster of G CTAs per sequence — per-CTA chunk summaries (tree of C x C products), one
 * DSMEM bulk exchange, boundary vectors, local forward/backward sweeps with fused marginals
 * (fb_cscan.cu).  0 (default) = the one-CTA-per-sequence kernels (fb_tiny measured faster
 * at cfg2: 6.25 vs 6.8 us/step); -1 = auto (G = 4 if 4B <= #SMs, else 2 if
 * 2B <= #SMs, else one CTA); 2 or 4 = force that G where the shape fits.  Results agree within the parity tolerances (gated inputs fall back to the
 * exact one-CTA body inside the same launch). */
TS_API void ts_set_small_cluster(int G);

/* Debug/testing knob (process-global): 1 (default) runs short log-semiring chains with
 * C % 4 == 0 and C <= 28 through the latency-optimised single-CTA kernel (bulk-copied
 * tiles, lagged-normaliser recursions, mbarrier-published nodes, overlapped marginals);
 * 0 = the general single-CTA kernel.  Results agree within the parity tolerances. */
TS_API void ts_set_tiny(int enable);

/* Debug/testing knob (process-global): 1 (default) streams the tiles of the wide-label log
 * path (128 < C <= 256, C % 4 == 0) through a bulk-copy SMEM ring; 0 = plain coalesced
 * loads into registers (the path odd widths always take).  Results agree within the
 * parity tolerances. */
TS_API void ts_set_wide_ring(int enable);

/* Debug/testing knob (process-global): 1 (default) lets the short-chain kernel fb_tiny read
 * its inputs before waiting for a still-running earlier call on the stream (programmatic
 * dependent launch), so consecutive calls overlap everything but their global writes — when
 * the library has not recorded a recent call whose outputs overlap this call's pot / lengths
 * (then it waits before reading, as with 0).  Results are identical either way.
 * Contract: only this library's kernels are assumed to trigger programmatic dependents
 * (griddepcontrol.launch_dependents / cudaTriggerProgrammaticLaunchCompletion); if a caller's
 * own kernel that does so writes a buffer a following ts_* call reads, without an event or
 * other stream operation in between, set 0. */
TS_API void ts_set_tiny_early(int enable);

/* Debug/testing knob (process-global): 1 (default) runs ts_marginals for C = 64 with one
 * serial chunk per sequence as the meet-in-the-middle kernel (forward and backward
 * recursions concurrently from both ends, marginals fused); 0 = separate forward and
 * backward sweep kernels.  Results agree within the parity tolerances. */
TS_API void ts_set_meet(int enable);

/* Debug/testing knob (process-global) for the time-chunked Viterbi (ts_set_plan_chunk, and
 * the automatic choice for long chains with C in {32, 64, 128}): 1 (default) = chunk
 * summaries by the register-blocked max-plus product kernel where C in {32, 64, 128} and
 * the potentials are 16-byte aligned; 0 = the row-chain summary kernel for every C (the
 * automatic plan then keeps the serial sweep).  Results are bit-identical. */
TS_API void ts_set_vchunk_mm(int enable);

/* Debug/testing knob (process-global) for ts_kbest: lanes per label column S in {1, 2, 4, 8}
 * (0 = automatic: 2 when B >= #SMs, else 8; capped so that C * S <= 512).  Results are
 * bit-identical for every S. */
TS_API void ts_set_kbest_split(int S);

/* Debug/testing knob (process-global) for the Viterbi forward with C in {128, 256}:
 * 0 (default) = automatic cluster column split (the largest G in {1,2,4,8} with B*G CTAs
 * fitting the SMs, C/G >= 32); G in {1,2,4,8} = forced cluster size; -1 = the
 * one-CTA-per-sequence kernel used for every other C.  Results are bit-identical. */
TS_API void ts_set_viterbi_split(int G);

/* Number of kernel launches the most recent successful call on this host thread
 * enqueued (bench accounting). */
/* Name of the dominant (time-wise) kernel enqueued by this thread's last successful
 * ts_logpartition / ts_marginals / ts_viterbi call ("" before any): for measurement and
 * profiling (bench.py roofline line).  Static string, never freed. */
TS_API const char *ts_last_kernel(void);
TS_API int ts_last_launch_count(void);

TS_API const char *ts_status_str(ts_status s);
TS_API const char *ts_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TS_B200_H */
