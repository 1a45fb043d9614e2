// kernels.cuh — argument blocks and launchers of the sm_100a kernels (internal to the
// library; the public surface is include/ts_b200.h, implemented in abi.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ts_b200.h"

namespace tsb {

// Per-sequence scratch flags accumulated by the kernels that read l (device, [B]).
enum : uint32_t { WF_NONFINITE = 2u };

// ---- short chains, C <= 32: one CTA per sequence, whole chain in SMEM (fb_small.cu),
// or the chunked-scan variant on a cluster of G CTAs per sequence (fb_cluster.cu) ---------
struct SmallArgs {
  const float* pot;
  const int32_t* lengths;
  int64_t B, N, C;
  float* marg;      // [B][N-1][C][C] or nullptr (logZ only)
  float* logz;      // [B]
  uint32_t* flags;  // [B] or nullptr
  // fused f1 epilogue (fb_tiny only): xmode 1 = entropy H = A - Σ mu·l, 2 = expectation
  // Σ mu·xr (terms with mu = 0 skipped); xout [B], NaN for flagged sequences
  const float* xr;
  int xmode;
  float* xout;
  // fb_tiny: bit 0 = no programmatic (PDL) predecessor that may still run writes pot /
  // lengths / xr (checked by the launcher against its recent PDL launches), so the inputs are
  // read at once and the wait for the previous grid moves to just before the first global
  // write; bit 1 = none reads or writes the marginal range either, so the marginals are
  // written before the wait too; bit 2 = the same for logZ / flags / xout; every thread
  // still waits before it exits (the call completes after its predecessor)
  int early;
};
size_t small_smem_bytes(int64_t N, int64_t C);
bool small_fits(int64_t N, int64_t C);
cudaError_t launch_small(const SmallArgs& a, cudaStream_t st);
// latency-optimised variant for C % 4 == 0, C <= 28 (fb_tiny.cu)
size_t tiny_smem_bytes(int64_t N, int64_t C);
bool tiny_fits(const SmallArgs& a);
cudaError_t launch_tiny(const SmallArgs& a, cudaStream_t st);
// PDL bookkeeping shared by fb_tiny / fb_cscan launches (fb_tiny.cu): records the inputs and
// outputs of a dependents-triggering launch, returns its SmallArgs::early value
int pdl_launch_note(const SmallArgs& a);
void set_tiny_early(int on);  // fb_tiny early input reads (default 1)
int get_tiny_early();
// the chunked scan of §6(a) on a G-CTA cluster per sequence (fb_cscan.cu), same shapes
size_t cscan_smem_bytes(int64_t N, int64_t C, int G);
bool cscan_fits(const SmallArgs& a, int G);
int cscan_g(const SmallArgs& a, int sms);  // G for the auto plan (0 = do not use)
cudaError_t launch_cscan(const SmallArgs& a, int G, cudaStream_t st);

// ---- streaming (time-chunked) forward / backward sweeps, log semiring (C <= 128) ----
// Chunk k of sequence b covers edges [k*L, min((k+1)*L, E_b)), E_b = len_b - 1.
// Vectors crossing chunk boundaries are "LogVec": C fp32 log2-domain values relative
// to one fp64 natural-log offset.
struct SweepArgs {
  const float* pot;
  const int32_t* lengths;
  int64_t B, N, C;
  int64_t L, P;             // chunk length and chunks per sequence
  // forward
  const float* alpha_in;    // [B*P][C] log2-relative start vector per chunk, or nullptr (=0)
  const double* alpha_in_off;  // [B*P] natural offsets, or nullptr (=0)
  float* alpha_hat;         // [B][N][C] node vectors (nodes [s_k, e_k) written by chunk k)
  float* alpha_end;         // [B*P][C] chunk-end vector in the chunk's own frame
  double* alpha_end_off;    // [B*P] its natural offset
  float* mlag;              // [B][N] lag bound m_t used at step t (forward frame)
  float* tmax;              // [B][N-1] per-edge tile max (natural units)
  // backward
  const float* beta_out;    // [B*P][C] chunk-end beta vector, or nullptr (=0, last chunk)
  const double* beta_out_off;  // [B*P] or nullptr
  float* marg;              // [B][N-1][C][C] or nullptr
  // bookkeeping
  uint32_t* wflags;         // [B] scratch flags (zeroed before the forward launch)
  float* logz;              // [B] (written by the last chunk's forward CTA when P == 1)
  uint32_t* flags;          // [B] or nullptr
  int final_in_fwd;         // 1: forward writes logz/flags (logZ-only call, P == 1)
  int no_final;             // 1: backward must not write logz/flags (time-sharded segment)
};
size_t fwd_smem_bytes(int64_t C, int stages);
size_t bwd_smem_bytes(int64_t C, int stages);
cudaError_t launch_fwd(const SweepArgs& a, cudaStream_t st);
cudaError_t launch_bwd(const SweepArgs& a, cudaStream_t st);
// register-blocked variants for C in {32, 64, 128} (fb_stream2.cu)
bool stream2_ok(const SweepArgs& a);
cudaError_t launch_fwd2(const SweepArgs& a, cudaStream_t st);
cudaError_t launch_bwd2(const SweepArgs& a, cudaStream_t st);

// ---- meet-in-the-middle fused forward/backward + marginals, one CTA per sequence
// (fb_meet.cu): two 256-thread engines sweep from both ends at once, exchange their node
// vectors through HBM/L2 at the midpoint and each finishes the other half with marginals.
struct MeetArgs {
  const float* pot;
  const int32_t* lengths;
  int64_t B, N;
  float* marg;       // [B][N-1][C][C]
  float* logz;       // [B]
  uint32_t* flags;   // [B] or nullptr
  float* alpha_hat;  // [B][N][C] forward node vectors, nodes 0..h (scratch)
  float* beta_hat;   // [B][N][C] backward node vectors, nodes h..E_b (scratch)
  float* mlag;       // [B][N]  forward lag bound per edge t < h (scratch)
  float* tshift;     // [B][N-1] natural-unit shift used for edge t (scratch)
  // fused f1 epilogue: xmode 1 = Σ mu·l (entropy), 2 = Σ mu·xr (expectation);
  // terms with mu = 0 skipped; per-engine fp64 partials xsum[2b + engine], fixed order
  const float* xr;
  int xmode;
  double* xsum;
};
bool meet_ok(int64_t C, const float* pot, const float* marg);
cudaError_t launch_meet(const MeetArgs& a, int64_t C, cudaStream_t st);

// ---- time-chunked scan (scan.cu): leaf summaries, up-sweep tree, down-sweep ---------
// Tree of one sequence: levels 0..H, level l holds Ppad >> l nodes (Ppad = 2^H >= P),
// `nodes` = 2*Ppad - 1 node slots per sequence.  LogMat node: mat [C][C] log2 values +
// off [C] fp64 natural row offsets; ident = 1 marks the identity I (padding).
struct ScanArgs {
  const float* pot;
  const int32_t* lengths;
  int64_t B, N, C;
  int64_t L, P, Ppad, nodes;
  int H;
  float* mat;
  double* off;
  uint8_t* ident;
  uint32_t* cflag;  // [B][Ppad] leaf chunks needing the exact log-space recomputation
  float* valpha;    // [B][nodes][C] alpha_in vector of every node
  double* oalpha;
  float* vbeta;     // [B][nodes][C] beta_out vector of every node
  double* obeta;
  float* leaf_alpha;  // [B][P][C] leaf copies read by the leaf sweeps
  double* leaf_alpha_off;
  float* leaf_beta;
  double* leaf_beta_off;
  uint32_t* wflags;
  float* logz;
  uint32_t* flags;
};
__host__ __device__ int64_t level_off(int l, int64_t Ppad);
size_t scan_mat_smem(int64_t C);
cudaError_t launch_scan_up(const ScanArgs& a, cudaStream_t st, int* launches);
cudaError_t launch_scan_down(const ScanArgs& a, cudaStream_t st, int* launches, bool set_root);
// Segment summary layout (ts_segment_summary_bytes): [B][C][C] fp32, padded to a multiple
// of 4 floats so the fp64 offsets that follow are 16-byte aligned whatever B*C*C is, then
// [B][C] fp64 padded to an even count so every gathered slice stays 16-byte aligned.
__host__ __device__ inline int64_t seg_mat_floats(int64_t B, int64_t C) {
  return (B * C * C + 3) & ~int64_t(3);
}
__host__ __device__ inline int64_t seg_total_floats(int64_t B, int64_t C) {
  return seg_mat_floats(B, C) + 2 * ((B * C + 1) & ~int64_t(1));
}
cudaError_t launch_segment_export(const ScanArgs& a, float* summ, cudaStream_t st);
cudaError_t launch_segment_combine(const ScanArgs& a, const float* all_summ, int rank, int world,
                                   bool write_root, cudaStream_t st);
cudaError_t launch_scan_logz(const ScanArgs& a, cudaStream_t st);
// tensor-core (tcgen05 kind::tf32, 3xTF32) leaf summaries for 64 < C <= 128 (scan_tc.cu)
bool summary_tc_ok(const ScanArgs& a);
cudaError_t launch_summary_tc(const ScanArgs& a, cudaStream_t st);
void set_tc_summary(int mode);  // 0 SIMT, 1 1xTF32, 3 3xTF32
int get_tc_summary();

// ---- Viterbi (max-plus) -------------------------------------------------------------
struct VitArgs {
  const float* pot;
  const int32_t* lengths;
  int64_t B, N, C;
  uint8_t* bp;      // [B][N-1][C] backpointers
  int32_t* zend;    // [B] final label (first argmax), -1 if none
  float* score;     // [B]
  uint32_t* flags;  // [B] or nullptr
  int32_t* path;    // [B][N] or nullptr
  float* marg;      // [B][N-1][C][C] indicator or nullptr
  float* logz;      // [B] copy of the score for ts_logpartition/ts_marginals(TS_MAX), or nullptr
  const float* delta_in;  // [B][C] start vector (time-sharded segment), or nullptr (= 0)
};
size_t vit_smem_bytes(int64_t C, int stages, int rows_per_stage);
// vsplit: -1 = one-CTA-per-sequence kernel for every C; 0 = auto (cluster column split for
// C in {128, 256}); 1/2/4/8 = forced cluster size for C in {128, 256}.
cudaError_t launch_viterbi(const VitArgs& a, cudaStream_t st, int* launches, int vsplit);
cudaError_t launch_backtrack(const VitArgs& a, cudaStream_t st);
// one-hot dA*/dl from a.path into a.marg (ts_marginals(TS_MAX)); no-op without marg
cudaError_t launch_indicator(const VitArgs& a, cudaStream_t st);
cudaError_t launch_vit1(const VitArgs& a, cudaStream_t st);
// cluster column-split forward (viterbi2.cu)
bool vit2_ok(const VitArgs& a);
cudaError_t launch_vit2(const VitArgs& a, int g_force, cudaStream_t st);

// ---- distribution properties (dist_ops.cu) ---------------------------
struct DistArgs {
  const float* pot;
  const int32_t* lengths;
  int64_t B, N, C;
  const float* marg;       // entropy / expectation: marginals [B][N-1][C][C]
  const float* r;          // expectation: additive feature [B][N-1][C][C] (NULL: entropy)
  const float* logz;       // [B] (entropy: required; score: NULL -> Score(z))
  const uint32_t* flags;   // [B] or NULL
  float* out;              // [B] entropy / log_prob
  double* partial;         // entropy partials [B][S]
  int64_t Ls;              // entropy slice length (edges)
  const int32_t* z;        // score: labels [B][N]
  int32_t* zout;           // sample: [K][B][N]
  const float* uniforms;   // sample: [K][B][N]
  int64_t K;
  const float* ah;         // sample: forward node vectors [B][N][C] (log2, per-node frame)
  const float* aend;       // sample: node Eb vector [B][C]
  int aend_in_ah;          // sample: node len-1 vector is row len-1 of ah (fb_wide, C > 128)
};
int entropy_slices(const DistArgs& a);
cudaError_t launch_entropy(DistArgs a, cudaStream_t st);
// the final stage alone: out[b] from partial[b][0..S) (a fused marginal epilogue's partials)
cudaError_t launch_entropy_final(const DistArgs& a, int S, cudaStream_t st);
cudaError_t launch_score(const DistArgs& a, cudaStream_t st);
cudaError_t launch_sample(const DistArgs& a, cudaStream_t st);

// ---- semi-Markov CRF (semimarkov.cu, reading R17) -----------------------
struct SemiArgs {
  const float* pot;        // [B][N-1][K][C][C]
  const int32_t* lengths;
  int64_t B, N, C, K;
  float* marg;             // same layout as pot, or nullptr
  float* logz;
  uint32_t* flags;
  float* ah;               // [B][N][C] normalised forward vectors (workspace)
  float* bh;               // [B][N][C] normalised backward vectors
  double* ao;              // [B][N] natural offsets
  double* bo;
  double* zbuf;            // [B] logZ in fp64
  int staged;              // semimarkov_kernel: tiles staged in SMEM one step ahead (launcher)
};
cudaError_t launch_semimarkov(const SemiArgs& a, cudaStream_t st);
// linear chain, 128 < C <= 256 (fb_wide.cu): the SemiArgs workspace of K = 1
cudaError_t launch_fb_wide(const SemiArgs& a, cudaStream_t st);
extern int g_wide_ring;  // debug knob: 1 = SMEM ring (C % 4 == 0), 0 = register path
// semi-Markov Viterbi (reading R18): seg [B][N] int32 out, score [B] out, bp [B][N][C] uint16
// workspace ((k-1) * C + c'), flags as the other entry points
struct SemiVitArgs {
  const float* pot;        // [B][N-1][K][C][C]
  const int32_t* lengths;
  int64_t B, N, C, K;
  int32_t* seg;
  float* score;
  uint32_t* flags;
  uint16_t* bp;
  int staged;              // set by the launcher: tiles staged in SMEM one step ahead
};
cudaError_t launch_semimarkov_viterbi(const SemiVitArgs& a, cudaStream_t st);

// ---- K-best Viterbi (kbest.cu) -------------------------------------------
struct KbestArgs {
  const float* pot;
  const int32_t* lengths;
  int64_t B, N, C, K;
  uint16_t* bp;      // [B][N-1][C][KM] (i | r << 8)
  int32_t* paths;    // [B][K][N]
  float* scores;     // [B][K]
  uint32_t* flags;   // [B] or nullptr
};
int kbest_km(int64_t K);
size_t kbest_smem(int64_t C, int64_t K, int S);
void set_kbest_split(int S);  // debug: lanes per column (0 auto, 1/2/4/8)
cudaError_t launch_kbest(const KbestArgs& a, cudaStream_t st);

// ---- time-sharded Viterbi segments (vseg.cu) -------------------------------
struct VsegArgs {
  const float* pot;       // local edges [B][E_loc][C][C]
  int64_t B, N, C;        // local chain (N = E_loc + 1 nodes)
  float* summary;         // [B][C][C] max-plus transfer matrix of the local edges
  const float* all_summ;  // [world][B][C][C]
  int rank, world;
  float* delta_in;        // [B][C] boundary vector of this segment
  float* score;           // [B] global A*
  int32_t* zglob;         // [B] global final label (first argmax)
  uint32_t* flags;        // [B] or nullptr
  const uint8_t* bp;      // local backpointers [B][E_loc][C]
  int32_t* maps;          // [B][C] end label -> start label of the local segment
  const int32_t* all_maps;  // [world][B][C]
  int32_t* zend;          // [B] this segment's end label
};
cudaError_t launch_vseg_summary(const VsegArgs& a, cudaStream_t st);

// ---- semi-Markov through the expanded-state chain (semi_expand.cu) ------------------------
struct SemiExpandArgs {
  const float* pot;        // [B][N-1][K][C][C]
  const int32_t* lengths;
  int64_t B, N, C, K;
  float* xpot;             // [B][N-1][S][S], S = C K (expanded chain potentials)
  const float* xmarg;      // [B][N-1][S][S] expanded marginals (gather input)
  float* marg;             // [B][N-1][K][C][C] or nullptr
  float* logz;             // [B] (len = 1 fix-up) or nullptr
  const int32_t* xpath;    // [B][N] expanded Viterbi path (seg input)
  int32_t* seg;            // [B][N] semi-Markov Viterbi output
};
cudaError_t launch_semi_expand(const SemiExpandArgs& a, cudaStream_t st);
cudaError_t launch_semi_gather(const SemiExpandArgs& a, cudaStream_t st);
cudaError_t launch_semi_seg(const SemiExpandArgs& a, cudaStream_t st);

// ---- single-GPU time-chunked Viterbi (vchunk.cu) -------------------------------------------
struct VChunkArgs {
  const float* pot;
  const int32_t* lengths;
  int64_t B, N, C;
  int64_t L, P;        // chunk length, chunks per sequence (P = ceil((N-1) / L))
  float* summ;         // [B P][C][C] chunk max-plus summaries
  float* din;          // [B P][C] boundary vectors
  uint8_t* bp;         // [B][N-1][C] backpointers
  int32_t* maps;       // [B P][C] end label -> first-node label of the chunk
  int32_t* zend;       // [B P] chunk end labels
  int32_t* zglob;      // [B] final label
  float* score;        // [B]
  float* logz;         // [B] or nullptr (copy of the score)
  uint32_t* flags;     // [B] or nullptr
  int32_t* path;       // [B][N]
};
size_t vchunk_ws_floats(const VChunkArgs& a);
bool vchunk_ok(int64_t C);
cudaError_t launch_vchunk(const VChunkArgs& a, bool want_path, cudaStream_t st, int* launches);
void set_vchunk_mm(int enable);  // debug: 0 = row-chain summaries for every C
bool vchunk_mm(int64_t C);        // the register-blocked summary kernel serves this C
cudaError_t launch_vseg_combine(const VsegArgs& a, cudaStream_t st);
cudaError_t launch_vseg_maps(const VsegArgs& a, cudaStream_t st);
cudaError_t launch_vseg_endlabel(const VsegArgs& a, cudaStream_t st);

}  // namespace tsb
