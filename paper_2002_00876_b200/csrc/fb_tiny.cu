// fb_tiny.cu — the fb_tiny kernel (one CTA per sequence) and its launcher; the
// device code lives in tiny.cuh (shared with the cluster scan's exact fallback).
#include <mutex>

#include "tiny.cuh"

namespace tsb {

template <int C, int XM>
__global__ void __launch_bounds__(kTinyThreads, 2) fb_tiny_kernel(SmallArgs a) {
  extern __shared__ __align__(16) float sm[];
  tiny_body<C, true, XM>(a, blockIdx.x, sm);
}

size_t tiny_smem_bytes(int64_t N, int64_t C) {
  return (size_t)tiny_layout(N, (int)C).total * sizeof(float);
}

bool tiny_fits(const SmallArgs& a) {
  const int64_t C = a.C;
  if (C % 4 != 0 || C < 4 || C > 28 || a.N < 1) return false;
  if ((reinterpret_cast<uintptr_t>(a.pot) & 15) != 0) return false;
  if (a.marg && (reinterpret_cast<uintptr_t>(a.marg) & 15) != 0) return false;
  return tiny_smem_bytes(a.N, C) <= (size_t)200 * 1024;
}

// ---- early input reads / early marginal writes (SmallArgs::early) --------------------------
// fb_tiny and fb_cscan trigger their dependents (griddepcontrol.launch_dependents) as they
// start, so a call may begin while earlier calls on the stream still run — at most the last
// kPdlWindow such launches (a device holds at most 128 resident grids, and a grid triggers only
// once all of its CTAs are resident).  The input and output ranges of recent launches are kept
// here: a launch may read its inputs before its PDL wait if no launch in the window writes
// them, and may also write its marginals before the wait if no launch in the window reads or
// writes that range (every thread still waits before the per-sequence scalars and before it
// exits, so a call completes only after its predecessor).
namespace {
struct PdlRange {
  uintptr_t lo, hi;
  int64_t seq;
  bool out;
};
constexpr int kPdlRing = 2048;
constexpr int64_t kPdlWindow = 130;
std::mutex g_pdl_mu;
PdlRange g_pdl_ring[kPdlRing];
int64_t g_pdl_n = 0;    // ranges recorded
int64_t g_pdl_seq = 0;  // launches recorded
std::atomic<int> g_tiny_early{1};

PdlRange range_of(const void* p, int64_t bytes, bool out) {
  const uintptr_t lo = reinterpret_cast<uintptr_t>(p);
  return PdlRange{lo, p ? lo + (uintptr_t)(bytes > 0 ? bytes : 0) : lo, g_pdl_seq, out};
}
// any range of a launch in the window overlapping r (outputs only, or inputs and outputs)?
bool window_hit(const PdlRange& r, bool outputs_only) {
  if (r.hi <= r.lo) return false;
  const int64_t n = g_pdl_n < kPdlRing ? g_pdl_n : kPdlRing;
  for (int64_t i = 0; i < n; ++i) {
    const PdlRange& q = g_pdl_ring[i];
    if (q.seq <= g_pdl_seq - kPdlWindow || (outputs_only && !q.out)) continue;
    if (r.lo < q.hi && q.lo < r.hi) return true;
  }
  return false;
}
void ring_add(const PdlRange& r) {
  if (r.hi <= r.lo) return;
  g_pdl_ring[g_pdl_n % kPdlRing] = r;
  ++g_pdl_n;
}
}  // namespace

void set_tiny_early(int on) { g_tiny_early.store(on ? 1 : 0); }
int get_tiny_early() { return g_tiny_early.load(); }

// Records the inputs and outputs of a dependents-triggering launch; returns SmallArgs::early
// for it (0: wait first; bit 0: read early; bit 1: also write the marginals early; bit 2: also
// write logZ / flags / the fused output early), checked against the launches before it.  (A ring this size never drops an entry of the window.)
int pdl_launch_note(const SmallArgs& a) {
  const int64_t E = a.N - 1 > 0 ? a.N - 1 : 0, nel = a.B * E * a.C * a.C;
  std::lock_guard<std::mutex> lock(g_pdl_mu);
  const PdlRange in_pot = range_of(a.pot, nel * 4, false);
  const PdlRange in_len = range_of(a.lengths, a.B * 4, false);
  const PdlRange in_xr = range_of(a.xmode == 2 ? a.xr : nullptr, nel * 4, false);
  const PdlRange out_m = range_of(a.marg, nel * 4, true);
  const PdlRange out_l = range_of(a.logz, a.B * 4, true);
  const PdlRange out_f = range_of(a.flags, a.B * 4, true);
  const PdlRange out_x = range_of(a.xmode ? a.xout : nullptr, a.B * 4, true);
  int early = 0;
  if (!window_hit(in_pot, true) && !window_hit(in_len, true) && !window_hit(in_xr, true)) {
    early = 1;
    if (a.marg && !window_hit(out_m, false)) early |= 2;
    if (!window_hit(out_l, false) && !window_hit(out_f, false) && !window_hit(out_x, false)) early |= 4;
  }
  ring_add(in_pot);
  ring_add(in_len);
  ring_add(in_xr);
  ring_add(out_m);
  ring_add(out_l);
  ring_add(out_f);
  ring_add(out_x);
  ++g_pdl_seq;
  return early;
}

namespace {
template <int C, int XM>
cudaError_t launch_tiny_cx(const SmallArgs& a, size_t smem, cudaStream_t st) {
  static std::atomic<uint64_t> attr_mask{0};  // one-time attribute setup per device
  cudaError_t e = smem_optin_once(fb_tiny_kernel<C, XM>, attr_mask, 200 * 1024);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)a.B);
  cfg.blockDim = dim3(kTinyThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, fb_tiny_kernel<C, XM>, a);
}
// XM: the fused f1 epilogue variant (0 = plain marginals, the default instantiation)
template <int C>
cudaError_t launch_tiny_c(const SmallArgs& a, size_t smem, cudaStream_t st) {
  if (a.xmode == 1) return launch_tiny_cx<C, 1>(a, smem, st);
  if (a.xmode == 2) return launch_tiny_cx<C, 2>(a, smem, st);
  return launch_tiny_cx<C, 0>(a, smem, st);
}
}  // namespace

cudaError_t launch_tiny(const SmallArgs& a0, cudaStream_t st) {
  SmallArgs a = a0;
  const int early = pdl_launch_note(a);
  a.early = g_tiny_early.load() ? early : 0;
  const size_t smem = tiny_smem_bytes(a.N, a.C);
  switch (a.C) {
    case 4: return launch_tiny_c<4>(a, smem, st);
    case 8: return launch_tiny_c<8>(a, smem, st);
    case 12: return launch_tiny_c<12>(a, smem, st);
    case 16: return launch_tiny_c<16>(a, smem, st);
    case 20: return launch_tiny_c<20>(a, smem, st);
    case 24: return launch_tiny_c<24>(a, smem, st);
    case 28: return launch_tiny_c<28>(a, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tsb
