// fb_tiny.cu — the fb_tiny kernel (one CTA per sequence) and its launcher; the
// device code lives in tiny.cuh (shared with the cluster scan's exact fallback).
#include <mutex>

#include "tiny.cuh"

namespace tsb {

template <int C, int XM>
__global__ void __launch_bounds__(kTinyThreads, 1) fb_tiny_kernel(SmallArgs a) {
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

// ---- early input reads (SmallArgs::early) --------------------------------------------------
// fb_tiny and fb_cscan trigger their dependents (griddepcontrol.launch_dependents) as they
// start, so a call may begin while earlier calls on the stream still run.  A call may read its
// inputs before its PDL wait only if none of those calls writes them: the outputs of the most
// recent PDL launches (more than the device can hold resident at once) are kept here and a
// launch whose pot / lengths ranges meet one of them waits before reading, as before.
namespace {
struct ByteRange {
  uintptr_t lo, hi;
};
constexpr int kPdlRing = 512;
std::mutex g_pdl_mu;
ByteRange g_pdl_ring[kPdlRing];
int64_t g_pdl_count = 0;
std::atomic<int> g_tiny_early{1};

ByteRange range_of(const void* p, int64_t bytes) {
  const uintptr_t lo = reinterpret_cast<uintptr_t>(p);
  return ByteRange{lo, lo + (uintptr_t)(bytes > 0 ? bytes : 0)};
}
bool ring_hit(const ByteRange& r) {
  if (r.hi <= r.lo) return false;
  const int64_t n = g_pdl_count < kPdlRing ? g_pdl_count : kPdlRing;
  for (int64_t i = 0; i < n; ++i)
    if (r.lo < g_pdl_ring[i].hi && g_pdl_ring[i].lo < r.hi) return true;
  return false;
}
void ring_add(const ByteRange& r) {
  if (r.hi <= r.lo) return;
  g_pdl_ring[g_pdl_count % kPdlRing] = r;
  ++g_pdl_count;
}
}  // namespace

void set_tiny_early(int on) { g_tiny_early.store(on ? 1 : 0); }
int get_tiny_early() { return g_tiny_early.load(); }

// Records the outputs of a PDL-triggering launch; returns whether its inputs are clear of
// every recorded output (checked before this launch's own outputs are added).
bool pdl_launch_note(const SmallArgs& a) {
  const int64_t E = a.N - 1 > 0 ? a.N - 1 : 0, nel = a.B * E * a.C * a.C;
  std::lock_guard<std::mutex> lock(g_pdl_mu);
  const bool clear = !ring_hit(range_of(a.pot, nel * 4)) &&
                     !(a.lengths && ring_hit(range_of(a.lengths, a.B * 4)));
  if (a.marg) ring_add(range_of(a.marg, nel * 4));
  ring_add(range_of(a.logz, a.B * 4));
  if (a.flags) ring_add(range_of(a.flags, a.B * 4));
  if (a.xmode && a.xout) ring_add(range_of(a.xout, a.B * 4));
  return clear;
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
  const bool clear = pdl_launch_note(a);
  a.early = (clear && g_tiny_early.load()) ? 1 : 0;
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
