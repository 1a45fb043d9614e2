// fb_tiny.cu — the fb_tiny kernel (one CTA per sequence) and its launcher; the
// device code lives in tiny.cuh (shared with the cluster scan's exact fallback).
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

cudaError_t launch_tiny(const SmallArgs& a, cudaStream_t st) {
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
