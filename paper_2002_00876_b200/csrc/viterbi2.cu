// viterbi2.cu — max-plus forward with backpointers for C in {128, 256} (BASELINE cfg4:
// B=64, N=1024, C=256), columns of each sequence split across a thread-block cluster of G
// CTAs so that B*G CTAs fill the GPU (paper P:160/P:265, reading R5, SURVEY §8(e) "cluster
// column-split per sequence").
//
// CTA h of the cluster owns columns [h C/G, (h+1) C/G) of every tile:
//   delta_{t+1}[j] = max_i (delta_t[i] + l_t[i][j]),  bp_t[j] = smallest maximising i.
// Each step streams the CTA's C x C/G column slab in 32-row blocks through a TMA ring (one
// 2-D tensor copy per block, issued by a dedicated producer warp; full/empty mbarriers).  The
// CTA first processes the row blocks of its own part (delta rows it computed itself), then
// waits for the peers' delta slices (written into its shared memory through DSMEM and
// signalled on a cluster-scope mbarrier) and processes the remaining parts, so the exchange
// overlaps half a step of streaming.  Thread (g, q) keeps (best, arg) for 4 columns over
// rows g + RG x: strict '>' within a part (rows ascending), (value, smaller index) merges
// across parts and row groups.  fp32 adds of dyadic inputs are exact, so delta and bp
// equal the fp64 oracle bit for bit.
#include <cuda.h>

#include <atomic>

#include "common.cuh"
#include "kernels.cuh"

namespace tsb {

namespace {
constexpr int kVT = 256;        // consumer threads
constexpr int kVW = kVT / 32;   // consumer warps
constexpr int kRB = 32;         // rows per staged block (one 2-D tensor copy)
constexpr int kRingBytes = 160 * 1024;

__device__ __forceinline__ float max_nan2(float a, float b) {
  float r;
  asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

template <int C, int G>
struct VL {
  static constexpr int CP = C / G;             // columns per CTA
  static constexpr int Q = CP / 4;             // column quads
  static constexpr int RG = kVT / Q;           // row groups
  static constexpr int RPT = kRB / RG;         // rows per thread per block
  static constexpr int NB = C / kRB;           // blocks per step
  static constexpr int NBP = NB / G;           // blocks per part
  static constexpr int BLK = kRB * CP;         // floats per block
  static constexpr int S = kRingBytes / (BLK * 4) > 16 ? 16 : kRingBytes / (BLK * 4);
  static_assert(CP % 4 == 0 && kVT % Q == 0 && RG <= kRB && kRB % RG == 0, "layout");
  static_assert(NBP >= 1 && NB % G == 0, "parts");
  static constexpr size_t ring_f = (size_t)S * BLK;
  static constexpr size_t smem = (ring_f + 2 * C + 3 * RG * CP + 3 * kVW + 2) * 4 +
                                 (2 * S + 2) * 8 + 16;
};

template <int C, int G>
__global__ void __launch_bounds__(kVT + 32, 1) vit2_kernel(VitArgs a, const __grid_constant__ CUtensorMap tm) {
  using L = VL<C, G>;
  extern __shared__ __align__(128) unsigned char smraw[];
  float* ring = reinterpret_cast<float*>(smraw);
  float* dl = ring + L::ring_f;          // [2][C] delta_t, delta_{t+1}
  float* pv = dl + 2 * C;                // [RG][CP] partial best
  int* pi = reinterpret_cast<int*>(pv + L::RG * L::CP);
  float* pc = reinterpret_cast<float*>(pi + L::RG * L::CP);  // NaN probes
  float* redv = pc + L::RG * L::CP;
  int* redi = reinterpret_cast<int*>(redv + kVW);
  float* redb = reinterpret_cast<float*>(redi + kVW);
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(redb + kVW) + 15) & ~static_cast<uintptr_t>(15));
  uint64_t* full = bars;
  uint64_t* empty = bars + L::S;
  uint64_t* dbar = bars + 2 * L::S;  // [2] peers' delta slices landed (cluster scope)

  const int tid = threadIdx.x;
  int h = 0;
  if (G > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(h));
  const int64_t N = a.N, E = N - 1;
  const int64_t b = blockIdx.x / G;
  const int64_t len = seq_len(a.lengths, b, N);
  if (len < 0) {  // uniform over the cluster: nothing staged, no DSMEM traffic
    if (h == 0 && tid == 0) {
      a.zend[b] = -1;
      a.score[b] = qnan();
      if (a.logz) a.logz[b] = qnan();
      if (a.flags) a.flags[b] = TS_F_BADLEN;
    }
    return;
  }
  const int64_t Eb = len - 1;
  if (tid == 0) {
    for (int s = 0; s < L::S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kVW);
    }
    mbar_init(&dbar[0], G > 1 ? G - 1 : 1);
    mbar_init(&dbar[1], G > 1 ? G - 1 : 1);
    fence_mbar_init();
  }
  for (int c = tid; c < C; c += kVT + 32) dl[c] = 0.f;
  if (G > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
  } else {
    __syncthreads();
  }

  if (tid >= kVT) {
    // ---------------- producer warp: one 2-D tensor copy (32 rows x CP columns) per block ---
    const int lane = tid - kVT;
    if (lane == 0) {
      const int64_t total = Eb * L::NB;
      for (int64_t gb = 0; gb < total; ++gb) {
        const int slot = (int)(gb % L::S);
        mbar_wait(&empty[slot], (uint32_t)(((gb / L::S) & 1) ^ 1));
        const int64_t t = gb / L::NB;
        const int k = (int)(gb - t * L::NB);
        const int part = (h + k / L::NBP) % G;
        const int row0 = part * (C / G) + (k % L::NBP) * kRB;
        const int32_t y = (int32_t)((b * E + t) * C + row0), x = h * L::CP;
        mbar_expect_tx(&full[slot], (uint32_t)(L::BLK * 4));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(ring + (size_t)slot * L::BLK)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x), "r"(y), "r"(smem_u32(&full[slot]))
            : "memory");
      }
    }
  } else {
    // ---------------- consumers ------------------------------------------------------------
    const int q = tid % L::Q, g = tid / L::Q, lane = tid & 31, w = tid >> 5;
    int64_t gb = 0;
    for (int64_t t = 0; t < Eb; ++t) {
      const float* d = dl + (t & 1) * C;
      float best[4], chk[4];
      int arg[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        best[c] = neg_inf();
        chk[c] = neg_inf();
        arg[c] = 0x7fffffff;
      }
      for (int kp = 0; kp < G; ++kp) {
        const int part = (h + kp) % G;
        if (G > 1 && kp == 1 && t > 0) mbar_wait_cluster(&dbar[t & 1], (uint32_t)(((t - 1) >> 1) & 1));
        float pb[4];
        int pa[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          pb[c] = neg_inf();
          pa[c] = part * (C / G);
        }
        for (int kb = 0; kb < L::NBP; ++kb, ++gb) {
          const int slot = (int)(gb % L::S);
          mbar_wait(&full[slot], (uint32_t)((gb / L::S) & 1));
          const float* tile = ring + (size_t)slot * L::BLK;
          const int row0 = part * (C / G) + kb * kRB;
#pragma unroll
          for (int x = 0; x < L::RPT; ++x) {
            const int rl = g + L::RG * x;
            const int r = row0 + rl;
            const float dr = d[r];
            const float4 l4 = *reinterpret_cast<const float4*>(tile + rl * L::CP + 4 * q);
            const float v[4] = {dr + l4.x, dr + l4.y, dr + l4.z, dr + l4.w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              chk[c] = max_nan2(chk[c], v[c]);
              if (v[c] > pb[c]) {
                pb[c] = v[c];
                pa[c] = r;
              }
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[slot]);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (pb[c] > best[c] || (pb[c] == best[c] && pa[c] < arg[c])) {
            best[c] = pb[c];
            arg[c] = pa[c];
          }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        pv[g * L::CP + 4 * q + c] = best[c];
        pi[g * L::CP + 4 * q + c] = arg[c];
        pc[g * L::CP + 4 * q + c] = chk[c];
      }
      named_bar(1, kVT);
      if (tid < L::CP) {
        const int j = tid;
        float bv = pv[j], bc = pc[j];
        int bi = pi[j];
        for (int x = 1; x < L::RG; ++x) {
          const float v = pv[x * L::CP + j];
          const int i = pi[x * L::CP + j];
          if (v > bv || (v == bv && i < bi)) {
            bv = v;
            bi = i;
          }
          bc = max_nan2(bc, pc[x * L::CP + j]);
        }
        const float nd = (bc != bc) ? qnan() : bv;
        const int col = h * L::CP + j;
        a.bp[(b * E + t) * C + col] = (uint8_t)bi;
        float* dn = dl + ((t + 1) & 1) * C;
        dn[col] = nd;
        if (G > 1) {
#pragma unroll
          for (int p = 1; p < G; ++p) st_cluster_f32(dn + col, (h + p) % G, nd);
        }
      }
      named_bar(1, kVT);
      // one release-arrive per peer after the barrier covers every thread's DSMEM stores
      if (G > 1 && tid < G - 1) mbar_arrive_cluster(&dbar[(t + 1) & 1], (h + 1 + tid) % G);
    }
    // ---------------- final argmax (rank 0): smallest j attaining max delta_E -------------
    if (h == 0) {
      if (G > 1 && Eb > 0) mbar_wait_cluster(&dbar[Eb & 1], (uint32_t)(((Eb - 1) >> 1) & 1));
      const float* d = dl + (Eb & 1) * C;
      float v = neg_inf(), bad = neg_inf();
      int idx = 0x7fffffff;
      for (int c = tid; c < C; c += kVT) {
        const float x = d[c];
        bad = max_nan2(bad, x);
        if (x > v || (x == v && c < idx)) {
          v = x;
          idx = c;
        }
      }
      if (idx == 0x7fffffff) idx = 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        bad = max_nan2(bad, __shfl_xor_sync(0xffffffffu, bad, o));
        if (ov > v || (ov == v && oi < idx)) {
          v = ov;
          idx = oi;
        }
      }
      if (lane == 0) {
        redv[w] = v;
        redi[w] = idx;
        redb[w] = bad;
      }
      named_bar(1, kVT);
      if (tid == 0) {
        float bv = redv[0], bb = redb[0];
        int bi = redi[0];
        for (int x = 1; x < kVW; ++x) {
          if (redv[x] > bv || (redv[x] == bv && redi[x] < bi)) {
            bv = redv[x];
            bi = redi[x];
          }
          bb = max_nan2(bb, redb[x]);
        }
        uint32_t fl = 0;
        float sc = bv;
        int z = bi;
        if (bb != bb || bb == pos_inf()) {
          fl = TS_F_NONFINITE;
          sc = qnan();
          z = -1;
        } else if (bv == neg_inf()) {
          fl = TS_F_EMPTY;
          z = -1;
        }
        a.zend[b] = z;
        a.score[b] = sc;
        if (a.logz) a.logz[b] = sc;
        if (a.flags) a.flags[b] = fl;
      }
    }
  }
  if (G > 1)  // no CTA leaves while a peer may still write into its shared memory
    asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}

std::atomic<uint64_t> g_vit2_attr{0};

// cuTensorMapEncodeTiled through the runtime's driver entry point: the library then has no
// link-time dependency on libcuda.so (it loads on hosts without a driver; the CPU ABI tests).
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
PFN_encodeTiled resolve_encode_tiled() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<PFN_encodeTiled>(fn);
}

template <int C, int G>
cudaError_t launch_cg(const VitArgs& a, cudaStream_t st, int bit) {
  using L = VL<C, G>;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t m = 1ull << ((dev & 7) * 8 + bit);
  if (!(g_vit2_attr.load() & m)) {
    cudaError_t e = cudaFuncSetAttribute(vit2_kernel<C, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)L::smem);
    if (e != cudaSuccess) return e;
    if (G > 1) {
      e = cudaFuncSetAttribute(vit2_kernel<C, G>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    g_vit2_attr.fetch_or(m);
  }
  CUtensorMap tm;
  {
    const cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)(a.B * (a.N - 1) * C)};
    const cuuint64_t strides[1] = {(cuuint64_t)C * 4};
    const cuuint32_t box[2] = {(cuuint32_t)L::CP, (cuuint32_t)kRB};
    const cuuint32_t estr[2] = {1, 1};
    static PFN_encodeTiled encode = resolve_encode_tiled();
    if (!encode) return cudaErrorNotSupported;
    if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a.pot), dims,
                               strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.B * G), 1, 1);
  cfg.blockDim = dim3(kVT + 32, 1, 1);
  cfg.dynamicSmemBytes = L::smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, vit2_kernel<C, G>, a, tm);
}
}  // namespace

bool vit2_ok(const VitArgs& a) {
  // tensor-map row coordinates are int32: B*(N-1)*C rows must fit
  return (a.C == 128 || a.C == 256) && (reinterpret_cast<uintptr_t>(a.pot) & 15) == 0 &&
         a.N > 1 && a.B * (a.N - 1) * a.C < ((int64_t)1 << 31);
}

// cluster size: the largest G in {1, 2, 4} with B*G <= #SMs (C/G >= 32 columns per CTA),
// or the debug override g_force (0 = auto).
cudaError_t launch_vit2(const VitArgs& a, int g_force, cudaStream_t st) {
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int G = 1;
  if (g_force > 0) {
    G = g_force;
  } else {
    // at most 4 CTAs per sequence: G = 8 measured slower than G = 4 at every batch
    // (cfg4 shape, B = 8..64; profiles/r2_shard_shapes.jsonl)
    const int gmax = (int)(a.C / 32) < 4 ? (int)(a.C / 32) : 4;
    while (2 * G <= gmax && a.B * 2 * G <= sms) G *= 2;
  }
  if (a.C == 256) {
    switch (G) {
      case 1: return launch_cg<256, 1>(a, st, 0);
      case 2: return launch_cg<256, 2>(a, st, 1);
      case 4: return launch_cg<256, 4>(a, st, 2);
      case 8: return launch_cg<256, 8>(a, st, 3);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (G) {
    case 1: return launch_cg<128, 1>(a, st, 4);
    case 2: return launch_cg<128, 2>(a, st, 5);
    case 4: return launch_cg<128, 4>(a, st, 6);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tsb
