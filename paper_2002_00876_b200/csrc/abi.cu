// abi.cu — the C ABI (include/ts_b200.h): validation, plan selection, workspace layout
// and dispatch to the sm_100a kernels.  No CPU compute path exists: on a non-sm_100
// device every entry point returns TS_E_UNSUPPORTED.
#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "kernels.cuh"
#include "ts_b200.h"

using namespace tsb;

namespace {

std::atomic<int64_t> g_plan_chunk{0};
std::atomic<int> g_small_cluster{0};  // short chains: 0 one CTA (default), -1 auto cluster scan, 2/4 forced G
std::atomic<int> g_meet{1};
std::atomic<int> g_tiny{1};    // short chains: 1 = fb_tiny when eligible, 0 = fb_small only
std::atomic<int> g_vsplit{0};  // Viterbi: -1 one CTA per sequence, 0 auto, G forced cluster size  // meet-in-the-middle marginals kernel for C = 64  // debug: run short C<=32 chains on G-CTA clusters
thread_local int t_launches = 0;
thread_local const char* t_kernel = "";  // dominant kernel of the last call (bench / profiling)

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

// Bump allocator over the caller's workspace.
struct Carve {
  char* base;
  size_t off = 0;
  explicit Carve(void* p) : base(static_cast<char*>(p)) {}
  template <typename T>
  T* take(size_t n) {
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off = align_up(off + n * sizeof(T));
    return p;
  }
};

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

bool chain_ok(const ts_chain* c) {
  if (!c) return false;
  if (c->B < 1 || c->N < 1 || c->C < 1 || c->C > 256) return false;
  if (c->B > (int64_t)1 << 31 || c->N > (int64_t)1 << 40) return false;
  const double elems = (double)c->B * (double)(c->N - 1) * (double)c->C * (double)c->C;
  if (elems > 9.0e18) return false;
  if (c->N > 1 && (!c->pot || !aligned(c->pot, 16))) return false;
  if (c->lengths && !aligned(c->lengths, 4)) return false;
  return true;
}

// sm_100 (B200) check, cached per device.
std::atomic<int> g_dev_ok[64];
bool device_ok() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  if (dev < 0 || dev >= 64) return false;
  int v = g_dev_ok[dev].load();
  if (v == 0) {
    int maj = 0, min = 0;
    cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&min, cudaDevAttrComputeCapabilityMinor, dev);
    v = (maj == 10 && min == 0) ? 1 : 2;
    g_dev_ok[dev].store(v);
  }
  return v == 1;
}

enum class PlanKind { Small, Stream, Unsupported };
struct Plan {
  PlanKind kind;
  int64_t L, P, Ppad;
  int H;
};

// Plan selection: the fused small kernel for short chains with C <= 32;
// otherwise the streaming sweeps, time-chunked with the scan tree when the batch alone
// cannot fill the GPU (or when the debug knob asks for a chunk length).
// SM count of the current device (cached per device: the plan is chosen on every call).
int device_sms() {
  static std::atomic<int> cache[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev >= 0 && dev < 64) {
    const int v = cache[dev].load(std::memory_order_relaxed);
    if (v > 0) return v;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cache[dev].store(sms, std::memory_order_relaxed);
  return sms;
}

// Chunk length of the auto plan, 0 = serial (P = 1).  Calibrated on B200 (tools/plan_calib.py,
// profiles/r2_plan_calib.jsonl; ms = one ts_marginals call):
//   serial:  meet64 (C = 64) ~1.2 us per edge, fwd2+bwd2 ~2.6 us (C <= 32) / ~4.9 us (C = 128)
//            per edge, times ceil(B / #SMs) waves;
//   chunked: C <= 64 (SIMT summaries, C^3 per edge): ~0.39 + 4.5e-5 B E ms (C = 64) and
//            ~0.45 + 1.1e-5 B E ms (C = 32) with L = 64 (the best of 32..1024 in every shape);
//            C <= 32 beyond the one-CTA kernels' shared memory: always chunked, L = 16 / 32
//            (profiles/r2_ablations.jsonl X4: 5-8x faster than the serial sweeps at N >= 128);
//            C = 128 (tensor-core summaries): best L = E / floor(#SMs / B), at least 128
//            (one wave of chunk summaries; cfg5: 37 chunks of 1772 edges, 17.7 ms, vs 32
//            chunks of 2048, 20.1 ms).
// The serial plan wins for C = 64 once B >~ 30 (e.g. every per-rank shape of cfg3's batch
// sharding: B = 256 / G); chunking pays for few long sequences (cfg5).
int64_t auto_chunk(int64_t B, int64_t E, int64_t C, int sms) {
  if (E < 64 && C > 32) return 0;
  const double waves = (double)((B + sms - 1) / sms);
  if (C > 64) {
    if (2 * B > sms) return 0;
    const int64_t per = sms / B;  // chunks per sequence that keep one wave of summaries
    const int64_t L = (E + per - 1) / per;
    return L < 128 ? 128 : L;
  }
  if (C <= 32) {  // the generic serial sweeps cost 2.6-4.3 us per edge here: chunk from E >= 32
    if (E < 32) return 0;
    return E <= 1024 ? 16 : 32;  // X4 ablation (B16 C20 N 64..512): L = 16 best, 0.20-0.38 ms
  }
  const bool meet = (C == 64);
  const double serial_ms = (meet ? 1.2e-3 : 2.6e-3) * (double)E * waves;
  const double chunk_ms = 0.39 + 4.5e-5 * (double)(B * E);
  return chunk_ms < serial_ms ? 64 : 0;
}

Plan log_plan(const ts_chain* c) {
  const int64_t knob = g_plan_chunk.load();
  const int64_t E = c->N - 1;
  Plan p{PlanKind::Stream, E > 0 ? E : 1, 1, 1, 0};
  int64_t P = 1;
  if (knob == 0) {
    if (small_fits(c->N, c->C)) {
      p.kind = PlanKind::Small;
      return p;
    }
    const int sms = device_sms();
    const int64_t L = auto_chunk(c->B, E, c->C, sms);
    if (L > 0 && L < E) P = (E + L - 1) / L;
  } else if (knob < E) {
    P = (E + knob - 1) / knob;
  } else if (small_fits(c->N, c->C)) {
    p.kind = PlanKind::Small;
    return p;
  }
  if (c->C > 128) {
    p.kind = PlanKind::Unsupported;
    return p;
  }
  if (P > 1) {
    p.P = P;
    p.L = (knob > 0 && knob < E) ? knob : (E + P - 1) / P;
    p.P = (E + p.L - 1) / p.L;
    int64_t pp = 1;
    int h = 0;
    while (pp < p.P) {
      pp <<= 1;
      ++h;
    }
    p.Ppad = pp;
    p.H = h;
  }
  return p;
}

// Workspace layout of the streaming log path.
struct StreamWs {
  float* alpha_hat = nullptr;
  float* mlag = nullptr;
  float* tmax = nullptr;
  float* alpha_end = nullptr;
  double* alpha_end_off = nullptr;
  uint32_t* wflags = nullptr;
  float* beta_hat = nullptr;  // meet-in-the-middle kernel only (P == 1, C == 64)
};
struct ScanWs {
  float* mat = nullptr;
  double* off = nullptr;
  uint8_t* ident = nullptr;
  uint32_t* cflag = nullptr;
  float* valpha = nullptr;
  double* oalpha = nullptr;
  float* vbeta = nullptr;
  double* obeta = nullptr;
  float* leaf_alpha = nullptr;
  double* leaf_alpha_off = nullptr;
  float* leaf_beta = nullptr;
  double* leaf_beta_off = nullptr;
};
size_t stream_ws(const ts_chain* c, const Plan& pl, bool marg, void* ws, StreamWs* out,
                 ScanWs* sout, bool force_tree = false) {
  Carve cv(ws);
  StreamWs w;
  ScanWs s;
  const int64_t B = c->B, N = c->N, C = c->C, E = N - 1, P = pl.P;
  if (marg) {
    w.alpha_hat = cv.take<float>((size_t)(B * N * C));
    w.mlag = cv.take<float>((size_t)(B * N));
    w.tmax = cv.take<float>((size_t)(B * (E > 0 ? E : 1)));
    if (P == 1 && !force_tree && C == 64) w.beta_hat = cv.take<float>((size_t)(B * N * C));
  }
  w.alpha_end = cv.take<float>((size_t)(B * P * C));
  w.alpha_end_off = cv.take<double>((size_t)(B * P));
  w.wflags = cv.take<uint32_t>((size_t)B);
  if (P > 1 || force_tree) {
    const int64_t nodes = 2 * pl.Ppad - 1;
    s.mat = cv.take<float>((size_t)(B * nodes * C * C));
    s.off = cv.take<double>((size_t)(B * nodes * C));
    s.ident = cv.take<uint8_t>((size_t)(B * nodes));
    s.cflag = cv.take<uint32_t>((size_t)(B * pl.Ppad));
    if (marg) {
      s.valpha = cv.take<float>((size_t)(B * nodes * C));
      s.oalpha = cv.take<double>((size_t)(B * nodes));
      s.vbeta = cv.take<float>((size_t)(B * nodes * C));
      s.obeta = cv.take<double>((size_t)(B * nodes));
      s.leaf_alpha = cv.take<float>((size_t)(B * P * C));
      s.leaf_alpha_off = cv.take<double>((size_t)(B * P));
      s.leaf_beta = cv.take<float>((size_t)(B * P * C));
      s.leaf_beta_off = cv.take<double>((size_t)(B * P));
    }
  }
  if (out) *out = w;
  if (sout) *sout = s;
  return cv.off;
}

// Chunk length of the single-GPU time-chunked Viterbi (vchunk.cu), 0 = the serial sweep.
// Knob (ts_set_plan_chunk): 1 <= L < E forces chunks of L edges.  Auto (calibrated,
// tools/vchunk_calib.py -> profiles/r2_vchunk_calib.jsonl): the serial sweeps cost ~1.5 us
// per edge whatever B (one dependent step per edge: vit2 for C = 128, viterbi_fwd below);
// the chunked scan with the register-blocked summaries (C in {32, 64, 128}) costs, once its
// chunks fill the GPU, K(C) us per (sequence x edge) — 0.145 (C = 128, one 256-thread CTA
// per SM), 0.020 (C = 64, four per SM), 0.007 (C = 32) — so it is chosen when
// B K(C) < 0.7 x 1.5 us and the chains are long (E >= 256), with enough chunks per sequence
// for one wave of NSEG(C) = #SMs x {1, 4, 8} CTAs.
int64_t vit_chunk(const ts_chain* c) {
  const int64_t knob = g_plan_chunk.load();
  const int64_t B = c->B, C = c->C, E = c->N - 1;
  if (E < 2 || !vchunk_ok(C)) return 0;
  if (knob > 0) return knob < E ? knob : 0;
  if (E < 256 || !vchunk_mm(C) || B < 1 || (reinterpret_cast<uintptr_t>(c->pot) & 15) != 0) return 0;
  const double K = C == 128 ? 0.145 : C == 64 ? 0.020 : 0.007;
  if ((double)B * K >= 0.7 * 1.5) return 0;
  const int64_t nseg = (int64_t)device_sms() * (C == 128 ? 1 : C == 64 ? 4 : 8);
  const int64_t per = nseg / B;
  if (per < 2) return 0;
  return (E + per - 1) / per;
}

struct VitWs {
  uint8_t* bp = nullptr;
  int32_t* zend = nullptr;
  int32_t* path = nullptr;
  float* score = nullptr;
  // chunked plan
  int64_t L = 0, P = 0;
  float* summ = nullptr;
  float* din = nullptr;
  int32_t* maps = nullptr;
  int32_t* czend = nullptr;
  int32_t* zglob = nullptr;
};
size_t vit_ws(const ts_chain* c, bool need_path, bool need_score, void* ws, VitWs* out) {
  Carve cv(ws);
  VitWs w;
  const int64_t B = c->B, N = c->N, C = c->C, E = N - 1;
  w.bp = cv.take<uint8_t>((size_t)(B * (E > 0 ? E : 1) * C));
  w.zend = cv.take<int32_t>((size_t)B);
  if (need_path) w.path = cv.take<int32_t>((size_t)(B * N));
  if (need_score) w.score = cv.take<float>((size_t)B);
  const int64_t L = vit_chunk(c);
  if (L > 0) {
    w.L = L;
    w.P = (E + L - 1) / L;
    w.summ = cv.take<float>((size_t)(B * w.P * C * C));
    w.din = cv.take<float>((size_t)(B * w.P * C));
    w.maps = cv.take<int32_t>((size_t)(B * w.P * C));
    w.czend = cv.take<int32_t>((size_t)(B * w.P));
    w.zglob = cv.take<int32_t>((size_t)B);
    if (!w.path) w.path = cv.take<int32_t>((size_t)(B * N));  // the chunked backtrack's target
  }
  if (out) *out = w;
  return cv.off;
}

// workspace of the exact SIMT segmental kernel (semimarkov.cu), also the K = 1 fallback of
// the log semiring for long chains with 128 < C <= 256
size_t semi_ws(const ts_chain* c, int64_t K, void* ws, SemiArgs* a) {
  Carve cv(ws);
  const int64_t B = c->B, N = c->N, C = c->C;
  float* ah = cv.take<float>((size_t)(B * N * C));
  float* bh = cv.take<float>((size_t)(B * N * C));
  double* ao = cv.take<double>((size_t)(B * N));
  double* bo = cv.take<double>((size_t)(B * N));
  double* zb = cv.take<double>((size_t)B);
  if (a) {
    a->ah = ah;
    a->bh = bh;
    a->ao = ao;
    a->bo = bo;
    a->zbuf = zb;
    a->K = K;
  }
  return cv.off;
}

size_t op_ws(const ts_chain* c, int op, ts_semiring s, void* ws, StreamWs* sw, VitWs* vw) {
  if (s == TS_MAX) {
    switch (op) {
      case TS_OP_LOGZ: return vit_ws(c, false, true, ws, vw);
      case TS_OP_MARG: return vit_ws(c, true, true, ws, vw);
      case TS_OP_VITERBI: return vit_ws(c, false, false, ws, vw);
      default: return 0;
    }
  }
  if (op == TS_OP_VITERBI) return vit_ws(c, false, false, ws, vw);
  const Plan p = log_plan(c);
  if (p.kind == PlanKind::Unsupported) return c->C <= 256 ? semi_ws(c, 1, ws, nullptr) : 0;
  if (p.kind != PlanKind::Stream) return 0;
  return stream_ws(c, p, op == TS_OP_MARG, ws, sw, nullptr);
}

ts_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return TS_OK;
  cudaGetLastError();  // clear sticky launch error state where possible
  return TS_E_CUDA;
}

// A request to fuse the f1 reduction (entropy: Σ mu·l, expectation: Σ mu·r) into the marginal
// kernel of the plan.  run_log sets `fused` when the plan's kernel did it:
// with `final_partials` > 0 the kernel left that many fp64 partials per sequence in `partial`
// (the caller runs the final stage), else it wrote `out` itself.
struct FusedX {
  int mode;          // 1 entropy, 2 expectation
  const float* r;    // expectation feature
  float* out;        // [B]
  double* partial;   // [B][final_partials]
  bool fused = false;
  int final_partials = 0;
};

ts_status run_log(const ts_chain* c, float* marg, float* logz, uint32_t* flags, void* ws,
                  size_t ws_bytes, cudaStream_t st, FusedX* fx = nullptr) {
  const Plan p = log_plan(c);
  if (p.kind == PlanKind::Unsupported) {
    if (c->C > 256) return TS_E_UNSUPPORTED;
    // long chains with 128 < C <= 256: forward and backward recursion CTAs concurrently
    // (exact per-cell LSE), then a machine-wide marginal pass (fb_wide.cu); the workspace is
    // the segmental kernel's with K = 1
    SemiArgs sa{};
    const size_t need = semi_ws(c, 1, ws, &sa);
    if (ws_bytes < need || !ws || !aligned(ws, kAlign)) return TS_E_WORKSPACE;
    sa.pot = c->pot;
    sa.lengths = c->lengths;
    sa.B = c->B;
    sa.N = c->N;
    sa.C = c->C;
    sa.marg = marg;
    sa.logz = logz;
    sa.flags = flags;
    ts_status r = cuda_status(launch_fb_wide(sa, st));
    if (r == TS_OK) {
      t_launches = (marg && c->N > 1) ? 2 : 1;
      t_kernel = "fb_wide_sweep_kernel";
    }
    return r;
  }
  if (p.kind == PlanKind::Small) {
    SmallArgs a{c->pot, c->lengths, c->B, c->N, c->C, marg, logz, flags};
    const int knob = g_small_cluster.load();
    const bool fuse = fx && marg && g_tiny.load() && tiny_fits(a);
    int G = 0;
    if (fuse)
      G = 0;  // the fused epilogue lives in the one-CTA body
    else if (knob < 0)
      G = g_tiny.load() ? cscan_g(a, device_sms()) : 0;
    else if (cscan_fits(a, knob))
      G = knob;
    ts_status r;
    if (G > 1) {
      r = cuda_status(launch_cscan(a, G, st));
      t_kernel = "fb_cscan_kernel";
    } else if (g_tiny.load() && tiny_fits(a)) {
      if (fuse) {
        a.xmode = fx->mode;
        a.xr = fx->r;
        a.xout = fx->out;
        fx->fused = true;
        fx->final_partials = 0;
      }
      r = cuda_status(launch_tiny(a, st));
      t_kernel = "fb_tiny_kernel";
    } else {
      r = cuda_status(launch_small(a, st));
      t_kernel = "fb_small_kernel";
    }
    if (r == TS_OK) t_launches = 1;
    return r;
  }
  StreamWs w;
  ScanWs sw;
  const size_t need = stream_ws(c, p, marg != nullptr, ws, &w, &sw);
  if (ws_bytes < need || (need && (!ws || !aligned(ws, kAlign)))) return TS_E_WORKSPACE;
  cudaError_t e;
  if (marg && p.P == 1 && w.beta_hat && meet_ok(c->C, c->pot, marg) && g_meet.load()) {
    MeetArgs m{c->pot, c->lengths, c->B, c->N, marg, logz, flags,
               w.alpha_hat, w.beta_hat, w.mlag, w.tmax};
    if (fx) {
      m.xmode = fx->mode;
      m.xr = fx->r;
      m.xsum = fx->partial;
      fx->fused = true;
      fx->final_partials = 2;  // one per engine
    }
    if ((e = launch_meet(m, c->C, st)) != cudaSuccess) return cuda_status(e);
    t_launches = 1;
    t_kernel = "meet64_kernel";
    return TS_OK;
  }
  e = cudaMemsetAsync(w.wflags, 0, sizeof(uint32_t) * (size_t)c->B, st);
  if (e != cudaSuccess) return cuda_status(e);
  int n = 0;
  ScanArgs sa{};
  if (p.P > 1) {
    sa.pot = c->pot;
    sa.lengths = c->lengths;
    sa.B = c->B;
    sa.N = c->N;
    sa.C = c->C;
    sa.L = p.L;
    sa.P = p.P;
    sa.Ppad = p.Ppad;
    sa.nodes = 2 * p.Ppad - 1;
    sa.H = p.H;
    sa.mat = sw.mat;
    sa.off = sw.off;
    sa.ident = sw.ident;
    sa.cflag = sw.cflag;
    sa.valpha = sw.valpha;
    sa.oalpha = sw.oalpha;
    sa.vbeta = sw.vbeta;
    sa.obeta = sw.obeta;
    sa.leaf_alpha = sw.leaf_alpha;
    sa.leaf_alpha_off = sw.leaf_alpha_off;
    sa.leaf_beta = sw.leaf_beta;
    sa.leaf_beta_off = sw.leaf_beta_off;
    sa.wflags = w.wflags;
    sa.logz = logz;
    sa.flags = flags;
    t_kernel = summary_tc_ok(sa) ? "summary_tc_kernel" : "summary_fast_kernel";
    if ((e = launch_scan_up(sa, st, &n)) != cudaSuccess) return cuda_status(e);
    if (!marg) {  // logZ from the root of the Fig. 4 tree
      if ((e = launch_scan_logz(sa, st)) != cudaSuccess) return cuda_status(e);
      t_launches = n + 1;
      return TS_OK;
    }
    if ((e = launch_scan_down(sa, st, &n, true)) != cudaSuccess) return cuda_status(e);
  }
  SweepArgs a{};
  a.pot = c->pot;
  a.lengths = c->lengths;
  a.B = c->B;
  a.N = c->N;
  a.C = c->C;
  a.L = p.L;
  a.P = p.P;
  a.alpha_in = sw.leaf_alpha;
  a.alpha_in_off = sw.leaf_alpha_off;
  a.beta_out = sw.leaf_beta;
  a.beta_out_off = sw.leaf_beta_off;
  a.alpha_hat = w.alpha_hat;
  a.alpha_end = w.alpha_end;
  a.alpha_end_off = w.alpha_end_off;
  a.mlag = w.mlag;
  a.tmax = w.tmax;
  a.marg = marg;
  a.wflags = w.wflags;
  a.logz = logz;
  a.flags = flags;
  a.final_in_fwd = marg ? 0 : 1;
  if (p.P == 1)
    t_kernel = stream2_ok(a) ? (marg ? "bwd2_kernel" : "fwd2_kernel")
                             : (marg ? "bwd_sweep_kernel" : "fwd_sweep_kernel");
  e = launch_fwd(a, st);
  if (e != cudaSuccess) return cuda_status(e);
  ++n;
  if (marg) {
    e = launch_bwd(a, st);
    if (e != cudaSuccess) return cuda_status(e);
    ++n;
  }
  t_launches = n;
  return TS_OK;
}

ts_status run_max(const ts_chain* c, int op, float* marg, float* logz, int32_t* path,
                  float* score, uint32_t* flags, void* ws, size_t ws_bytes, cudaStream_t st) {
  VitWs w;
  const bool need_path = (op == TS_OP_MARG);
  const size_t need = vit_ws(c, need_path, op != TS_OP_VITERBI, ws, &w);
  if (ws_bytes < need || !ws || !aligned(ws, kAlign)) return TS_E_WORKSPACE;
  VitArgs a{};
  a.pot = c->pot;
  a.lengths = c->lengths;
  a.B = c->B;
  a.N = c->N;
  a.C = c->C;
  a.bp = w.bp;
  a.zend = w.zend;
  a.score = score ? score : w.score;
  a.flags = flags;
  a.path = path ? path : w.path;
  a.marg = marg;
  a.logz = logz;
  if (w.P > 0) {  // time-chunked max-plus scan (vchunk.cu)
    VChunkArgs v{};
    v.pot = c->pot;
    v.lengths = c->lengths;
    v.B = c->B;
    v.N = c->N;
    v.C = c->C;
    v.L = w.L;
    v.P = w.P;
    v.summ = w.summ;
    v.din = w.din;
    v.bp = w.bp;
    v.maps = w.maps;
    v.zend = w.czend;
    v.zglob = w.zglob;
    v.score = a.score;
    v.logz = logz;
    v.flags = flags;
    v.path = a.path;
    const bool want_path = (path != nullptr) || (marg != nullptr);
    int n = 0;
    cudaError_t e = launch_vchunk(v, want_path, st, &n);
    if (e == cudaSuccess && marg) {
      e = launch_indicator(a, st);
      ++n;
    }
    if (e != cudaSuccess) return cuda_status(e);
    t_launches = n;
    t_kernel = vchunk_mm(c->C) ? "vch_summary_mm_kernel" : "vch_summary_kernel";
    return TS_OK;
  }
  int n = 0;
  ts_status r = cuda_status(launch_viterbi(a, st, &n, g_vsplit.load()));
  if (r == TS_OK) t_launches = n;
  t_kernel = (g_vsplit.load() >= 0 && vit2_ok(a)) ? "vit2_kernel" : "viterbi_fwd_kernel";
  return r;
}

// Plan of a time-sharded segment: always the scan tree (P >= 1), chunked like log_plan.
Plan seg_plan(const ts_chain* c) {
  Plan p = log_plan(c);
  const int64_t E = c->N - 1;
  if (p.kind == PlanKind::Small) {  // segments always run through the tree
    p.kind = PlanKind::Stream;
    p.P = 1;
    p.L = E > 0 ? E : 1;
  }
  if (p.P <= 1) {
    p.P = 1;
    p.Ppad = 1;
    p.H = 0;
    p.L = E > 0 ? E : 1;
  }
  return p;
}

ScanArgs make_scan(const ts_chain* c, const Plan& p, const StreamWs& w, const ScanWs& sw,
                   float* logz, uint32_t* flags) {
  ScanArgs sa{};
  sa.pot = c->pot;
  sa.lengths = c->lengths;
  sa.B = c->B;
  sa.N = c->N;
  sa.C = c->C;
  sa.L = p.L;
  sa.P = p.P;
  sa.Ppad = p.Ppad;
  sa.nodes = 2 * p.Ppad - 1;
  sa.H = p.H;
  sa.mat = sw.mat;
  sa.off = sw.off;
  sa.ident = sw.ident;
  sa.cflag = sw.cflag;
  sa.valpha = sw.valpha;
  sa.oalpha = sw.oalpha;
  sa.vbeta = sw.vbeta;
  sa.obeta = sw.obeta;
  sa.leaf_alpha = sw.leaf_alpha;
  sa.leaf_alpha_off = sw.leaf_alpha_off;
  sa.leaf_beta = sw.leaf_beta;
  sa.leaf_beta_off = sw.leaf_beta_off;
  sa.wflags = w.wflags;
  sa.logz = logz;
  sa.flags = flags;
  return sa;
}

bool seg_ok(const ts_chain* c, int64_t edge_begin, int64_t n_global) {
  return chain_ok(c) && c->lengths == nullptr && edge_begin >= 0 &&
         edge_begin + (c->N - 1) <= n_global - 1 && c->C <= 128;
}

// ts_marginals_host pipelining: the batch is cut into K chunks, each on its own library
// stream (H2D -> kernels -> D2H), so chunk k's copy back overlaps chunk k+1's kernels and
// copy in (the two copy directions run on separate engines).  Chunks of >= 4 MB.
#ifndef TS_HOST_MAX_CHUNKS
#define TS_HOST_MAX_CHUNKS 4
#endif
constexpr int kHostMaxChunks = TS_HOST_MAX_CHUNKS;
int host_chunks(int64_t B, int64_t per_seq_floats) {
  // >= 4 MB per chunk: splitting a 1.2 MB transfer into 4 streams measured slower on the
  // GPU boxes (cfg2 e2e 103 -> 77 us/step with one chunk; tools/e2e_ab.py)
  const int64_t bytes = B * per_seq_floats * 4;
  int64_t k = bytes / (4 << 20);
  if (k > kHostMaxChunks) k = kHostMaxChunks;
  if (k > B) k = B;
  return k < 1 ? 1 : (int)k;
}

std::atomic<int> g_host_graphs{1};
std::atomic<int> g_host_pipeline{2};  // 2 = three-stage, 1 = two-stream, 0 = stream order

struct HostKey {
  int64_t B, N, C;
  const float* pot;
  const int32_t* lengths;
  int s;
  float* marg;
  float* logz;
  uint32_t* flags;
  void* ws;
  size_t ws_bytes;
  int64_t plan_chunk;
  int64_t knobs;  // every kernel-selection knob (knob_word): a toggle never replays a stale graph
  bool operator==(const HostKey& o) const {
    return B == o.B && N == o.N && C == o.C && pot == o.pot && lengths == o.lengths && s == o.s &&
           marg == o.marg && logz == o.logz && flags == o.flags && ws == o.ws &&
           ws_bytes == o.ws_bytes && plan_chunk == o.plan_chunk && knobs == o.knobs;
  }
};

// All debug knobs that change which kernels a call enqueues, packed into one key word.
int64_t knob_word() {
  return (int64_t)g_meet.load() | ((int64_t)g_small_cluster.load() << 1) |
         ((int64_t)tsb::get_tc_summary() << 4) | ((int64_t)g_tiny.load() << 8) |
         ((int64_t)(g_vsplit.load() + 1) << 9) | ((int64_t)(tsb::g_wide_ring != 0) << 14) |
         ((int64_t)tsb::get_tiny_early() << 15);
}

struct HostGraph {
  HostKey key;
  cudaGraphExec_t exec = nullptr;
  int launches = 0;
  uint64_t used = 0;
};

constexpr int kHostGraphs = 16;

struct HostPipe {
  std::mutex mu;
  cudaStream_t side[kHostMaxChunks];
  cudaStream_t cap;
  cudaEvent_t fork, join[kHostMaxChunks];
  // cross-call pipeline (single-chunk payloads): inputs copied on `cin` into one of two
  // staging buffers; ev_in[p] = copy-in done, ev_done[p] = the call that used buffer p done
  cudaStream_t cin;
  cudaEvent_t ev_in[2], ev_done[2];
  // three-stage pipeline (pipeline mode 2): copy-in on `cin`, kernels on `ck`, copy-back on
  // `cout`, input and output staging double-buffered; e3_in / e3_k / e3_out[p] = the copy-in,
  // kernels, copy-back of the last call that used buffer set p
  cudaStream_t ck, cout;
  cudaEvent_t e3_in[2], e3_k[2], e3_out[2], e3_fork;
  bool p3_primed[2] = {false, false};
  int p3_parity = 0;
  int64_t p3_sig[5] = {0, 0, 0, 0, 0};
  // the previous call (any path) and its stream: a call on another stream orders after it,
  // since all calls share the device staging buffers and the inner workspace
  cudaEvent_t ev_last;
  cudaStream_t last_st = nullptr;
  bool has_last = false;
  int parity = 0;
  bool primed[2] = {false, false};
  int64_t sig[5] = {0, 0, 0, 0, 0};  // (B, N, C, ws, semiring) of the last pipelined call
  HostGraph graphs[kHostGraphs];
  int n_graphs = 0;
  uint64_t clock = 0;
  HostGraph* find(const HostKey& k) {
    for (int i = 0; i < n_graphs; ++i)
      if (graphs[i].key == k) {
        graphs[i].used = ++clock;
        return &graphs[i];
      }
    return nullptr;
  }
  void insert(const HostKey& k) {
    int slot = n_graphs;
    if (n_graphs == kHostGraphs) {  // evict the least recently used binding
      slot = 0;
      for (int i = 1; i < kHostGraphs; ++i)
        if (graphs[i].used < graphs[slot].used) slot = i;
      if (graphs[slot].exec) cudaGraphExecDestroy(graphs[slot].exec);
    } else {
      ++n_graphs;
    }
    graphs[slot].key = k;
    graphs[slot].exec = nullptr;
    graphs[slot].launches = 0;
    graphs[slot].used = ++clock;
  }
};

// One-time per-device setup (streams + events; never allocated in the hot call again).
HostPipe* host_pipe() {
  static std::mutex init_mu;
  static HostPipe* pipes[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(init_mu);
  if (!pipes[dev]) {
    HostPipe* p = new HostPipe;
    bool ok = cudaEventCreateWithFlags(&p->fork, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventCreateWithFlags(&p->ev_last, cudaEventDisableTiming) == cudaSuccess &&
              cudaStreamCreateWithFlags(&p->cap, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&p->cin, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&p->ck, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamCreateWithFlags(&p->cout, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&p->e3_fork, cudaEventDisableTiming) == cudaSuccess;
    for (int k = 0; k < 2 && ok; ++k)
      ok = cudaEventCreateWithFlags(&p->ev_in[k], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&p->ev_done[k], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&p->e3_in[k], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&p->e3_k[k], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&p->e3_out[k], cudaEventDisableTiming) == cudaSuccess;
    for (int k = 0; k < kHostMaxChunks && ok; ++k)
      ok = cudaStreamCreateWithFlags(&p->side[k], cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&p->join[k], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
      delete p;
      return nullptr;
    }
    pipes[dev] = p;
  }
  return pipes[dev];
}


// ---- distribution properties ------------------------------------------
size_t entropy_ws(const ts_chain* c, void* ws, size_t* marg_part, double** partial) {
  const size_t m = align_up(op_ws(c, TS_OP_MARG, TS_LOG, nullptr, nullptr, nullptr));
  DistArgs d{};
  d.B = c->B;
  d.N = c->N;
  const int S = entropy_slices(d) < 2 ? 2 : entropy_slices(d);  // >= 2: fused meet64 partials
  if (marg_part) *marg_part = m;
  if (partial) *partial = ws ? reinterpret_cast<double*>(static_cast<char*>(ws) + m) : nullptr;
  return m + align_up(sizeof(double) * (size_t)(c->B * S));
}

Plan serial_plan(const ts_chain* c) {
  const int64_t E = c->N - 1;
  return Plan{PlanKind::Stream, E > 0 ? E : 1, 1, 1, 0};
}

size_t sample_ws(const ts_chain* c, void* ws, StreamWs* w, uint32_t** fl) {
  const size_t m = align_up(stream_ws(c, serial_plan(c), true, ws, w, nullptr));
  if (fl) *fl = ws ? reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + m) : nullptr;
  return m + align_up(sizeof(uint32_t) * (size_t)c->B);
}


// ---- time-sharded Viterbi segments (vseg.cu) ----------------------------------------------
struct VsegWs {
  uint8_t* bp = nullptr;
  float* delta_in = nullptr;
  float* lscore = nullptr;   // local forward's score (unused)
  int32_t* lzend = nullptr;  // local forward's argmax, then this segment's end label
  int32_t* zglob = nullptr;
  float* gscore = nullptr;
  uint32_t* gflags = nullptr;
};
size_t vseg_ws(const ts_chain* c, void* ws, VsegWs* out) {
  Carve cv(ws);
  VsegWs w;
  const int64_t B = c->B, C = c->C, E = c->N - 1;
  w.bp = cv.take<uint8_t>((size_t)(B * (E > 0 ? E : 1) * C));
  w.delta_in = cv.take<float>((size_t)(B * C));
  w.lscore = cv.take<float>((size_t)B);
  w.lzend = cv.take<int32_t>((size_t)B);
  w.zglob = cv.take<int32_t>((size_t)B);
  w.gscore = cv.take<float>((size_t)B);
  w.gflags = cv.take<uint32_t>((size_t)B);
  if (out) *out = w;
  return cv.off;
}
bool vseg_ok(const ts_chain* c, int64_t edge_begin, int64_t n_global) {
  return chain_ok(c) && c->lengths == nullptr && edge_begin >= 0 &&
         edge_begin + (c->N - 1) <= n_global - 1 && c->C <= 128;
}

}  // namespace

extern "C" {

TS_API size_t ts_workspace_bytes(const ts_chain* c, int op, ts_semiring s) {
  if (!chain_ok(c) || (s != TS_LOG && s != TS_MAX)) return 0;
  if (op == TS_OP_MARG_HOST) {
    // K batch chunks, each with its own device staging + inner workspace (ts_marginals_host)
    Carve cv(nullptr);
    const int64_t B = c->B, N = c->N, C = c->C, E = N - 1, per = E * C * C;
    const int K = host_chunks(B, per);
    for (int k = 0; k < K; ++k) {
      const int64_t Bk = B * (k + 1) / K - B * k / K;
      ts_chain dc{Bk, N, C, c->pot, c->lengths};
      cv.take<float>((size_t)(Bk * per));  // pot
      cv.take<int32_t>((size_t)Bk);         // lengths
      cv.take<float>((size_t)(Bk * per + 2 * Bk));  // marg (+ logZ, flags for one copy-back)
      cv.take<float>((size_t)Bk);           // logz
      cv.take<uint32_t>((size_t)Bk);        // flags
      cv.take<char>(op_ws(&dc, TS_OP_MARG, s, nullptr, nullptr, nullptr));
    }
    if (K == 1) {  // second input staging buffer of the cross-call pipeline
      cv.take<float>((size_t)(B * per));
      cv.take<int32_t>((size_t)B);
      cv.take<float>((size_t)(B * per + 2 * B));  // second output staging (three-stage mode)
    }
    return cv.off;
  }
  if (op == TS_OP_SEGMENT) {
    if (c->C > 128) return 0;
    return stream_ws(c, seg_plan(c), true, nullptr, nullptr, nullptr, true);
  }
  if (op == TS_OP_KBEST) return 0;  // use ts_kbest_workspace_bytes (depends on K)
  if (op == TS_OP_SEGMENT_VITERBI) return c->C <= 128 ? vseg_ws(c, nullptr, nullptr) : 0;
  if (op == TS_OP_ENTROPY || op == TS_OP_EXPECTATION)
    return s == TS_LOG ? entropy_ws(c, nullptr, nullptr, nullptr) : 0;
  if (op == TS_OP_SAMPLE) {
    if (s != TS_LOG) return 0;
    if (c->C <= 128) return sample_ws(c, nullptr, nullptr, nullptr);
    return align_up(semi_ws(c, 1, nullptr, nullptr)) + align_up(sizeof(uint32_t) * (size_t)c->B);
  }
  if (op < TS_OP_LOGZ || op > TS_OP_VITERBI) return 0;
  return op_ws(c, op, s, nullptr, nullptr, nullptr);
}

// Semi-Markov plan (semi_expand.cu): the expanded-state chain (S = C K states) whenever the
// plan knob asks for a chunk length, or automatically for long chains (E >= 256) with
// S <= 128 (tensor-core chunk summaries); otherwise the segmental one-CTA kernels.
bool semi_expanded(const ts_chain* c, int64_t K) {
  const int64_t S = c->C * K, E = c->N - 1;
  if (K < 1 || S > 256 || E < 1) return false;
  if (g_plan_chunk.load() > 0) return true;
  return S <= 128 && E >= 256;
}
ts_chain semi_xchain(const ts_chain* c, int64_t K, const float* xpot) {
  ts_chain x = *c;
  x.C = c->C * K;
  x.pot = xpot;
  return x;
}
// layout: xpot | xmarg (log) or xpath (max) | the chain workspace of the expanded call
size_t semi_x_ws(const ts_chain* c, int64_t K, bool maxsemi, bool want_marg, void* ws,
                 float** xpot, float** xmarg, int32_t** xpath, void** inner, size_t* inner_bytes) {
  Carve cv(ws);
  const int64_t S = c->C * K, E = c->N - 1 > 0 ? c->N - 1 : 1;
  float* xp = cv.take<float>((size_t)(c->B * E * S * S));
  float* xm = nullptr;
  int32_t* xa = nullptr;
  if (!maxsemi && want_marg) xm = cv.take<float>((size_t)(c->B * E * S * S));
  if (maxsemi) xa = cv.take<int32_t>((size_t)(c->B * c->N));
  const ts_chain x = semi_xchain(c, K, xp);
  const size_t in_b = align_up(maxsemi ? op_ws(&x, TS_OP_VITERBI, TS_MAX, nullptr, nullptr, nullptr)
                                       : op_ws(&x, want_marg ? TS_OP_MARG : TS_OP_LOGZ, TS_LOG,
                                               nullptr, nullptr, nullptr));
  void* in = cv.take<uint8_t>(in_b);
  if (xpot) *xpot = xp;
  if (xmarg) *xmarg = xm;
  if (xpath) *xpath = xa;
  if (inner) *inner = in;
  if (inner_bytes) *inner_bytes = in_b;
  return cv.off;
}

TS_API size_t ts_semimarkov_workspace_bytes(const ts_chain* c, int64_t K) {
  if (!chain_ok(c) || K < 1 || K > 16) return 0;
  if (semi_expanded(c, K))
    return semi_x_ws(c, K, false, true, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  return semi_ws(c, K, nullptr, nullptr);
}

TS_API ts_status ts_semimarkov(const ts_chain* c, int64_t K, float* marg, float* logz,
                               uint32_t* flags, void* ws, size_t ws_bytes, void* stream) {
  if (!chain_ok(c) || K < 1 || K > 16 || !logz || !aligned(logz, 4) ||
      (marg && !aligned(marg, 4)) || (flags && !aligned(flags, 4)))
    return TS_E_INVALID;
  if (!device_ok()) return TS_E_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (semi_expanded(c, K)) {  // the expanded-state chain through the log plans (scan, tree)
    float *xpot, *xmarg;
    void* inner;
    size_t inner_b;
    const size_t need = semi_x_ws(c, K, false, marg != nullptr, ws, &xpot, &xmarg, nullptr,
                                  &inner, &inner_b);
    if (ws_bytes < need || !ws || !aligned(ws, kAlign)) return TS_E_WORKSPACE;
    SemiExpandArgs x{};
    x.pot = c->pot;
    x.lengths = c->lengths;
    x.B = c->B;
    x.N = c->N;
    x.C = c->C;
    x.K = K;
    x.xpot = xpot;
    x.xmarg = xmarg;
    x.marg = marg;
    x.logz = logz;
    cudaError_t e = launch_semi_expand(x, st);
    if (e != cudaSuccess) return cuda_status(e);
    const ts_chain xc = semi_xchain(c, K, xpot);
    ts_status r = run_log(&xc, xmarg, logz, flags, inner, inner_b, st);
    if (r != TS_OK) return r;
    const int n = t_launches;
    const char* kern = t_kernel;
    if ((e = launch_semi_gather(x, st)) != cudaSuccess) return cuda_status(e);
    t_launches = n + 2;
    t_kernel = kern;
    return TS_OK;
  }
  SemiArgs a{};
  const size_t need = semi_ws(c, K, ws, &a);
  if (ws_bytes < need || !ws || !aligned(ws, kAlign)) return TS_E_WORKSPACE;
  a.pot = c->pot;
  a.lengths = c->lengths;
  a.B = c->B;
  a.N = c->N;
  a.C = c->C;
  a.marg = marg;
  a.logz = logz;
  a.flags = flags;
  ts_status r = cuda_status(launch_semimarkov(a, st));
  if (r == TS_OK) {
    t_launches = 1;
    t_kernel = "semimarkov_kernel";
  }
  return r;
}

TS_API size_t ts_semimarkov_viterbi_workspace_bytes(const ts_chain* c, int64_t K) {
  if (!chain_ok(c) || K < 1 || K > 16) return 0;
  if (semi_expanded(c, K))
    return semi_x_ws(c, K, true, false, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  return align_up(sizeof(uint16_t) * (size_t)(c->B * c->N * c->C));
}

TS_API ts_status ts_semimarkov_viterbi(const ts_chain* c, int64_t K, int32_t* seg, float* score,
                                       uint32_t* flags, void* ws, size_t ws_bytes, void* stream) {
  if (!chain_ok(c) || K < 1 || K > 16 || !seg || !aligned(seg, 4) || !score ||
      !aligned(score, 4) || (flags && !aligned(flags, 4)))
    return TS_E_INVALID;
  if (!device_ok()) return TS_E_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (semi_expanded(c, K)) {  // the expanded-state chain through the max plans (serial, chunked)
    float* xpot;
    int32_t* xpath;
    void* inner;
    size_t inner_b;
    const size_t need = semi_x_ws(c, K, true, false, ws, &xpot, nullptr, &xpath, &inner, &inner_b);
    if (ws_bytes < need || !ws || !aligned(ws, kAlign)) return TS_E_WORKSPACE;
    SemiExpandArgs x{};
    x.pot = c->pot;
    x.lengths = c->lengths;
    x.B = c->B;
    x.N = c->N;
    x.C = c->C;
    x.K = K;
    x.xpot = xpot;
    x.xpath = xpath;
    x.seg = seg;
    cudaError_t e = launch_semi_expand(x, st);
    if (e != cudaSuccess) return cuda_status(e);
    const ts_chain xc = semi_xchain(c, K, xpot);
    ts_status r = run_max(&xc, TS_OP_VITERBI, nullptr, nullptr, xpath, score, flags, inner, inner_b, st);
    if (r != TS_OK) return r;
    const int n = t_launches;
    const char* kern = t_kernel;
    if ((e = launch_semi_seg(x, st)) != cudaSuccess) return cuda_status(e);
    t_launches = n + 2;
    t_kernel = kern;
    return TS_OK;
  }
  const size_t need = ts_semimarkov_viterbi_workspace_bytes(c, K);
  if (ws_bytes < need || !ws || !aligned(ws, kAlign)) return TS_E_WORKSPACE;
  SemiVitArgs a{};
  a.pot = c->pot;
  a.lengths = c->lengths;
  a.B = c->B;
  a.N = c->N;
  a.C = c->C;
  a.K = K;
  a.seg = seg;
  a.score = score;
  a.flags = flags;
  a.bp = static_cast<uint16_t*>(ws);
  ts_status r = cuda_status(launch_semimarkov_viterbi(a, st));
  if (r == TS_OK) {
    t_launches = 1;
    t_kernel = "semimarkov_viterbi_kernel";
  }
  return r;
}

TS_API size_t ts_kbest_workspace_bytes(const ts_chain* c, int64_t K) {
  if (!chain_ok(c) || K < 1 || K > 16) return 0;
  const int64_t E = c->N - 1 > 0 ? c->N - 1 : 1;
  return align_up(sizeof(uint16_t) * (size_t)(c->B * E * c->C * kbest_km(K)));
}

TS_API ts_status ts_kbest(const ts_chain* c, int64_t K, int32_t* paths, float* scores,
                          uint32_t* flags, void* ws, size_t ws_bytes, void* stream) {
  if (!chain_ok(c) || K < 1 || K > 16 || !paths || !aligned(paths, 4) || !scores ||
      !aligned(scores, 4) || (flags && !aligned(flags, 4)))
    return TS_E_INVALID;
  if (!device_ok()) return TS_E_UNSUPPORTED;
  const size_t need = ts_kbest_workspace_bytes(c, K);
  if (ws_bytes < need || !ws || !aligned(ws, kAlign)) return TS_E_WORKSPACE;
  KbestArgs a{};
  a.pot = c->pot;
  a.lengths = c->lengths;
  a.B = c->B;
  a.N = c->N;
  a.C = c->C;
  a.K = K;
  a.bp = static_cast<uint16_t*>(ws);
  a.paths = paths;
  a.scores = scores;
  a.flags = flags;
  ts_status r = cuda_status(launch_kbest(a, static_cast<cudaStream_t>(stream)));
  if (r == TS_OK) {
    t_launches = 1;
    t_kernel = "kbest_kernel";
  }
  return r;
}

TS_API size_t ts_segment_viterbi_summary_bytes(const ts_chain* local) {
  if (!chain_ok(local)) return 0;
  return sizeof(float) * (size_t)(local->B * local->C * local->C);
}

TS_API ts_status ts_segment_viterbi_summary(const ts_chain* local, int64_t edge_begin,
                                            int64_t n_global, float* summary, void* stream) {
  if (!vseg_ok(local, edge_begin, n_global) || !summary || !aligned(summary, 16))
    return TS_E_INVALID;
  if (!device_ok()) return TS_E_UNSUPPORTED;
  VsegArgs v{};
  v.pot = local->pot;
  v.B = local->B;
  v.N = local->N;
  v.C = local->C;
  v.summary = summary;
  ts_status r = cuda_status(launch_vseg_summary(v, static_cast<cudaStream_t>(stream)));
  if (r == TS_OK) {
    t_launches = 1;
    t_kernel = "vseg_summary_kernel";
  }
  return r;
}

TS_API ts_status ts_segment_viterbi_maps(const ts_chain* local, int64_t edge_begin,
                                         int64_t n_global, int rank, int world,
                                         const float* all_summaries, int32_t* maps, float* score,
                                         uint32_t* flags, void* ws, size_t ws_bytes, void* stream) {
  if (!vseg_ok(local, edge_begin, n_global) || world < 1 || rank < 0 || rank >= world ||
      !all_summaries || !maps || !aligned(maps, 4) || (score && !aligned(score, 4)) ||
      (flags && !aligned(flags, 4)))
    return TS_E_INVALID;
  if (!device_ok()) return TS_E_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  VsegWs w;
  const size_t need = vseg_ws(local, ws, &w);
  if (ws_bytes < need || !ws || !aligned(ws, kAlign)) return TS_E_WORKSPACE;
  VsegArgs v{};
  v.pot = local->pot;
  v.B = local->B;
  v.N = local->N;
  v.C = local->C;
  v.all_summ = all_summaries;
  v.rank = rank;
  v.world = world;
  v.delta_in = w.delta_in;
  v.score = w.gscore;
  v.zglob = w.zglob;
  v.flags = w.gflags;
  v.bp = w.bp;
  v.maps = maps;
  cudaError_t e;
  if ((e = launch_vseg_combine(v, st)) != cudaSuccess) return cuda_status(e);
  VitArgs a{};
  a.pot = local->pot;
  a.B = local->B;
  a.N = local->N;
  a.C = local->C;
  a.bp = w.bp;
  a.zend = w.lzend;
  a.score = w.lscore;
  a.delta_in = w.delta_in;
  if ((e = launch_vit1(a, st)) != cudaSuccess) return cuda_status(e);
  if ((e = launch_vseg_maps(v, st)) != cudaSuccess) return cuda_status(e);
  if (score && (e = cudaMemcpyAsync(score, w.gscore, sizeof(float) * (size_t)local->B,
                                    cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
    return cuda_status(e);
  if (flags && (e = cudaMemcpyAsync(flags, w.gflags, sizeof(uint32_t) * (size_t)local->B,
                                    cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
    return cuda_status(e);
  t_launches = 3;
  t_kernel = "viterbi_fwd_kernel";
  return TS_OK;
}

TS_API ts_status ts_segment_viterbi_finish(const ts_chain* local, int64_t edge_begin,
                                           int64_t n_global, int rank, int world,
                                           const int32_t* all_maps, int32_t* path, void* ws,
                                           size_t ws_bytes, void* stream) {
  if (!vseg_ok(local, edge_begin, n_global) || world < 1 || rank < 0 || rank >= world ||
      !all_maps || !path || !aligned(path, 4))
    return TS_E_INVALID;
  if (!device_ok()) return TS_E_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  VsegWs w;
  const size_t need = vseg_ws(local, ws, &w);
  if (ws_bytes < need || !ws || !aligned(ws, kAlign)) return TS_E_WORKSPACE;
  VsegArgs v{};
  v.B = local->B;
  v.N = local->N;
  v.C = local->C;
  v.rank = rank;
  v.world = world;
  v.zglob = w.zglob;
  v.all_maps = all_maps;
  v.zend = w.lzend;
  cudaError_t e;
  if ((e = launch_vseg_endlabel(v, st)) != cudaSuccess) return cuda_status(e);
  VitArgs a{};
  a.pot = local->pot;
  a.B = local->B;
  a.N = local->N;
  a.C = local->C;
  a.bp = w.bp;
  a.zend = w.lzend;
  a.path = path;
  if ((e = launch_backtrack(a, st)) != cudaSuccess) return cuda_status(e);
  t_launches = 2;
  t_kernel = "backtrack_kernel";
  return TS_OK;
}

namespace {
ts_status entropy_or_expectation(const ts_chain* c, const float* r, float* marg, float* logz,
                                 float* out, uint32_t* flags, void* ws, size_t ws_bytes,
                                 void* stream) {
  if (!chain_ok(c) || (c->N > 1 && !marg) || (marg && !aligned(marg, 16)) || !logz ||
      !aligned(logz, 4) || !out || !aligned(out, 4) || (flags && !aligned(flags, 4)))
    return TS_E_INVALID;
  if (!device_ok()) return TS_E_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  size_t mpart = 0;
  double* partial = nullptr;
  const size_t need = entropy_ws(c, ws, &mpart, &partial);
  if (ws_bytes < need || !ws || !aligned(ws, kAlign)) return TS_E_WORKSPACE;
  FusedX fx{r ? 2 : 1, r, out, partial};
  ts_status st_r = run_log(c, marg, logz, flags, ws, mpart, st, &fx);
  if (st_r != TS_OK) return st_r;
  const int n = t_launches;
  const char* k = t_kernel;
  if (fx.fused && fx.final_partials == 0) return TS_OK;  // the marginal kernel wrote `out`
  DistArgs d{};
  d.pot = c->pot;
  d.lengths = c->lengths;
  d.B = c->B;
  d.N = c->N;
  d.C = c->C;
  d.marg = marg;
  d.logz = logz;
  d.flags = flags;
  d.out = out;
  d.r = r;
  d.partial = partial;
  if (fx.fused) {  // per-sequence partials from the marginal kernel: the final stage only
    st_r = cuda_status(launch_entropy_final(d, fx.final_partials, st));
    if (st_r == TS_OK) {
      t_launches = n + 1;
      t_kernel = k;
    }
    return st_r;
  }
  st_r = cuda_status(launch_entropy(d, st));
  if (st_r == TS_OK) {
    t_launches = n + 2;
    t_kernel = k;
  }
  return st_r;
}
}  // namespace

TS_API ts_status ts_entropy(const ts_chain* c, float* marg, float* logz, float* entropy,
                            uint32_t* flags, void* ws, size_t ws_bytes, void* stream) {
  return entropy_or_expectation(c, nullptr, marg, logz, entropy, flags, ws, ws_bytes, stream);
}

TS_API ts_status ts_expectation(const ts_chain* c, const float* r, float* marg, float* logz,
                                float* out, uint32_t* flags, void* ws, size_t ws_bytes,
                                void* stream) {
  if (!r || !aligned(r, 16)) return TS_E_INVALID;
  return entropy_or_expectation(c, r, marg, logz, out, flags, ws, ws_bytes, stream);
}

TS_API ts_status ts_log_prob(const ts_chain* c, const int32_t* z, const float* logz, float* out,
                             void* stream) {
  if (!chain_ok(c) || !z || !aligned(z, 4) || !out || !aligned(out, 4) ||
      (logz && !aligned(logz, 4)))
    return TS_E_INVALID;
  if (!device_ok()) return TS_E_UNSUPPORTED;
  DistArgs d{};
  d.pot = c->pot;
  d.lengths = c->lengths;
  d.B = c->B;
  d.N = c->N;
  d.C = c->C;
  d.logz = logz;
  d.z = z;
  d.out = out;
  ts_status r = cuda_status(launch_score(d, static_cast<cudaStream_t>(stream)));
  if (r == TS_OK) {
    t_launches = 1;
    t_kernel = "score_kernel";
  }
  return r;
}

TS_API ts_status ts_sample(const ts_chain* c, const float* uniforms, int64_t K, int32_t* z,
                           float* logz, uint32_t* flags, void* ws, size_t ws_bytes, void* stream) {
  if (!chain_ok(c) || !uniforms || !aligned(uniforms, 4) || K < 1 || K > ((int64_t)1 << 31) ||
      !z || !aligned(z, 4) || !logz || !aligned(logz, 4) || (flags && !aligned(flags, 4)))
    return TS_E_INVALID;
  if (!device_ok()) return TS_E_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (c->C > 128) {
    // wide labels: the forward recursion of fb_wide (exact per-cell LSE) stores every node
    // vector (log2, normalised) and writes logZ + flags; then the same backward sampler
    SemiArgs sa{};
    const size_t m = align_up(semi_ws(c, 1, ws, &sa));
    const size_t need = m + align_up(sizeof(uint32_t) * (size_t)c->B);
    if (ws_bytes < need || !ws || !aligned(ws, kAlign)) return TS_E_WORKSPACE;
    uint32_t* fl = flags ? flags : reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + m);
    sa.pot = c->pot;
    sa.lengths = c->lengths;
    sa.B = c->B;
    sa.N = c->N;
    sa.C = c->C;
    sa.marg = nullptr;
    sa.logz = logz;
    sa.flags = fl;
    ts_status r = cuda_status(launch_fb_wide(sa, st));
    if (r != TS_OK) return r;
    DistArgs d{};
    d.pot = c->pot;
    d.lengths = c->lengths;
    d.B = c->B;
    d.N = c->N;
    d.C = c->C;
    d.flags = fl;
    d.zout = z;
    d.uniforms = uniforms;
    d.K = K;
    d.ah = sa.ah;
    d.aend_in_ah = 1;
    r = cuda_status(launch_sample(d, st));
    if (r == TS_OK) {
      t_launches = 2;
      t_kernel = "sample_kernel";
    }
    return r;
  }
  StreamWs w;
  uint32_t* wfl = nullptr;
  const size_t need = sample_ws(c, ws, &w, &wfl);
  if (ws_bytes < need || !ws || !aligned(ws, kAlign)) return TS_E_WORKSPACE;
  uint32_t* fl = flags ? flags : wfl;
  cudaError_t e = cudaMemsetAsync(w.wflags, 0, sizeof(uint32_t) * (size_t)c->B, st);
  if (e != cudaSuccess) return cuda_status(e);
  // forward filtering: the serial streaming forward sweep (one chunk per sequence) stores
  // every node vector; it also writes logZ and the flags (logZ-only epilogue)
  SweepArgs a{};
  a.pot = c->pot;
  a.lengths = c->lengths;
  a.B = c->B;
  a.N = c->N;
  a.C = c->C;
  a.L = c->N - 1 > 0 ? c->N - 1 : 1;
  a.P = 1;
  a.alpha_hat = w.alpha_hat;
  a.alpha_end = w.alpha_end;
  a.alpha_end_off = w.alpha_end_off;
  a.mlag = w.mlag;
  a.tmax = w.tmax;
  a.wflags = w.wflags;
  a.logz = logz;
  a.flags = fl;
  a.final_in_fwd = 1;
  if ((e = launch_fwd(a, st)) != cudaSuccess) return cuda_status(e);
  DistArgs d{};
  d.pot = c->pot;
  d.lengths = c->lengths;
  d.B = c->B;
  d.N = c->N;
  d.C = c->C;
  d.flags = fl;
  d.zout = z;
  d.uniforms = uniforms;
  d.K = K;
  d.ah = w.alpha_hat;
  d.aend = w.alpha_end;
  ts_status r = cuda_status(launch_sample(d, st));
  if (r == TS_OK) {
    t_launches = 2;
    t_kernel = "sample_kernel";
  }
  return r;
}

TS_API ts_status ts_logpartition(const ts_chain* c, ts_semiring s, float* logz, uint32_t* flags,
                                 void* ws, size_t ws_bytes, void* stream) {
  if (!chain_ok(c) || !logz || !aligned(logz, 4) || (flags && !aligned(flags, 4)))
    return TS_E_INVALID;
  if (s != TS_LOG && s != TS_MAX) return TS_E_INVALID;
  if (!device_ok()) return TS_E_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (s == TS_MAX) return run_max(c, TS_OP_LOGZ, nullptr, logz, nullptr, nullptr, flags, ws, ws_bytes, st);
  return run_log(c, nullptr, logz, flags, ws, ws_bytes, st);
}

TS_API ts_status ts_marginals(const ts_chain* c, ts_semiring s, float* marg, float* logz,
                              uint32_t* flags, void* ws, size_t ws_bytes, void* stream) {
  // N == 1: there are no edges, the marginal tensor is empty and `marg` may be NULL
  if (!chain_ok(c) || (c->N > 1 && !marg) || (marg && !aligned(marg, 16)) ||
      (logz && !aligned(logz, 4)) || (flags && !aligned(flags, 4)))
    return TS_E_INVALID;
  if (s != TS_LOG && s != TS_MAX) return TS_E_INVALID;
  if (!device_ok()) return TS_E_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (s == TS_MAX) return run_max(c, TS_OP_MARG, marg, logz, nullptr, nullptr, flags, ws, ws_bytes, st);
  // logz is required internally by the log path; use a workspace slot if the caller passed NULL
  if (!logz) return TS_E_INVALID;
  return run_log(c, marg, logz, flags, ws, ws_bytes, st);
}

TS_API ts_status ts_viterbi(const ts_chain* c, int32_t* path, float* score, uint32_t* flags,
                            void* ws, size_t ws_bytes, void* stream) {
  if (!chain_ok(c) || !path || !score || !aligned(path, 4) || !aligned(score, 4) ||
      (flags && !aligned(flags, 4)))
    return TS_E_INVALID;
  if (!device_ok()) return TS_E_UNSUPPORTED;
  return run_max(c, TS_OP_VITERBI, nullptr, nullptr, path, score, flags, ws, ws_bytes,
                 static_cast<cudaStream_t>(stream));
}

// Enqueue the chunked host pipeline of ts_marginals_host on `st` (fork -> K chunk streams
// of H2D, kernels, D2H -> join).  Caller holds hp->mu.
static ts_status host_enqueue(HostPipe* hp, const ts_chain* hc, ts_semiring s, float* host_marg,
                              float* host_logz, uint32_t* host_flags, void* ws, cudaStream_t st) {
  const int64_t B = hc->B, N = hc->N, C = hc->C, E = N - 1;
  const int64_t per = E * C * C;  // floats per sequence
  const int K = host_chunks(B, per);
  cudaError_t e;
  if ((e = cudaEventRecord(hp->fork, st)) != cudaSuccess) return cuda_status(e);
  Carve cv(ws);
  int launches = 0;
  for (int k = 0; k < K; ++k) {
    const int64_t b0 = B * k / K, b1 = B * (k + 1) / K, Bk = b1 - b0;
    const size_t nel = (size_t)(Bk * per);
    cudaStream_t sk = hp->side[k];
    if ((e = cudaStreamWaitEvent(sk, hp->fork, 0)) != cudaSuccess) return cuda_status(e);
    float* d_pot = cv.take<float>(nel);
    int32_t* d_len = cv.take<int32_t>((size_t)Bk);
    float* d_marg = cv.take<float>(nel + 2 * (size_t)Bk);
    float* d_logz = cv.take<float>((size_t)Bk);
    uint32_t* d_flags = cv.take<uint32_t>((size_t)Bk);
    ts_chain dc{Bk, N, C, nel ? d_pot : nullptr, hc->lengths ? d_len : nullptr};
    const size_t inner_bytes = op_ws(&dc, TS_OP_MARG, s, nullptr, nullptr, nullptr);
    void* inner = cv.take<char>(inner_bytes);
    if (nel && (e = cudaMemcpyAsync(d_pot, hc->pot + b0 * per, nel * 4, cudaMemcpyHostToDevice,
                                    sk)) != cudaSuccess)
      return cuda_status(e);
    if (hc->lengths && (e = cudaMemcpyAsync(d_len, hc->lengths + b0, (size_t)Bk * 4,
                                            cudaMemcpyHostToDevice, sk)) != cudaSuccess)
      return cuda_status(e);
    ts_status r = ts_marginals(&dc, s, d_marg, d_logz, d_flags, inner, inner_bytes, sk);
    if (r != TS_OK) return r;
    launches += t_launches;
    if (nel && (e = cudaMemcpyAsync(host_marg + b0 * per, d_marg, nel * 4, cudaMemcpyDeviceToHost,
                                    sk)) != cudaSuccess)
      return cuda_status(e);
    if ((e = cudaMemcpyAsync(host_logz + b0, d_logz, (size_t)Bk * 4, cudaMemcpyDeviceToHost, sk)) !=
        cudaSuccess)
      return cuda_status(e);
    if (host_flags && (e = cudaMemcpyAsync(host_flags + b0, d_flags, (size_t)Bk * 4,
                                           cudaMemcpyDeviceToHost, sk)) != cudaSuccess)
      return cuda_status(e);
    if ((e = cudaEventRecord(hp->join[k], sk)) != cudaSuccess) return cuda_status(e);
    if ((e = cudaStreamWaitEvent(st, hp->join[k], 0)) != cudaSuccess) return cuda_status(e);
  }
  t_launches = launches;
  return TS_OK;
}

// Single-chunk payloads: the copy-in of call k runs on hp->cin into staging buffer k % 2 and
// overlaps call k-1's copy-back on `st` (PCIe is full duplex: tools/duplex_probe.py); the
// scan + copy-back run on `st` after the copy-in (graph-replayed for a repeated binding).
static ts_status host_compute_d2h(const ts_chain* dc, ts_semiring s, float* d_marg,
                                  float* d_logz, uint32_t* d_flags, void* inner, size_t inner_bytes,
                                  float* host_marg, float* host_logz, uint32_t* host_flags,
                                  cudaStream_t st) {
  const int64_t B = dc->B, per = (dc->N - 1) * dc->C * dc->C;
  // host outputs laid out back to back (marg | logZ | flags): the kernel writes logZ / flags
  // right behind the device marginals (the workspace keeps 2B floats there) and one copy
  // brings all three back (each small copy costs ~3.5 us per call, tools/pipe_probe2.py)
  const bool contig = host_logz == host_marg + B * per &&
                      (!host_flags || reinterpret_cast<float*>(host_flags) == host_logz + B);
  if (contig) {
    float* k_logz = d_marg + B * per;
    uint32_t* k_flags = host_flags ? reinterpret_cast<uint32_t*>(k_logz + B) : nullptr;
    ts_status r = ts_marginals(dc, s, d_marg, k_logz, k_flags, inner, inner_bytes, st);
    if (r != TS_OK) return r;
    const size_t n = (size_t)(B * per + B + (host_flags ? B : 0));
    const cudaError_t e = cudaMemcpyAsync(host_marg, d_marg, n * 4, cudaMemcpyDeviceToHost, st);
    return e == cudaSuccess ? TS_OK : cuda_status(e);
  }
  ts_status r = ts_marginals(dc, s, d_marg, d_logz, d_flags, inner, inner_bytes, st);
  if (r != TS_OK) return r;
  cudaError_t e;
  if (B * per && (e = cudaMemcpyAsync(host_marg, d_marg, (size_t)(B * per) * 4,
                                      cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return cuda_status(e);
  if ((e = cudaMemcpyAsync(host_logz, d_logz, (size_t)B * 4, cudaMemcpyDeviceToHost, st)) !=
      cudaSuccess)
    return cuda_status(e);
  if (host_flags && (e = cudaMemcpyAsync(host_flags, d_flags, (size_t)B * 4,
                                         cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return cuda_status(e);
  return TS_OK;
}

static ts_status host_pipelined(HostPipe* hp, const ts_chain* hc, ts_semiring s, float* host_marg,
                                float* host_logz, uint32_t* host_flags, void* ws, size_t ws_bytes,
                                cudaStream_t st) {
  const int64_t B = hc->B, N = hc->N, C = hc->C, per = (N - 1) * C * C;
  const size_t nel = (size_t)(B * per);
  Carve cv(ws);
  float* d_pot0 = cv.take<float>(nel);
  int32_t* d_len0 = cv.take<int32_t>((size_t)B);
  float* d_marg = cv.take<float>(nel + 2 * (size_t)B);
  float* d_logz = cv.take<float>((size_t)B);
  uint32_t* d_flags = cv.take<uint32_t>((size_t)B);
  ts_chain probe{B, N, C, nel ? d_pot0 : nullptr, hc->lengths ? d_len0 : nullptr};
  const size_t inner_bytes = op_ws(&probe, TS_OP_MARG, s, nullptr, nullptr, nullptr);
  void* inner = cv.take<char>(inner_bytes);
  float* d_pot1 = cv.take<float>(nel);
  int32_t* d_len1 = cv.take<int32_t>((size_t)B);
  // a different binding lays the workspace out differently: order this call's copy-in after
  // everything on `st` (the staging buffers of the new layout may overlap the old one's)
  const int64_t sig[5] = {B, N, C, (int64_t)reinterpret_cast<uintptr_t>(ws), (int64_t)s};
  if (std::memcmp(sig, hp->sig, sizeof sig) != 0) {
    std::memcpy(hp->sig, sig, sizeof sig);
    hp->primed[0] = hp->primed[1] = false;
  }
  const int p = hp->parity;
  hp->parity ^= 1;
  float* d_pot = p ? d_pot1 : d_pot0;
  int32_t* d_len = p ? d_len1 : d_len0;
  cudaError_t e;
  // copy-in: after the call that last used this staging buffer; the very first use of a
  // buffer is ordered after the work already on `st`
  if (hp->primed[p]) {
    if ((e = cudaStreamWaitEvent(hp->cin, hp->ev_done[p], 0)) != cudaSuccess) return cuda_status(e);
  } else {
    if ((e = cudaEventRecord(hp->fork, st)) != cudaSuccess) return cuda_status(e);
    if ((e = cudaStreamWaitEvent(hp->cin, hp->fork, 0)) != cudaSuccess) return cuda_status(e);
  }
  if (nel && (e = cudaMemcpyAsync(d_pot, hc->pot, nel * 4, cudaMemcpyHostToDevice, hp->cin)) !=
                 cudaSuccess)
    return cuda_status(e);
  if (hc->lengths && (e = cudaMemcpyAsync(d_len, hc->lengths, (size_t)B * 4,
                                          cudaMemcpyHostToDevice, hp->cin)) != cudaSuccess)
    return cuda_status(e);
  if ((e = cudaEventRecord(hp->ev_in[p], hp->cin)) != cudaSuccess) return cuda_status(e);
  if ((e = cudaStreamWaitEvent(st, hp->ev_in[p], 0)) != cudaSuccess) return cuda_status(e);
  ts_chain dc{B, N, C, nel ? d_pot : nullptr, hc->lengths ? d_len : nullptr};
  // scan + copy-back: graph replay for a repeated binding (parity is part of the key)
  HostKey key{hc->B, hc->N, hc->C, hc->pot, hc->lengths, (int)s + 8 * (p + 1), host_marg,
              host_logz, host_flags, ws, ws_bytes, g_plan_chunk.load(), knob_word()};
  HostGraph* g = hp->find(key);
  ts_status r = TS_OK;
  if (g && g->exec) {
    if ((e = cudaGraphLaunch(g->exec, st)) != cudaSuccess) return cuda_status(e);
    t_launches = g->launches;
  } else if (!g || !g_host_graphs.load()) {
    r = host_compute_d2h(&dc, s, d_marg, d_logz, d_flags, inner, inner_bytes, host_marg,
                         host_logz, host_flags, st);
    if (r == TS_OK && g_host_graphs.load()) hp->insert(key);
  } else {
    if ((e = cudaStreamBeginCapture(hp->cap, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
      return cuda_status(e);
    r = host_compute_d2h(&dc, s, d_marg, d_logz, d_flags, inner, inner_bytes, host_marg,
                         host_logz, host_flags, hp->cap);
    const int n = t_launches;
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(hp->cap, &graph);
    if (r != TS_OK) {
      if (graph) cudaGraphDestroy(graph);
      return r;
    }
    if (e != cudaSuccess) return cuda_status(e);
    e = cudaGraphInstantiate(&g->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      g->exec = nullptr;
      return cuda_status(e);
    }
    g->launches = n;
    if ((e = cudaGraphLaunch(g->exec, st)) != cudaSuccess) return cuda_status(e);
    t_launches = n;
  }
  if (r != TS_OK) return r;
  if ((e = cudaEventRecord(hp->ev_done[p], st)) != cudaSuccess) return cuda_status(e);
  hp->primed[p] = true;
  return TS_OK;
}

// Three-stage pipeline across calls (single-chunk payloads, pipeline mode 2): call k's
// copy-in (`cin`), kernels (`ck`) and copy-back (`cout`) run on library streams into buffer set
// p = k % 2 (input staging and output staging [marg | logZ | flags] each double-buffered), so
// call k+1's copy-in, call k's kernels and call k-1's copy-back overlap (PCIe full duplex);
// `stream` waits for the call's copy-back.  The copy-in of buffer set p waits for the kernels
// of the call that last read it, the kernels for the copy-back of the call that last read its
// output staging (tools/pipe_probe3.py: 42 vs 51 us per call at cfg2).
static ts_status host_pipe3(HostPipe* hp, const ts_chain* hc, ts_semiring s, float* host_marg,
                            float* host_logz, uint32_t* host_flags, void* ws, cudaStream_t st) {
  const int64_t B = hc->B, N = hc->N, C = hc->C, per = (N - 1) * C * C;
  const size_t nel = (size_t)(B * per);
  Carve cv(ws);
  float* d_pot0 = cv.take<float>(nel);
  int32_t* d_len0 = cv.take<int32_t>((size_t)B);
  float* d_out0 = cv.take<float>(nel + 2 * (size_t)B);
  cv.take<float>((size_t)B);     // (logz / flags of the two-stream path)
  cv.take<uint32_t>((size_t)B);
  ts_chain probe{B, N, C, nel ? d_pot0 : nullptr, hc->lengths ? d_len0 : nullptr};
  const size_t inner_bytes = op_ws(&probe, TS_OP_MARG, s, nullptr, nullptr, nullptr);
  void* inner = cv.take<char>(inner_bytes);
  float* d_pot1 = cv.take<float>(nel);
  int32_t* d_len1 = cv.take<int32_t>((size_t)B);
  float* d_out1 = cv.take<float>(nel + 2 * (size_t)B);
  cudaError_t e;
  const int64_t sig[5] = {B, N, C, (int64_t)reinterpret_cast<uintptr_t>(ws), (int64_t)s};
  if (std::memcmp(sig, hp->p3_sig, sizeof sig) != 0) {
    std::memcpy(hp->p3_sig, sig, sizeof sig);
    hp->p3_primed[0] = hp->p3_primed[1] = false;
  }
  const int p = hp->p3_parity;
  hp->p3_parity ^= 1;
  float* d_pot = p ? d_pot1 : d_pot0;
  int32_t* d_len = p ? d_len1 : d_len0;
  float* d_out = p ? d_out1 : d_out0;
  const bool primed = hp->p3_primed[p];
  if (!primed) {  // first use of this set (or a new layout): after everything on `stream`
    if ((e = cudaEventRecord(hp->e3_fork, st)) != cudaSuccess) return cuda_status(e);
    if ((e = cudaStreamWaitEvent(hp->cin, hp->e3_fork, 0)) != cudaSuccess) return cuda_status(e);
    if ((e = cudaStreamWaitEvent(hp->ck, hp->e3_fork, 0)) != cudaSuccess) return cuda_status(e);
  } else if ((e = cudaStreamWaitEvent(hp->cin, hp->e3_k[p], 0)) != cudaSuccess) {
    return cuda_status(e);
  }
  // 1. copy-in
  if (nel && (e = cudaMemcpyAsync(d_pot, hc->pot, nel * 4, cudaMemcpyHostToDevice, hp->cin)) !=
                 cudaSuccess)
    return cuda_status(e);
  if (hc->lengths && (e = cudaMemcpyAsync(d_len, hc->lengths, (size_t)B * 4,
                                          cudaMemcpyHostToDevice, hp->cin)) != cudaSuccess)
    return cuda_status(e);
  if ((e = cudaEventRecord(hp->e3_in[p], hp->cin)) != cudaSuccess) return cuda_status(e);
  // 2. kernels (logZ and flags land right behind the device marginals)
  if ((e = cudaStreamWaitEvent(hp->ck, hp->e3_in[p], 0)) != cudaSuccess) return cuda_status(e);
  if (primed && (e = cudaStreamWaitEvent(hp->ck, hp->e3_out[p], 0)) != cudaSuccess)
    return cuda_status(e);
  ts_chain dc{B, N, C, nel ? d_pot : nullptr, hc->lengths ? d_len : nullptr};
  float* k_logz = d_out + nel;
  uint32_t* k_flags = reinterpret_cast<uint32_t*>(k_logz + B);
  const ts_status r = ts_marginals(&dc, s, d_out, k_logz, k_flags, inner, inner_bytes, hp->ck);
  if (r != TS_OK) return r;
  if ((e = cudaEventRecord(hp->e3_k[p], hp->ck)) != cudaSuccess) return cuda_status(e);
  // 3. copy-back: one copy when the host outputs are back to back
  if ((e = cudaStreamWaitEvent(hp->cout, hp->e3_k[p], 0)) != cudaSuccess) return cuda_status(e);
  const bool contig = host_logz == host_marg + nel &&
                      (!host_flags || reinterpret_cast<float*>(host_flags) == host_logz + B);
  if (contig) {
    const size_t n = nel + (size_t)B + (host_flags ? (size_t)B : 0);
    if ((e = cudaMemcpyAsync(host_marg, d_out, n * 4, cudaMemcpyDeviceToHost, hp->cout)) != cudaSuccess)
      return cuda_status(e);
  } else {
    if (nel && (e = cudaMemcpyAsync(host_marg, d_out, nel * 4, cudaMemcpyDeviceToHost, hp->cout)) !=
                   cudaSuccess)
      return cuda_status(e);
    if ((e = cudaMemcpyAsync(host_logz, k_logz, (size_t)B * 4, cudaMemcpyDeviceToHost, hp->cout)) !=
        cudaSuccess)
      return cuda_status(e);
    if (host_flags && (e = cudaMemcpyAsync(host_flags, k_flags, (size_t)B * 4, cudaMemcpyDeviceToHost,
                                           hp->cout)) != cudaSuccess)
      return cuda_status(e);
  }
  if ((e = cudaEventRecord(hp->e3_out[p], hp->cout)) != cudaSuccess) return cuda_status(e);
  // 4. the caller's stream sees the results once it is past this event
  if ((e = cudaStreamWaitEvent(st, hp->e3_out[p], 0)) != cudaSuccess) return cuda_status(e);
  hp->p3_primed[p] = true;
  return TS_OK;
}

// ts_marginals_host body, under hp->mu, after the cross-stream ordering.
ts_status marginals_host_locked(HostPipe* hp, const ts_chain* hc, ts_semiring s,
                                float* host_marg, float* host_logz, uint32_t* host_flags,
                                void* ws, size_t ws_bytes, cudaStream_t st) {
  const bool one_chunk = host_chunks(hc->B, (hc->N - 1) * hc->C * hc->C) == 1;
  if (g_host_pipeline.load() == 2 && one_chunk) {
    hp->primed[0] = hp->primed[1] = false;  // (the two-stream path's buffers are reused here)
    return host_pipe3(hp, hc, s, host_marg, host_logz, host_flags, ws, st);
  }
  hp->p3_primed[0] = hp->p3_primed[1] = false;
  if (g_host_pipeline.load() == 1 && one_chunk)
    return host_pipelined(hp, hc, s, host_marg, host_logz, host_flags, ws, ws_bytes, st);
  // a stream-ordered call: the next pipelined call must order its copy-in after it again
  hp->primed[0] = hp->primed[1] = false;
  // Replay path: the same I/O binding seen before -> one graph launch (all copies and
  // kernels of the call are nodes of the instantiated graph; nothing is skipped).
  HostKey key{hc->B, hc->N, hc->C, hc->pot, hc->lengths, (int)s, host_marg, host_logz,
              host_flags, ws, ws_bytes, g_plan_chunk.load(), knob_word()};
  HostGraph* g = hp->find(key);
  if (g && g->exec) {
    cudaError_t e = cudaGraphLaunch(g->exec, st);
    if (e != cudaSuccess) return cuda_status(e);
    t_launches = g->launches;
    return TS_OK;
  }
  if (!g || !g_host_graphs.load()) {
    // first sighting: enqueue eagerly (also performs one-time kernel attribute setup)
    ts_status r = host_enqueue(hp, hc, s, host_marg, host_logz, host_flags, ws, st);
    if (r == TS_OK && g_host_graphs.load()) hp->insert(key);
    return r;
  }
  // second sighting: capture the pipeline on the private stream, instantiate, launch
  cudaError_t e = cudaStreamBeginCapture(hp->cap, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) return cuda_status(e);
  ts_status r = host_enqueue(hp, hc, s, host_marg, host_logz, host_flags, ws, hp->cap);
  cudaGraph_t graph = nullptr;
  e = cudaStreamEndCapture(hp->cap, &graph);
  if (r != TS_OK) {
    if (graph) cudaGraphDestroy(graph);
    return r;
  }
  if (e != cudaSuccess) return cuda_status(e);
  e = cudaGraphInstantiate(&g->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) {
    g->exec = nullptr;
    return cuda_status(e);
  }
  g->launches = t_launches;
  if ((e = cudaGraphLaunch(g->exec, st)) != cudaSuccess) return cuda_status(e);
  t_launches = g->launches;
  return TS_OK;
}

TS_API ts_status ts_marginals_host(const ts_chain* hc, ts_semiring s, float* host_marg,
                                   float* host_logz, uint32_t* host_flags, void* ws,
                                   size_t ws_bytes, void* stream) {
  if (!chain_ok(hc) || !host_marg || !host_logz) return TS_E_INVALID;
  if (s != TS_LOG && s != TS_MAX) return TS_E_INVALID;
  if (!device_ok()) return TS_E_UNSUPPORTED;
  const size_t need = ts_workspace_bytes(hc, TS_OP_MARG_HOST, s);
  if (ws_bytes < need || !ws || !aligned(ws, kAlign)) return TS_E_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  HostPipe* hp = host_pipe();
  if (!hp) return TS_E_CUDA;
  std::lock_guard<std::mutex> lock(hp->mu);
  cudaError_t e;
  // every call shares the device staging buffers, d_marg/d_logz/d_flags and the inner
  // workspace: a call on a different stream than the previous one first waits for it
  if (hp->has_last && hp->last_st != st &&
      (e = cudaStreamWaitEvent(st, hp->ev_last, 0)) != cudaSuccess)
    return cuda_status(e);
  const ts_status r =
      marginals_host_locked(hp, hc, s, host_marg, host_logz, host_flags, ws, ws_bytes, st);
  if (r != TS_OK) return r;
  if ((e = cudaEventRecord(hp->ev_last, st)) != cudaSuccess) return cuda_status(e);
  hp->last_st = st;
  hp->has_last = true;
  return TS_OK;
}

TS_API void ts_set_host_graphs(int on) { g_host_graphs.store(on ? 1 : 0); }
TS_API void ts_set_host_pipeline(int mode) { g_host_pipeline.store(mode <= 0 ? 0 : (mode == 1 ? 1 : 2)); }

TS_API void ts_set_tc_summary(int mode) { tsb::set_tc_summary(mode); }
TS_API int ts_get_tc_summary(void) { return tsb::get_tc_summary(); }

TS_API void* ts_host_alloc(size_t bytes) {
  // Blocks are rounded up to >= 32 MB: on the GPU boxes' virtualised PCIe, host->device DMA
  // from small page-locked allocations measured ~13-16 GB/s vs ~25 GB/s from slices of
  // large ones (tools/e2e_probe.py, gpurun_out/s12_*).
  void* p = nullptr;
  if (bytes == 0) return nullptr;
  const size_t kMin = (size_t)32 << 20, kGran = (size_t)2 << 20;
  size_t sz = (bytes + kGran - 1) / kGran * kGran;
  if (sz < kMin) sz = kMin;
  if (cudaHostAlloc(&p, sz, cudaHostAllocPortable) != cudaSuccess) return nullptr;
  return p;
}

TS_API void ts_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

TS_API size_t ts_segment_summary_bytes(const ts_chain* local) {
  if (!chain_ok(local)) return 0;
  return (size_t)seg_total_floats(local->B, local->C) * sizeof(float);
}

TS_API ts_status ts_segment_summary(const ts_chain* local, int64_t edge_begin, int64_t n_global,
                                    ts_semiring s, void* summary, void* ws, size_t ws_bytes,
                                    void* stream) {
  if (!seg_ok(local, edge_begin, n_global) || !summary || !aligned(summary, 16)) return TS_E_INVALID;
  if (s != TS_LOG) return TS_E_UNSUPPORTED;
  if (!device_ok()) return TS_E_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Plan p = seg_plan(local);
  StreamWs w;
  ScanWs sw;
  const size_t need = stream_ws(local, p, true, ws, &w, &sw, true);
  if (ws_bytes < need || !ws || !aligned(ws, kAlign)) return TS_E_WORKSPACE;
  cudaError_t e = cudaMemsetAsync(w.wflags, 0, sizeof(uint32_t) * (size_t)local->B, st);
  if (e != cudaSuccess) return cuda_status(e);
  ScanArgs sa = make_scan(local, p, w, sw, nullptr, nullptr);
  int n = 0;
  if ((e = launch_scan_up(sa, st, &n)) != cudaSuccess) return cuda_status(e);
  if ((e = launch_segment_export(sa, static_cast<float*>(summary), st)) != cudaSuccess)
    return cuda_status(e);
  t_launches = n + 1;
  return TS_OK;
}

TS_API ts_status ts_segment_finish(const ts_chain* local, int64_t edge_begin, int64_t n_global,
                                   int rank, int world, ts_semiring s, const void* all_summaries,
                                   float* marg, float* logz, uint32_t* flags, void* ws,
                                   size_t ws_bytes, void* stream) {
  if (!seg_ok(local, edge_begin, n_global) || !all_summaries || !logz || world < 1 || rank < 0 ||
      rank >= world || (marg && !aligned(marg, 16)) || !aligned(all_summaries, 16))
    return TS_E_INVALID;
  if (s != TS_LOG) return TS_E_UNSUPPORTED;
  if (!device_ok()) return TS_E_UNSUPPORTED;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const Plan p = seg_plan(local);
  StreamWs w;
  ScanWs sw;
  const size_t need = stream_ws(local, p, true, ws, &w, &sw, true);
  if (ws_bytes < need || !ws || !aligned(ws, kAlign)) return TS_E_WORKSPACE;
  ScanArgs sa = make_scan(local, p, w, sw, logz, flags);
  cudaError_t e;
  int n = 0;
  // prefix / suffix over the gathered segment summaries (same order on every rank) and logZ
  if ((e = launch_segment_combine(sa, static_cast<const float*>(all_summaries), rank, world,
                                  marg != nullptr, st)) != cudaSuccess)
    return cuda_status(e);
  ++n;
  if (!marg) {
    t_launches = n;
    return TS_OK;
  }
  if ((e = launch_scan_down(sa, st, &n, false)) != cudaSuccess) return cuda_status(e);
  SweepArgs a{};
  a.pot = local->pot;
  a.lengths = nullptr;
  a.B = local->B;
  a.N = local->N;
  a.C = local->C;
  a.L = p.L;
  a.P = p.P;
  a.alpha_in = sw.leaf_alpha;
  a.alpha_in_off = sw.leaf_alpha_off;
  a.beta_out = sw.leaf_beta;
  a.beta_out_off = sw.leaf_beta_off;
  a.alpha_hat = w.alpha_hat;
  a.alpha_end = w.alpha_end;
  a.alpha_end_off = w.alpha_end_off;
  a.mlag = w.mlag;
  a.tmax = w.tmax;
  a.marg = marg;
  a.wflags = w.wflags;
  a.logz = logz;
  a.flags = flags;
  a.final_in_fwd = 0;
  a.no_final = 1;
  if ((e = launch_fwd(a, st)) != cudaSuccess) return cuda_status(e);
  if ((e = launch_bwd(a, st)) != cudaSuccess) return cuda_status(e);
  t_launches = n + 2;
  return TS_OK;
}

TS_API void ts_set_meet(int enable) { g_meet.store(enable ? 1 : 0); }
TS_API void ts_set_vchunk_mm(int enable) { set_vchunk_mm(enable); }
TS_API void ts_set_kbest_split(int S) { set_kbest_split(S); }
TS_API void ts_set_viterbi_split(int G) {
  g_vsplit.store((G == -1 || G == 1 || G == 2 || G == 4 || G == 8) ? G : 0);
}
TS_API void ts_set_plan_chunk(int64_t L) { g_plan_chunk.store(L < 0 ? 0 : L); }
TS_API int64_t ts_get_plan_chunk(void) { return g_plan_chunk.load(); }
TS_API void ts_set_small_cluster(int G) {
  g_small_cluster.store((G == 2 || G == 4) ? G : (G < 0 ? -1 : 0));
}
TS_API void ts_set_tiny(int enable) { g_tiny.store(enable ? 1 : 0); }
TS_API void ts_set_wide_ring(int enable) { g_wide_ring = enable ? 1 : 0; }
TS_API void ts_set_tiny_early(int enable) { tsb::set_tiny_early(enable); }
TS_API int ts_last_launch_count(void) { return t_launches; }
TS_API const char* ts_last_kernel(void) { return t_kernel; }

TS_API const char* ts_status_str(ts_status s) {
  switch (s) {
    case TS_OK: return "TS_OK";
    case TS_E_INVALID: return "TS_E_INVALID: invalid argument";
    case TS_E_UNSUPPORTED: return "TS_E_UNSUPPORTED: needs an sm_100 (B200) device / unsupported case";
    case TS_E_WORKSPACE: return "TS_E_WORKSPACE: workspace too small or misaligned";
    case TS_E_CUDA: return "TS_E_CUDA: CUDA launch/copy failure";
  }
  return "unknown ts_status";
}

TS_API const char* ts_version(void) { return "ts_b200 0.1 (sm_100a)"; }

}  // extern "C"
