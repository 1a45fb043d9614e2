// tsgen_device.cu — device-side fill of the seeded synthetic potentials (tsgen.h).
// Test/bench infrastructure: fills l[b][t][i][j] for t in [t_begin, t_begin+E_local)
// of a chain with E_global edges, using GLOBAL indices so a time-sharded rank
// generates exactly its slice of the unsharded input.
#include <cuda_runtime.h>
#include <stdint.h>

#include "tsgen.h"

__global__ void tsgen_fill_kernel(float* __restrict__ out, int64_t B, int64_t E_local,
                                  int64_t C, uint64_t seed, int s, int64_t t_begin,
                                  int64_t E_global) {
  const int64_t CC = C * C;
  const int64_t per_b = E_local * CC;
  const int64_t total = B * per_b;
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < total;
       n += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = n / per_b;
    int64_t r = n - b * per_b;
    int64_t t = r / CC;
    int64_t ij = r - t * CC;
    uint64_t idx = ((uint64_t)b * (uint64_t)E_global + (uint64_t)(t_begin + t)) * (uint64_t)CC +
                   (uint64_t)ij;
    out[n] = tsgen_value(seed, s, idx);
  }
}

extern "C" __attribute__((visibility("default"))) int tsgen_fill_device(float* out, int64_t B, int64_t E_local, int64_t C,
                                 uint64_t seed, int s, int64_t t_begin, int64_t E_global,
                                 void* stream) {
  if (B <= 0 || E_local <= 0 || C <= 0) return 0;
  if (out == nullptr || s < 0 || s > 15 || t_begin < 0 || t_begin + E_local > E_global) return 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t total = B * E_local * C * C;
  int64_t blocks = (total + 255) / 256;
  int64_t cap = (int64_t)sms * 16;
  if (blocks > cap) blocks = cap;
  tsgen_fill_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(out, B, E_local, C, seed,
                                                                         s, t_begin, E_global);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
