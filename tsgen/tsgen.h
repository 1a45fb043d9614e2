/*
 * tsgen.h — the seeded synthetic-input generator, shared by the oracle (host C)
 * and the GPU bench/tests (device CUDA).  It holds NONE of the method's
 * arithmetic: it only maps a global element index to a dyadic fp32 value.
 *
 * Recipe ("Synthetic inputs"):
 *   idx = ((b*E_global + t)*C + i)*C + j                (uint64, global edge index t)
 *   x   = splitmix64(seed + (idx+1) * 0x9E3779B97F4A7C15)
 *   k   = (x&0xFFFF) + (x>>16&0xFFFF) + (x>>32&0xFFFF) + (x>>48) - 131070
 *                                                         (Irwin-Hall(4) of 16-bit uniforms)
 *   l   = (float)(k >> (15 - s)) * 2^-s                  (arithmetic shift, |l| <= 4, sd ~ 1.15)
 * `s` (the dyadic quantum) is chosen so that E*4*2^s <= 2^24: every partial path
 * sum is then exactly representable in fp32 and fp64, so max-plus (Viterbi) is
 * exact in any association order.
 *
 * Pure integer arithmetic: bit-identical on host and device.
 */
#ifndef TSGEN_H
#define TSGEN_H
#include <stdint.h>

#if defined(__CUDACC__)
#define TSGEN_FN __host__ __device__ __forceinline__
#else
#define TSGEN_FN static inline
#endif

#define TSGEN_GOLDEN 0x9E3779B97F4A7C15ULL
#define TSGEN_SEED_BASE 0x200200876ULL /* seed = TSGEN_SEED_BASE + cfg_no */

TSGEN_FN uint64_t tsgen_splitmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* Irwin-Hall(4) integer in [-131070, 131070] for one global index. */
TSGEN_FN int32_t tsgen_irwin_hall(uint64_t seed, uint64_t idx) {
  uint64_t x = tsgen_splitmix64(seed + (idx + 1ULL) * TSGEN_GOLDEN);
  int32_t k = (int32_t)(x & 0xFFFFULL) + (int32_t)((x >> 16) & 0xFFFFULL) +
              (int32_t)((x >> 32) & 0xFFFFULL) + (int32_t)(x >> 48);
  return k - 131070;
}

/* The dyadic value: (k >> (15-s)) * 2^-s, computed exactly (power-of-two scale). */
TSGEN_FN float tsgen_value(uint64_t seed, int s, uint64_t idx) {
  int32_t k = tsgen_irwin_hall(seed, idx) >> (15 - s); /* arithmetic shift (floor) */
  /* 2^-s as an exact float; s in [0,15] */
  float scale = 1.0f / (float)(1u << s);
  return (float)k * scale;
}

/* Largest s in [0,15] with E*4*2^s <= 2^24 (E >= 1). */
TSGEN_FN int tsgen_quantum(int64_t E) {
  int s = 15;
  if (E < 1) E = 1;
  while (s > 0 && (int64_t)E * 4 * ((int64_t)1 << s) > ((int64_t)1 << 24)) --s;
  return s;
}

TSGEN_FN uint64_t tsgen_index(int64_t b, int64_t t, int64_t i, int64_t j, int64_t E_global,
                              int64_t C) {
  return (((uint64_t)b * (uint64_t)E_global + (uint64_t)t) * (uint64_t)C + (uint64_t)i) *
             (uint64_t)C + (uint64_t)j;
}

#endif /* TSGEN_H */
